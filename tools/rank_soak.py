"""Random multi-rank soak: solve(workers=R) vs solve() bitwise on random
shapes / block widths / fields / rank counts, deferred Z on every other
case (python tools/rank_soak.py; 14 cases, 0 mismatches in round 1)."""
import sys, os, numpy as np
sys.path.insert(0, os.getcwd())
import paper_1909_00101_b200 as hz
from oracle import oracle as O
rng = np.random.default_rng(11)
fails = 0
for t in range(14):
    w = int(rng.choice([4, 8, 16]))
    nb = int(rng.integers(4, 40)) * 2
    n = nb * w - int(rng.integers(0, w))
    cplx = bool(rng.integers(0, 2))
    R = int(rng.integers(2, 9))
    if t % 2: os.environ["HZG_WAVE_DEFER_Z"] = "1"
    else: os.environ.pop("HZG_WAVE_DEFER_Z", None)
    g = O.gaussian_stream(100 + t, 4 * n * n)
    F = g[:n*n].reshape((n, n), order="F"); G = g[n*n:2*n*n].reshape((n, n), order="F")
    if cplx:
        F = F + 1j * g[2*n*n:3*n*n].reshape((n, n), order="F"); G = G + 1j * g[3*n*n:].reshape((n, n), order="F")
    cfg = hz.SolverConfig(block_width=w, max_outer_sweeps=8)
    a = hz.solve(F, G, cfg); b = hz.solve(F, G, cfg, workers=R)
    ok = np.array_equal(a.sigma, b.sigma) and np.array_equal(a.Z.to_dense(), b.Z.to_dense()) and a.total_transforms == b.total_transforms
    fails += not ok
    print(t, n, w, cplx, R, b.workers, os.environ.get("HZG_WAVE_DEFER_Z", "0"), "ok" if ok else "MISMATCH", flush=True)
print("fails", fails)
