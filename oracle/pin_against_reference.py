# Pins the C oracle against the reference package (needs /root/reference; build container only).
import sys, time, math
sys.path.insert(0, "/root/reference/pkg/src"); sys.path.insert(0, "/root/repo")
import numpy as np
import hzgsvd as hz
from hzgsvd import harness
from oracle import oracle as O
# generator parity
for seed in (1, 12345, 2**63+5):
    a = harness.uniform_stream(seed, 1000); b = O.uniform_stream(seed, 1000)
    assert np.array_equal(a, b), "uniform"
    a = harness.gaussian_stream(seed, 1001); b = O.gaussian_stream(seed, 1001)
    assert np.array_equal(a, b), "gauss"
print("generators bitwise ok")
for kind in ("me", "mm"):
    for n in range(2, 40, 2):
        assert np.array_equal(hz.gen_table(kind, n).as_array(), O.gen_table(kind, n)), (kind, n)
print("tables ok")
def run(F, G, w, field, **kw):
    cfg = hz.SolverConfig(block_width=w, **kw)
    t0 = time.time(); r = hz.solve(F, G, cfg); t1 = time.time()
    o = O.solve(F, G, O.cfg_from(cfg), threads=4); t2 = time.time()
    same = all(np.array_equal(x, y) for x, y in [(r.sigma, o["sigma"]), (r.sigmaF, o["sigmaF"]), (r.U.to_dense(), o["U"]), (r.Z.to_dense(), o["Z"]), (r.V.to_dense(), o["V"])])
    print(f"{field} n={F.shape[1]} w={w} {kw}: bitwise={same} sweeps {r.sweeps}/{o['sweeps']} tot {r.total_transforms}/{o['total']} big {r.big_transforms}/{o['big']} ref {t1-t0:.2f}s oracle {t2-t1:.2f}s maxdiff {np.abs(r.sigma-o['sigma']).max():.2e}")
    return same
eye = np.eye(4); hz.solve(eye, eye, hz.SolverConfig(block_width=1))
for field in ("real", "complex"):
    for n, w in ((16, 2), (32, 4), (40, 8), (64, 8)):
        pair, ref = hz.gen_pair(hz.random_genspec(n, 777 + n, field))
        F = pair.F.to_dense(); G = pair.G.to_dense()
        run(F, G, w, field)
    pair, ref = hz.gen_pair(hz.random_genspec(48, 99, field))
    F = pair.F.to_dense(); G = pair.G.to_dense()
    for vid in range(8):
        run(F, G, 4, field, variant_id=vid)
    run(F, G, 4, field, blocking="bo")
    run(F, G, 4, field, outer_kind="mm", inner_kind="mm")
    run(F, G, 4, field, shorten="qr")
    run(F, G, 4, field, sorting=False)
