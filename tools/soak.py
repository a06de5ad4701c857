"""Randomised parity soak (run on the GPU box): random shapes, block widths,
fields, variants and options; exact mode must equal the oracle bitwise
(sigma, U, V, Z, counters), the default mode must stay within the stated
tolerances.  Usage: python tools/soak.py [cases] [seed]"""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_1909_00101_b200 as hz
from oracle import oracle as O

EPS = 2.0 ** -52
cases = int(sys.argv[1]) if len(sys.argv) > 1 else 60
rng = np.random.default_rng(int(sys.argv[2]) if len(sys.argv) > 2 else 1)
fails = 0
t0 = time.time()
for c in range(cases):
    n = int(rng.integers(2, 200))
    mF = n + int(rng.integers(0, 60))
    mG = n + int(rng.integers(0, 30))
    cplx = bool(rng.integers(0, 2))
    w = int(rng.choice([1, 2, 3, 4, 5, 6, 7, 8, 10, 12, 16, 24, 32]))
    kw = dict(block_width=w, variant_id=int(rng.integers(0, 8)), sorting=bool(rng.integers(0, 4) > 0),
              blocking="bo" if rng.integers(0, 4) == 0 else "fb",
              outer_kind="mm" if rng.integers(0, 4) == 0 else "me", inner_kind="mm" if rng.integers(0, 4) == 0 else "me")
    F = rng.standard_normal((mF, n)) + (1j * rng.standard_normal((mF, n)) if cplx else 0)
    G = rng.standard_normal((mG, n)) + (1j * rng.standard_normal((mG, n)) if cplx else 0)
    cfg = hz.SolverConfig(**kw)
    try:
        ref = O.solve(F, G, O.cfg_from(cfg))
    except O.OracleError as e:
        print("case %d oracle error %s (%s)" % (c, e, kw))
        continue
    msg = []
    try:
        r = hz.solve(F, G, hz.SolverConfig(exact=True, **kw))
        same = (np.array_equal(r.sigma, ref["sigma"]) and np.array_equal(r.Z.to_dense(), ref["Z"])
                and np.array_equal(r.U.to_dense(), ref["U"]) and np.array_equal(r.V.to_dense(), ref["V"])
                and (r.sweeps, r.total_transforms, r.big_transforms) == (ref["sweeps"], ref["total"], ref["big"]))
        if not same:
            msg.append("exact mode not bitwise")
        d = hz.solve(F, G, cfg)
        nn = max(n, 64)
        rel = np.abs(d.sigma - ref["sigma"]) / ref["sigma"]
        # the tests' DMMA-mode bound: every sigma within 1e-10 (the
        # reference's variant-agreement bound), 99 % within 8 n eps
        err = rel.max() if np.mean(rel <= 8 * nn * EPS) < 0.99 or rel.max() > 1e-10 else 0.0
        U, V, Z = d.U.to_dense(), d.V.to_dense(), d.Z.to_dense()
        resF = np.linalg.norm(F @ Z - U * d.sigmaF[None, :]) / np.linalg.norm(F)
        oU = np.linalg.norm(U.conj().T @ U - np.eye(n))
        if not (err <= 8 * nn * EPS and resF <= 4 * nn * EPS and oU <= 32 * nn * EPS):
            msg.append("default mode out of tolerance: err %.2e resF %.2e orthU %.2e" % (err, resF, oU))
    except Exception as e:  # noqa
        msg.append("exception %r" % e)
    if msg:
        fails += 1
        print("FAIL case %d n=%d mF=%d mG=%d cplx=%s %s: %s" % (c, n, mF, mG, cplx, kw, "; ".join(msg)), flush=True)
print("soak: %d cases, %d failures, %.0f s" % (cases, fails, time.time() - t0))
