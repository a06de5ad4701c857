"""Full-solve wall time with the short-chain 2x2 forms on / off (DMMA mode):
config 4 (real 4096^2, sigma 1e-8..1e8), config 3 (complex 3072x2048 /
2048^2), config 2 (real 1024^2).  Prints sweeps, seconds and the sigma
difference to the oracle fixtures when present."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1909_00101_b200 as hz  # noqa: E402
from oracle import oracle as O  # noqa: E402

names = sys.argv[1:] or ["config2", "config4", "config3"]
for name in names:
    F, G, kw, extra = O.ns_inputs(name)
    fx = os.path.join(os.path.dirname(__file__), "..", "tests", "golden", "ns_%s.npz" % name)
    ref = dict(np.load(fx)) if os.path.exists(fx) else None
    for approx in (True, False):
        cfg = hz.SolverConfig(approx_2x2=approx, **kw)
        hz.solve(F, G, cfg)  # warm (graph capture)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        r = hz.solve(F, G, cfg)
        dt = time.perf_counter() - t0
        line = "%s approx=%d: %d sweeps, %.3f s e2e" % (name, approx, r.sweeps, dt)
        if ref is not None:
            rel = np.abs(r.sigma - ref["sigma"]) / ref["sigma"]
            line += ", max rel sigma vs oracle %.2e (median %.2e), oracle sweeps %d" % (
                rel.max(), np.median(rel), int(ref["sweeps"]))
        print(line, flush=True)
    hz.clear_cache()
