"""Stripe scheme (solve(workers=s)) wall time on the GPU vs single worker."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1909_00101_b200 as hz  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
rng = np.random.default_rng(3)
F, G = rng.standard_normal((n, n)), rng.standard_normal((n, n))
cfg = hz.SolverConfig(block_width=16)
for s in (1, 2, 4, 8):
    hz.solve(F, G, cfg, workers=s)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    r = hz.solve(F, G, cfg, workers=s)
    print("n=%d workers=%d: %d outermost sweeps, %.3f s" % (n, s, r.sweeps, time.perf_counter() - t0), flush=True)
