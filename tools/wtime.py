"""Full-solve wall time vs block width (DMMA mode, short-chain 2x2):
python tools/wtime.py config4 16 32 -- inputs of the north-star fixtures."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1909_00101_b200 as hz  # noqa: E402
from oracle import oracle as O  # noqa: E402

name = sys.argv[1]
ws = [int(x) for x in sys.argv[2:] if "=" not in x] or [16, 32]
# extra SolverConfig fields as key=value (integers), e.g. split_rows=256
over = {k: int(v) for k, v in (x.split("=") for x in sys.argv[2:] if "=" in x)}
F, G, kw, extra = O.ns_inputs(name)
fx = os.path.join(os.path.dirname(__file__), "..", "tests", "golden", "ns_%s.npz" % name)
ref = dict(np.load(fx)) if os.path.exists(fx) else None
for w in ws:
    kw2 = dict(kw, block_width=w, **over)
    cfg = hz.SolverConfig(**kw2)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    hz.solve(F, G, cfg)  # first call: context, sweep-graph capture and instantiation
    first = time.perf_counter() - t0
    t0 = time.perf_counter()
    r = hz.solve(F, G, cfg)
    dt = time.perf_counter() - t0
    line = "%s w=%d: %d sweeps, %.3f s e2e (first call %.3f s), converged %s" % (name, w, r.sweeps, dt, first,
                                                                              r.converged)
    if ref is not None:
        rel = np.abs(r.sigma - ref["sigma"]) / ref["sigma"]
        line += ", max rel sigma vs oracle(w=16) %.2e (median %.2e)" % (rel.max(), np.median(rel))
    print(line, flush=True)
    hz.clear_cache()
