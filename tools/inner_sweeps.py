"""Inner-sweep load balance per outer sweep (DMMA mode):
python tools/inner_sweeps.py config4 [w]

For each outer sweep prints the sum over outer steps of the max (over the
step's pairs) and of the mean inner-sweep count, and the sweep's wall time.
The max/mean ratio is the load imbalance a step-synchronous schedule pays
for the latency-bound inner solves."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1909_00101_b200 as hz  # noqa: E402
from paper_1909_00101_b200 import solver as S  # noqa: E402
from paper_1909_00101_b200.core import MatrixPlanePair, ProblemPair, border_pair  # noqa: E402
from oracle import oracle as O  # noqa: E402

name = sys.argv[1]
w = int(sys.argv[2]) if len(sys.argv) > 2 else 16
F, G, kw, extra = O.ns_inputs(name)
cfg = hz.SolverConfig(**dict(kw, block_width=w))
p = ProblemPair(MatrixPlanePair.from_dense(F), MatrixPlanePair.from_dense(G))
p = border_pair(p, 2 * w, 2 * w)
planes, n, mF, mG = S.upload_bordered(p.F, p.G, w)
dev = S.DeviceGsvd(planes, cfg)
dev.init()
tot_max = tot_mean = 0
pos_sum = None
arg_hist = None
t_all = 0.0
for sw in range(cfg.max_outer_sweeps):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    t, b = dev.sweep()
    dt = time.perf_counter() - t0
    t_all += dt
    c = dev.step_counters()  # (osteps, npairs, 4)
    isw = c[:, :, 3].astype(np.int64)
    smax = int(isw.max(axis=1).sum())
    pos_sum = isw.sum(axis=0) if pos_sum is None else pos_sum + isw.sum(axis=0)
    am = np.bincount(isw.argmax(axis=1), minlength=isw.shape[1])
    arg_hist = am if arg_hist is None else arg_hist + am
    smean = float(isw.mean(axis=1).sum())
    tot_max += smax
    tot_mean += smean
    print("sweep %2d: %6.1f ms  inner sweeps per step: sum(max) %5d  sum(mean) %8.1f  ratio %.2f  "
          "max %d  big %d" % (sw + 1, dt * 1e3, smax, smean, smax / max(smean, 1e-9), isw.max(), b), flush=True)
    if b == 0:
        break
print("total %.3f s; sum(max) %d sum(mean) %.1f ratio %.3f" % (t_all, tot_max, tot_mean, tot_max / tot_mean))
np.set_printoptions(linewidth=160)
print("mean inner sweeps per circle position (over steps and sweeps):")
print(np.round(pos_sum / pos_sum.mean(), 2))
print("how often each position holds the step's max:")
print(arg_hist)
