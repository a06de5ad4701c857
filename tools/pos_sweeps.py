"""Inner sweeps per circle position (single-GPU schedule): mean over the
steps of each outer sweep, for the first and last positions and the rest."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import bench
import paper_1909_00101_b200 as hz

n = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
nsw = int(sys.argv[2]) if len(sys.argv) > 2 else 4


class A:
    pass


a = A()
a.n, a.kind, a.seed, a.w = n, "gauss", 7, 16
F0, G0, _ = bench.gen_pair(a, torch, torch.device("cuda"))
dev = hz.DeviceGsvd({"Fr": F0, "Gr": G0, "Fi": None, "Gi": None}, hz.SolverConfig(block_width=16))
dev.init()
np.set_printoptions(precision=2, linewidth=200)
for s in range(nsw):
    dev.sweep()
    c = dev.step_counters()            # (steps, npairs, 4): total, big, status, inner sweeps
    isw = c[:, :, 3].astype(np.float64)
    m = isw.mean(axis=0)
    print(f"sweep {s + 1}: mean inner sweeps {isw.mean():.2f}; first positions {m[:4]}; last {m[-4:]}; "
          f"interior max {m[4:-4].max():.2f}; per-step max over pairs mean {isw.max(axis=1).mean():.2f}", flush=True)
