"""Device sweep time of the bench workload (no e2e / roofline passes), for
quick A/B of HZG_* knobs and configuration fields:
python tools/sweep_time.py [n] [warmup] [timed] [w] [split_rows]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import bench
import paper_1909_00101_b200 as hz

n = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
W = int(sys.argv[2]) if len(sys.argv) > 2 else 3
K = int(sys.argv[3]) if len(sys.argv) > 3 else 3
w = int(sys.argv[4]) if len(sys.argv) > 4 else 16
split = int(sys.argv[5]) if len(sys.argv) > 5 else 0


class A:
    pass


a = A()
a.n, a.kind, a.seed, a.w = n, "gauss", 7, w
F0, G0, _ = bench.gen_pair(a, torch, torch.device("cuda"))
dev = hz.DeviceGsvd({"Fr": F0, "Gr": G0, "Fi": None, "Gi": None}, hz.SolverConfig(block_width=w, max_outer_sweeps=100, split_rows=split))
dev.init()
import time
torch.cuda.synchronize()
t0 = time.perf_counter()
dev.sweep()                       # includes the sweep graph capture + instantiation
first = time.perf_counter() - t0
for _ in range(W - 1):
    dev.sweep()
clk = bench.ClockSampler(0)
torch.cuda.synchronize()
clk.start()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(K):
    dev.sweep()
e1.record()
torch.cuda.synchronize()
c = clk.stop()
ms = e0.elapsed_time(e1) / K
tf = bench.flops_per_sweep(n, n, n, w) / (ms / 1e3) / 1e12
knobs = " ".join(f"{k}={v}" for k, v in sorted(os.environ.items()) if k.startswith("HZG_"))
print(f"n={n} w={w} split_rows={split} {knobs or 'default'}: first sweep {first * 1e3:.0f} ms; {ms:.1f} ms/sweep {tf:.2f} TF/s sm {c['sm_mhz']} MHz -> {tf / c['sm_mhz'] * 1e3:.2f} TF/s/GHz",
      flush=True)
