"""Inner-sweep statistics per outer sweep (max / mean over the pairs of a step)."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1909_00101_b200 as hz
import bench
n = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
kind = sys.argv[2] if len(sys.argv) > 2 else "gauss"
class A: pass
a = A(); a.n = n; a.kind = kind; a.seed = 7; a.w = 16
F0, G0, _ = bench.gen_pair(a, torch, torch.device("cuda"))
dev = hz.DeviceGsvd({"Fr": F0, "Gr": G0, "Fi": None, "Gi": None}, hz.SolverConfig(block_width=16))
dev.set_timing(True)
dev.init()
for sw in range(40):
    dev.kernel_times(reset=True)
    t, b = dev.sweep()
    kt = dev.kernel_times()
    c = dev.step_counters()
    isw = c[:, :, 3]
    stepmax = isw.max(axis=1)
    print(f"sweep {sw}: total {t} big {b} inner sweeps mean {isw.mean():.2f} max {isw.max()} "
          f"mean-of-step-max {stepmax.mean():.2f}  inner {kt['inner'][0]/kt['inner'][1]*1e3:.0f}us/launch "
          f"-> {kt['inner'][0]/kt['inner'][1]*1e3/(stepmax.mean()*(2*16-1)):.2f}us per inner step", flush=True)
    if b == 0:
        break
