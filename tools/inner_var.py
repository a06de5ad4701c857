"""Distribution of inner sweeps per pair within outer steps (why a step
costs the max over its pairs): runs a few outer sweeps of the config-4
pair and prints, per sweep, mean / max of the per-pair inner sweep counts."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1909_00101_b200 as hz
import bench
n = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
kind = sys.argv[2] if len(sys.argv) > 2 else "cond"
class A: pass
a = A(); a.n = n; a.kind = kind; a.seed = 7; a.w = 16
F0, G0, _ = bench.gen_pair(a, torch, torch.device("cuda"))
dev = hz.DeviceGsvd({"Fr": F0, "Gr": G0, "Fi": None, "Gi": None}, hz.SolverConfig(block_width=16, max_outer_sweeps=100))
dev.init()
for sw in range(100):
    t, b = dev.sweep()
    c = dev.step_counters()  # (osteps, npairs, 4)
    s = c[:, :, 3].astype(float)
    g = s.reshape(s.shape[0], 8, -1)
    print("sweep %2d big %8d  inner sweeps/pair mean %.2f  step-max mean %.2f  group-max mean %.2f  total-max %d" %
          (sw + 1, b, s.mean(), s.max(axis=1).mean(), g.max(axis=2).mean(), s.max()), flush=True)
    if sw + 1 in (1, 20, 40, 60):
        np.save(os.path.join("gpurun_out", "counts_sweep%d.npy" % (sw + 1)), c)
    if b == 0:
        break

