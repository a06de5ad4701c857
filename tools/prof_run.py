"""Small driver for ncu captures: a few outer steps of sweep 1 (no graph)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1909_00101_b200 as hz
import bench
n = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 4
kind = sys.argv[3] if len(sys.argv) > 3 else "gauss"
class A: pass
a = A(); a.n = n; a.kind = kind; a.seed = 7; a.w = int(sys.argv[4]) if len(sys.argv) > 4 else 16
F0, G0, _ = bench.gen_pair(a, torch, torch.device("cuda"))
dev = hz.DeviceGsvd({"Fr": F0, "Gr": G0, "Fi": None, "Gi": None}, hz.SolverConfig(block_width=a.w))
dev.init()
dev.run_steps(0, steps)
torch.cuda.synchronize()
print("done")
