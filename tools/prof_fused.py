"""A few fused sweeps-worth of steps for ncu: one hzg_sweep at n (real Gaussian)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1909_00101_b200 as hz
n = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
g = torch.Generator(device="cuda"); g.manual_seed(3)
F = torch.randn((n, n), generator=g, dtype=torch.float64, device="cuda")
G = torch.randn((n, n), generator=g, dtype=torch.float64, device="cuda")
dev = hz.DeviceGsvd({"Fr": F, "Gr": G, "Fi": None, "Gi": None}, hz.SolverConfig(block_width=16))
dev.init()
dev.sweep()
torch.cuda.synchronize()
print("done")
