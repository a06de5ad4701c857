"""Config 3 (complex F 3072x2048, G 2048^2) sweep-1 steps for ncu."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1909_00101_b200 as hz
n, mF = 2048, 3072
steps = int(sys.argv[1]) if len(sys.argv) > 1 else 127
g = torch.Generator(device="cuda"); g.manual_seed(5)
kw = dict(dtype=torch.float64, device="cuda")
pl = {"Fr": torch.randn((n, mF), generator=g, **kw), "Fi": torch.randn((n, mF), generator=g, **kw),
      "Gr": torch.randn((n, n), generator=g, **kw), "Gi": torch.randn((n, n), generator=g, **kw)}
dev = hz.DeviceGsvd(pl, hz.SolverConfig(block_width=16))
dev.init()
dev.run_steps(0, steps)
torch.cuda.synchronize()
print("done")
