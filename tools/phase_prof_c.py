"""Per-phase cycle counts of the complex inner kernel (CTA 0, warp 0), config 3 shapes."""
import sys, os, ctypes
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1909_00101_b200 as hz
n, mF = 2048, 3072
g = torch.Generator(device="cuda"); g.manual_seed(5)
kw = dict(dtype=torch.float64, device="cuda")
pl = {"Fr": torch.randn((n, mF), generator=g, **kw), "Fi": torch.randn((n, mF), generator=g, **kw),
      "Gr": torch.randn((n, n), generator=g, **kw), "Gi": torch.randn((n, n), generator=g, **kw)}
dev = hz.DeviceGsvd(pl, hz.SolverConfig(block_width=16))
dev.init()
out = np.zeros(4, dtype=np.int64)
dev.lib.hzg_debug_phases(dev.ctx, 1, None)
dev.run_steps(0, 20)
torch.cuda.synchronize()
dev.lib.hzg_debug_phases(dev.ctx, 0, out.ctypes.data_as(ctypes.c_void_p))
print("complex: steps", out[3], "cycles per inner step: A %.0f  B %.0f  C %.0f  total %.0f" % tuple(list(out[:3] / out[3]) + [out[:3].sum() / out[3]]))
print("raw phase[0] (fallbacks x 1e9 when built with HZG_EXP_FALLBACK):", int(out[0]))
