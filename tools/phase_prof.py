"""Per-phase cycle counts of the inner kernel (CTA 0, warp 0) over a few outer steps."""
import sys, os, ctypes
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1909_00101_b200 as hz
import bench
n = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
class A: pass
a = A(); a.n = n; a.kind = "gauss"; a.seed = 7; a.w = 16
F0, G0, _ = bench.gen_pair(a, torch, torch.device("cuda"))
dev = hz.DeviceGsvd({"Fr": F0, "Gr": G0, "Fi": None, "Gi": None}, hz.SolverConfig(block_width=16))
dev.init()
out = np.zeros(4, dtype=np.int64)
dev.lib.hzg_debug_phases(dev.ctx, 1, None)
dev.run_steps(0, 20)
torch.cuda.synchronize()
dev.lib.hzg_debug_phases(dev.ctx, 0, out.ctypes.data_as(ctypes.c_void_p))
print("steps", out[3], "cycles per inner step: A %.0f  B %.0f  C %.0f  total %.0f" % tuple(list(out[:3] / out[3]) + [out[:3].sum() / out[3]]))
print("raw phase[0] (fallbacks x 1e9 when built with HZG_EXP_FALLBACK):", int(out[0]))
