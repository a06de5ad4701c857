"""Per-phase cycle counts of the inner kernel (CTA 0, warp 0) over a few outer
steps: python tools/phase_prof.py [n] [gauss|cond|complex] [approx 0/1] [steps]."""
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_1909_00101_b200 as hz  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
kind = sys.argv[2] if len(sys.argv) > 2 else "gauss"
approx = bool(int(sys.argv[3])) if len(sys.argv) > 3 else True
steps = int(sys.argv[4]) if len(sys.argv) > 4 else 20
w = int(sys.argv[5]) if len(sys.argv) > 5 else 16


class A:
    pass


a = A()
a.n, a.kind, a.seed, a.w = n, ("cond" if kind == "cond" else "gauss"), 7, w
F0, G0, _ = bench.gen_pair(a, torch, torch.device("cuda"))
planes = {"Fr": F0, "Gr": G0, "Fi": None, "Gi": None}
if kind == "complex":
    planes["Fi"] = torch.flip(F0, [1]).contiguous()
    planes["Gi"] = torch.flip(G0, [1]).contiguous()
dev = hz.DeviceGsvd(planes, hz.SolverConfig(block_width=w, approx_2x2=approx))
dev.init()
out = np.zeros(4, dtype=np.int64)
dev.lib.hzg_debug_phases(dev.ctx, 1, None)
dev.run_steps(0, min(steps, n // w - 1))
torch.cuda.synchronize()
dev.lib.hzg_debug_phases(dev.ctx, 0, out.ctypes.data_as(ctypes.c_void_p))
fb = int(out[0]) // 1000000000
out[0] -= fb * 1000000000
print("w %d n %d %s approx=%d: steps %d, cycles per inner step: A %.0f  B %.0f  C %.0f  total %.0f; approx fallbacks %d"
      % tuple([w, n, kind, approx, out[3]] + list(out[:3] / out[3]) + [out[:3].sum() / out[3], fb]))
