"""Device preprocess_tall time on a config-3-shaped pair (complex F m x n,
G n x n): python tools/tall_time.py [m] [n]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_1909_00101_b200 as hz

m = int(sys.argv[1]) if len(sys.argv) > 1 else 3072
n = int(sys.argv[2]) if len(sys.argv) > 2 else 2048
rng = np.random.default_rng(3)
F = rng.standard_normal((m, n)) + 1j * rng.standard_normal((m, n))
G = rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n))
Fm, Gm = hz.MatrixPlanePair.from_dense(np.asfortranarray(F)), hz.MatrixPlanePair.from_dense(np.asfortranarray(G))
hz.preprocess_tall(Fm, Gm)  # warm
torch.cuda.synchronize()
t0 = time.perf_counter()
hz.preprocess_tall(Fm, Gm)
torch.cuda.synchronize()
print(f"preprocess_tall complex F {m}x{n}, G {n}x{n}: {time.perf_counter() - t0:.3f} s (host in/out included)", flush=True)

# device-only: the column-pivoted R factor of F on resident planes (median of 3)
from paper_1909_00101_b200 import ops
ts = []
for _ in range(3):
    Fr = torch.from_numpy(np.ascontiguousarray(F.real.T)).cuda()
    Fi = torch.from_numpy(np.ascontiguousarray(F.imag.T)).cuda()
    jp = torch.arange(n, dtype=torch.int64, device="cuda")
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    ops.qr_rfactor(Fr, Fi, True, jp, n * 2.0 ** -52)
    e1.record()
    torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1) / 1e3)
print(f"qr_rfactor complex {m}x{n} with pivoting, device only: {sorted(ts)[1]:.3f} s (median of 3)", flush=True)
