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
