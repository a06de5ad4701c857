"""Where the time of one end-to-end solve() goes (the bench's e2e call:
pinned numpy inputs, max_outer_sweeps=2): python tools/e2e_breakdown.py [n] [w]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import bench
import paper_1909_00101_b200 as hz
from paper_1909_00101_b200 import solver as S

n = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
w = int(sys.argv[2]) if len(sys.argv) > 2 else 32


class A:
    pass


a = A()
a.n, a.kind, a.seed, a.w = n, "gauss", 7, w
F0, G0, _ = bench.gen_pair(a, torch, torch.device("cuda"))
Fh = torch.empty(F0.shape, dtype=torch.float64, pin_memory=True)
Gh = torch.empty(G0.shape, dtype=torch.float64, pin_memory=True)
Fh.copy_(F0)
Gh.copy_(G0)
Fnp, Gnp = Fh.numpy().T, Gh.numpy().T
cfg = hz.SolverConfig(block_width=w, max_outer_sweeps=2)
hz.solve(Fnp, Gnp, cfg)
for rep in range(2):
    T = {}
    torch.cuda.synchronize()
    t = time.perf_counter()
    F = hz.MatrixPlanePair.from_dense(Fnp)
    G = hz.MatrixPlanePair.from_dense(Gnp)
    p = hz.ProblemPair(F, G)
    T["from_dense+ProblemPair"] = time.perf_counter() - t
    t = time.perf_counter()
    dev = S._cached_solver(p, cfg)
    torch.cuda.synchronize()
    T["upload"] = time.perf_counter() - t
    t = time.perf_counter()
    dev.init()
    torch.cuda.synchronize()
    T["init(prescale)"] = time.perf_counter() - t
    t = time.perf_counter()
    for _ in range(2):
        dev.sweep()
    torch.cuda.synchronize()
    T["2 sweeps"] = time.perf_counter() - t
    t = time.perf_counter()
    out = dev.finalize(p.n, p.F.rows, p.G.rows, sort=True)
    torch.cuda.synchronize()
    T["finalize"] = time.perf_counter() - t
    t = time.perf_counter()
    r = S._result_from_device(dev, out, False)
    T["to host"] = time.perf_counter() - t
    t = time.perf_counter()
    r2 = hz.solve(Fnp, Gnp, cfg)
    T["solve() total"] = time.perf_counter() - t
    print("  ".join(f"{k} {v * 1e3:.0f} ms" for k, v in T.items()), flush=True)
    del r, r2
