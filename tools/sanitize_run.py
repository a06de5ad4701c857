"""Small solves that exercise every step kernel for compute-sanitizer
(racecheck / synccheck / memcheck): DMMA mode real and complex (k_gram_ws,
k_inner, k_post_ws, deferred Z on low-priority streams, 2 wavefront
groups), exact mode, the stripe scheme and the fused postgram path."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ.setdefault("HZG_GROUPS", "2")
import paper_1909_00101_b200 as hz  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 256
rng = np.random.default_rng(1)
F = rng.standard_normal((n, n))
G = rng.standard_normal((n, n))
cfg = hz.SolverConfig(block_width=16, max_outer_sweeps=2)
r = hz.solve(F, G, cfg)
print("dmma real", r.sweeps)
Fc = F + 1j * rng.standard_normal((n, n))
Gc = G + 1j * rng.standard_normal((n, n))
r = hz.solve(Fc[:, : n // 2], Gc[:, : n // 2], cfg)
print("dmma complex", r.sweeps)
r = hz.solve(F[:, :128], G[:, :128], hz.SolverConfig(block_width=16, max_outer_sweeps=2, exact=True))
print("exact", r.sweeps)
r = hz.solve(F[:, :128], G[:, :128], hz.SolverConfig(block_width=8, max_outer_sweeps=2), workers=2)
print("stripes", r.sweeps)
os.environ["HZG_FUSED"] = "1"
r = hz.solve(F, G, hz.SolverConfig(block_width=16, max_outer_sweeps=2, split_rows=256))
print("fused", r.sweeps)
os.environ["HZG_FUSED"] = "0"
r = hz.solve(F, G, hz.SolverConfig(block_width=32, max_outer_sweeps=2))
print("dmma 2w=64 (m16n8k8 postmultiply)", r.sweeps)
p = hz.ProblemPair(hz.MatrixPlanePair.from_dense(F[:, :64]), hz.MatrixPlanePair.from_dense(G[:, :64]))
r = hz.solve(F[:, :64], G[:, :64], hz.SolverConfig(block_width=16))
print("accuracy report", hz.accuracy_report(p, r))
from paper_1909_00101_b200 import dist as D  # noqa: E402
planes, nb, mF, mG = hz.upload_bordered(hz.MatrixPlanePair.from_dense(F), hz.MatrixPlanePair.from_dense(G), 16)
dev = hz.DeviceGsvd(planes, hz.SolverConfig(block_width=16))
dev.comm_attach(1, 0, D.unique_id())
dev.comm_set_moves([[(k % (nb // 16), 0, 0)] for k in range(nb // 16 - 1)])
dev.init()
print("nccl rank sweep", dev.dist_sweep())
dev.close()
print("sanitize run done")
