"""Config 3 (complex, tall F) on the GPU: half scale (F 1536x1024, G 1024^2)
against the oracle outputs made in the build container
(scratch/c3_*_1024.npy), then the full config 3 (F 3072x2048, G 2048^2)
timed with its self-consistency metrics."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_1909_00101_b200 as hz
from oracle import oracle as O

F = np.load("scratch/c3_F_1024.npy"); G = np.load("scratch/c3_G_1024.npy"); s_ref = np.load("scratch/c3_sigma_1024.npy")
for exact in (False, True):
    r = hz.solve(F, G, hz.SolverConfig(block_width=16, exact=exact))
    print("half-scale config 3 exact=%s: sweeps %d total %d big %d, max rel sigma vs oracle %.2e, bitwise %s" % (
        exact, r.sweeps, r.total_transforms, r.big_transforms, np.max(np.abs(r.sigma - s_ref) / s_ref),
        np.array_equal(r.sigma, s_ref)), flush=True)

n, mF = 2048, 3072
g = O.gaussian_stream
F = (g(41, mF * n) + 1j * g(42, mF * n)).reshape((mF, n), order="F")
G = (g(43, n * n) + 1j * g(44, n * n)).reshape((n, n), order="F")
cfg = hz.SolverConfig(block_width=16)
r = hz.solve(F, G, cfg)  # warm
torch.cuda.synchronize()
t0 = time.perf_counter()
r = hz.solve(F, G, cfg)
torch.cuda.synchronize()
dt = time.perf_counter() - t0
nb = n // 16
P = nb * (nb - 1) // 2
fl = r.sweeps * P * 4 * (12 * 256 * (mF + n) + 8 * 256 * n)
U, V, Z = r.U.to_dense(), r.V.to_dense(), r.Z.to_dense()
resF = np.linalg.norm(F @ Z - U * r.sigmaF[None, :]) / np.linalg.norm(F)
resG = np.linalg.norm(G @ Z - V * r.sigmaG[None, :]) / np.linalg.norm(G)
oU = np.linalg.norm(U.conj().T @ U - np.eye(n)); oV = np.linalg.norm(V.conj().T @ V - np.eye(n))
print("config 3 (complex F 3072x2048, G 2048^2, w=16): e2e solve() %.2f s, %d sweeps, %.2f TFLOP/s; "
      "resF %.2e resG %.2e orthU %.2e orthV %.2e" % (dt, r.sweeps, fl / dt / 1e12, resF, resG, oU, oV), flush=True)
