out=gpurun_out
tag=${1:-x}
python tools/phase_prof_c.py > $out/${tag}_phase.txt 2>&1
python - > $out/${tag}_c3.txt 2>&1 <<'PY'
import sys, os, time
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import paper_1909_00101_b200 as hz
from oracle import oracle as O
n, mF = 2048, 3072
g = O.gaussian_stream
F = (g(41, mF * n) + 1j * g(42, mF * n)).reshape((mF, n), order="F")
G = (g(43, n * n) + 1j * g(44, n * n)).reshape((n, n), order="F")
cfg = hz.SolverConfig(block_width=16)
r = hz.solve(F, G, cfg)
torch.cuda.synchronize(); t0 = time.perf_counter()
r = hz.solve(F, G, cfg)
torch.cuda.synchronize(); dt = time.perf_counter() - t0
nb = n // 16; P = nb * (nb - 1) // 2
fl = r.sweeps * P * 4 * (12 * 256 * (mF + n) + 8 * 256 * n)
print("config 3 e2e %.2f s, %d sweeps, %.2f TFLOP/s" % (dt, r.sweeps, fl / dt / 1e12))
PY
