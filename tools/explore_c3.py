"""Config 3: complex F 3072x2048, G 2048x2048 (iid Gaussian re/im), w=16, full solve."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1909_00101_b200 as hz
import bench
mF, mG, n, w = 3072, 2048, 2048, int(sys.argv[1]) if len(sys.argv) > 1 else 16
g = torch.Generator(device="cuda"); g.manual_seed(3)
kw = dict(dtype=torch.float64, device="cuda")
planes = {"Fr": torch.randn((n, mF), generator=g, **kw), "Fi": torch.randn((n, mF), generator=g, **kw),
          "Gr": torch.randn((n, mG), generator=g, **kw), "Gi": torch.randn((n, mG), generator=g, **kw)}
orig = {k: v.clone() for k, v in planes.items()}
dev = hz.DeviceGsvd(planes, hz.SolverConfig(block_width=w))
dev.set_timing(True)
for rep in range(2):
    for k in planes: planes[k].copy_(orig[k])
    dev.kernel_times(reset=True)
    torch.cuda.synchronize(); t0 = time.perf_counter()
    dev.run(); out = dev.finalize()
    torch.cuda.synchronize(); dt = time.perf_counter() - t0
kt = dev.kernel_times()
fl = dev.sweeps * bench.flops_per_sweep(n, mF, mG, w, cplx=True)
print(f"config3 complex {mF}x{n}/{mG}x{n} w={w}: sweeps {dev.sweeps} conv {dev.converged} time {dt:.3f}s {fl/dt/1e12:.2f} TF/s  "
      + "  ".join(f"{k}: {v[0]:.1f}ms/{v[1]} ({v[0]/max(1,v[1])*1e3:.1f}us)" for k, v in kt.items()))
F = torch.complex(orig["Fr"], orig["Fi"]).T; G = torch.complex(orig["Gr"], orig["Gi"]).T
U = torch.complex(out["Ur"], out["Ui"]).T; V = torch.complex(out["Vr"], out["Vi"]).T; Z = torch.complex(out["Zr"], out["Zi"]).T
resF = torch.linalg.norm(F @ Z - U * out["sigmaF"][None, :]) / torch.linalg.norm(F)
resG = torch.linalg.norm(G @ Z - V * out["sigmaG"][None, :]) / torch.linalg.norm(G)
eye = torch.eye(n, dtype=torch.complex128, device="cuda")
print("resF %.2e resG %.2e orthU %.2e orthV %.2e" % (resF, resG, torch.linalg.norm(U.conj().T @ U - eye), torch.linalg.norm(V.conj().T @ V - eye)))
