"""Quick per-size timing of the device solve with per-kernel event times."""
import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1909_00101_b200 as hz
import bench

sizes = [int(x) for x in sys.argv[1].split(",")] if len(sys.argv) > 1 else [1024, 2048, 4096]
kind = sys.argv[2] if len(sys.argv) > 2 else "gauss"
w = int(sys.argv[3]) if len(sys.argv) > 3 else 16
blocking = sys.argv[4] if len(sys.argv) > 4 else "fb"
cap = int(sys.argv[5]) if len(sys.argv) > 5 else 30
for n in sizes:
    class A: pass
    a = A(); a.n = n; a.kind = kind; a.seed = 7; a.w = w
    F0, G0, truth = bench.gen_pair(a, torch, torch.device("cuda"))
    Fw, Gw = F0.clone(), G0.clone()
    dev = hz.DeviceGsvd({"Fr": Fw, "Gr": Gw, "Fi": None, "Gi": None}, hz.SolverConfig(block_width=w, blocking=blocking, max_outer_sweeps=cap))
    dev.set_timing(True)
    for rep in range(2):
        Fw.copy_(F0); Gw.copy_(G0)
        dev.kernel_times(reset=True)
        torch.cuda.synchronize(); t0 = time.perf_counter()
        dev.run()
        out = dev.finalize()
        torch.cuda.synchronize(); dt = time.perf_counter() - t0
    kt = dev.kernel_times()
    fl = dev.sweeps * bench.flops_per_sweep(n, n, n, w)
    print(f"n={n} {kind} w={w} {blocking}: sweeps {dev.sweeps} conv {dev.converged} time {dt:.3f}s  {fl/dt/1e12:.2f} TF/s  "
          + "  ".join(f"{k}: {v[0]:.1f}ms/{v[1]} ({v[0]/max(1,v[1])*1e3:.1f}us)" for k, v in kt.items()), flush=True)
    if truth is not None:
        tr = torch.sort(truth, descending=True).values
        print("   max rel sigma vs generator %.2e" % float(torch.max(torch.abs(out['sigma'] - tr) / tr)))
    del dev
