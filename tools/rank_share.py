"""Per-rank sweep time of the block-partitioned schedule, measured on one GPU.

One rank r of an R-rank job runs its slot range of every step (Grammian,
inner, postmultiply of its pairs) on the GPU alone; the block exchange is
replaced by event bookkeeping only (blocks are not copied: the columns that
would arrive keep stale, valid values, so the per-step work has the same
shape).  The slowest rank's sweep time bounds the R-GPU sweep from below
(NCCL moves at most 2 blocks per rank and step, overlapped with the
interior groups), so F_sweep / max_r(t_r) estimates strong scaling on R
B200s where only one GPU is available.

usage: python tools/rank_share.py N R[,R...] [wave|serial|timed|vtimed|graph] [sweeps] [w]

graph: the library data plane -- the rank's sweep as ONE captured CUDA graph
(hzg_dist_sweep) on a 1-rank NCCL communicator with its block moves removed
(they are the only part that needs the other GPUs); host issue is one graph
launch per sweep.
"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import bench
import paper_1909_00101_b200 as hz
from paper_1909_00101_b200 import dist as D


class NullTransport:
    def exchange(self, moves):
        pass

    def exchange_on(self, moves, stream, zstream=None):
        pass


def main():
    n = int(sys.argv[1])
    Rs = [int(x) for x in sys.argv[2].split(",")]
    mode = sys.argv[3] if len(sys.argv) > 3 else "wave"
    nsw = int(sys.argv[4]) if len(sys.argv) > 4 else 2
    w = int(sys.argv[5]) if len(sys.argv) > 5 else 16

    class A:
        pass
    a = A()
    a.n, a.kind, a.seed, a.w = n, "gauss", 7, w
    F0, G0, _ = bench.gen_pair(a, torch, torch.device("cuda"))
    Fsw = bench.flops_per_sweep(n, n, n, w)
    cfg = hz.SolverConfig(block_width=w, max_outer_sweeps=100)
    for R in Rs:
        if mode == "vtimed":   # R virtual ranks with real block exchange, per-rank kernel times
            job = D.PartitionedGsvd({"Fr": F0.clone(), "Gr": G0.clone(), "Fi": None, "Gi": None}, cfg, R,
                                    wavefront=False)
            job.init()
            job.sweep()
            for d in job.devs:
                d.set_timing(True)
                d.kernel_times(reset=True)
            job.sweep()
            for r, d in enumerate(job.devs):
                kt = d.kernel_times()
                print(f"n={n} R={R} rank {r} (real exchange): " + "  ".join(
                    f"{k} {v[0] / max(1, v[1]) * 1e3:.1f} us" for k, v in kt.items()), flush=True)
            job.close()
            del job
            continue
        sched = D.BlockSchedule(n // w, R)
        worst = 0.0
        if mode == "graph":
            for r in sorted({0, R // 2, R - 1}):
                Fw, Gw = F0.clone(), G0.clone()
                dev = hz.DeviceGsvd({"Fr": Fw, "Gr": Gw, "Fi": None, "Gi": None}, cfg, epsn=D.epsn_of(cfg, n),
                                    schedule=sched.colpairs(r, w))
                dev.comm_attach(1, 0, D.unique_id())
                dev.comm_set_moves([[] for _ in range(sched.steps)])
                dev.init()
                dev.dist_sweep()  # warm-up (graph capture)
                times, hs = [], []
                for _ in range(nsw):
                    torch.cuda.synchronize()
                    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    e0.record()
                    h0 = time.perf_counter()
                    dev.lib.hzg_dist_sweep_launch(dev.ctx)
                    hs.append(time.perf_counter() - h0)   # host time to issue the whole sweep
                    dev.dist_sweep_wait()
                    e1.record()
                    torch.cuda.synchronize()
                    times.append(e0.elapsed_time(e1) / 1e3)
                t = sorted(times)[len(times) // 2]
                worst = max(worst, t)
                lo, hi = sched.ranges[r]
                print(f"n={n} w={w} R={R} rank {r}: {hi - lo} pairs/step, graph: sweep {t * 1e3:.1f} ms "
                      f"(host issue {min(hs) * 1e3:.3f} ms = {100 * min(hs) / t:.3f} % of the sweep)", flush=True)
                dev.close()
                del dev, Fw, Gw
            print(f"n={n} w={w} R={R} graph: slowest rank {worst * 1e3:.1f} ms/sweep -> "
                  f"{Fsw / worst / 1e12:.2f} TF/s job, {Fsw / worst / 1e12 / R:.2f} TF/s per GPU", flush=True)
            continue
        for r in sorted({0, R // 2, R - 1}):
            Fw, Gw = F0.clone(), G0.clone()
            dev = hz.DeviceGsvd({"Fr": Fw, "Gr": Gw, "Fi": None, "Gi": None}, cfg, epsn=D.epsn_of(cfg, n),
                                schedule=sched.colpairs(r, w))
            lo, hi = sched.ranges[r]
            wave = D.Wavefront([dev], [hi - lo], split_z=D.split_z_default()) if mode == "wave" else None
            dev.init()
            D.sweep_ranks([dev], sched, NullTransport(), None, wave)   # warm-up sweep
            if mode == "timed":   # isolated per-kernel times (serialised, synchronous)
                dev.set_timing(True)
                dev.kernel_times(reset=True)
                D.sweep_ranks([dev], sched, NullTransport(), None, None)
                kt = dev.kernel_times()
                dev.set_timing(False)
                print(f"n={n} R={R} rank {r}: " + "  ".join(
                    f"{k} {v[0] / max(1, v[1]) * 1e3:.1f} us" for k, v in kt.items()), flush=True)
            times, hs = [], []
            for _ in range(nsw):
                torch.cuda.synchronize()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                h0 = time.perf_counter()
                if wave is not None:
                    D._sweep_wavefront([dev], sched, NullTransport(), wave)
                else:
                    for k in range(sched.steps):
                        dev.run_steps(k, 1)
                hs.append(time.perf_counter() - h0)   # host time to issue the sweep's steps
                _, big = dev.collect()
                if big:
                    dev.rescale_z()
                e1.record()
                torch.cuda.synchronize()
                times.append(e0.elapsed_time(e1) / 1e3)
            t = sorted(times)[len(times) // 2]
            worst = max(worst, t)
            g = wave.groups[0] if wave else 1
            print(f"n={n} R={R} rank {r}: {hi - lo} pairs/step, {g} groups, {mode}: sweep {t * 1e3:.1f} ms "
                  f"(host issue {min(hs) * 1e3:.1f} ms)", flush=True)
            dev.close()
            del dev, Fw, Gw
        print(f"n={n} R={R} {mode}: slowest rank {worst * 1e3:.1f} ms/sweep -> "
              f"{Fsw / worst / 1e12:.2f} TF/s job, {Fsw / worst / 1e12 / R:.2f} TF/s per GPU", flush=True)


if __name__ == "__main__":
    main()
