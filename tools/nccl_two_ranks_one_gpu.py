"""Can two processes form an NCCL communicator on the same GPU?  If yes,
run the block-partitioned solve with the library data plane (hzg_dist_sweep)
on 2 ranks sharing cuda:0 and compare with the single-rank solve bitwise.
torch.distributed (gloo) is used only to broadcast the ncclUniqueId."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def worker(rank, world, port, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    import paper_1909_00101_b200 as hz
    from paper_1909_00101_b200 import dist as D
    n = 512
    rng = np.random.default_rng(5)
    F = rng.standard_normal((n, n))
    G = rng.standard_normal((n, n))
    cfg = hz.SolverConfig(block_width=16)
    p = hz.ProblemPair(hz.MatrixPlanePair.from_dense(F), hz.MatrixPlanePair.from_dense(G))
    planes, nb, mF, mG = hz.upload_bordered(p.F, p.G, 16)
    sched = D.BlockSchedule(nb // 16, world)
    dev = hz.DeviceGsvd(planes, cfg, epsn=D.epsn_of(cfg, nb), schedule=sched.colpairs(rank, 16))
    uid = [D.unique_id() if rank == 0 else None]
    dist.broadcast_object_list(uid, src=0)
    try:
        dev.comm_attach(world, rank, uid[0])
    except Exception as exc:
        torch.save({"error": repr(exc)}, "%s.%d" % (out, rank))
        return
    dev.comm_set_moves([sched.moves(k) for k in range(sched.steps)])
    dev.init()
    sweeps = total = big = 0
    for _ in range(cfg.max_outer_sweeps):
        t, b = dev.dist_sweep()
        sweeps += 1
        total += t
        big += b
        if b == 0:
            break
    dev.comm_exchange(D.gather_blocks(sched))
    res = {"sweeps": sweeps, "total": total, "big": big}
    if rank == 0:
        dev.sweeps, dev.total, dev.big, dev.converged = sweeps, total, big, big == 0
        outp = dev.finalize(n, n, n)
        res["sigma"] = outp["sigma"].cpu().numpy()
        res["Z"] = outp["Zr"].cpu().numpy()
        ref = hz.solve(F, G, cfg)
        res["ref_sigma"] = ref.sigma
        res["ref_Z"] = np.ascontiguousarray(ref.Z.re.T)
        res["ref_counts"] = (ref.sweeps, ref.total_transforms, ref.big_transforms)
    torch.save(res, "%s.%d" % (out, rank))
    dev.close()
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    import socket
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    out = "/tmp/nccl2"
    mp.spawn(worker, args=(2, port, out), nprocs=2, join=True)
    r0 = torch.load(out + ".0", weights_only=False)
    if "error" in r0:
        print("NCCL 2 ranks on one GPU: not possible here:", r0["error"])
        sys.exit(0)
    same = (np.array_equal(r0["sigma"], r0["ref_sigma"]) and np.array_equal(r0["Z"], r0["ref_Z"])
            and (r0["sweeps"], r0["total"], r0["big"]) == tuple(r0["ref_counts"]))
    print("2 NCCL ranks on one GPU, library data plane: sweeps %d, bitwise equal to 1 rank: %s"
          % (r0["sweeps"], same))
