"""The NCCL data plane inside libhzg (hzg_comm_*, hzg_dist_sweep) on the one
GPU of the test box: a 1-rank communicator runs the captured rank-sweep
graph (steps + grouped ncclSend/ncclRecv + counter all-reduce + gated
rescale), with and without self-addressed block moves, and must reproduce
the single-GPU sweep graph bitwise.  Multi-rank routing is covered by the
gloo tests (tests/test_dist.py, tests/test_gpu_dist.py)."""

import os
import socket

import numpy as np
import pytest

import paper_1909_00101_b200 as hz
from paper_1909_00101_b200 import dist as D
from oracle import oracle as O

pytestmark = pytest.mark.gpu


def _pair(n, seed):
    g = O.gaussian_stream(seed, 2 * n * n)
    return g[: n * n].reshape((n, n), order="F"), g[n * n:].reshape((n, n), order="F")


def _device_solve(F, G, cfg, moves=None):
    """Full solve through hzg_dist_sweep on a 1-rank communicator; moves:
    None (no exchange) or a function k -> [(block, 0, 0), ...]."""
    p = hz.ProblemPair(hz.MatrixPlanePair.from_dense(F), hz.MatrixPlanePair.from_dense(G))
    planes, n, mF, mG = hz.upload_bordered(p.F, p.G, cfg.block_width)
    dev = hz.DeviceGsvd(planes, cfg)
    try:
        dev.comm_attach(1, 0, D.unique_id())
        osteps = n // cfg.block_width - 1
        dev.comm_set_moves([moves(k) if moves else [] for k in range(osteps)])
        dev.init()
        for _ in range(cfg.max_outer_sweeps):
            t, b = dev.dist_sweep()
            dev.sweeps += 1
            dev.total += t
            dev.big += b
            if b == 0:
                dev.converged = True
                break
        out = dev.finalize(p.n, p.F.rows, p.G.rows, sort=True)
        from paper_1909_00101_b200.solver import _result_from_device
        return _result_from_device(dev, out, False)
    finally:
        dev.close()


def _same(a, b):
    assert (a.sweeps, a.total_transforms, a.big_transforms) == (b.sweeps, b.total_transforms, b.big_transforms)
    for x, y in ((a.sigma, b.sigma), (a.U.re, b.U.re), (a.V.re, b.V.re), (a.Z.re, b.Z.re)):
        assert np.array_equal(x, y)


@pytest.mark.parametrize("n", [256, 1024])
def test_one_rank_nccl_sweep_graph_bitwise(n):
    F, G = _pair(n, 300 + n)
    cfg = hz.SolverConfig(block_width=16)
    _same(_device_solve(F, G, cfg), hz.solve(F, G, cfg))


def test_one_rank_nccl_self_exchange_bitwise():
    """Every step sends one block (all planes) to this rank itself inside the
    captured graph: the data must come back unchanged."""
    n = 512
    F, G = _pair(n, 77)
    cfg = hz.SolverConfig(block_width=16)
    nblk = n // 16
    r = _device_solve(F, G, cfg, moves=lambda k: [(k % nblk, 0, 0), ((k + 7) % nblk, 0, 0)])
    _same(r, hz.solve(F, G, cfg))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def test_torch_distributed_nccl_world_one_uses_library_plane():
    """solve_blocks(comm="dist") under an NCCL process group: the library
    data plane attaches (uid broadcast through torch.distributed) and the
    result is bitwise the single-GPU solve."""
    import torch.distributed as dist
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ["MASTER_PORT"] = str(_free_port())
    dist.init_process_group("nccl", rank=0, world_size=1)
    try:
        F, G = _pair(512, 91)
        cfg = hz.SolverConfig(block_width=16)
        p = hz.ProblemPair(hz.MatrixPlanePair.from_dense(F), hz.MatrixPlanePair.from_dense(G))
        planes, n, mF, mG = hz.upload_bordered(p.F, p.G, 16)
        job = D.PartitionedGsvd(planes, cfg, 1, comm="dist")
        assert job.nccl
        job.close()
        r = D.solve_blocks(F, G, cfg, 1, comm="dist")
        _same(r, hz.solve(F, G, cfg))
    finally:
        dist.destroy_process_group()


def test_one_process_driving_devices_bitwise():
    """solve(..., scheme="blocks", devices=[...]): one process, one context
    and ncclCommInitAll communicator per device, every rank's sweep graph
    launched before any is waited for (hzg_dist_sweep_launch / _wait), the
    gather by hzg_comm_exchange_all.  With the box's single GPU: devices=[0],
    bitwise the single-GPU solve."""
    F, G = _pair(512, 123)
    cfg = hz.SolverConfig(block_width=16)
    r = hz.solve(F, G, cfg, workers=1, scheme="blocks", devices=[0])
    _same(r, hz.solve(F, G, cfg))
