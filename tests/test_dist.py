"""The multi-GPU block schedule and its block exchange, on CPU: two gloo
ranks run a toy block computation along the circle-position schedule and
must reproduce a single-process run exactly (same routing logic and
transport code as the NCCL path, tensors on the CPU)."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1909_00101_b200.dist import BlockSchedule, DistTransport, LocalTransport, gather_blocks

W = 2


def _toy_step(planes, sched, k, rank):
    """Deterministic, order-sensitive update of the rank's pairs at step k."""
    lo, hi = sched.ranges[rank]
    for p, q in sched.pos[k, lo:hi]:
        for key in ("Fr", "Gr", "Zr"):
            t = planes[key]
            a = t[p * W:(p + 1) * W].clone()
            b = t[q * W:(q + 1) * W].clone()
            t[p * W:(p + 1) * W] = a * 1.5 + b + (k + 1)
            t[q * W:(q + 1) * W] = b * 0.5 - a


def _initial(nblk, m):
    g = torch.Generator().manual_seed(5)
    return {key: torch.randn((nblk * W, m), generator=g, dtype=torch.float64) for key in ("Fr", "Gr", "Zr")}


def _reference(nblk, m, sweeps):
    planes = _initial(nblk, m)
    sched = BlockSchedule(nblk, 1)
    for _ in range(sweeps):
        for k in range(sched.steps):
            _toy_step(planes, sched, k, 0)
    return planes


def _worker(rank, world, port, nblk, m, sweeps, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    planes = _initial(nblk, m)
    sched = BlockSchedule(nblk, world)
    tr = DistTransport(planes, W, rank)
    for _ in range(sweeps):
        for k in range(sched.steps):
            _toy_step(planes, sched, k, rank)
            tr.exchange(sched.moves(k))
    tr.exchange(gather_blocks(sched))
    if rank == 0:
        torch.save({k: v.clone() for k, v in planes.items()}, out)
    dist.barrier()
    dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


@pytest.mark.parametrize("nblk,world", [(12, 3)])
def test_gloo_block_exchange_matches_single_process(tmp_path, nblk, world):
    out = str(tmp_path / "planes.pt")
    mp.spawn(_worker, args=(world, _free_port(), nblk, 5, 2, out), nprocs=world, join=True)
    got = torch.load(out)
    ref = _reference(nblk, 5, 2)
    for key in ("Fr", "Gr", "Zr"):
        assert torch.equal(got[key], ref[key]), key


@pytest.mark.parametrize("nblk,world", [(16, 4), (64, 8), (256, 8), (1024, 8)])
def test_local_transport_matches_single_process(nblk, world):
    sched = BlockSchedule(nblk, world)
    m = 3
    planes = [_initial(nblk, m) for _ in range(world)]
    tr = LocalTransport(planes, W)
    for k in range(sched.steps):
        for r in range(world):
            _toy_step(planes[r], sched, k, r)
        tr.exchange(sched.moves(k))
    tr.exchange(gather_blocks(sched))
    ref = _initial(nblk, m)
    s1 = BlockSchedule(nblk, 1)
    for k in range(s1.steps):
        _toy_step(ref, s1, k, 0)
    for key in ("Fr", "Gr", "Zr"):
        assert torch.equal(planes[0][key], ref[key])


@pytest.mark.parametrize("end_weight", [1.0, 0.6])
def test_schedule_moves_per_rank_and_step(end_weight):
    for nblk, world in ((64, 2), (1024, 8), (2048, 8), (96, 5)):
        sched = BlockSchedule(nblk, world, end_weight=end_weight)
        for k in range(sched.steps):
            mv = sched.moves(k)
            out_per_rank = np.bincount([s for (_, s, _) in mv], minlength=world)
            assert out_per_rank.max() <= 2  # at most two blocks leave a rank per step
            for (b, s, d) in mv:
                assert abs(s - d) == 1 or {s, d} == {0, world - 1} or world == 2


def test_colpairs_cover_every_pair_once_per_sweep():
    nblk, world, w = 32, 4, 16
    sched = BlockSchedule(nblk, world)
    seen = set()
    for r in range(world):
        cp = sched.colpairs(r, w)
        for k in range(sched.steps):
            for c0, c1 in cp[k]:
                assert c0 < c1
                seen.add((c0 // w, c1 // w))
    assert len(seen) == nblk * (nblk - 1) // 2


def test_weighted_slot_ranges_partition():
    from paper_1909_00101_b200.strategies import weighted_slot_ranges
    for npos in range(1, 70):
        for world in range(1, npos + 1):
            for f in (0.1, 0.6, 1.0, 1.7):
                r = weighted_slot_ranges(npos, world, f)
                assert r[0][0] == 0 and r[-1][1] == npos and len(r) == world
                assert all(lo < hi for lo, hi in r)
                assert all(r[i][1] == r[i + 1][0] for i in range(world - 1))
    r = weighted_slot_ranges(512, 8, 0.6)
    assert r[0][1] - r[0][0] < r[1][1] - r[1][0] and r[-1][1] - r[-1][0] == r[0][1] - r[0][0]


def test_weighted_schedule_covers_every_pair():
    nblk, world, w = 40, 4, 8
    sched = BlockSchedule(nblk, world, end_weight=0.5)
    seen = set()
    for r in range(world):
        cp = sched.colpairs(r, w)
        for k in range(sched.steps):
            for c0, c1 in cp[k]:
                seen.add((c0 // w, c1 // w))
    assert len(seen) == nblk * (nblk - 1) // 2


class _FakeDev:
    """A rank whose inner solve reports `code` (0 ok, 1 RankError, 2 not PD)."""

    def __init__(self, code):
        self.code = code
        self.rescaled = 0

    def run_steps(self, k, count):
        pass

    def collect_status(self):
        return 10, 3, self.code

    def rescale_z(self):
        self.rescaled += 1


class _NoTransport:
    def exchange(self, moves, keys=None):
        pass


def _status_worker(rank, world, port, codes, out):
    from paper_1909_00101_b200 import NotPositiveDefiniteError, RankError
    from paper_1909_00101_b200.dist import counter_allreduce, sweep_ranks
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    sched = BlockSchedule(4 * world, world)
    dev = _FakeDev(codes[rank])
    try:
        t, b = sweep_ranks([dev], sched, _NoTransport(), counter_allreduce("cpu"))
        res = ("ok", t, b, dev.rescaled)
    except NotPositiveDefiniteError:
        res = ("notpd",)
    except RankError:
        res = ("rank",)
    # every rank reaches this collective: nobody left the job early
    dist.barrier()
    torch.save(res, "%s.%d" % (out, rank))
    dist.destroy_process_group()


@pytest.mark.parametrize("codes,expect", [((0, 0, 0), ("ok", 30, 9, 1)), ((0, 1, 0), ("rank",)),
                                          ((2, 1, 0), ("notpd",))])
def test_gloo_status_agreed_before_raising(tmp_path, codes, expect):
    """A failing block pair on one rank raises the same error on EVERY rank
    (the status is all-reduced with the counters) instead of leaving the
    others waiting in the next exchange (dist.py)."""
    out = str(tmp_path / "res")
    mp.spawn(_status_worker, args=(3, _free_port(), codes, out), nprocs=3, join=True)
    for r in range(3):
        assert torch.load("%s.%d" % (out, r)) == expect
