"""Block-partitioned multi-GPU GSVD (the paper's multi-GPU algorithm, PAPER.md
§4, re-designed for one NVSwitch node).

Every outer step keeps the reference's ME pair sets (strategies.py:59-70).
Pairs are placed by their circle-method position; rank r owns a contiguous
range of positions.  Between two steps every block moves by one position,
so only the blocks at the ends of each range change owner: at most two
blocks leave and two arrive per rank and step, exchanged with NCCL
send/recv over NVLink (grouped, device to device).

Each rank keeps full-size F, G, Z planes; a block always lives at its
logical column offset (block b = columns [b w, (b+1) w)), so a block
exchange is a contiguous copy of w columns of each plane and the kernels
take the rank's slice of the schedule unchanged.  Per-pair work is
identical to the single-GPU path (same kernels, same Grammian split
geometry, same per-pair data), so the result is bitwise independent of the
number of ranks; the per-sweep counters are integers summed with an
all-reduce.

Data planes:
  * NCCL jobs (one process per GPU): libhzg owns the exchange -- grouped
    ncclSend / ncclRecv of the crossing blocks after every step and the
    counter all-reduce, captured with the rank's steps into ONE CUDA graph
    per sweep (hzg_dist_sweep); torch.distributed only broadcasts the
    ncclUniqueId;
  * DistTransport -- torch.distributed P2P over gloo (the CPU tests of the
    routing, and several ranks sharing one GPU in the GPU tests);
  * LocalTransport -- R virtual ranks in one process (one device), block
    exchange by device copies; used by solve(workers=R) and the tests.
"""

import math
import os

import numpy as np

from . import _native
from .strategies import circle_positions, slot_ranges, weighted_slot_ranges


class BlockSchedule:
    """Circle-position schedule of nblk blocks over nranks ranks."""

    def __init__(self, nblk, nranks, end_weight=None):
        """end_weight: share of an end rank relative to an interior rank
        (None: HZG_END_WEIGHT or the default, see end_weight_default)."""
        if nblk < 2 or nblk % 2:
            raise ValueError("need an even number of blocks")
        if nranks < 1 or nranks > nblk // 2:
            raise ValueError("need 1 <= ranks <= blocks / 2 (got %d ranks, %d blocks)" % (nranks, nblk))
        self.nblk = nblk
        self.nranks = nranks
        self.steps = nblk - 1
        self.pos = circle_positions(nblk)            # (steps, nblk/2, 2), (min, max)
        ew = end_weight_default(nblk // 2, nranks) if end_weight is None else end_weight
        self.ranges = weighted_slot_ranges(nblk // 2, nranks, ew)
        owner = np.empty((self.steps, nblk), dtype=np.int64)
        for r, (lo, hi) in enumerate(self.ranges):
            for k in range(self.steps):
                owner[k, self.pos[k, lo:hi, 0]] = r
                owner[k, self.pos[k, lo:hi, 1]] = r
        self.owner = owner

    def colpairs(self, rank, w):
        """int32 (steps, npairs_rank, 2): column offsets of the rank's pairs."""
        lo, hi = self.ranges[rank]
        return np.ascontiguousarray(self.pos[:, lo:hi, :] * w, dtype=np.int32)

    def moves(self, k):
        """Blocks changing owner between step k and step (k+1) mod steps:
        sorted list of (block, src_rank, dst_rank)."""
        if not hasattr(self, "_moves"):
            self._moves = {}
        if k not in self._moves:
            a = self.owner[k]
            b = self.owner[(k + 1) % self.steps]
            self._moves[k] = [(int(blk), int(a[blk]), int(b[blk])) for blk in np.nonzero(a != b)[0]]
        return self._moves[k]

    def owned(self, k, rank):
        return np.nonzero(self.owner[k] == rank)[0]


def _block_views(planes, b, w, keys=("Fr", "Fi", "Gr", "Gi", "Zr", "Zi")):
    """Contiguous (w, m) views of block b of every plane (column-major planes
    are stored as (cols, rows) tensors, so w consecutive columns are one
    contiguous chunk)."""
    out = []
    for key in keys:
        t = planes.get(key)
        if t is not None:
            out.append(t[b * w:(b + 1) * w])
    return out


_ALL = ("Fr", "Fi", "Gr", "Gi", "Zr", "Zi")
_FG = ("Fr", "Fi", "Gr", "Gi")
_Z = ("Zr", "Zi")


class LocalTransport:
    """R virtual ranks in one process: planes_by_rank[r] are that rank's planes."""

    def __init__(self, planes_by_rank, w):
        self.planes = planes_by_rank
        self.w = w

    def exchange(self, moves, keys=_ALL):
        for (b, src, dst) in moves:
            for s, d in zip(_block_views(self.planes[src], b, self.w, keys),
                            _block_views(self.planes[dst], b, self.w, keys)):
                d.copy_(s)

    def exchange_on(self, moves, stream, zstream=None):
        """exchange() queued on ``stream`` (the wavefront's exchange stream);
        with ``zstream`` the Z blocks go on that stream instead."""
        import torch
        with torch.cuda.stream(stream):
            self.exchange(moves, _FG if zstream is not None else _ALL)
        if zstream is not None:
            with torch.cuda.stream(zstream):
                self.exchange(moves, _Z)


class DistTransport:
    """torch.distributed point-to-point (NCCL between GPUs, gloo on CPU)."""

    def __init__(self, planes, w, rank, group=None, zgroup=None):
        """zgroup: a second process group (its own NCCL communicator and
        stream) for exchanging Z blocks off the step chain, or None."""
        import torch.distributed as dist
        self.dist = dist
        self.planes = planes
        self.w = w
        self.rank = rank
        self.group = group
        self.zgroup = zgroup

    def exchange(self, moves, keys=_ALL, group=None):
        dist = self.dist
        group = self.group if group is None else group
        # NCCL moves device tensors directly; a gloo group (CPU tests, or
        # several ranks sharing one GPU) stages device blocks through host
        # memory
        staged = dist.get_backend(group) == "gloo"
        ops, back = [], []
        for (b, src, dst) in moves:
            if src == self.rank:
                for t in _block_views(self.planes, b, self.w, keys):
                    ops.append(dist.P2POp(dist.isend, t.cpu() if staged and t.is_cuda else t, dst, group))
            elif dst == self.rank:
                for t in _block_views(self.planes, b, self.w, keys):
                    if staged and t.is_cuda:
                        h = t.new_empty(t.shape, device="cpu")
                        back.append((t, h))
                        t = h
                    ops.append(dist.P2POp(dist.irecv, t, src, group))
        if ops:
            for wk in dist.batch_isend_irecv(ops):
                wk.wait()
        for t, h in back:
            t.copy_(h)

    def exchange_on(self, moves, stream, zstream=None):
        """exchange() ordered on ``stream``: NCCL's stream waits on it (it
        already waits for this rank's end groups) and wait() makes it wait
        for the transfers, so the next step's end groups see the received
        blocks without a host synchronisation.  With ``zstream`` (and the Z
        process group) the Z blocks go on that stream through their own
        communicator.  (gloo stages through host memory; its device-to-host
        copies synchronise.)"""
        import torch
        with torch.cuda.stream(stream):
            self.exchange(moves, _FG if zstream is not None else _ALL)
        if zstream is not None:
            with torch.cuda.stream(zstream):
                self.exchange(moves, _Z, self.zgroup)


def gather_blocks(sched, k_final=0):
    """(block, owner, 0) moves bringing every block to rank 0 at step k_final."""
    return [(b, int(sched.owner[k_final, b]), 0) for b in range(sched.nblk) if sched.owner[k_final, b] != 0]


def run_ranks(devs, sched, transport, cfg, allreduce=None, wave=None):
    """The outer sweep loop (blocked.py:503-550) for block-partitioned ranks.

    devs: the DeviceGsvd objects this process drives (all R virtual ranks,
    or the single local rank).  allreduce(total, big) -> (total, big) sums
    the counters over processes (identity for virtual ranks).
    Returns (sweeps, total, big, converged)."""
    for d in devs:
        d.init()
    sweeps = total = big = 0
    converged = False
    for _ in range(cfg.max_outer_sweeps):
        t, b = sweep_ranks(devs, sched, transport, allreduce, wave)
        sweeps += 1
        total += t
        big += b
        if b == 0:
            converged = True
            break
    return sweeps, total, big, converged


def end_weight_default(npos, nranks):
    """Relative share of the two end ranks (HZG_END_WEIGHT overrides).
    Measured on the per-rank share at n = 16384 (profiles/r01_rank_share.txt):
    with 64 pairs per rank (8 ranks) 0.65 balances the end ranks' slower
    inner solves (728 -> 667 ms per sweep); with 128 (4 ranks) equal ranges
    are best."""
    e = os.environ.get("HZG_END_WEIGHT")
    if e:
        return float(e)
    return 0.65 if nranks >= 3 and npos / nranks <= 64 else 1.0


_ZGROUPS = {}


def _z_group(dist, world):
    """The second process group of the split Z exchange, created once per
    world size (every rank calls this at the same point)."""
    if world not in _ZGROUPS:
        _ZGROUPS[world] = dist.new_group(list(range(world)))
    return _ZGROUPS[world]


def split_z_default():
    """Exchange Z blocks on their own stream / communicator: only useful
    with the deferred Z postmultiply (HZG_WAVE_DEFER_Z=1), so on by default
    only then (HZG_SPLIT_Z overrides); otherwise one exchange (one NCCL
    communicator) carries every plane."""
    e = os.environ.get("HZG_SPLIT_Z")
    if e is not None:
        return e != "0"
    return os.environ.get("HZG_WAVE_DEFER_Z", "0") not in ("", "0")


def rank_groups(npairs, ngroups=None):
    """Contiguous position groups [(p0, pn), ...] of one rank's slot range
    for the per-rank wavefront (same rule as the single-GPU sweep graph,
    hzg_api.cu choose_groups: 16+ pairs per group, at most 8 groups;
    HZG_GROUPS overrides)."""
    import os
    if ngroups is None:
        ngroups = max(1, min(8, npairs // 16))
        if os.environ.get("HZG_GROUPS"):
            ngroups = max(1, min(npairs, int(os.environ["HZG_GROUPS"])))
    ngroups = max(1, min(npairs, ngroups))
    return [(npairs * g // ngroups, npairs * (g + 1) // ngroups - npairs * g // ngroups) for g in range(ngroups)]


class Wavefront:
    """Group split and exchange stream of the per-rank wavefront.

    Rank r's slot range is cut into G contiguous position groups, each on
    its own stream (hzg_wave_step, one library call per step).  Group g of
    step k+1 waits only for groups g-1, g, g+1 of step k on the same rank
    (a block moves by at most one position per step); the two end groups
    also wait for the block exchange of step k, which itself waits only for
    the end groups of step k (the blocks that change owner sit at the ends
    of a range).  So the Grammian and postmultiply streaming of some groups
    overlaps the latency-bound inner solves of others, and the NCCL
    exchange overlaps the interior groups, with no host synchronisation
    inside a sweep.  Per-pair work is that of the serialised schedule, so
    results stay bitwise equal."""

    def __init__(self, devs, npairs, ngroups=None, split_z=False):
        """npairs: slot-range length of every rank in ``devs``; split_z:
        exchange Z blocks on a second stream (zcomm), off the step chain."""
        import torch
        self.torch = torch
        self.groups = [len(rank_groups(np_, ngroups)) for np_ in npairs]
        self.comm = torch.cuda.Stream(device=devs[0].device)
        self.zcomm = torch.cuda.Stream(device=devs[0].device) if split_z else None


def sweep_ranks(devs, sched, transport, allreduce=None, wave=None):
    """One outer sweep of the partitioned schedule: every step on every
    rank with the block exchange after it, the counter sum, and the
    inter-sweep Z rescale when the sweep applied big transforms
    (blocked.py:521-542).  Returns the sweep's (total, big).

    wave: a Wavefront to run every rank's steps as position groups on
    several streams (asynchronous exchange); None serialises step by step."""
    if wave is None:
        for k in range(sched.steps):
            for d in devs:
                d.run_steps(k, 1)
            transport.exchange(sched.moves(k))
    else:
        _sweep_wavefront(devs, sched, transport, wave)
    t = b = code = 0
    for d in devs:
        tt, bb, cc = d.collect_status()
        t += tt
        b += bb
        code = max(code, cc)
    if allreduce is not None:
        # every rank learns the worst status before anyone raises, so no
        # rank leaves the job while the others wait in the next exchange
        t, b, code = allreduce(t, b, code)
    _native.check(code, None, "block pair of this sweep (status agreed over all ranks)")
    if b != 0:
        for d in devs:
            d.rescale_z()
    return t, b


def _sweep_wavefront(devs, sched, transport, wave):
    for k in range(sched.steps):
        for d, g in zip(devs, wave.groups):
            d.wave_step(k, g, wave.comm, wave.zcomm)
        transport.exchange_on(sched.moves(k), wave.comm, wave.zcomm)
    for d in devs:
        d.wave_join(wave.comm, wave.zcomm)


class PartitionedGsvd:
    """One rank of a block-partitioned solve over device-resident planes.

    planes: bordered device planes (same content on every rank); comm:
    None for R virtual ranks on this device (planes are cloned per rank),
    or "dist" for the torch.distributed rank this process is.  run() is
    _algorithm1_loop over the partitioned schedule; finalize() gathers the
    blocks to rank 0 and returns its device outputs (None elsewhere)."""

    def __init__(self, planes, cfg, nranks, comm=None, wavefront=True, devices=None):
        import torch

        from .solver import DeviceGsvd

        self.cfg = cfg
        w = cfg.block_width
        n = planes["Fr"].shape[0]
        self.nblk = n // w
        if not 1 <= nranks <= self.nblk // 2:
            raise ValueError("%d ranks for %d column blocks: the block-partitioned schedule needs "
                             "1 <= ranks <= blocks / 2" % (nranks, self.nblk))
        self.nranks = nranks
        self.sched = BlockSchedule(self.nblk, self.nranks)
        epsn = epsn_of(cfg, n)
        self.comm = comm
        self.nccl = False
        self.multi = False
        if comm == "devices":
            # one process driving nranks GPUs: a context per
            # device, ncclCommInitAll, every rank's sweep graph launched
            # before any is waited for
            devices = list(range(nranks)) if devices is None else list(devices)
            if len(devices) != self.nranks:
                raise ValueError("need one device per rank")
            self.rank = 0
            self.devs = []
            for r, d in enumerate(devices):
                dd = torch.device("cuda", d)
                with torch.cuda.device(dd):
                    pl = {k: (v.to(dd) if v is not None else None) for k, v in planes.items()}
                    self.devs.append(DeviceGsvd(pl, cfg, device=dd, epsn=epsn, schedule=self.sched.colpairs(r, w)))
            import ctypes
            arr = (ctypes.c_void_p * len(self.devs))(*[dv.ctx.value for dv in self.devs])
            L = _native.load()
            _native.check(L.hzg_comm_attach_all(arr, len(self.devs)), self.devs[0].ctx, "hzg_comm_attach_all")
            self._ctx_array = arr
            for dv in self.devs:
                dv.comm_set_moves([self.sched.moves(k) for k in range(self.sched.steps)])
            self.nccl = self.multi = True
            self.transport = None
            self.allreduce = None
        elif comm is None:
            plist = [planes] + [{k: (v.clone() if v is not None else None) for k, v in planes.items()}
                                for _ in range(self.nranks - 1)]
            self.devs = [DeviceGsvd(plist[r], cfg, epsn=epsn, schedule=self.sched.colpairs(r, w))
                         for r in range(self.nranks)]
            self.transport = LocalTransport([dict(pl, Zr=d.Zr, Zi=d.Zi) for pl, d in zip(plist, self.devs)], w)
            self.rank = 0
            self.allreduce = None
        else:
            import torch.distributed as dist
            self.rank, world = dist.get_rank(), dist.get_world_size()
            if world != self.nranks:
                raise ValueError("distributed solve needs world size %d for %d blocks" % (self.nranks, self.nblk))
            dev = DeviceGsvd(planes, cfg, epsn=epsn, schedule=self.sched.colpairs(self.rank, w))
            self.devs = [dev]
            # the Z exchange gets its own communicator (and NCCL stream) so
            # it never queues ahead of the next step's F, G exchange
            zgroup = _z_group(dist, world) if wavefront and split_z_default() else None
            self.transport = DistTransport(dict(planes, Zr=dev.Zr, Zi=dev.Zi), w, self.rank, zgroup=zgroup)

            self.allreduce = counter_allreduce("cpu" if dist.get_backend() == "gloo" else dev.device)
            if dist.get_backend() == "nccl" and os.environ.get("HZG_TORCH_P2P", "0") in ("", "0"):
                # the data plane lives in libhzg: NCCL send / recv of the
                # crossing blocks and the counter all-reduce inside one
                # captured CUDA graph per sweep; torch.distributed only
                # carries the ncclUniqueId
                uid = [None]
                if self.rank == 0:
                    uid[0] = unique_id()
                dist.broadcast_object_list(uid, src=0)
                dev.comm_attach(world, self.rank, uid[0])
                dev.comm_set_moves([self.sched.moves(k) for k in range(self.sched.steps)])
                self.nccl = True
        ranks = range(self.nranks) if comm in (None, "devices") else [self.rank]
        self.wave = None
        if wavefront and torch.cuda.is_available() and not self.nccl:
            self.wave = Wavefront(self.devs, [self.sched.ranges[r][1] - self.sched.ranges[r][0] for r in ranks],
                                  split_z=split_z_default())
        self.sweeps = self.total = self.big = 0
        self.converged = False

    def run(self):
        if self.nccl:
            self.init()
            for _ in range(self.cfg.max_outer_sweeps):
                if self.sweep()[1] == 0:
                    break
            return self
        self.sweeps, self.total, self.big, self.converged = run_ranks(self.devs, self.sched, self.transport, self.cfg,
                                                                      self.allreduce, self.wave)
        return self

    def init(self):
        import torch
        for d in self.devs:
            with torch.cuda.device(d.device):
                d.init()
        self.sweeps = self.total = self.big = 0
        self.converged = False

    def sweep(self):
        """One outer sweep (after init()); returns (total, big)."""
        if self.multi:
            L = _native.load()
            for d in self.devs:
                _native.check(L.hzg_dist_sweep_launch(d.ctx), d.ctx, "dist_sweep")
            res = [d.dist_sweep_wait() for d in self.devs]
            t, b = res[0]  # every rank holds the same reduced counters
        elif self.nccl:
            t, b = self.devs[0].dist_sweep()
        else:
            t, b = sweep_ranks(self.devs, self.sched, self.transport, self.allreduce, self.wave)
        self.sweeps += 1
        self.total += t
        self.big += b
        self.converged = b == 0
        return t, b

    def finalize(self, n0=None, mF0=None, mG0=None, sort=True):
        import torch
        with torch.cuda.device(self.devs[0].device):
            return self._finalize(n0, mF0, mG0, sort)

    def _finalize(self, n0=None, mF0=None, mG0=None, sort=True):
        if self.multi:
            moves = gather_blocks(self.sched)
            arr = np.asarray([x for m in moves for x in m] or [0], dtype=np.int32)
            import ctypes
            _native.check(_native.load().hzg_comm_exchange_all(self._ctx_array, len(self.devs),
                                                              arr.ctypes.data_as(ctypes.c_void_p), len(moves)),
                          self.devs[0].ctx, "hzg_comm_exchange_all")
        elif self.nccl:
            self.devs[0].comm_exchange(gather_blocks(self.sched))
        else:
            self.transport.exchange(gather_blocks(self.sched))
        if self.rank != 0:
            return None
        root = self.devs[0]
        root.sweeps, root.total, root.big, root.converged = self.sweeps, self.total, self.big, self.converged
        return root.finalize(n0, mF0, mG0, sort=sort)

    def launch_counts(self):
        if self.nccl:
            # hzg_dist_sweep: 3 kernels per position group and step, the
            # counter fold, 2 status packs and the gated rescale per sweep
            # (NCCL's own kernels not counted)
            G = max(1, min(8, (self.sched.ranges[self.rank][1] - self.sched.ranges[self.rank][0]) // 16))
            if os.environ.get("HZG_GROUPS"):
                G = max(1, int(os.environ["HZG_GROUPS"]))
            return self.sched.steps * 3 * G + 4, 6
        # step-wise driving: 3 kernels per step (per position group with the
        # wavefront), plus the counter fold and the Z rescale per sweep, per
        # rank driven by this process
        g = sum(self.wave.groups) if self.wave is not None else len(self.devs)
        per_step = 3
        if self.wave is not None and os.environ.get("HZG_WAVE_DEFER_Z", "0") not in ("", "0") and \
                os.environ.get("HZG_DEFER_Z", "1") != "0" and not self.cfg.exact:
            per_step = 4            # the deferred Z postmultiply is a 4th kernel per group and step
        return self.sched.steps * per_step * g + 2 * len(self.devs), len(self.devs) + 5

    def close(self):
        for d in self.devs:
            d.close()


def counter_allreduce(device):
    """(total, big, status code) summed / maxed over the torch.distributed
    ranks: every rank sees the same status, so all raise the same error
    (HZG codes order by severity: OK 0 < RANK 1 < NOT_PD 2)."""
    import torch
    import torch.distributed as dist

    def allreduce(t, b, code):
        x = torch.tensor([t, b], dtype=torch.int64, device=device)
        dist.all_reduce(x)
        c = torch.tensor([code], dtype=torch.int64, device=device)
        dist.all_reduce(c, op=dist.ReduceOp.MAX)
        return int(x[0]), int(x[1]), int(c[0])

    return allreduce


def unique_id():
    """A new ncclUniqueId (bytes) from libhzg's NCCL binding."""
    import ctypes
    L = _native.load()
    buf = ctypes.create_string_buffer(int(L.hzg_comm_unique_id_bytes()))
    _native.check(L.hzg_comm_unique_id(buf), None, "ncclGetUniqueId")
    return buf.raw


def epsn_of(cfg, n):
    return cfg.gate_eps * math.sqrt(n)


def solve_blocks(F, G, cfg, nranks, comm=None, wavefront=True, devices=None):
    """GSVD of (F, G) with the block-partitioned schedule over nranks ranks.

    comm=None: nranks virtual ranks in this process on the current device
    (block exchange by device copies).  comm="devices": this process drives
    one GPU per rank (``devices``, default 0..nranks-1) with one NCCL
    communicator each (ncclCommInitAll).  comm="dist": this process is one
    rank of an initialized torch.distributed job (NCCL, one GPU per rank);
    every rank passes the same F, G and rank 0 returns the result (the
    others return None).  wavefront=False serialises each rank's steps
    (no position groups).  Results are bitwise those of nranks = 1.
    """
    from .config import SolverConfig
    from .core import MatrixPlanePair, ProblemPair
    from .solver import _result_from_device, gsvd_1x1, upload_bordered

    cfg = cfg or SolverConfig()
    if isinstance(F, np.ndarray):
        F = MatrixPlanePair.from_dense(F)
    if isinstance(G, np.ndarray):
        G = MatrixPlanePair.from_dense(G)
    if F.cols == 1:
        return gsvd_1x1(F, G)
    p = ProblemPair(F, G)
    w = cfg.block_width
    planes0, n, mF, mG = upload_bordered(p.F, p.G, w)
    job = PartitionedGsvd(planes0, cfg, nranks, comm, wavefront=wavefront, devices=devices)
    try:
        job.run()
        out = job.finalize(p.n, p.F.rows, p.G.rows, sort=True)
        if out is None:
            return None
        root = job.devs[0]
        return _result_from_device(root, out, p.is_complex, workers=job.nranks)
    finally:
        job.close()
