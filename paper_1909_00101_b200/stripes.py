"""The reference's stripe-distributed scheme (distsim.py) on the device.

``solve(F, G, cfg, workers=s)`` and ``run_distributed(p, cfg, s, s_inner)``
of the reference do NOT return the single-worker result: the columns are cut
into 2s stripes, worker r joins the two stripes of step k of the outermost
strategy table (gen_table(kind, 2s)) into one slab, runs the blocked sweep
loop on that slab for up to ``s_inner`` sweeps (``_algorithm1_loop`` with a
trailing Z rescale, blocked.py:503-550), then the stripes move along the
communication mapping (strategies.py:117-143).  The generalized singular
values agree with the single-worker solve to ~1e-13, but the bits, the
sweep count and the transform counters depend on s.  This module rebuilds
that scheme so ``workers=s`` is a drop-in:

* every worker's slab is a device problem of its own (a libhzg context of
  n_local = 2W columns whose Z keeps the n global rows, hzg_set_z_rows), so
  the per-slab work runs on the same sm_100a kernels as the single-GPU path;
* the stripe exchange is a device copy per stripe plane, routed and checked
  with the reference's tag protocol (ProtocolError on a missing or
  duplicate tag, distsim.py:103-144);
* all s workers live on one GPU here, as the reference's simulation keeps
  them in one process; each slab's sweep is its own captured CUDA graph on
  the worker's own stream, and the s sweeps of an outermost step run
  concurrently (hzg_sweep_launch / hzg_sweep_wait).

In exact mode (SolverConfig(exact=True)) the result is bitwise the
reference's run_distributed (tests/golden/dist_*.npz).

Planes are torch tensors.  StripeState exposes them as (rows, cols)
column-major views (``t.T`` of the (cols, rows) storage the kernels use), so
``st.Fr[i, j]`` indexes row i, column j as in the reference.
"""

import ctypes
import dataclasses
import math
from typing import Optional

import numpy as np

from . import _native
from .config import SolverConfig
from .core import GsvdResult, MatrixPlanePair
from .errors import ProtocolError, RankError
from .strategies import comm_mapping, gen_table

# the reference's per-stripe message order (distsim.py:57-58)
_PLANES_CPLX = ("Fr", "Fi", "Gr", "Gi", "Zr", "Zi")
_PLANES_REAL = ("Fr", "Gr", "Zr")
# outermost sweeps of run_distributed: a fixed 30 in the reference
# (distsim.py:196), independent of cfg.max_outer_sweeps
OUTERMOST_SWEEPS = 30


@dataclasses.dataclass
class StripeState:
    """Worker ``rank``'s slab: stripes p (left half) and q (right half) of
    width ``width``; F, G are m x 2W, Z is n x 2W (global rows)."""

    rank: int
    p: int
    q: int
    width: int
    Fr: object
    Fi: Optional[object]
    Gr: object
    Gi: Optional[object]
    Zr: object
    Zi: Optional[object]
    is_complex: bool = False

    def storage(self, key):
        """The (cols, rows) contiguous tensor behind plane ``key``."""
        t = getattr(self, key)
        return None if t is None else t.T


def _device(device):
    import torch
    if device is not None:
        return torch.device(device)
    if torch.cuda.is_available():
        return torch.device("cuda", torch.cuda.current_device())
    return torch.device("cpu")


def _slab(plane, sp, sq, width, dev, rows):
    """(2W, rows) contiguous storage holding columns of stripes sp and sq
    (zero rows appended up to ``rows``)."""
    import torch
    cols = np.concatenate([np.arange(sp * width, (sp + 1) * width), np.arange(sq * width, (sq + 1) * width)])
    host = np.zeros((2 * width, rows))
    src = np.asarray(plane)
    host[:, :src.shape[0]] = src[:, cols].T
    return torch.from_numpy(host).to(dev)


def partition_stripes(p, s, block_width=1, kind="me", device=None, row_multiple=1):
    """Cut the bordered pair p into 2s stripes; worker r gets the two
    stripes of step 0 of gen_table(kind, 2s) (distsim.py:62-95).  Z slabs
    start at zero.  ``row_multiple``: zero rows are appended to F and G up
    to a multiple of it (the device kernels need multiples of 2w; zero rows
    change no inner product and are cropped again on assembly)."""
    import torch
    n = p.n
    if n % (2 * s) != 0:
        raise ValueError("n=%d is not divisible into 2*%d stripes" % (n, s))
    width = n // (2 * s)
    if width % block_width != 0:
        raise ValueError("stripe width %d is not a multiple of the block width %d" % (width, block_width))
    dev = _device(device)
    step0 = gen_table(kind, 2 * s).steps[0]
    cplx = p.is_complex
    states = []
    for r in range(s):
        sp, sq = step0[r]
        planes = {}
        for key, mat in (("F", p.F), ("G", p.G)):
            rows = -(-mat.rows // row_multiple) * row_multiple
            planes[key + "r"] = _slab(mat.re, sp, sq, width, dev, rows)
            planes[key + "i"] = _slab(mat.im, sp, sq, width, dev, rows) if cplx else None
        planes["Zr"] = torch.zeros((2 * width, n), dtype=torch.float64, device=dev)
        planes["Zi"] = torch.zeros((2 * width, n), dtype=torch.float64, device=dev) if cplx else None
        views = {k: (v.T if v is not None else None) for k, v in planes.items()}
        states.append(StripeState(r, sp, sq, width, is_complex=cplx, **views))
    return states


def exchange_step(states, mapping, k):
    """The tagged stripe exchange after outermost step k (distsim.py:103-144):
    every worker sends one message per stripe plane, tag = base tag of the
    plane (+ half when the stripe lands in the destination's second slot);
    every worker must receive exactly one message per tag.  Stripe ids
    advance to step (k + 1) mod steps."""
    cplx = states[0].is_complex
    order = _PLANES_CPLX if cplx else _PLANES_REAL
    half = len(order)
    inbox = {}
    for st in states:
        p, q, t0, t1 = mapping.entries[k][st.rank]
        if (p, q) != (st.p, st.q):
            raise ProtocolError("worker %d holds stripes (%d, %d) but the mapping says (%d, %d)"
                                % (st.rank, st.p, st.q, p, q))
        for slot, enc in ((0, t0), (1, t1)):
            dest = abs(enc) - 1
            offset = half if enc > 0 else 0
            for i, key in enumerate(order):
                tag = i + 1 + offset
                if (dest, tag) in inbox:
                    raise ProtocolError("duplicate tag %d at worker %d" % (tag, dest))
                # a clone: the destination slot may be this worker's own,
                # overwritten before the message is consumed
                src = st.storage(key)[slot * st.width:(slot + 1) * st.width]
                inbox[(dest, tag)] = (src.clone(), st.rank)
    for st in states:
        for tag in range(1, 2 * half + 1):
            msg = inbox.pop((st.rank, tag), None)
            if msg is None:
                raise ProtocolError("missing tag %d at worker %d" % (tag, st.rank))
            slot = 0 if tag <= half else 1
            key = order[(tag - 1) % half]
            st.storage(key)[slot * st.width:(slot + 1) * st.width].copy_(msg[0])
        st.p, st.q = mapping.entries[(k + 1) % mapping.steps][st.rank][:2]
    return states


def _logical_rows(st):
    """Global row of the initial Z entry of each slab column."""
    w = st.width
    return np.concatenate([np.arange(st.p * w, (st.p + 1) * w), np.arange(st.q * w, (st.q + 1) * w)])


class _Worker:
    """One stripe slab as a device problem (libhzg context with Z of n
    global rows)."""

    def __init__(self, st, cfg, epsn, n):
        import torch
        from .solver import DeviceGsvd
        self.st = st
        planes = {k: st.storage(k) for k in ("Fr", "Fi", "Gr", "Gi")}
        # every worker's context is bound to its own stream, so the slabs of
        # one outermost step sweep concurrently on the GPU
        self.stream = torch.cuda.Stream(device=st.Fr.device)
        with torch.cuda.stream(self.stream):
            self.dev = DeviceGsvd(planes, cfg, epsn=epsn, zrows=n, Z=(st.storage("Zr"), st.storage("Zi")))

    def init(self):
        """Per-slab prescale (column-local, distsim.py:183-193); the library
        places z0[j] at local row j, the reference at the column's logical
        row."""
        import torch
        self.dev.init()
        with torch.cuda.stream(self.stream):
            idx = torch.arange(2 * self.st.width, device=self.dev.device)
            rows = torch.from_numpy(_logical_rows(self.st)).to(self.dev.device)
            for key in ("Zr", "Zi"):
                z = self.st.storage(key)
                if z is None:
                    continue
                diag = z[idx, idx].clone()
                z[idx, idx] = 0.0
                z[idx, rows] = diag


    def final(self):
        """Final rescale of the slab: (sigmaF, sigmaG, sigma) device vectors."""
        import torch
        st, d = self.st, self.dev
        kw = dict(dtype=torch.float64, device=d.device)
        sig = [torch.empty(2 * st.width, **kw) for _ in range(3)]
        P = lambda t: ctypes.c_void_p(t.data_ptr()) if t is not None else None  # noqa: E731
        rc = d.lib.hzg_op_rescale(d.mF, d.mG, 2 * st.width, int(st.is_complex), int(d.cfg.compensated), 1,
                                  P(st.storage("Fr")), P(st.storage("Fi")), P(st.storage("Gr")),
                                  P(st.storage("Gi")), P(st.storage("Zr")), P(st.storage("Zi")), d.Zr.shape[1],
                                  P(sig[0]), P(sig[1]), P(sig[2]), ctypes.c_void_p(d.stream.cuda_stream))
        if rc == _native.HZG_RANK:
            raise RankError("zero column at extraction on worker %d" % st.rank)
        _native.check(rc, None, "final rescale on worker %d" % st.rank)
        return sig

    def close(self):
        self.dev.close()


def _loops(workers, sweep_cap):
    """_algorithm1_loop(..., sweep_cap, trailing_rescale=True) on every
    worker's slab (blocked.py:503-550), the workers' sweeps queued together
    on their streams and waited for together.  Returns the per-worker
    (total, big) sums."""
    import torch
    tot = [0] * len(workers)
    big = [0] * len(workers)
    active = list(range(len(workers)))
    for _ in range(sweep_cap):
        for q in active:
            workers[q].dev.sweep_launch()  # the inter-sweep rescale is gated on big != 0 in the graph
        still = []
        for q in active:
            t, b = workers[q].dev.sweep_wait()
            tot[q] += t
            big[q] += b
            if b != 0:
                still.append(q)
        active = still
        if not active:
            break
    for wk in workers:
        wk.dev.rescale_z()  # the trailing rescale
    torch.cuda.synchronize()  # the stripe exchange reads and writes every slab
    return tot, big



def run_distributed(p, cfg=None, s=2, s_inner=1, pool=1):
    """Stripe-distributed solve of a bordered pair with s workers
    (distsim.py:147-259).  s = 1 delegates to gsvd_blocked.  ``pool`` is
    accepted for signature compatibility (the result is pool-invariant in
    the reference too; the slabs here share one GPU)."""
    from .solver import gsvd_blocked
    cfg = cfg or SolverConfig()
    if s < 1:
        raise ValueError("need at least one worker")
    if s == 1:
        r = gsvd_blocked(p, cfg)
        r.workers = 1
        return r
    n = p.n
    w = cfg.block_width
    if n % (2 * w * s) != 0:
        raise ValueError("n=%d not divisible for %d workers at block width %d" % (n, s, w))
    table = gen_table(cfg.outer_kind, 2 * s)
    mapping = comm_mapping(table)
    from .solver import _torch
    torch = _torch()  # no device: fail loudly (no CPU fallback)
    states = partition_stripes(p, s, w, cfg.outer_kind, row_multiple=2 * w)
    epsn = cfg.gate_eps * math.sqrt(n)
    torch.cuda.synchronize()  # slabs built on the current stream, used on the workers' streams
    workers = [_Worker(st, cfg, epsn, n) for st in states]
    try:
        for wk in workers:
            wk.init()
        total = big = sweeps = 0
        converged = False
        torch.cuda.synchronize()
        for _ in range(OUTERMOST_SWEEPS):
            t_sw = b_sw = 0
            for k in range(len(table.steps)):
                tot, big_w = _loops(workers, s_inner)
                t_sw += sum(tot)
                b_sw += sum(big_w)
                exchange_step(states, mapping, k)
                torch.cuda.synchronize()  # the next sweeps run on the workers' streams
            sweeps += 1
            total += t_sw
            big += b_sw
            if b_sw == 0:
                converged = True
                break
        return _assemble(p, states, [wk.final() for wk in workers], sweeps, total, big, converged, s)
    finally:
        for wk in workers:
            wk.close()


def _assemble(p, states, sigs, sweeps, total, big, converged, s):
    """Reassemble the global U, V, Z and sigma vectors by stripe id
    (distsim.py:226-259)."""
    import torch
    torch.cuda.synchronize()
    n, mF, mG = p.n, p.F.rows, p.G.rows
    cplx = p.is_complex
    out = {k: np.zeros(shape, order="F") for k, shape in
           (("Ur", (mF, n)), ("Vr", (mG, n)), ("Zr", (n, n)), ("Ui", (mF, n)), ("Vi", (mG, n)), ("Zi", (n, n)))}
    sv = {k: np.zeros(n) for k in ("sigmaF", "sigmaG", "sigma")}
    for st, sig in zip(states, sigs):
        w = st.width
        host = {k: (st.storage(k).cpu().numpy() if st.storage(k) is not None else None)
                for k in ("Fr", "Fi", "Gr", "Gi", "Zr", "Zi")}
        hs = [x.cpu().numpy() for x in sig]
        for slot, stripe in ((0, st.p), (1, st.q)):
            lo, g0 = slot * w, stripe * w
            for dst, src in (("Ur", "Fr"), ("Vr", "Gr"), ("Zr", "Zr"), ("Ui", "Fi"), ("Vi", "Gi"), ("Zi", "Zi")):
                if host[src] is not None:
                    rows = out[dst].shape[0]
                    out[dst][:, g0:g0 + w] = host[src][lo:lo + w, :rows].T
            for name, v in zip(("sigmaF", "sigmaG", "sigma"), hs):
                sv[name][g0:g0 + w] = v[lo:lo + w]

    def wrap(kr, ki):
        re = out[kr]
        return MatrixPlanePair(re.shape[0], re.shape[1], re, out[ki] if cplx else None, cplx)

    return GsvdResult(wrap("Ur", "Ui"), wrap("Vr", "Vi"), wrap("Zr", "Zi"), sv["sigmaF"], sv["sigmaG"],
                      sv["sigma"], sweeps=sweeps, total_transforms=total, big_transforms=big,
                      converged=converged, workers=s)


def unborder(r, pb):
    """_unborder (blocked.py:593-620) on a host GsvdResult: keep the columns
    whose Z support in the padded rows is exactly zero."""
    n, n0 = pb.n, pb.original_n
    mF0, mG0 = pb.original_mF, pb.original_mG
    if n == n0 and r.U.rows == mF0 and r.V.rows == mG0:
        return r
    if n > n0:
        pad = np.abs(r.Z.re[n0:, :])
        if r.Z.is_complex:
            pad = pad + np.abs(r.Z.im[n0:, :])
        keep = np.flatnonzero(pad.sum(axis=0) == 0.0)
    else:
        keep = np.arange(n)
    if keep.size != n0:
        raise RankError("bordered solve mixed padded and original columns")
    return _select(r, keep, (mF0, mG0, n0))


def sort_descending(r):
    """_sort_descending (blocked.py:623-637): stable sort by -sigma."""
    order = np.argsort(-r.sigma, kind="stable")
    return _select(r, order, (r.U.rows, r.V.rows, r.Z.rows))


def _select(r, cols, rows):
    def cut(m, nr):
        im = np.asfortranarray(m.im[:nr, cols]) if m.is_complex else None
        return MatrixPlanePair(nr, len(cols), np.asfortranarray(m.re[:nr, cols]), im, m.is_complex)

    return GsvdResult(cut(r.U, rows[0]), cut(r.V, rows[1]), cut(r.Z, rows[2]), r.sigmaF[cols], r.sigmaG[cols],
                      r.sigma[cols], sweeps=r.sweeps, total_transforms=r.total_transforms,
                      big_transforms=r.big_transforms, converged=r.converged, workers=r.workers)
