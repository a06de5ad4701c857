"""The GSVD entry points on the B200 path.

``solve`` keeps the reference's contract (blocked.py:640-663): numpy or
MatrixPlanePair inputs, bordering, unbordering and a stable descending sort,
a GsvdResult of numpy planes.  Underneath, the pair is copied to the GPU,
bordered there, and every outer sweep runs in libhzg.so (hzg_sweep); only
the two sweep counters come back to the host per sweep.

``DeviceGsvd`` is the device-resident form used by the benchmark and by
callers that already hold torch tensors: planes stay in HBM from input to
output.
"""

import ctypes
import dataclasses
import math
import os
import threading

import numpy as np

from . import _native
from .config import SolverConfig
from .core import GsvdResult, MatrixPlanePair, ProblemPair, bordered_shape
from .errors import DeviceError, RankError


def _torch():
    import torch
    if not torch.cuda.is_available():
        raise DeviceError("no CUDA device: the B200 path has no CPU fallback")
    return torch


def _ptr(t):
    return ctypes.c_void_p(t.data_ptr()) if t is not None else None


class DeviceGsvd:
    """One bordered problem resident on a GPU.

    planes: dict with keys Fr, Fi, Gr, Gi (torch float64 tensors of shape
    (n, m) -- column-major planes; imaginary ones None for real problems)
    already bordered to multiples of 2w.  Z planes and the workspace are
    allocated here unless ``Z`` = (Zr, Zi) tensors of shape (n, zrows) are
    given; ``zrows`` (default n) is the height of Z -- a stripe slab of
    the reference's distributed scheme keeps the n global rows of Z for its
    2W columns (stripes.py).
    """

    def __init__(self, planes, cfg, device=None, epsn=None, schedule=None, zrows=None, Z=None):
        torch = _torch()
        self.cfg = cfg
        self.torch = torch
        Fr, Gr = planes["Fr"], planes["Gr"]
        self.device = Fr.device if device is None else torch.device(device)
        self.n, self.mF = Fr.shape
        self.mG = Gr.shape[1]
        self.cplx = planes.get("Fi") is not None
        self.planes = planes
        lib = _native.load()
        self.lib = lib
        ccfg = _native.make_config(cfg)
        ctx = ctypes.c_void_p()
        _native.check(lib.hzg_create(ctypes.byref(ctx), self.device.index or 0, self.mF, self.mG, self.n,
                                     int(self.cplx), ctypes.byref(ccfg), float(epsn or 0.0)),
                      None, "hzg_create (n=%d, mF=%d, mG=%d, w=%d)" % (self.n, self.mF, self.mG, cfg.block_width))
        self.ctx = ctx
        if schedule is not None:
            sched = np.ascontiguousarray(schedule, dtype=np.int32)
            _native.check(lib.hzg_set_schedule(ctx, sched.ctypes.data_as(ctypes.c_void_p), sched.shape[0],
                                               sched.shape[1]), ctx, "hzg_set_schedule")
        zrows = self.n if zrows is None else int(zrows)
        if zrows != self.n:
            _native.check(lib.hzg_set_z_rows(ctx, zrows), ctx, "hzg_set_z_rows")
        kw = dict(dtype=torch.float64, device=self.device)
        if Z is not None:
            self.Zr, self.Zi = Z
            if tuple(self.Zr.shape) != (self.n, zrows) or not self.Zr.is_contiguous():
                raise ValueError("Z planes must be contiguous (n, zrows) tensors")
        else:
            self.Zr = torch.empty((self.n, zrows), **kw)
            self.Zi = torch.empty((self.n, zrows), **kw) if self.cplx else None
        self.ws = torch.empty(int(lib.hzg_workspace_bytes(ctx)), dtype=torch.uint8, device=self.device)
        self.stream = torch.cuda.current_stream(self.device)
        _native.check(lib.hzg_bind(ctx, _ptr(Fr), _ptr(planes.get("Fi")), _ptr(Gr), _ptr(planes.get("Gi")),
                                   _ptr(self.Zr), _ptr(self.Zi), _ptr(self.ws),
                                   ctypes.c_void_p(self.stream.cuda_stream)), ctx, "hzg_bind")
        self.sweeps = 0
        self.total = 0
        self.big = 0
        self.converged = False

    def close(self):
        if getattr(self, "ctx", None) is not None:
            self.lib.hzg_destroy(self.ctx)
            self.ctx = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def init(self):
        self.sweeps = 0
        self.total = 0
        self.big = 0
        self.converged = False
        _native.check(self.lib.hzg_init_fgz(self.ctx), self.ctx, "prescale")

    def set_timing(self, on=True):
        _native.check(self.lib.hzg_set_timing(self.ctx, int(bool(on))), self.ctx, "set_timing")

    def kernel_times(self, reset=False):
        """{kind: (ms, launches)} for kind in grammian / inner / postmult."""
        ms = np.zeros(3)
        cnt = np.zeros(3, dtype=np.int64)
        _native.check(self.lib.hzg_kernel_times(self.ctx, ms.ctypes.data_as(ctypes.c_void_p),
                                                cnt.ctypes.data_as(ctypes.c_void_p), int(bool(reset))),
                      self.ctx, "kernel_times")
        return {k: (float(ms[i]), int(cnt[i])) for i, k in enumerate(("grammian", "inner", "postmult"))}

    def sweep(self):
        tot = ctypes.c_int64(0)
        big = ctypes.c_int64(0)
        _native.check(self.lib.hzg_sweep(self.ctx, ctypes.byref(tot), ctypes.byref(big)), self.ctx, "sweep")
        return tot.value, big.value

    def sweep_launch(self):
        """Queue one sweep on the bound stream (returns immediately)."""
        _native.check(self.lib.hzg_sweep_launch(self.ctx), self.ctx, "sweep")

    def sweep_wait(self):
        """Wait for the queued sweep: (total, big)."""
        tot = ctypes.c_int64(0)
        big = ctypes.c_int64(0)
        _native.check(self.lib.hzg_sweep_wait(self.ctx, ctypes.byref(tot), ctypes.byref(big)), self.ctx, "sweep")
        return tot.value, big.value

    def run(self, max_sweeps=None):
        """_algorithm1_loop (blocked.py:503-550) with the device doing the work."""
        self.init()
        cap = self.cfg.max_outer_sweeps if max_sweeps is None else max_sweeps
        for _ in range(cap):
            t, b = self.sweep()
            self.sweeps += 1
            self.total += t
            self.big += b
            if b == 0:
                self.converged = True
                break
        return self

    def collect(self):
        """Fold the per-pair counters of the schedule's steps (one sweep run
        step by step): (total, big)."""
        tot = ctypes.c_int64(0)
        big = ctypes.c_int64(0)
        _native.check(self.lib.hzg_collect(self.ctx, ctypes.byref(tot), ctypes.byref(big)), self.ctx, "collect")
        return tot.value, big.value

    def collect_status(self):
        """collect() without raising: (total, big, status code), so a
        multi-process caller can agree on the error before raising it."""
        tot = ctypes.c_int64(0)
        big = ctypes.c_int64(0)
        rc = self.lib.hzg_collect(self.ctx, ctypes.byref(tot), ctypes.byref(big))
        if rc not in (_native.HZG_OK, _native.HZG_RANK, _native.HZG_NOT_PD):
            _native.check(rc, self.ctx, "collect")
        return tot.value, big.value, rc

    def dist_sweep(self):
        """One outer sweep of this rank with the NCCL block exchange and
        counter all-reduce inside the library (hzg_dist_sweep): global
        (total, big)."""
        tot = ctypes.c_int64(0)
        big = ctypes.c_int64(0)
        _native.check(self.lib.hzg_dist_sweep(self.ctx, ctypes.byref(tot), ctypes.byref(big)), self.ctx,
                      "dist_sweep")
        return tot.value, big.value

    def dist_sweep_wait(self):
        """Wait for a sweep queued with hzg_dist_sweep_launch: global (total, big)."""
        tot = ctypes.c_int64(0)
        big = ctypes.c_int64(0)
        _native.check(self.lib.hzg_dist_sweep_wait(self.ctx, ctypes.byref(tot), ctypes.byref(big)), self.ctx,
                      "dist_sweep")
        return tot.value, big.value

    def comm_attach(self, nranks, rank, unique_id):
        """Attach an NCCL communicator (hzg_comm_attach; collective)."""
        buf = ctypes.create_string_buffer(bytes(unique_id), len(unique_id))
        _native.check(self.lib.hzg_comm_attach(self.ctx, nranks, rank, buf), self.ctx, "comm_attach")

    def comm_set_moves(self, moves_per_step):
        """moves_per_step[k] = [(block, src, dst), ...] after step k."""
        offs = np.zeros(len(moves_per_step) + 1, dtype=np.int32)
        flat = []
        for k, mv in enumerate(moves_per_step):
            flat.extend(x for m in mv for x in m)
            offs[k + 1] = offs[k] + len(mv)
        arr = np.asarray(flat if flat else [0], dtype=np.int32)
        _native.check(self.lib.hzg_comm_set_moves(self.ctx, arr.ctypes.data_as(ctypes.c_void_p),
                                                  offs.ctypes.data_as(ctypes.c_void_p), len(moves_per_step)),
                      self.ctx, "comm_set_moves")

    def comm_exchange(self, moves):
        """Immediate grouped NCCL exchange of whole blocks (block, src, dst)."""
        arr = np.asarray([x for m in moves for x in m] or [0], dtype=np.int32)
        _native.check(self.lib.hzg_comm_exchange(self.ctx, arr.ctypes.data_as(ctypes.c_void_p), len(moves)),
                      self.ctx, "comm_exchange")

    def rescale_z(self):
        _native.check(self.lib.hzg_rescale_z(self.ctx), self.ctx, "rescale_z")

    def step_counters(self):
        """int32 (osteps, npairs, 4): total, big, status, inner sweeps of the last sweep."""
        cnt = ctypes.c_int64(0)
        self.lib.hzg_step_counters(self.ctx, None, 0, ctypes.byref(cnt))
        out = np.zeros(cnt.value, dtype=np.int32)
        _native.check(self.lib.hzg_step_counters(self.ctx, out.ctypes.data_as(ctypes.c_void_p), out.size,
                                                 ctypes.byref(cnt)), self.ctx, "step_counters")
        return out.reshape(-1, self.n // self.cfg.block_width // 2, 4)

    def launch_counts(self):
        """(kernel launches per sweep, launches per solve outside the sweeps)."""
        a = ctypes.c_int64(0)
        b = ctypes.c_int64(0)
        _native.check(self.lib.hzg_launch_counts(self.ctx, ctypes.byref(a), ctypes.byref(b)), self.ctx,
                      "launch_counts")
        return a.value, b.value

    def run_steps(self, first, count):
        _native.check(self.lib.hzg_run_steps(self.ctx, first, count), self.ctx, "run_steps")

    def run_pairs(self, step, p0, pn, stream=None):
        """Pairs [p0, p0 + pn) of outer step ``step`` on ``stream`` (a torch
        stream; None: the bound stream), asynchronously."""
        s = ctypes.c_void_p(stream.cuda_stream) if stream is not None else None
        _native.check(self.lib.hzg_run_pairs(self.ctx, step, p0, pn, s), self.ctx, "run_pairs")

    def wave_step(self, step, groups, comm=None, zcomm=None):
        """Step ``step`` as ``groups`` position groups on library streams,
        ordered against the exchange streams ``comm`` (F, G and, without
        ``zcomm``, Z blocks) and ``zcomm`` (Z blocks) (hzg_wave_step)."""
        _native.check(self.lib.hzg_wave_step(self.ctx, step, groups, _sptr(comm), _sptr(zcomm)), self.ctx,
                      "wave_step")

    def wave_join(self, comm=None, zcomm=None):
        _native.check(self.lib.hzg_wave_join(self.ctx, _sptr(comm), _sptr(zcomm)), self.ctx, "wave_join")

    def finalize(self, n0=None, mF0=None, mG0=None, sort=True):
        """Final rescale, unborder, sort; returns device output tensors."""
        torch = self.torch
        n0 = self.n if n0 is None else n0
        mF0 = self.mF if mF0 is None else mF0
        mG0 = self.mG if mG0 is None else mG0
        kw = dict(dtype=torch.float64, device=self.device)
        out = dict(Ur=torch.empty((n0, mF0), **kw), Vr=torch.empty((n0, mG0), **kw),
                   Zr=torch.empty((n0, n0), **kw), sigmaF=torch.empty(n0, **kw), sigmaG=torch.empty(n0, **kw),
                   sigma=torch.empty(n0, **kw))
        for k, shape in (("Ui", (n0, mF0)), ("Vi", (n0, mG0)), ("Zi", (n0, n0))):
            out[k] = torch.empty(shape, **kw) if self.cplx else None
        _native.check(self.lib.hzg_finalize(self.ctx, n0, mF0, mG0, int(bool(sort)), _ptr(out["Ur"]),
                                            _ptr(out["Ui"]), _ptr(out["Vr"]), _ptr(out["Vi"]), _ptr(out["Zr"]),
                                            _ptr(out["Zi"]), _ptr(out["sigmaF"]), _ptr(out["sigmaG"]),
                                            _ptr(out["sigma"])), self.ctx, "finalize")
        return out


def _sptr(stream):
    return ctypes.c_void_p(stream.cuda_stream) if stream is not None else None


def _planes_of(m):
    """numpy (re, im or None) Fortran planes of a MatrixPlanePair."""
    return m.re, (m.im if m.is_complex else None)


def upload_bordered(F, G, w, device=None, torch=None, out=None):
    """Copy (F, G) to the GPU and border them there exactly like
    border_pair(p, 2w, 2w) (core.py:186-218): pad columns carry a single 1
    on the extended diagonal, pad rows are zero.  ``out``: planes of the
    same bordered shape to fill instead of allocating."""
    torch = torch or _torch()
    dev = torch.device("cuda", torch.cuda.current_device()) if device is None else torch.device(device)
    n0 = F.cols
    padF, mF = bordered_shape(n0, F.rows, 2 * w, 2 * w)
    padG, mG = bordered_shape(n0, G.rows, 2 * w, 2 * w)
    n = n0 + padF
    dst = out
    out = {}
    for key, M, m in (("F", F, mF), ("G", G, mG)):
        re, im = _planes_of(M)
        for suffix, host in (("r", re), ("i", im)):
            if host is None:
                out[key + suffix] = None
                continue
            if dst is not None:
                d = dst[key + suffix]
                if n0 < n or M.rows < m:
                    d.zero_()
            else:
                d = torch.zeros((n, m), dtype=torch.float64, device=dev)
            h = torch.from_numpy(np.asfortranarray(host).T)
            d[:n0, :M.rows].copy_(h, non_blocking=True)
            if suffix == "r" and padF:
                k = torch.arange(padF, device=dev)
                d[n0 + k, M.rows + k] = 1.0
            out[key + suffix] = d
    return out, n, mF, mG


def _to_host(t):
    """Start the copy of a device tensor into pinned host memory (torch's
    caching host allocator: blocks freed with the caller's arrays are reused
    by the next solve).  Synchronize before reading."""
    torch = _torch()
    h = torch.empty(t.shape, dtype=t.dtype, pin_memory=True)
    h.copy_(t, non_blocking=True)
    return h


def gsvd_1x1(F, G):
    """Closed form for a single-column pair (pointwise.py:324-345)."""
    from .reftree import norm_sq
    f = F.to_dense()[:, 0]
    g = G.to_dense()[:, 0]
    nf2 = norm_sq(f, F.field)
    ng2 = norm_sq(g, G.field)
    if not (nf2 > 0.0 and ng2 > 0.0):
        raise RankError("zero column in a 1x1 problem")
    nf = math.sqrt(nf2)
    ng = math.sqrt(ng2)
    rt = math.sqrt(nf2 + ng2)
    z = 1.0 / rt
    U = MatrixPlanePair.from_dense((f * (1.0 / nf)).reshape(-1, 1))
    V = MatrixPlanePair.from_dense((g * (1.0 / ng)).reshape(-1, 1))
    Z = MatrixPlanePair.from_dense(np.array([[z]]) if not F.is_complex else np.array([[complex(z, 0.0)]]))
    return GsvdResult(U, V, Z, np.array([nf / rt]), np.array([ng / rt]), np.array([nf / ng]), sweeps=0,
                      total_transforms=0, big_transforms=0, converged=True)


def _result_from_device(dev, out, cplx, workers=1):
    host = {k: _to_host(v) for k, v in out.items() if v is not None}
    _torch().cuda.current_stream().synchronize()

    def plane(kr, ki):
        re = host[kr].numpy().T
        im = host[ki].numpy().T if cplx else None
        return MatrixPlanePair(re.shape[0], re.shape[1], re, im, cplx)

    return GsvdResult(plane("Ur", "Ui"), plane("Vr", "Vi"), plane("Zr", "Zi"), host["sigmaF"].numpy(),
                      host["sigmaG"].numpy(), host["sigma"].numpy(), sweeps=dev.sweeps,
                      total_transforms=dev.total, big_transforms=dev.big, converged=dev.converged,
                      workers=workers)


def gsvd_blocked(p, cfg=None, epsn=None):
    """Full blocked solve of a bordered pair (column count a multiple of 2w),
    without unbordering or sorting (blocked.py:553-586)."""
    cfg = cfg or SolverConfig()
    w = cfg.block_width
    if p.n % (2 * w) != 0:
        raise ValueError("blocked solver needs n divisible by 2w; border first")
    # row counts that are not multiples of 2w are zero-padded on the device
    # (zero rows change no inner product) and cropped again by finalize
    planes, n, mF, mG = upload_bordered(p.F, p.G, w)
    dev = DeviceGsvd(planes, cfg, epsn=epsn)
    dev.run()
    out = dev.finalize(n, p.F.rows, p.G.rows, sort=False)
    r = _result_from_device(dev, out, p.is_complex)
    dev.close()
    return r


def solve(F, G, cfg=None, workers=1, worker_sweeps=1, scheme="stripes", keep_context=True, devices=None):
    """Border, solve on the GPU, unborder, and sort a GSVD problem
    (blocked.py:640-663).

    F and G may be MatrixPlanePair values or numpy arrays.  ``workers`` > 1
    selects a multi-worker schedule with ``scheme``:

    * "stripes" (default, the reference's semantics): the stripe-distributed
      scheme of distsim.py -- the pair is bordered to a multiple of
      2w * workers, each outermost step runs up to ``worker_sweeps`` sweeps
      on every worker's two-stripe slab, then the stripes move along the
      communication mapping.  Results depend on ``workers`` exactly as the
      reference's do (stripes.py);
    * "blocks": the B200 block-partitioned schedule (dist.py) -- the
      single-worker ME schedule with its block pairs split over ``workers``
      ranks; bitwise the single-worker result for any rank count (the
      multi-GPU production path; the ranks are virtual ranks on the current
      device, or -- with ``devices`` -- one GPU each driven from this
      process with the NCCL exchange inside libhzg; a torchrun job uses
      dist.solve_blocks(comm="dist")).

    ``keep_context`` (single worker): keep the device context (planes,
    workspace, captured sweep graph: about 3.3 n^2 doubles plus the inputs)
    for the next solve of the same shape and configuration, so the sweep
    graph is captured once; False releases it before returning
    (clear_cache() does the same at any time).
    """
    cfg = cfg or SolverConfig()
    if isinstance(F, np.ndarray):
        F = MatrixPlanePair.from_dense(F)
    if isinstance(G, np.ndarray):
        G = MatrixPlanePair.from_dense(G)
    if workers < 1:
        raise ValueError("need at least one worker")
    if scheme not in ("stripes", "blocks"):
        raise ValueError("scheme must be 'stripes' or 'blocks'")
    _torch()  # no device or no libhzg.so: fail loudly, also for the 1x1 closed form
    _native.load()
    if F.cols == 1:
        return gsvd_1x1(F, G)
    if (workers > 1 or devices is not None) and scheme == "blocks":
        from .dist import solve_blocks
        if devices is not None:  # one process driving one GPU per worker
            return solve_blocks(F, G, cfg, workers, comm="devices", devices=devices)
        return solve_blocks(F, G, cfg, workers)
    p = ProblemPair(F, G)
    if workers > 1:
        from .core import border_pair
        from .stripes import run_distributed, sort_descending, unborder
        w = cfg.block_width
        pb = border_pair(p, 2 * w * workers, 2 * w)
        return sort_descending(unborder(run_distributed(pb, cfg, workers, worker_sweeps), pb))
    with _cache_lock:
        dev = _cached_solver(p, cfg)
        try:
            dev.run()
            out = dev.finalize(p.n, p.F.rows, p.G.rows, sort=True)
            return _result_from_device(dev, out, p.is_complex, workers)
        finally:
            if not keep_context:
                clear_cache()


# The last solve's device context (planes, workspace, captured sweep graph)
# is kept for the next solve of the same shape and configuration: the graph
# is captured once instead of per call.
_cache_lock = threading.Lock()
_cache = {"key": None, "dev": None}


def _cached_solver(p, cfg):
    torch = _torch()
    w = cfg.block_width
    # the HZG_* performance variables shape the context too (graph layout,
    # stream use; none of them changes result bits), and so does the stream
    # the context was bound to
    knobs = tuple(sorted((k, v) for k, v in os.environ.items() if k.startswith("HZG_")))
    stream = torch.cuda.current_stream().cuda_stream
    key = (torch.cuda.current_device(), stream, p.n, p.F.rows, p.G.rows, p.is_complex,
           dataclasses.astuple(cfg), knobs)
    if _cache["key"] == key:
        dev = _cache["dev"]
        upload_bordered(p.F, p.G, w, out=dev.planes)
        return dev
    clear_cache()
    planes, n, mF, mG = upload_bordered(p.F, p.G, w)
    dev = DeviceGsvd(planes, cfg)
    _cache["key"], _cache["dev"] = key, dev
    return dev


def clear_cache():
    """Release the device context (planes, workspace, sweep graph: ~3.3 n^2
    doubles plus the inputs' size) that solve() keeps for the next call of
    the same shape."""
    dev = _cache["dev"]
    _cache["key"], _cache["dev"] = None, None
    if dev is not None:
        dev.close()
