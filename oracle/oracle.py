"""CPU ORACLE -- test infrastructure, NOT product code.

ctypes front end of ``hzg_oracle.c`` plus a numpy restatement of the
reference's driver glue (``solve`` / bordering / unbordering / sorting,
pkg/src/hzgsvd/blocked.py:593-663, core.py:186-218).  Only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py``'s CPU legs may import this
module, and only as the checker or the timed CPU baseline.

Parity status: pinned.  ``tests/golden/make_golden.py`` runs the reference
package itself (imported from /root/reference in the build container) on
fixed inputs and stores its outputs; ``tests/test_oracle.py`` requires this
oracle to reproduce them bitwise.
"""

import ctypes
import math
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "_build", "libhzg_oracle.so")

OK, RANK, NOT_PD, INVALID = 0, 1, 2, 4
EPS = 2.0 ** -52


class OracleError(Exception):
    def __init__(self, code, msg=""):
        super().__init__("oracle status %d %s" % (code, msg))
        self.code = code


class _Cfg(ctypes.Structure):
    _fields_ = [("prescale", ctypes.c_int), ("compensated", ctypes.c_int), ("crit_c2", ctypes.c_int),
                ("sorting", ctypes.c_int), ("max_inner_sweeps", ctypes.c_int),
                ("max_outer_sweeps", ctypes.c_int), ("block_width", ctypes.c_int),
                ("outer_mm", ctypes.c_int), ("inner_mm", ctypes.c_int), ("fallback_qr", ctypes.c_int),
                ("shorten_qr", ctypes.c_int), ("gate_eps", ctypes.c_double)]


class _Stats(ctypes.Structure):
    _fields_ = [("sweeps", ctypes.c_int64), ("total", ctypes.c_int64), ("big", ctypes.c_int64),
                ("converged", ctypes.c_int), ("fail_pair", ctypes.c_int), ("step_seconds", ctypes.c_double)]


def build():
    """Compile the oracle with its Makefile (gcc only)."""
    subprocess.run(["make", "-s", "-C", HERE], check=True)


_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            build()
        L = ctypes.CDLL(LIB_PATH)
        P = ctypes.c_void_p
        L.hzo_gsvd_blocked.argtypes = [ctypes.c_int64, ctypes.c_int64, ctypes.c_int64, ctypes.c_int,
                                       P, P, P, P, P, P, ctypes.POINTER(_Cfg), ctypes.c_double,
                                       P, P, P, ctypes.POINTER(_Stats), ctypes.c_int, ctypes.c_int64]
        L.hzo_block_inner.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.POINTER(_Cfg), ctypes.c_double,
                                      P, P, P, P, P, P, ctypes.POINTER(ctypes.c_int64),
                                      ctypes.POINTER(ctypes.c_int64)]
        L.hzo_cholesky_upper.argtypes = [ctypes.c_int, ctypes.c_int, P, P]
        L.hzo_gen_table.argtypes = [ctypes.c_int, ctypes.c_int, P]
        L.hzo_transform.argtypes = [ctypes.c_int] + [ctypes.c_double] * 6 + [P]
        L.hzo_grammian.argtypes = [ctypes.c_int64, ctypes.c_int64, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                   P, P, ctypes.c_int64, ctypes.c_int64, P, P]
        L.hzo_qr_shorten.argtypes = [ctypes.c_int64, ctypes.c_int, ctypes.c_int, P, P, P, P]
        L.hzo_qr_rfactor.argtypes = [ctypes.c_int64, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_double,
                                     P, P, P]
        L.hzo_tree_reduce.argtypes = [P, ctypes.c_int64]
        L.hzo_tree_reduce.restype = ctypes.c_double
        _lib = L
    return _lib


def _p(a):
    return ctypes.c_void_p(a.ctypes.data)


def make_cfg(variant_id=0, outer_kind="me", inner_kind="me", blocking="fb", sorting=True,
             max_inner_sweeps=0, max_outer_sweeps=30, block_width=8, gate_eps=EPS,
             fallback_qr=True, shorten="grammian"):
    """SolverConfig decode (pointwise.py:40-81) into the C struct."""
    if max_inner_sweeps <= 0:
        max_inner_sweeps = 30 if blocking == "fb" else 1
    return _Cfg(int(variant_id in (0, 1, 4, 5)), int(variant_id % 2 == 1), int(variant_id >= 4),
                int(bool(sorting)), max_inner_sweeps, max_outer_sweeps, block_width,
                int(outer_kind == "mm"), int(inner_kind == "mm"), int(bool(fallback_qr)),
                int(shorten == "qr"), gate_eps)


def cfg_from(cfg):
    """C struct from any object with SolverConfig's fields."""
    return make_cfg(cfg.variant_id, cfg.outer_kind, cfg.inner_kind, cfg.blocking, cfg.sorting,
                    cfg.max_inner_sweeps, cfg.max_outer_sweeps, cfg.block_width, cfg.gate_eps,
                    cfg.fallback_qr, cfg.shorten)


def sample_steps(Fp, Gp, cfg, steps, threads=None):
    """bench.py's CPU sample: prescale the bordered real planes, run the
    listed outer steps of sweep 1 (reference task pool, all threads),
    return the seconds spent in the steps (hzo_sample_steps)."""
    L = lib()
    P = ctypes.c_void_p
    L.hzo_sample_steps.argtypes = [ctypes.c_int64, ctypes.c_int64, ctypes.c_int64, ctypes.c_int, P, P, P, P, P, P,
                                   ctypes.POINTER(_Cfg), ctypes.c_int, P, ctypes.c_int,
                                   ctypes.POINTER(ctypes.c_double)]
    Fr = np.asfortranarray(Fp, dtype=np.float64).copy(order="F")
    Gr = np.asfortranarray(Gp, dtype=np.float64).copy(order="F")
    mF, n = Fr.shape
    Fi = np.zeros_like(Fr, order="F")
    Gi = np.zeros_like(Gr, order="F")
    Zr = np.zeros((n, n), order="F")
    Zi = np.zeros((n, n), order="F")
    st = np.ascontiguousarray(steps, dtype=np.int32)
    sec = ctypes.c_double(0.0)
    rc = L.hzo_sample_steps(mF, Gr.shape[0], n, 0, _p(Fr), _p(Fi), _p(Gr), _p(Gi), _p(Zr), _p(Zi), ctypes.byref(cfg),
                            threads or (os.cpu_count() or 1), _p(st), st.size, ctypes.byref(sec))
    if rc:
        raise OracleError(rc, "sample_steps")
    return sec.value


def gen_table(kind, n):
    """strategies.py:45-93 -> int32 (steps, n/2, 2)."""
    out = np.zeros((n, n // 2, 2), dtype=np.int32)
    steps = lib().hzo_gen_table(int(kind == "mm"), n, _p(out))
    return out[:steps].copy()


def tree_reduce(x):
    x = np.ascontiguousarray(x, dtype=np.float64)
    return lib().hzo_tree_reduce(_p(x), x.size)


def preprocess_tall(F, G):
    """Restatement of preprocess_tall (blocked.py:405-428) on dense numpy
    F (m x n), G (p x n): returns (F'', G'', piv) or raises OracleError
    (code 1) like the reference's RankError."""
    n = F.shape[1]
    EPSN = n * 2.0 ** -52

    def qr(A):
        cplx = np.iscomplexobj(A)
        Ar = np.array(np.real(A), dtype=np.float64, order="F", copy=True)
        Ai = np.array(np.imag(A), dtype=np.float64, order="F", copy=True) if cplx else np.zeros_like(Ar, order="F")
        jp = np.arange(n, dtype=np.int64)
        rc = lib().hzo_qr_rfactor(A.shape[0], n, int(cplx), 1, EPSN, _p(Ar), _p(Ai), _p(jp))
        R = Ar[:n, :] + 1j * Ai[:n, :] if cplx else Ar[:n, :].copy()
        return rc, R, jp

    rc, RF, jp1 = qr(F)
    if rc:
        raise OracleError(1, "numerically rank-deficient F in the preprocessing")
    rc, RG, jp2 = qr(G[:, jp1])
    if rc:
        raise OracleError(1, "numerically rank-deficient G in the preprocessing")
    return RF[:, jp2], RG, jp1[jp2]


def cholesky_upper(A):
    """blocked.py:59-94 on a dense (tw, tw) array; returns (R, status)."""
    A = np.asarray(A)
    cplx = np.iscomplexobj(A)
    Ar = np.asfortranarray(A.real.astype(np.float64))
    Ai = np.asfortranarray(A.imag.astype(np.float64)) if cplx else np.zeros_like(Ar, order="F")
    st = lib().hzo_cholesky_upper(A.shape[0], int(cplx), _p(Ar), _p(Ai))
    return (Ar + 1j * Ai if cplx else Ar), st


def grammian(Yr, Yi, c0, c1, w, cplx, comp=False):
    """blocked.py:40-56 for columns [c0, c0+w) u [c1, c1+w) of a Fortran plane."""
    Yr = np.asfortranarray(Yr, dtype=np.float64)
    Yi = np.asfortranarray(Yi if Yi is not None else np.zeros_like(Yr), dtype=np.float64)
    tw = 2 * w
    Ar = np.zeros((tw, tw), order="F")
    Ai = np.zeros((tw, tw), order="F")
    lib().hzo_grammian(Yr.shape[0], Yr.shape[0], w, int(cplx), int(comp), _p(Yr), _p(Yi), c0, c1, _p(Ar), _p(Ai))
    return Ar, Ai


def block_inner(Fh, Gh, cfg, epsn):
    """Prescale -> pointwise sweeps -> theta rescale on tw x tw factors
    (blocked.py:463-479).  Returns (F', G', Z~, total, big, status)."""
    Fh = np.asarray(Fh)
    cplx = np.iscomplexobj(Fh) or np.iscomplexobj(Gh)
    tw = Fh.shape[0]

    def planes(a):
        a = np.asarray(a, dtype=np.complex128 if cplx else np.float64)
        re = np.asfortranarray(a.real.copy())
        im = np.asfortranarray(a.imag.copy()) if cplx else np.zeros((tw, tw), order="F")
        return re, im

    Fr, Fi = planes(Fh)
    Gr, Gi = planes(Gh)
    Zr = np.zeros((tw, tw), order="F")
    Zi = np.zeros((tw, tw), order="F")
    tot = ctypes.c_int64(0)
    big = ctypes.c_int64(0)
    st = lib().hzo_block_inner(tw, int(cplx), ctypes.byref(cfg), epsn, _p(Fr), _p(Fi), _p(Gr), _p(Gi),
                               _p(Zr), _p(Zi), ctypes.byref(tot), ctypes.byref(big))
    j = (lambda r, i: r + 1j * i) if cplx else (lambda r, i: r)
    return j(Fr, Fi), j(Gr, Gi), j(Zr, Zi), tot.value, big.value, st


def transform(cplx, a11, a12r, a12i, a22, b12r, b12i):
    o = np.zeros(8)
    lib().hzo_transform(int(cplx), a11, a12r, a12i, a22, b12r, b12i, _p(o))
    return o


# ---------------------------------------------------------------------------
# driver glue (numpy restatement of blocked.py:593-663 and core.py:186-218)
# ---------------------------------------------------------------------------

def _planes_of(a):
    a = np.asarray(a)
    if np.iscomplexobj(a):
        return (np.asfortranarray(a.real.astype(np.float64)),
                np.asfortranarray(a.imag.astype(np.float64)), True)
    return np.asfortranarray(a.astype(np.float64)), None, False


def border_one(re, im, pad_cols, row_multiple):
    """core.py:186-200."""
    rows, cols = re.shape
    rows_new = -(-(rows + pad_cols) // row_multiple) * row_multiple
    cols_new = cols + pad_cols
    R = np.zeros((rows_new, cols_new), order="F")
    R[:rows, :cols] = re
    for k in range(pad_cols):
        R[rows + k, cols + k] = 1.0
    I = None
    if im is not None:
        I = np.zeros((rows_new, cols_new), order="F")
        I[:rows, :cols] = im
    return R, I


def gsvd_blocked(Fr, Fi, Gr, Gi, cplx, cfg, threads=None, step_limit=-1, epsn=0.0):
    """blocked.py:553-586 on bordered planes; returns a dict of results."""
    mF, n = Fr.shape
    mG = Gr.shape[0]
    Fr = np.asfortranarray(Fr.copy())
    Gr = np.asfortranarray(Gr.copy())
    Fi = np.asfortranarray(Fi.copy()) if Fi is not None else np.zeros_like(Fr, order="F")
    Gi = np.asfortranarray(Gi.copy()) if Gi is not None else np.zeros_like(Gr, order="F")
    Zr = np.zeros((n, n), order="F")
    Zi = np.zeros((n, n), order="F")
    sF = np.zeros(n)
    sG = np.zeros(n)
    s = np.zeros(n)
    st = _Stats()
    thr = threads if threads else (os.cpu_count() or 1)
    code = lib().hzo_gsvd_blocked(mF, mG, n, int(cplx), _p(Fr), _p(Fi), _p(Gr), _p(Gi), _p(Zr), _p(Zi),
                                  ctypes.byref(cfg), epsn, _p(sF), _p(sG), _p(s), ctypes.byref(st), thr,
                                  step_limit)
    return dict(status=code, U=(Fr, Fi), V=(Gr, Gi), Z=(Zr, Zi), sigmaF=sF, sigmaG=sG, sigma=s,
                sweeps=st.sweeps, total=st.total, big=st.big, converged=bool(st.converged),
                step_seconds=st.step_seconds)


def solve(F, G, cfg=None, threads=None):
    """blocked.py:640-663 for workers=1: border, solve, unborder, stable
    descending sort.  F, G dense numpy arrays.  Returns a dict with dense
    U, V, Z (complex when the pair is) and the sigma vectors."""
    cfg = cfg if cfg is not None else make_cfg()
    Fr, Fi, cplx = _planes_of(F)
    Gr, Gi, _ = _planes_of(G)
    mF0, n0 = Fr.shape
    mG0 = Gr.shape[0]
    if n0 == 1:
        raise NotImplementedError("n = 1 uses the closed form (pointwise.py:324-345)")
    w = cfg.block_width
    pad = (-n0) % (2 * w)
    if pad or mF0 % (2 * w) or mG0 % (2 * w):
        Fr, Fi = border_one(Fr, Fi, pad, 2 * w)
        Gr, Gi = border_one(Gr, Gi, pad, 2 * w)
    r = gsvd_blocked(Fr, Fi, Gr, Gi, cplx, cfg, threads)
    if r["status"] != OK:
        raise OracleError(r["status"])
    n = Fr.shape[1]
    Zr, Zi = r["Z"]
    if n > n0:
        padm = np.abs(Zr[n0:, :])
        if cplx:
            padm = padm + np.abs(Zi[n0:, :])
        keep = np.where(padm.sum(axis=0) == 0.0)[0]
        if keep.size != n0:
            raise OracleError(RANK, "unborder")
    else:
        keep = np.arange(n)
    sig = r["sigma"][keep]
    order = keep[np.argsort(-sig, kind="stable")]

    def dense(pl, rows):
        re, im = pl
        out = re[:rows, order]
        if cplx:
            out = out + 1j * im[:rows, order]
        return np.asfortranarray(out)

    return dict(U=dense(r["U"], mF0), V=dense(r["V"], mG0), Z=dense(r["Z"], n0),
                sigmaF=r["sigmaF"][order], sigmaG=r["sigmaG"][order], sigma=r["sigma"][order],
                sweeps=r["sweeps"], total=r["total"], big=r["big"], converged=r["converged"])


# ---------------------------------------------------------------------------
# generators (harness.py:43-71, numpy restatement; gaussian_stream is numpy
# code in the reference too, so this is bitwise the same stream)
# ---------------------------------------------------------------------------

def uniform_stream(seed, count):
    """splitmix64 uniforms on (0, 1) (harness.py:43-63)."""
    gamma = np.uint64(0x9E3779B97F4A7C15)
    idx = np.arange(1, count + 1, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = np.uint64(int(seed) % (1 << 64)) + idx * gamma
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        z = z ^ (z >> np.uint64(31))
    return ((z >> np.uint64(11)).astype(np.float64) + 0.5) * (2.0 ** -53)


def gaussian_stream(seed, count):
    """Box-Muller over the splitmix64 uniforms (harness.py:66-71)."""
    u = uniform_stream(seed, 2 * count)
    r = np.sqrt(-2.0 * np.log(u[0::2]))
    a = 2.0 * math.pi * u[1::2]
    return r * np.cos(a)


# ---------------------------------------------------------------------------
# deterministic fixture inputs for the north-star configurations (hzo_gen.c).
# numpy's SIMD log/cos differ between hosts in the last bit (1,680 of 2^20
# values here vs glibc), so the fixtures regenerate their inputs in C.
# ---------------------------------------------------------------------------

def gaussian_c(seed, count):
    """harness.py:66-71 with glibc log/cos (host-independent bytes)."""
    L = lib()
    L.hzo_gaussian_fill.argtypes = [ctypes.c_uint64, ctypes.c_int64, ctypes.c_void_p]
    out = np.empty(int(count))
    L.hzo_gaussian_fill(int(seed) % (1 << 64), out.size, _p(out))
    return out


def gen_cond(n, seed):
    """SURVEY 8(d) config 4 pair (sigma in [1e-8, 1e8]); returns (F, G, sigma_true)."""
    L = lib()
    L.hzo_gen_cond.argtypes = [ctypes.c_int64, ctypes.c_uint64, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p]
    F = np.empty((n, n), order="F")
    G = np.empty((n, n), order="F")
    s = np.empty(n)
    if L.hzo_gen_cond(n, int(seed), _p(F), _p(G), _p(s)):
        raise MemoryError("hzo_gen_cond")
    return F, G, s


NS_CONFIGS = {
    # name: (BASELINE.json config index, description)
    "config2": (1, "real 1024 x 1024, iid Gaussian (hzo_gaussian_fill seed 1024), w=16"),
    "config3": (2, "complex F 3072 x 2048, G 2048 x 2048, iid Gaussian re/im (seeds 31..34), w=16"),
    "config4": (3, "real 4096 x 4096, sigma = shuffled logspace(-8, 8) (hzo_gen_cond seed 4), w=16, "
                   "max_outer_sweeps=100"),
}


def ns_inputs(name, scale=1):
    """Inputs of a north-star fixture: (F, G, cfg kwargs, extra).  `scale`
    divides every dimension (for quick self-tests of the machinery)."""
    if name == "config2":
        n = 1024 // scale
        g = gaussian_c(1024, 2 * n * n)
        return (g[: n * n].reshape((n, n), order="F"), g[n * n:].reshape((n, n), order="F"),
                dict(block_width=16), {})
    if name == "config3":
        m, n = 3072 // scale, 2048 // scale
        F = (gaussian_c(31, m * n) + 1j * gaussian_c(32, m * n)).reshape((m, n), order="F")
        G = (gaussian_c(33, n * n) + 1j * gaussian_c(34, n * n)).reshape((n, n), order="F")
        return F, G, dict(block_width=16), {}
    if name == "config4":
        n = 4096 // scale
        F, G, s = gen_cond(n, 4)
        return F, G, dict(block_width=16, max_outer_sweeps=100), {"sigma_true": np.sort(s)[::-1].copy()}
    raise KeyError(name)


def sha256_planes(*arrays):
    """SHA-256 over the Fortran-order bytes of real planes (complex arrays
    contribute their real then imaginary plane)."""
    import hashlib
    h = hashlib.sha256()
    for a in arrays:
        a = np.asarray(a)
        parts = (a.real, a.imag) if np.iscomplexobj(a) else (a,)
        for p in parts:
            h.update(np.asfortranarray(p, dtype=np.float64).tobytes(order="F"))
    return h.hexdigest()
