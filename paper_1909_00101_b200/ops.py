"""Single block operations of the reference's public API on the device.

form_grammians, cholesky_upper, qr_shorten, postmultiply, rescale_z and
preprocess_tall keep the reference's signatures and results
(pkg/src/hzgsvd/blocked.py:328-428)
and run the same reference-order kernels the solver uses (bitwise the
reference), through the C ABI (include/hzg.h, hzg_op_*).  run_distributed
(distsim.py:147) is the reference's stripe-distributed scheme (stripes.py).
"""

import ctypes

import numpy as np

from . import _native
from .core import GsvdResult, MatrixPlanePair
from .errors import DeviceError


def _torch():
    import torch
    if not torch.cuda.is_available():
        raise DeviceError("no CUDA device: the B200 path has no CPU fallback")
    return torch


def _as_cols(Y):
    Y = np.asarray(Y)
    return Y.reshape(Y.shape[0], -1)


def _dev_planes(a, cplx, torch):
    """numpy (rows, cols) -> device column-major planes (cols, rows)."""
    a = np.asarray(a)
    dev = torch.device("cuda", torch.cuda.current_device())
    re = torch.from_numpy(np.ascontiguousarray(np.real(a).T, dtype=np.float64)).to(dev)
    im = torch.from_numpy(np.ascontiguousarray(np.imag(a).T, dtype=np.float64)).to(dev) if cplx else None
    return re, im


def _host(re, im):
    r = re.cpu().numpy().T
    return r + 1j * im.cpu().numpy().T if im is not None else r.copy()


def _p(t):
    return ctypes.c_void_p(t.data_ptr()) if t is not None else None


def _stream(torch):
    return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)


def _gram(stack, compensated, torch):
    cplx = np.iscomplexobj(stack)
    m, tw = stack.shape
    Yr, Yi = _dev_planes(stack, cplx, torch)
    Ar = torch.empty((tw, tw), dtype=torch.float64, device=Yr.device)
    Ai = torch.empty((tw, tw), dtype=torch.float64, device=Yr.device) if cplx else None
    L = _native.load()
    _native.check(L.hzg_op_grammian(m, tw // 2, int(cplx), int(bool(compensated)), _p(Yr), _p(Yi), _p(Ar), _p(Ai),
                                    _stream(torch)), None, "form_grammians")
    return _host(Ar, Ai)


def form_grammians(Fp, Fq, Gp, Gq, compensated=False):
    """Grammians of the stacked block-column pairs [Fp Fq] and [Gp Gq]
    (blocked.py:328-332)."""
    torch = _torch()
    A = _gram(np.hstack([_as_cols(Fp), _as_cols(Fq)]), compensated, torch)
    B = _gram(np.hstack([_as_cols(Gp), _as_cols(Gq)]), compensated, torch)
    return A, B


# block orders the device block kernels are instantiated for (2w; hzg_inner.cu)
BLOCK_ORDERS = (2, 4, 6, 8, 10, 12, 14, 16, 20, 24, 32, 48, 64)


def _check_order(tw, what):
    if tw not in BLOCK_ORDERS:
        raise ValueError("%s: order %d is not supported on the device (2w in %s)" % (what, tw, BLOCK_ORDERS))


def cholesky_upper(M):
    """Upper Cholesky factor with positive real diagonal (blocked.py:350-355);
    NotPositiveDefiniteError when the factorization breaks down."""
    M = np.array(M)
    cplx = np.iscomplexobj(M)
    tw = M.shape[0]
    if M.ndim != 2 or M.shape[1] != tw:
        raise ValueError("cholesky_upper needs a square matrix")
    _check_order(tw, "cholesky_upper")
    torch = _torch()
    Ar, Ai = _dev_planes(M, cplx, torch)
    _native.check(_native.load().hzg_op_cholesky_upper(tw, int(cplx), _p(Ar), _p(Ai), _stream(torch)), None,
                  "matrix is not numerically positive definite")
    return _host(Ar, Ai)


def qr_shorten(Yp, Yq):
    """R factor (nonnegative diagonal) of the stacked block-column pair
    (blocked.py:358-367); RankError on rank deficiency."""
    Yp, Yq = _as_cols(Yp), _as_cols(Yq)
    if Yp.shape[1] != Yq.shape[1]:
        # the device kernel factors a pair of equal-width block columns
        # (2w columns); it never truncates to fewer columns
        raise ValueError("qr_shorten on the device needs block columns of equal width (got %d and %d)"
                         % (Yp.shape[1], Yq.shape[1]))
    stack = np.hstack([Yp, Yq])
    cplx = np.iscomplexobj(stack)
    m, tw = stack.shape
    _check_order(tw, "qr_shorten")
    torch = _torch()
    Yr, Yi = _dev_planes(stack, cplx, torch)
    Rr = torch.empty((tw, tw), dtype=torch.float64, device=Yr.device)
    Ri = torch.empty((tw, tw), dtype=torch.float64, device=Yr.device) if cplx else None
    _native.check(_native.load().hzg_op_qr_shorten(m, tw // 2, int(cplx), _p(Yr), _p(Yi), _p(Rr), _p(Ri),
                                                   _stream(torch)), None,
                  "rank-deficient block columns in the QR shortening")
    return _host(Rr, Ri)


def qr_rfactor(Ar, Ai, pivot, jpvt, tol_scale):
    """In-place Householder R factor of device planes (column-major (cols,
    rows) float64 tensors; Ai None for real), with column pivoting into the
    int64 device tensor jpvt; returns the reference's flag (blocked.py:97-217:
    1 = a column vanished or a diagonal fell below tol_scale x its entry
    norm)."""
    torch = _torch()
    nc, m = Ar.shape
    res = ctypes.c_int32(0)
    _native.check(_native.load().hzg_op_qr_rfactor(m, nc, int(Ai is not None), int(bool(pivot)), float(tol_scale),
                                                    _p(Ar), _p(Ai), _p(jpvt), ctypes.byref(res), _stream(torch)),
                  None, "qr_rfactor")
    return res.value


def preprocess_tall(F, G):
    """Shorten a tall pair to square via two column-pivoted QR
    factorizations on the device (blocked.py:405-428): returns (F'', G'',
    piv) with column k of the shortened problem = original column piv[k];
    a Z'' of the shortened pair maps back by Z[piv[k], :] = Z''[k, :].
    Bitwise the reference (same fma order, same pivot ties)."""
    from .config import EPS
    from .errors import RankError
    torch = _torch()
    n = F.cols
    dev = torch.device("cuda", torch.cuda.current_device())

    def planes(M):
        re = torch.from_numpy(np.ascontiguousarray(M.re.T, dtype=np.float64)).to(dev)
        im = torch.from_numpy(np.ascontiguousarray(M.im.T, dtype=np.float64)).to(dev) if M.is_complex else None
        return re, im

    Fr, Fi = planes(F)
    jp1 = torch.arange(n, dtype=torch.int64, device=dev)
    if qr_rfactor(Fr, Fi, True, jp1, n * EPS) != 0:
        raise RankError("numerically rank-deficient F in the preprocessing")
    Gr, Gi = planes(G)
    Gr = Gr[jp1].contiguous()                        # G[:, jp1]
    Gi = Gi[jp1].contiguous() if Gi is not None else None
    jp2 = torch.arange(n, dtype=torch.int64, device=dev)
    if qr_rfactor(Gr, Gi, True, jp2, n * EPS) != 0:
        raise RankError("numerically rank-deficient G in the preprocessing")
    Fpp = MatrixPlanePair.from_dense(_host(Fr[jp2, :n], Fi[jp2, :n] if Fi is not None else None))
    Gpp = MatrixPlanePair.from_dense(_host(Gr[:, :n], Gi[:, :n] if Gi is not None else None))
    piv = jp1[jp2].cpu().numpy()
    return Fpp, Gpp, piv


def postmultiply(Yp, Yq, Ztilde):
    """[Yp' Yq'] = [Yp Yq] Ztilde (blocked.py:370-381)."""
    torch = _torch()
    Yp = _as_cols(Yp)
    w = Yp.shape[1]
    stack = np.hstack([Yp, _as_cols(Yq)])
    Zt = np.asarray(Ztilde)
    cplx = np.iscomplexobj(stack) or np.iscomplexobj(Zt)
    if cplx:
        stack = stack.astype(np.complex128)
        Zt = Zt.astype(np.complex128)
    m = stack.shape[0]
    Yr, Yi = _dev_planes(stack, cplx, torch)
    Zr, Zi = _dev_planes(Zt, cplx, torch)
    _native.check(_native.load().hzg_op_postmultiply(m, w, int(cplx), _p(Yr), _p(Yi), _p(Zr), _p(Zi),
                                                     _stream(torch)), None, "postmultiply")
    out = _host(Yr, Yi)
    return out[:, :w], out[:, w:]


def rescale_z(F, G, Z, final=False, compensated=False):
    """Theta rescaling of Z; with ``final`` also returns (U, V, Z, sigF, sigG,
    sigma) (blocked.py:384-401).  F, G, Z are MatrixPlanePair values."""
    torch = _torch()
    cplx = F.is_complex
    dF = _dev_planes(F.to_dense(), cplx, torch)
    dG = _dev_planes(G.to_dense(), cplx, torch)
    dZ = _dev_planes(Z.to_dense().astype(np.complex128) if cplx else Z.to_dense(), cplx, torch)
    n = F.cols
    kw = dict(dtype=torch.float64, device=dF[0].device)
    sig = [torch.empty(n, **kw) for _ in range(3)]
    L = _native.load()
    _native.check(L.hzg_op_rescale(F.rows, G.rows, n, int(cplx), int(bool(compensated)), int(bool(final)),
                                   _p(dF[0]), _p(dF[1]), _p(dG[0]), _p(dG[1]), _p(dZ[0]), _p(dZ[1]), Z.rows,
                                   _p(sig[0]), _p(sig[1]), _p(sig[2]), _stream(torch)), None,
                  "zero column during rescaling")
    Zo = MatrixPlanePair.from_dense(_host(*dZ))
    if not final:
        return Zo
    return (MatrixPlanePair.from_dense(_host(*dF)), MatrixPlanePair.from_dense(_host(*dG)), Zo,
            sig[0].cpu().numpy(), sig[1].cpu().numpy(), sig[2].cpu().numpy())


def run_distributed(p, cfg=None, s=2, s_inner=1, pool=1):
    """Stripe-distributed solve of a bordered pair with s workers, the
    reference's scheme and results (distsim.py:147-259; stripes.py)."""
    from .stripes import run_distributed as _run
    return _run(p, cfg, s, s_inner, pool)
