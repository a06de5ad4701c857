"""The reference's accuracy report on the device (harness.py:246-465).

``accuracy_report(p, r, reference=None)`` keeps the reference's signature
and AccuracyReport fields:

* X = Z^{-1} from an LU factorization with complete pivoting
  (hzg_lu_complete: bitwise the reference's _k_lu_complete factors) and two
  triangular solves on the factors (the reference's per-column
  substitutions, here as triangular solves of the whole permuted identity);
* resF = ||F - U S_F X||_F / ||F||_F and resG likewise, the products with
  compensated dot products (hzg_gemm_comp) and the Frobenius norms as
  compensated sums of squares (hzg_sumsq_comp);
* orthU = ||U^H U - I||_F, orthV = ||V^H V - I||_F, compensated the same way;
* with ``reference`` sigma values: the max / mean relative error of the
  descending-sorted sigma.

``device_accuracy`` does the same on device tensors (column-major planes as
(cols, rows) torch tensors) for callers that keep the result in HBM, e.g.
bench.py at n = 16384.  A diagnostic beside the hot path; no CPU fallback.
"""

import ctypes
import dataclasses
import math
from typing import Optional

import numpy as np

from . import _native
from .errors import DeviceError, NotPositiveDefiniteError


@dataclasses.dataclass
class AccuracyReport:
    resF: float
    resG: float
    orthU: float
    orthV: float
    max_rel_sigma: Optional[float] = None
    avg_rel_sigma: Optional[float] = None


def _torch():
    import torch
    if not torch.cuda.is_available():
        raise DeviceError("no CUDA device: the B200 path has no CPU fallback")
    return torch


def _p(t):
    return ctypes.c_void_p(t.data_ptr()) if t is not None else None


def _stream(torch):
    return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)


def invert_via_lu(Zr, Zi=None):
    """X = Z^{-1} for a device matrix given as (cols, rows) planes; returns
    X the same way.  Raises NotPositiveDefiniteError on a singular Z (the
    reference's invert_via_lu, harness.py:422-433)."""
    torch = _torch()
    L = _native.load()
    n = Zr.shape[0]
    Ar = Zr.clone()
    Ai = Zi.clone() if Zi is not None else None
    dev = Ar.device
    rp = torch.arange(n, dtype=torch.int64, device=dev)
    cp = torch.arange(n, dtype=torch.int64, device=dev)
    ws = torch.empty(int(L.hzg_lu_workspace_bytes(n)), dtype=torch.uint8, device=dev)
    st = torch.zeros(1, dtype=torch.int32, device=dev)
    _native.check(L.hzg_lu_complete(n, int(Ai is not None), _p(Ar), _p(Ai), n, _p(rp), _p(cp), _p(ws), _p(st),
                                    _stream(torch)), None, "hzg_lu_complete")
    if int(st.item()) != 0:
        raise NotPositiveDefiniteError("singular Z")
    # P Z Q = L U with P e_i = e_rp[i]-row selection, Q: row i of the
    # solution goes to X row cp[i] (harness.py:374-419)
    LU = Ar.T if Ai is None else torch.complex(Ar.T, Ai.T)
    eye = torch.eye(n, dtype=LU.dtype, device=dev)
    P = eye[:, rp].T.contiguous()  # P[i, col] = 1 iff rp[i] == col
    Lm = torch.tril(LU, -1) + eye
    Um = torch.triu(LU)
    Y = torch.linalg.solve_triangular(Lm, P, upper=False, unitriangular=True)
    W = torch.linalg.solve_triangular(Um, Y, upper=True)
    X = torch.empty_like(W)
    X[cp] = W
    if Ai is None:
        return X.T.contiguous(), None
    return X.real.T.contiguous(), X.imag.T.contiguous()


def _gemm(A, B, trans_a=False):
    """Compensated op(A) B of (cols, rows) planes A = (Ar, Ai), B = (Br, Bi)."""
    torch = _torch()
    L = _native.load()
    Ar, Ai = A
    Br, Bi = B
    cplx = Ai is not None or Bi is not None
    if cplx:
        Ai = Ai if Ai is not None else torch.zeros_like(Ar)
        Bi = Bi if Bi is not None else torch.zeros_like(Br)
    lda, ka = Ar.shape[1], Ar.shape[0]  # A as rows x cols: lda rows, ka cols
    m, k = (ka, lda) if trans_a else (lda, ka)
    n = Br.shape[0]
    Cr = torch.empty((n, m), dtype=torch.float64, device=Ar.device)
    Ci = torch.empty((n, m), dtype=torch.float64, device=Ar.device) if cplx else None
    _native.check(L.hzg_gemm_comp(m, n, k, int(cplx), int(bool(trans_a)), _p(Ar), _p(Ai), lda, _p(Br), _p(Bi),
                                  Br.shape[1], _p(Cr), _p(Ci), m, _stream(torch)), None, "hzg_gemm_comp")
    return Cr, Ci


def _sumsq(A, B=None, eye=False):
    """Compensated sum of |A - B|^2 over (cols, rows) planes."""
    torch = _torch()
    L = _native.load()
    Ar, Ai = A
    Br, Bi = B if B is not None else (None, None)
    cols, rows = Ar.shape
    nb = 148 * 8
    part = torch.empty(2 * nb, dtype=torch.float64, device=Ar.device)
    _native.check(L.hzg_sumsq_comp(rows, cols, _p(Ar), _p(Ai), rows, _p(Br), _p(Bi), rows, int(bool(eye)),
                                   _p(part), nb, _stream(torch)), None, "hzg_sumsq_comp")
    return math.fsum(part.cpu().numpy().tolist())


def device_accuracy(F, G, U, V, Z, sigmaF, sigmaG):
    """Reference-form residuals and orthogonality of a device result.
    F, G, U, V, Z: (re, im-or-None) pairs of (cols, rows) float64 tensors;
    sigmaF, sigmaG: device vectors.  Returns (resF, resG, orthU, orthV)."""
    X = invert_via_lu(*Z)
    out = []
    for (Y, W, s) in ((F, U, sigmaF), (G, V, sigmaG)):
        WS = (W[0] * s[:, None], W[1] * s[:, None] if W[1] is not None else None)
        M = _gemm(WS, X)
        out.append(math.sqrt(_sumsq(Y, M)) / math.sqrt(_sumsq(Y)))
        del M
    for W in (U, V):
        WW = _gemm(W, W, trans_a=True)
        out.append(math.sqrt(_sumsq(WW, eye=True)))
        del WW
    return tuple(out)


def _dev_planes(m, torch, dev):
    re = torch.from_numpy(np.ascontiguousarray(m.re.T)).to(dev)
    im = torch.from_numpy(np.ascontiguousarray(m.im.T)).to(dev) if m.is_complex else None
    return re, im


def accuracy_report(p, r, reference=None):
    """Residuals, orthogonality defects and (with reference sigma) sigma
    errors of a GsvdResult r for the pair p (harness.py:436-465), computed
    on the device."""
    torch = _torch()
    dev = torch.device("cuda", torch.cuda.current_device())
    F, G = _dev_planes(p.F, torch, dev), _dev_planes(p.G, torch, dev)
    U, V, Z = (_dev_planes(m, torch, dev) for m in (r.U, r.V, r.Z))
    sF = torch.from_numpy(np.asarray(r.sigmaF, dtype=np.float64)).to(dev)
    sG = torch.from_numpy(np.asarray(r.sigmaG, dtype=np.float64)).to(dev)
    resF, resG, orthU, orthV = device_accuracy(F, G, U, V, Z, sF, sG)
    max_rel = avg_rel = None
    if reference is not None:
        c = np.sort(np.asarray(r.sigma))[::-1]
        ref = np.sort(np.asarray(reference))[::-1]
        rel = np.abs(c - ref) / ref
        max_rel, avg_rel = float(rel.max()), float(rel.mean())
    return AccuracyReport(resF, resG, orthU, orthV, max_rel, avg_rel)
