"""Host-side reference-shape reductions for the few scalars the driver forms
on the CPU (the n = 1 closed form, pointwise.py:324-345).

The pairwise tree over the input zero-padded to a power of two is the
reference's summation shape (dotprod.py:79-91); numpy's strided adds
evaluate each level exactly like the reference's loop.
"""

import numpy as np


def _tree(buf):
    n = buf.shape[0]
    m = 1
    while m < n:
        m *= 2
    x = np.zeros(m)
    x[:n] = buf
    while x.shape[0] > 1:
        x = x[0::2] + x[1::2]
    return float(x[0])


def tree_reduce(values):
    v = np.ascontiguousarray(np.asarray(values, dtype=np.float64)).ravel()
    if v.size < 1:
        raise ValueError("tree_reduce needs at least one value")
    return _tree(v)


def norm_sq(v, field="real"):
    """Squared Euclidean norm (dotprod.py:206-232, ordinary form)."""
    if len(v) < 1:
        raise ValueError("norm_sq: empty vector")
    if field == "real":
        x = np.asarray(v, dtype=np.float64)
        return _tree(x * x)
    z = np.asarray(v, dtype=np.complex128)
    vr, vi = z.real.copy(), z.imag.copy()
    # fma(vi, vi, vr*vr): exact product vi*vi added to the rounded vr*vr, one rounding
    return _tree(_fma(vi, vi, vr * vr))


def _fma(a, b, c):
    """Correctly rounded a*b + c elementwise (exact rational arithmetic,
    then one round-to-nearest-even by float())."""
    from fractions import Fraction
    a, b, c = np.broadcast_arrays(np.asarray(a, dtype=np.float64), np.asarray(b, dtype=np.float64),
                                  np.asarray(c, dtype=np.float64))
    out = np.empty(a.shape)
    for idx in np.ndindex(a.shape):
        x, y, z = float(a[idx]), float(b[idx]), float(c[idx])
        if not (np.isfinite(x) and np.isfinite(y) and np.isfinite(z)):
            out[idx] = x * y + z
        else:
            out[idx] = float(Fraction(x) * Fraction(y) + Fraction(z))
    return out
