"""The reference's single block operations (form_grammians, cholesky_upper,
qr_shorten, postmultiply, rescale_z, run_distributed; blocked.py:328-401,
distsim.py:147) on the device, against the oracle."""

import ctypes

import numpy as np
import pytest

import paper_1909_00101_b200 as hz
from oracle import oracle as O

pytestmark = pytest.mark.gpu


def _stack(m, tw, cplx, seed):
    rng = np.random.default_rng(seed)
    Y = rng.standard_normal((m, tw))
    if cplx:
        Y = Y + 1j * rng.standard_normal((m, tw))
    return Y


@pytest.mark.parametrize("cplx", [False, True])
@pytest.mark.parametrize("comp", [False, True])
@pytest.mark.parametrize("m,w", [(40, 4), (300, 8), (1000, 16)])
def test_form_grammians_bitwise(cplx, comp, m, w):
    Y = _stack(m, 2 * w, cplx, 3 + m)
    X = _stack(m, 2 * w, cplx, 4 + m)
    A, B = hz.form_grammians(Y[:, :w], Y[:, w:], X[:, :w], X[:, w:], compensated=comp)
    for M, ref in ((A, Y), (B, X)):
        Rr, Ri = O.grammian(np.asfortranarray(ref.real), np.asfortranarray(ref.imag) if cplx else None, 0, w, w,
                            cplx, comp)
        assert np.array_equal(M.real, Rr)
        if cplx:
            assert np.array_equal(M.imag, Ri)


@pytest.mark.parametrize("cplx", [False, True])
@pytest.mark.parametrize("tw", [4, 16, 32])
def test_cholesky_upper_bitwise(cplx, tw):
    Y = _stack(3 * tw, tw, cplx, tw)
    M = Y.conj().T @ Y
    R = hz.cholesky_upper(M)
    ref, st = O.cholesky_upper(M)
    assert st == 0
    assert np.array_equal(R, ref)
    bad = np.eye(tw)
    bad[1, 1] = -1.0
    with pytest.raises(hz.NotPositiveDefiniteError):
        hz.cholesky_upper(bad)


@pytest.mark.parametrize("cplx", [False, True])
@pytest.mark.parametrize("m,w", [(24, 4), (100, 8)])
def test_qr_shorten_bitwise(cplx, m, w):
    tw = 2 * w
    Y = _stack(m, tw, cplx, m + w)
    R = hz.qr_shorten(Y[:, :w], Y[:, w:])
    Sr = np.asfortranarray(Y.real.copy())
    Si = np.asfortranarray(Y.imag.copy() if cplx else np.zeros_like(Y.real))
    outR = np.zeros((tw, tw), order="F")
    outI = np.zeros((tw, tw), order="F")
    p = lambda a: a.ctypes.data_as(ctypes.c_void_p)
    st = O.lib().hzo_qr_shorten(m, tw, int(cplx), p(Sr), p(Si), p(outR), p(outI))
    assert st == 0
    assert np.array_equal(R.real, outR)
    if cplx:
        assert np.array_equal(R.imag, outI)
    with pytest.raises(hz.RankError):
        Z = np.zeros((m, tw))
        hz.qr_shorten(Z[:, :w], Z[:, w:])


@pytest.mark.parametrize("cplx", [False, True])
@pytest.mark.parametrize("m,w", [(200, 8), (1000, 16), (77, 2)])
def test_postmultiply_bitwise(cplx, m, w):
    """postmultiply runs the reference-order kernel: bitwise the oracle's
    _k_postmult (blocked.py:220-250)."""
    Y = _stack(m, 2 * w, cplx, 9 + m)
    Zt = _stack(2 * w, 2 * w, cplx, 10 + m)
    a, b = hz.postmultiply(Y[:, :w], Y[:, w:], Zt)
    Yr = np.asfortranarray(Y.real.copy())
    Yi = np.asfortranarray(Y.imag.copy() if cplx else np.zeros_like(Y.real))
    Br = np.asfortranarray(Zt.real.copy())
    Bi = np.asfortranarray(Zt.imag.copy() if cplx else np.zeros_like(Zt.real))
    p = lambda x: x.ctypes.data_as(ctypes.c_void_p)  # noqa: E731
    L = O.lib()
    L.hzo_postmult.argtypes = [ctypes.c_int64, ctypes.c_int, ctypes.c_int] + [ctypes.c_void_p] * 4
    L.hzo_postmult(m, w, int(cplx), p(Yr), p(Yi), p(Br), p(Bi))
    got = np.hstack([a, b])
    assert np.array_equal(got.real, Yr)
    if cplx:
        assert np.array_equal(got.imag, Yi)


def test_rescale_z_bitwise_real():
    rng = np.random.default_rng(11)
    n, m = 24, 40
    F = hz.MatrixPlanePair.from_dense(rng.standard_normal((m, n)))
    G = hz.MatrixPlanePair.from_dense(rng.standard_normal((m, n)))
    Z = hz.MatrixPlanePair.from_dense(rng.standard_normal((n, n)))
    Zo = hz.rescale_z(F, G, Z)
    theta = np.array([1.0 / np.sqrt(O.tree_reduce(F.re[:, j] * F.re[:, j]) + O.tree_reduce(G.re[:, j] * G.re[:, j]))
                      for j in range(n)])
    assert np.array_equal(Zo.re, Z.re * theta[None, :])
    U, V, Z2, sF, sG, s = hz.rescale_z(F, G, Z, final=True)
    assert np.allclose(np.linalg.norm(U.re, axis=0), 1.0) and np.allclose(sF ** 2 + sG ** 2, 1.0)
    assert np.array_equal(s, sF / sG)


def test_run_distributed_stripes_vs_block_partitioned():
    """run_distributed is the reference's stripe scheme (its bits depend on
    s); the B200 block-partitioned scheme is bitwise the single worker.
    Both agree to the reference's own distributed-vs-single bound (1e-10,
    test_distsim.py:100-109); the stripe scheme itself is pinned bitwise to
    the reference in tests/test_gpu_stripes.py."""
    g = O.gaussian_stream(5, 2 * 128 * 128)
    F = hz.MatrixPlanePair.from_dense(g[:128 * 128].reshape((128, 128), order="F"))
    G = hz.MatrixPlanePair.from_dense(g[128 * 128:].reshape((128, 128), order="F"))
    p = hz.ProblemPair(F, G)
    cfg = hz.SolverConfig(block_width=8)
    a = hz.run_distributed(p, cfg, s=4)
    b = hz.gsvd_blocked(p, cfg)
    assert a.workers == 4 and a.converged
    rel = np.abs(np.sort(a.sigma) - np.sort(b.sigma)) / np.sort(b.sigma)
    assert rel.max() <= 1e-10
    c = hz.solve(F, G, cfg, workers=4, scheme="blocks")
    d = hz.solve(F, G, cfg)
    assert np.array_equal(c.sigma, d.sigma) and np.array_equal(c.Z.re, d.Z.re)
    with pytest.raises(ValueError):
        hz.run_distributed(p, cfg, s=3)
