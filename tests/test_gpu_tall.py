"""preprocess_tall on the device (blocked.py:405-428) against
the reference's own outputs (tests/golden/tall_*.npz, made by
tests/golden/make_tall_golden.py): bitwise F'', G'', piv, and the same
RankError cases."""

import glob
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
CASES = sorted(os.path.basename(p)[:-4] for p in glob.glob(os.path.join(GOLDEN, "tall_*.npz")))


def _load(name):
    d = dict(np.load(os.path.join(GOLDEN, name + ".npz")))
    cplx = bool(d["cplx"])
    F = d["F_re"] + 1j * d["F_im"] if cplx else d["F_re"]
    G = d["G_re"] + 1j * d["G_im"] if cplx else d["G_re"]
    return d, F, G


@pytest.mark.parametrize("name", CASES)
def test_preprocess_tall_bitwise_vs_reference(name):
    import paper_1909_00101_b200 as hz
    d, F, G = _load(name)
    Fm, Gm = hz.MatrixPlanePair.from_dense(F), hz.MatrixPlanePair.from_dense(G)
    err = str(d["error"])
    if err:
        with pytest.raises(hz.RankError, match="rank-deficient %s" % err):
            hz.preprocess_tall(Fm, Gm)
        return
    Fpp, Gpp, piv = hz.preprocess_tall(Fm, Gm)
    assert np.array_equal(piv, d["piv"])
    a, b = Fpp.to_dense(), Gpp.to_dense()
    assert np.array_equal(np.real(a), d["Fpp_re"]) and np.array_equal(np.imag(a), d["Fpp_im"])
    assert np.array_equal(np.real(b), d["Gpp_re"]) and np.array_equal(np.imag(b), d["Gpp_im"])


def test_preprocess_tall_then_solve_recovers_sigma():
    """The shortened pair has the generalized singular values of the tall
    pair (config 3 shape scaled down): solve(F'', G'') vs solve(F, G)."""
    import paper_1909_00101_b200 as hz
    from oracle import oracle as O
    m, n = 192, 128
    g = O.gaussian_stream(31, 2 * m * n + 2 * n * n)
    F = (g[: m * n] + 1j * g[m * n: 2 * m * n]).reshape((m, n), order="F")
    G = (g[2 * m * n: 2 * m * n + n * n] + 1j * g[2 * m * n + n * n:]).reshape((n, n), order="F")
    Fm, Gm = hz.MatrixPlanePair.from_dense(F), hz.MatrixPlanePair.from_dense(G)
    Fpp, Gpp, piv = hz.preprocess_tall(Fm, Gm)
    assert sorted(piv.tolist()) == list(range(n))
    cfg = hz.SolverConfig(block_width=16)
    r_tall = hz.solve(Fm, Gm, cfg)
    r_short = hz.solve(Fpp, Gpp, cfg)
    rel = np.abs(r_short.sigma - r_tall.sigma) / r_tall.sigma
    assert rel.max() < 64 * n * 2.2e-16


@pytest.mark.parametrize("m,n,p,cplx", [(300, 200, 240, False), (260, 160, 200, True), (97, 97, 97, False)])
def test_preprocess_tall_bitwise_vs_oracle_random(m, n, p, cplx):
    """Larger seeded pairs than the golden cases: device vs the oracle's
    restatement (itself pinned to the reference's golden vectors)."""
    import paper_1909_00101_b200 as hz
    from oracle import oracle as O
    g = O.gaussian_stream(m + n + p, 2 * (m + p) * n)
    F = g[: m * n].reshape((m, n), order="F")
    G = g[m * n: (m + p) * n].reshape((p, n), order="F")
    if cplx:
        F = F + 1j * g[(m + p) * n: (2 * m + p) * n].reshape((m, n), order="F")
        G = G + 1j * g[(2 * m + p) * n:].reshape((p, n), order="F")
    Fo, Go, po = O.preprocess_tall(F, G)
    Fpp, Gpp, piv = hz.preprocess_tall(hz.MatrixPlanePair.from_dense(F), hz.MatrixPlanePair.from_dense(G))
    assert np.array_equal(piv, po)
    assert np.array_equal(Fpp.to_dense(), Fo) and np.array_equal(Gpp.to_dense(), Go)
