"""CPU checks of the preprocess_tall golden vectors (made from the reference
by tests/golden/make_tall_golden.py): the shortened pair has the Grammians
of the permuted tall pair, G'' is upper triangular with a real nonnegative
diagonal, piv is a permutation.  The device path is checked against them
bitwise in tests/test_gpu_tall.py."""

import glob
import os

import numpy as np
import pytest

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
CASES = sorted(os.path.basename(p)[:-4] for p in glob.glob(os.path.join(GOLDEN, "tall_*.npz")))


def test_tall_cases_present():
    assert len(CASES) >= 8
    errs = [str(np.load(os.path.join(GOLDEN, c + ".npz"))["error"]) for c in CASES]
    assert "F" in errs and "G" in errs and "" in errs


@pytest.mark.parametrize("name", CASES)
def test_tall_golden_consistent(name):
    d = dict(np.load(os.path.join(GOLDEN, name + ".npz")))
    if str(d["error"]):
        return
    F = d["F_re"] + 1j * d["F_im"]
    G = d["G_re"] + 1j * d["G_im"]
    Fpp = d["Fpp_re"] + 1j * d["Fpp_im"]
    Gpp = d["Gpp_re"] + 1j * d["Gpp_im"]
    piv = d["piv"]
    n = F.shape[1]
    assert sorted(piv.tolist()) == list(range(n))
    assert np.allclose(np.tril(Gpp, -1), 0) and np.all(np.imag(np.diag(Gpp)) == 0)
    assert np.all(np.real(np.diag(Gpp)) >= 0)
    Fp, Gp = F[:, piv], G[:, piv]
    for A, B in ((Fpp, Fp), (Gpp, Gp)):
        ga, gb = A.conj().T @ A, B.conj().T @ B
        assert np.max(np.abs(ga - gb)) <= 1e-12 * np.max(np.abs(gb))


@pytest.mark.parametrize("name", CASES)
def test_oracle_preprocess_tall_bitwise_vs_reference(name):
    """The oracle's restatement (hzo_qr_rfactor, hzg_oracle.c) reproduces
    the reference's preprocess_tall bitwise, errors included."""
    from oracle import oracle as O
    d = dict(np.load(os.path.join(GOLDEN, name + ".npz")))
    cplx = bool(d["cplx"])
    F = d["F_re"] + 1j * d["F_im"] if cplx else d["F_re"]
    G = d["G_re"] + 1j * d["G_im"] if cplx else d["G_re"]
    if str(d["error"]):
        with pytest.raises(O.OracleError, match="rank-deficient %s" % str(d["error"])):
            O.preprocess_tall(F, G)
        return
    Fpp, Gpp, piv = O.preprocess_tall(F, G)
    assert np.array_equal(piv, d["piv"])
    assert np.array_equal(np.real(Fpp), d["Fpp_re"]) and np.array_equal(np.imag(Fpp), d["Fpp_im"])
    assert np.array_equal(np.real(Gpp), d["Gpp_re"]) and np.array_equal(np.imag(Gpp), d["Gpp_im"])
