"""The CPU oracle against the reference's own outputs (golden fixtures made
by tests/golden/make_golden.py from the reference package).  Bitwise."""

import numpy as np
import pytest

from conftest import load_case, manifest
from oracle import oracle as O

CASES = sorted(manifest())


@pytest.mark.parametrize("name", CASES)
def test_oracle_reproduces_reference_bitwise(name):
    c = load_case(name)
    r = O.solve(c["F"], c["G"], O.make_cfg(**c["cfg"]), threads=4)
    assert np.array_equal(r["sigma"], c["sigma"])
    assert np.array_equal(r["sigmaF"], c["sigmaF"])
    assert np.array_equal(r["sigmaG"], c["sigmaG"])
    assert [r["sweeps"], r["total"], r["big"], int(r["converged"])] == list(c["counters"])
    if c["full"]:
        assert np.array_equal(r["U"], c["U"])
        assert np.array_equal(r["V"], c["V"])
        assert np.array_equal(r["Z"], c["Z"])


def test_oracle_thread_count_is_bitwise_invisible():
    c = load_case("corpus64_real_w8")
    a = O.solve(c["F"], c["G"], O.make_cfg(block_width=8), threads=1)
    b = O.solve(c["F"], c["G"], O.make_cfg(block_width=8), threads=8)
    assert np.array_equal(a["Z"], b["Z"]) and np.array_equal(a["sigma"], b["sigma"])


def test_oracle_known_4x4_values():
    # test_acceptance.py:25-28 of the reference
    ref = np.array([1.414213562302384e10, 9.999999999999997e-1, 9.999999999999997e-1, 7.071067812219032e-1])
    c = load_case("pitfall4x4_w2")
    r = O.solve(c["F"], c["G"], O.make_cfg(block_width=2))
    assert np.max(np.abs(r["sigma"] - ref) / ref) <= 1e-10


def test_tree_reduce_shape():
    # dotprod.py:79-91: pairwise over the zero-padded power of two
    x = np.array([1e16, 1.0, -1e16, 1.0, 3.0])
    assert O.tree_reduce(x) == ((1e16 + 1.0) + (-1e16 + 1.0)) + ((3.0 + 0.0) + 0.0)


def test_generators_match_reference_formulas():
    u = O.uniform_stream(7, 5)
    assert np.all((u > 0) & (u < 1))
    g = O.gaussian_stream(7, 1000)
    assert abs(g.mean()) < 0.15 and abs(g.std() - 1) < 0.1
