"""CPU tests of the stripe-distributed scheme's routing (stripes.py), ported
from the reference's pkg/tests/test_distsim.py:19-83.  The stripes live in
CPU torch tensors here; the solver tests are in test_gpu_stripes.py."""

import numpy as np
import pytest

import paper_1909_00101_b200 as hz


def _pair(n, seed, cplx=False):
    rng = np.random.default_rng(seed)
    F = rng.standard_normal((n, n))
    G = rng.standard_normal((n, n))
    if cplx:
        F = F + 1j * rng.standard_normal((n, n))
        G = G + 1j * rng.standard_normal((n, n))
    return hz.ProblemPair(hz.MatrixPlanePair.from_dense(F), hz.MatrixPlanePair.from_dense(G))


def test_partition_examples():
    pair = _pair(8, 50)
    states = hz.partition_stripes(pair, 2, block_width=2, device="cpu")
    assert [s.rank for s in states] == [0, 1]
    t = hz.gen_table("me", 4)
    assert (states[0].p, states[0].q) == t.steps[0][0]
    assert (states[1].p, states[1].q) == t.steps[0][1]
    assert states[0].width == 2
    # slab = [stripe p | stripe q] of F, Z all zero with the global rows
    F = pair.F.re
    p, q = states[1].p, states[1].q
    assert np.array_equal(states[1].Fr.numpy(), np.hstack([F[:, 2 * p:2 * p + 2], F[:, 2 * q:2 * q + 2]]))
    assert states[1].Zr.shape == (8, 4) and not states[1].Zr.any()
    one = hz.partition_stripes(pair, 1, block_width=2, device="cpu")
    assert len(one) == 1 and (one[0].p, one[0].q) == (0, 1)
    with pytest.raises(ValueError):
        hz.partition_stripes(_pair(6, 51), 2, block_width=1, device="cpu")
    with pytest.raises(ValueError):
        hz.partition_stripes(_pair(8, 51), 2, block_width=4, device="cpu")


def test_exchange_self_sends():
    pair = _pair(8, 52)
    states = hz.partition_stripes(pair, 1, block_width=2, device="cpu")
    before = states[0].Fr.clone()
    mapping = hz.comm_mapping(hz.gen_table("me", 2))
    hz.exchange_step(states, mapping, 0)
    assert np.array_equal(states[0].Fr.numpy(), before.numpy())
    assert (states[0].p, states[0].q) == (0, 1)


def test_exchange_tag_arithmetic_real():
    t = hz.gen_table("me", 4)
    mapping = hz.comm_mapping(t)
    p, q, t0, t1 = mapping.entries[0][0]
    assert (p, q) == t.steps[0][0]
    assert abs(t0) in (1, 2) and abs(t1) in (1, 2)
    enc = [e for row in mapping.entries for (_p, _q, a, b) in row for e in (a, b)]
    assert -2 in enc


@pytest.mark.parametrize("kind", ["me", "mm"])
@pytest.mark.parametrize("cplx", [False, True])
@pytest.mark.parametrize("s", [2, 3, 4])
def test_exchange_routing_matches_table(kind, cplx, s):
    pair = _pair(8 * s, 54, cplx)
    states = hz.partition_stripes(pair, s, block_width=2, kind=kind, device="cpu")
    t = hz.gen_table(kind, 2 * s)
    mapping = hz.comm_mapping(t)
    width = states[0].width
    # tag each stripe's first entries with its global id in every plane
    for st in states:
        for key in ("Fr", "Gr", "Zr") + (("Fi", "Gi", "Zi") if cplx else ()):
            getattr(st, key)[0, 0] = 1000.0 + st.p
            getattr(st, key)[0, width] = 1000.0 + st.q
    for k in range(len(t.steps)):
        hz.exchange_step(states, mapping, k)
        kk = (k + 1) % len(t.steps)
        for r, st in enumerate(states):
            assert (st.p, st.q) == tuple(t.steps[kk][r])
            for key in ("Fr", "Gr", "Zr") + (("Fi", "Gi", "Zi") if cplx else ()):
                assert float(getattr(st, key)[0, 0]) == 1000.0 + st.p
                assert float(getattr(st, key)[0, width]) == 1000.0 + st.q
    for r, st in enumerate(states):
        assert (st.p, st.q) == tuple(t.steps[0][r])


def test_exchange_protocol_violation():
    pair = _pair(16, 55)
    states = hz.partition_stripes(pair, 2, block_width=2, device="cpu")
    mapping = hz.comm_mapping(hz.gen_table("me", 4))
    states[0].p, states[0].q = states[0].q, states[0].p
    with pytest.raises(hz.ProtocolError):
        hz.exchange_step(states, mapping, 0)


def test_exchange_duplicate_and_missing_tags():
    pair = _pair(16, 56)
    states = hz.partition_stripes(pair, 2, block_width=2, device="cpu")
    mapping = hz.comm_mapping(hz.gen_table("me", 4))
    bad = hz.CommMapping(mapping.order, mapping.steps, [list(r) for r in mapping.entries])
    p, q, t0, t1 = bad.entries[0][0]
    bad.entries[0][0] = (p, q, t0, t0)  # both stripes to the same slot
    with pytest.raises(hz.ProtocolError):
        hz.exchange_step(states, bad, 0)


def test_solve_scheme_argument_checked():
    with pytest.raises(ValueError):
        hz.solve(np.eye(4), np.eye(4), hz.SolverConfig(block_width=1), workers=2, scheme="rings")
