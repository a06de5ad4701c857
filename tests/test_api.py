"""Host-side logic of the B200 package: configuration, storage model,
bordering, strategies and the multi-GPU block schedule, and the C ABI
library (loads and exports every declared symbol; no device calls)."""

import os
import re

import numpy as np
import pytest

import paper_1909_00101_b200 as hz
from paper_1909_00101_b200 import _native
from conftest import ROOT
from oracle import oracle as O


def test_config_decode_matches_reference():
    for vid in range(8):
        cfg = hz.SolverConfig(variant_id=vid)
        assert cfg.criterion == ("C1" if vid < 4 else "C2")
        assert cfg.prescale == (vid in (0, 1, 4, 5))
        assert cfg.compensated == (vid % 2 == 1)
    assert hz.SolverConfig(blocking="fb").max_inner_sweeps == 30
    assert hz.SolverConfig(blocking="bo").max_inner_sweeps == 1
    assert hz.SolverConfig().block_width == 8
    for bad in (dict(variant_id=8), dict(blocking="xx"), dict(outer_kind="zz"), dict(shorten="lu"),
                dict(block_width=0)):
        with pytest.raises(ValueError):
            hz.SolverConfig(**bad)
    with pytest.raises(ValueError):
        hz.SweepStats(total=1, big=2)


def test_error_hierarchy():
    assert issubclass(hz.NotPositiveDefiniteError, hz.RankError)
    assert issubclass(hz.RankError, hz.HzgsvdError)
    assert issubclass(hz.ProtocolError, hz.HzgsvdError)


def test_plane_pair_validation():
    with pytest.raises(ValueError):
        hz.MatrixPlanePair(2, 2, np.zeros((2, 3)))
    with pytest.raises(ValueError):
        hz.MatrixPlanePair(2, 2, np.zeros((2, 2)), None, True)
    with pytest.raises(ValueError):
        hz.ProblemPair(hz.MatrixPlanePair.from_dense(np.ones((2, 3))), hz.MatrixPlanePair.from_dense(np.ones((4, 3))))
    m = hz.MatrixPlanePair.from_dense(np.arange(6.0).reshape(3, 2) + 1j)
    assert m.is_complex and np.array_equal(m.to_dense(), np.arange(6.0).reshape(3, 2) + 1j)
    c = m.copy()
    c.re[0, 0] = 99.0
    assert m.re[0, 0] == 0.0
    flat = hz.MatrixPlanePair(2, 2, np.arange(4.0))
    assert np.array_equal(flat.re, np.arange(4.0).reshape((2, 2), order="F"))


@pytest.mark.parametrize("shape", [(5, 3, 2), (16, 16, 4), (70, 45, 8), (33, 20, 16)])
def test_border_pair_matches_oracle(shape):
    m, n, w = shape
    A = np.arange(m * n, dtype=float).reshape(m, n) + 1
    p = hz.ProblemPair(hz.MatrixPlanePair.from_dense(A), hz.MatrixPlanePair.from_dense(A))
    b = hz.border_pair(p, 2 * w, 2 * w)
    pad = (-n) % (2 * w)
    R, _ = O.border_one(A, None, pad, 2 * w)
    assert np.array_equal(b.F.re, R)
    Ac = A + 1j * A[::-1]
    pc = hz.ProblemPair(hz.MatrixPlanePair.from_dense(Ac), hz.MatrixPlanePair.from_dense(Ac))
    bc = hz.border_pair(pc, 2 * w, 2 * w)
    Rr, Ri = O.border_one(Ac.real.copy(), Ac.imag.copy(), pad, 2 * w)
    assert np.array_equal(bc.F.re, Rr) and np.array_equal(bc.G.im, Ri)
    assert (b.original_n, b.original_mF) == (n, m)
    assert hz.core.bordered_shape(n, m, 2 * w, 2 * w) == (pad, R.shape[0])


@pytest.mark.parametrize("kind", ["me", "mm"])
def test_tables_match_oracle_and_invariants(kind):
    for n in range(2, 66, 2):
        t = hz.gen_table(kind, n)
        assert np.array_equal(t.as_array(), O.gen_table(kind, n))
        rep = hz.validate_table(t)
        assert rep["coverage_ok"] and rep["disjoint_ok"]
        if kind == "me":
            assert rep["cyclic"] and len(t.steps) == n - 1
        m = hz.comm_mapping(t)
        half = n // 2
        want = [(r, s) for r in range(half) for s in (0, 1)]
        for row in m.entries:
            assert sorted((abs(e) - 1, 0 if e < 0 else 1) for ent in row for e in ent[2:]) == want


def test_circle_positions_are_the_me_step_sets():
    for n in (4, 8, 64, 256):
        pos = hz.circle_positions(n)
        t = hz.gen_table("me", n)
        for k in range(n - 1):
            assert sorted(map(tuple, pos[k].tolist())) == t.steps[k]


@pytest.mark.parametrize("nblk,nranks", [(16, 2), (64, 4), (256, 8), (1024, 8)])
def test_block_schedule_moves_are_bounded(nblk, nranks):
    moves = hz.block_moves(nblk, nranks)
    assert len(moves) == nblk - 1
    for mv in moves:
        assert len(mv) <= 2 * nranks
        per_rank_in = np.bincount([d for (_, _, d) in mv], minlength=nranks)
        per_rank_out = np.bincount([s for (_, s, _) in mv], minlength=nranks)
        assert np.array_equal(per_rank_in, per_rank_out)  # slots are conserved


def test_clib_exports_every_declared_symbol():
    with open(os.path.join(ROOT, "include", "hzg.h")) as fh:
        decl = set(re.findall(r"\b(hzg_[a-z_0-9]+)\s*\(", fh.read()))
    assert decl == set(_native.EXPORTS)
    lib = _native.load()
    for name in decl:
        assert hasattr(lib, name)


def test_make_config_layout():
    c = _native.make_config(hz.SolverConfig(variant_id=6, block_width=16, blocking="bo", outer_kind="mm",
                                            exact=True))
    assert (c.variant_id, c.block_width, c.max_inner_sweeps, c.outer_mm, c.inner_mm, c.exact) == (6, 16, 1, 1, 0, 1)


def test_gsvd_1x1_closed_form():
    # pointwise test_gsvd_1x1 of the reference
    r = hz.gsvd_1x1(hz.MatrixPlanePair.from_dense(np.array([[3.0]])),
                    hz.MatrixPlanePair.from_dense(np.array([[4.0]])))
    assert r.sigmaF[0] == 0.6 and r.sigmaG[0] == 0.8 and r.sigma[0] == 0.75
    assert r.Z.re[0, 0] == 0.2 and r.U.re[0, 0] == 1.0
    with pytest.raises(hz.RankError):
        hz.gsvd_1x1(hz.MatrixPlanePair.from_dense(np.array([[0.0]])),
                    hz.MatrixPlanePair.from_dense(np.array([[1.0]])))


def test_no_cpu_fallback_without_device():
    import torch
    if torch.cuda.is_available():
        pytest.skip("device present")
    with pytest.raises(hz.DeviceError):
        hz.solve(np.eye(4), np.eye(4), hz.SolverConfig(block_width=2))


def test_product_package_never_uses_the_oracle():
    """The oracle is test infrastructure: no module of the product package
    may import, load or execute anything under oracle/ (DESIGN.md section 2)."""
    import pathlib
    pkg = pathlib.Path(hz.__file__).parent
    offenders = []
    for path in list(pkg.rglob("*.py")) + list(pkg.rglob("*.cu")) + list(pkg.rglob("*.h")) + list(pkg.rglob("*.cuh")):
        text = path.read_text()
        for pat in ("import oracle", "from oracle", "hzg_oracle", "libhzg_oracle", "oracle/", "hzo_"):
            if pat in text:
                offenders.append("%s: %s" % (path.name, pat))
    assert not offenders, offenders


def test_block_operations_reject_unsupported_shapes():
    """unsupported or unequal block widths raise a clear
    ValueError before any device work (no silent truncation)."""
    from paper_1909_00101_b200 import ops
    with pytest.raises(ValueError, match="equal width"):
        ops.qr_shorten(np.ones((8, 2)), np.ones((8, 3)))
    with pytest.raises(ValueError, match="not supported"):
        ops.qr_shorten(np.ones((40, 9)), np.ones((40, 9)))
    with pytest.raises(ValueError, match="not supported"):
        ops.cholesky_upper(np.eye(3))
