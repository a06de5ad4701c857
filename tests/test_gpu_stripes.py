"""GPU parity of the stripe-distributed scheme (stripes.py) with the
reference's own distsim outputs (tests/golden/make_dist_golden.py runs the
reference's solve(F, G, cfg, workers=s, worker_sweeps=k)).

* exact mode: bitwise U, V, Z, sigma vectors, sweeps and counters;
* DMMA mode: sigma within the tolerance of the reference's own s-vs-single
  test (1e-10, test_distsim.py:100-109), residuals and normalization as in
  test_distsim.py:136-141;
* s = 1 delegates to the single-worker solver (test_distsim.py:80-86).
"""

import json
import os

import numpy as np
import pytest

import paper_1909_00101_b200 as hz
from conftest import GOLDEN, gsvd_metrics, rel_err_sorted

pytestmark = pytest.mark.gpu

with open(os.path.join(GOLDEN, "dist_manifest.json")) as fh:
    DIST = json.load(fh)


def _case(name):
    d = dict(np.load(os.path.join(GOLDEN, name + ".npz")))
    d.update(DIST[name])
    return d


@pytest.mark.parametrize("name", sorted(DIST))
def test_stripes_exact_mode_bitwise_vs_reference(name):
    c = _case(name)
    cfg = hz.SolverConfig(exact=True, **c["cfg"])
    r = hz.solve(c["F"], c["G"], cfg, workers=c["workers"], worker_sweeps=c["worker_sweeps"])
    sweeps, total, big, conv, workers = (int(x) for x in c["counters"])
    assert (r.sweeps, r.total_transforms, r.big_transforms, int(r.converged), r.workers) == \
        (sweeps, total, big, conv, workers)
    for got, want in ((r.sigma, c["sigma"]), (r.sigmaF, c["sigmaF"]), (r.sigmaG, c["sigmaG"]),
                      (r.U.to_dense(), c["U"]), (r.V.to_dense(), c["V"]), (r.Z.to_dense(), c["Z"])):
        assert np.array_equal(got, want)


@pytest.mark.parametrize("name", sorted(DIST))
def test_stripes_dmma_mode_within_tolerance(name):
    c = _case(name)
    cfg = hz.SolverConfig(**c["cfg"])
    r = hz.solve(c["F"], c["G"], cfg, workers=c["workers"], worker_sweeps=c["worker_sweeps"])
    assert r.converged and r.workers == c["workers"]
    n = c["n"]
    # sigma vs the reference's distributed run: 8 n eps, or 1e-10 (the
    # reference's own distributed-vs-single bound) for the pitfall pair
    # whose smallest sigma is conditioning-limited
    tol = 1e-10 if "pitfall" in name else 8 * n * 2.0 ** -52
    assert rel_err_sorted(r.sigma, c["sigma"]).max() <= tol
    assert abs(r.sweeps - int(c["counters"][0])) <= 2
    m = gsvd_metrics(c["F"], c["G"], r)
    assert m["resF"] <= 1e-12 and m["resG"] <= 1e-12
    assert m["pencil"] <= 1e-14


@pytest.mark.parametrize("s", [2, 4])
@pytest.mark.parametrize("cplx", [False, True])
def test_stripes_vs_single_worker(s, cplx):
    """test_distsim.py:98-109: workers = s agrees with workers = 1 to 1e-10."""
    rng = np.random.default_rng(57 + s + 10 * cplx)
    n = 64
    F = rng.standard_normal((n, n)) + (1j * rng.standard_normal((n, n)) if cplx else 0)
    G = rng.standard_normal((n, n)) + (1j * rng.standard_normal((n, n)) if cplx else 0)
    cfg = hz.SolverConfig(block_width=8)
    base = hz.solve(F, G, cfg)
    r = hz.solve(F, G, cfg, workers=s, worker_sweeps=1)
    assert r.workers == s and r.converged and r.sweeps <= 30
    assert rel_err_sorted(r.sigma, base.sigma).max() <= 1e-10
    # and the B200 block-partitioned scheme is bitwise the single worker
    b = hz.solve(F, G, cfg, workers=s, scheme="blocks")
    assert np.array_equal(b.sigma, base.sigma) and np.array_equal(b.Z.re, base.Z.re)


def test_run_distributed_single_worker_delegates():
    c = _case("dist64_real_s2_w8")
    p = hz.ProblemPair(hz.MatrixPlanePair.from_dense(c["F"]), hz.MatrixPlanePair.from_dense(c["G"]))
    pb = hz.border_pair(p, 16, 16)
    cfg = hz.SolverConfig(exact=True)
    a = hz.run_distributed(pb, cfg, 1, 30)
    b = hz.gsvd_blocked(pb, cfg)
    assert a.workers == 1
    assert np.array_equal(a.sigma, b.sigma) and np.array_equal(a.Z.re, b.Z.re) and np.array_equal(a.U.re, b.U.re)


def test_run_distributed_deterministic():
    c = _case("dist64_real_s2_w8")
    p = hz.ProblemPair(hz.MatrixPlanePair.from_dense(c["F"]), hz.MatrixPlanePair.from_dense(c["G"]))
    pb = hz.border_pair(p, 32, 16)
    cfg = hz.SolverConfig()
    a = hz.run_distributed(pb, cfg, 2, 1)
    b = hz.run_distributed(pb, cfg, 2, 1, pool=2)
    assert np.array_equal(a.sigma, b.sigma) and np.array_equal(a.Z.re, b.Z.re)


def test_run_distributed_rejects_bad_sizes():
    c = _case("dist64_real_s2_w8")
    p = hz.ProblemPair(hz.MatrixPlanePair.from_dense(c["F"]), hz.MatrixPlanePair.from_dense(c["G"]))
    with pytest.raises(ValueError):
        hz.run_distributed(p, hz.SolverConfig(block_width=8), 3, 1)
    with pytest.raises(ValueError):
        hz.run_distributed(p, hz.SolverConfig(), 0, 1)
