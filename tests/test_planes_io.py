"""File formats of the reference's pipelines (planes_io.py): round trips and
byte-level agreement with the reference's own writer/reader (core.py:126-179,
cli.py:94-137) -- the expected bytes are built here from the format
definition, and, when /root/reference is present, checked against the
reference's functions themselves."""

import os
import sys

import numpy as np
import pytest

import paper_1909_00101_b200 as hz

REF = "/root/reference/pkg/src"


def _mat(cplx, shape=(5, 3)):
    a = np.arange(np.prod(shape), dtype=float).reshape(shape) * 0.37 - 1.1
    return a + (1j * a[::-1] if cplx else 0)


@pytest.mark.parametrize("cplx", [False, True])
def test_matrix_round_trip_and_layout(tmp_path, cplx):
    A = _mat(cplx)
    m = hz.MatrixPlanePair.from_dense(A)
    path = str(tmp_path / "a.bin")
    hz.write_matrix(m, path)
    raw = np.fromfile(path, dtype="<f8")
    want = np.concatenate([A.real.ravel(order="F")] + ([A.imag.ravel(order="F")] if cplx else []))
    assert np.array_equal(raw, want)
    assert open(path + ".hdr").read() == "rows=5\ncols=3\nfield=%s\n" % ("complex" if cplx else "real")
    r = hz.read_matrix(path)
    assert r.is_complex == cplx and np.array_equal(r.to_dense(), A)


def test_matrix_format_errors(tmp_path):
    m = hz.MatrixPlanePair.from_dense(_mat(False))
    path = str(tmp_path / "a.bin")
    hz.write_matrix(m, path)
    with open(path, "ab") as fh:
        fh.write(b"x")
    with pytest.raises(hz.FileFormatError):
        hz.read_matrix(path)
    with open(path + ".hdr", "w") as fh:
        fh.write("rows=5\ncols=3\nfield=quaternion\n")
    with pytest.raises(hz.FileFormatError):
        hz.read_matrix(path)
    with pytest.raises(hz.FileFormatError):
        hz.read_matrix(str(tmp_path / "missing.bin"))


def test_result_directory(tmp_path):
    M = hz.MatrixPlanePair.from_dense
    r = hz.GsvdResult(M(np.eye(3)), M(np.eye(3)), M(np.eye(3)), np.array([0.6, 0.8, 1 / 3]),
                      np.array([0.8, 0.6, 0.1]), np.array([0.75, 4 / 3, 10 / 3]), sweeps=4, total_transforms=9,
                      big_transforms=2, converged=True, workers=2)
    line = hz.write_result(r, str(tmp_path / "out"))
    assert line == "sweeps=4 total=9 big=2 converged=1"
    assert open(tmp_path / "out" / "stats.txt").read() == line + "\nworkers=2\n"
    tsv = open(tmp_path / "out" / "sigma.tsv").read().splitlines()
    assert tsv[0] == "sigma_f\tsigma_g\tsigma"
    assert tsv[3].split("\t")[2] == "%.17g" % (10 / 3)
    back = hz.read_sigma_tsv(str(tmp_path / "out" / "sigma.tsv"))
    assert np.array_equal(back["sigma"], r.sigma) and np.array_equal(back["sigma_f"], r.sigmaF)
    assert np.array_equal(hz.read_matrix(str(tmp_path / "out" / "Z.bin")).to_dense(), np.eye(3))


@pytest.mark.skipif(not os.path.isdir(REF), reason="reference package not present")
@pytest.mark.parametrize("cplx", [False, True])
def test_bytes_identical_to_reference_writer(tmp_path, cplx):
    sys.path.insert(0, REF)
    try:
        from hzgsvd import core as rc
    except Exception as exc:  # pragma: no cover - numba import issues
        pytest.skip("reference import failed: %s" % exc)
    A = _mat(cplx, (7, 4))
    ours, theirs = str(tmp_path / "o.bin"), str(tmp_path / "t.bin")
    hz.write_matrix(hz.MatrixPlanePair.from_dense(A), ours)
    rc.write_matrix(rc.MatrixPlanePair.from_dense(A), theirs)
    assert open(ours, "rb").read() == open(theirs, "rb").read()
    assert open(ours + ".hdr").read() == open(theirs + ".hdr").read()
    assert np.array_equal(rc.read_matrix(ours, ours + ".hdr").to_dense(), hz.read_matrix(theirs).to_dense())
