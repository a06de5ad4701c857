"""File formats of the reference's pipelines (core.py:126-179, cli.py:94-137).

* a matrix is its real plane then (complex) its imaginary plane, each
  column-major little-endian binary64, with a text sidecar ``<file>.hdr`` of
  ``key=value`` lines: rows, cols, field (real | complex);
* a result directory holds U.bin, V.bin, Z.bin (+ sidecars), ``sigma.tsv``
  (header sigma_f, sigma_g, sigma; one row per value, 17 significant
  digits) and ``stats.txt`` (``sweeps=.. total=.. big=.. converged=0|1``,
  then ``workers=..``).

Planes are read straight into float64 arrays with ``np.fromfile`` (no
intermediate byte string), so a large input can be handed to the device
path without an extra host copy.  Errors are FileFormatError, as in the
reference.
"""

import os

import numpy as np

from .core import MatrixPlanePair
from .errors import FileFormatError

_FIELDS = ("real", "complex")


def read_sidecar(header):
    """(rows, cols, field) from a ``key=value`` sidecar."""
    try:
        with open(header, "r", encoding="utf-8") as fh:
            pairs = [ln.split("=", 1) for ln in (x.strip() for x in fh) if ln]
        kv = {k.strip(): v.strip() for k, v in pairs}
        rows, cols, field = int(kv["rows"]), int(kv["cols"]), kv["field"]
    except (OSError, KeyError, ValueError) as exc:
        raise FileFormatError("unreadable or malformed sidecar %s: %s" % (header, exc))
    if field not in _FIELDS:
        raise FileFormatError("sidecar %s: field must be real or complex" % header)
    if min(rows, cols) < 1:
        raise FileFormatError("sidecar %s: dimensions must be positive" % header)
    return rows, cols, field


def read_matrix(path, header=None):
    """MatrixPlanePair from a plane file and its sidecar (default path + '.hdr')."""
    rows, cols, field = read_sidecar(header or str(path) + ".hdr")
    nplanes = 1 + (field == "complex")
    want = rows * cols * nplanes
    try:
        size = os.path.getsize(path)
        flat = np.fromfile(path, dtype="<f8") if size == 8 * want else None
    except OSError as exc:
        raise FileFormatError("unreadable matrix file %s: %s" % (path, exc))
    if flat is None or flat.size != want:
        raise FileFormatError("size mismatch for %s: sidecar promises %d bytes, file has %d"
                              % (path, 8 * want, size))
    planes = flat.astype(np.float64, copy=False).reshape((nplanes, cols, rows))
    re = planes[0].T
    im = planes[1].T if nplanes == 2 else None
    return MatrixPlanePair(rows, cols, re, im, nplanes == 2)


def write_matrix(m, path):
    """Plane file + sidecar, the byte layout read_matrix expects."""
    with open(path, "wb") as fh:
        for plane in (m.re, m.im) if m.is_complex else (m.re,):
            np.asfortranarray(plane, dtype="<f8").T.tofile(fh)
    with open(str(path) + ".hdr", "w", encoding="utf-8") as fh:
        fh.write("".join("%s=%s\n" % kv for kv in (("rows", m.rows), ("cols", m.cols), ("field", m.field))))


def write_sigma_tsv(path, sigmaF, sigmaG, sigma):
    cols = np.column_stack([np.asarray(v, dtype=np.float64) for v in (sigmaF, sigmaG, sigma)])
    with open(path, "w", encoding="utf-8") as fh:
        fh.write("sigma_f\tsigma_g\tsigma\n")
        for row in cols:
            fh.write("\t".join("%.17g" % x for x in row) + "\n")


def read_sigma_tsv(path):
    """{column name: array} of a sigma.tsv."""
    with open(path, "r", encoding="utf-8") as fh:
        names = fh.readline().strip().split("\t")
        data = np.loadtxt(fh, delimiter="\t", ndmin=2)
    return {k: data[:, q].copy() for q, k in enumerate(names)}


def stats_line(r):
    return "sweeps=%d total=%d big=%d converged=%d" % (r.sweeps, r.total_transforms, r.big_transforms,
                                                       int(bool(r.converged)))


def write_result(r, out_dir):
    """A GsvdResult in the reference CLI's output layout; returns the stats line."""
    os.makedirs(out_dir, exist_ok=True)
    for name, m in (("U", r.U), ("V", r.V), ("Z", r.Z)):
        write_matrix(m, os.path.join(out_dir, name + ".bin"))
    write_sigma_tsv(os.path.join(out_dir, "sigma.tsv"), r.sigmaF, r.sigmaG, r.sigma)
    line = stats_line(r)
    with open(os.path.join(out_dir, "stats.txt"), "w", encoding="utf-8") as fh:
        fh.write("%s\nworkers=%d\n" % (line, r.workers))
    return line
