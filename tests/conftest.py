import json
import os
import sys

import numpy as np
import pytest

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)
GOLDEN = os.path.join(HERE, "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (run on the B200 box)")


def manifest():
    with open(os.path.join(GOLDEN, "manifest.json")) as fh:
        return json.load(fh)


def load_case(name):
    d = dict(np.load(os.path.join(GOLDEN, name + ".npz")))
    d.update(manifest()[name])
    return d


def sorted_desc(x):
    return np.sort(np.asarray(x))[::-1].copy()


def rel_err_sorted(computed, reference):
    c = sorted_desc(computed)
    r = sorted_desc(reference)
    return np.abs(c - r) / np.abs(r)


def gsvd_metrics(F, G, r):
    """North-star self-consistency metrics of a GsvdResult (dense numpy)."""
    U, V, Z = r.U.to_dense(), r.V.to_dense(), r.Z.to_dense()
    n = Z.shape[1]
    resF = np.linalg.norm(F @ Z - U * r.sigmaF[None, :]) / np.linalg.norm(F)
    resG = np.linalg.norm(G @ Z - V * r.sigmaG[None, :]) / np.linalg.norm(G)
    orthU = np.linalg.norm(U.conj().T @ U - np.eye(n))
    orthV = np.linalg.norm(V.conj().T @ V - np.eye(n))
    pencil = np.abs(r.sigmaF ** 2 + r.sigmaG ** 2 - 1.0).max()
    return dict(resF=resF, resG=resG, orthU=orthU, orthV=orthV, pencil=pencil)
