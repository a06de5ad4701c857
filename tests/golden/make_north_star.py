"""Oracle fixtures for BASELINE.json configurations 2-4 (north-star shapes).

Run once in the build container (CPU, all cores; config 4 takes about an hour):
    python tests/golden/make_north_star.py [config2 config3 config4]

The inputs are regenerated bit-for-bit on any host by oracle/hzo_gen.c
(oracle.ns_inputs), so only the results are stored: the oracle's sorted
sigma vectors, sweep and transform counters, and SHA-256 digests of the
inputs and of the U, V, Z output planes (the exact-mode GPU path must
reproduce those bytes).  The oracle itself is pinned bitwise to the
reference's outputs (tests/test_oracle.py, make_golden.py).
"""

import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from oracle import oracle as O  # noqa: E402


def make(name, threads=None):
    F, G, kw, extra = O.ns_inputs(name)
    t0 = time.time()
    r = O.solve(F, G, O.make_cfg(**kw), threads=threads)
    dt = time.time() - t0
    out = dict(sigma=r["sigma"], sigmaF=r["sigmaF"], sigmaG=r["sigmaG"], sweeps=r["sweeps"],
               total=r["total"], big=r["big"], converged=r["converged"],
               input_sha=O.sha256_planes(F, G), U_sha=O.sha256_planes(r["U"]),
               V_sha=O.sha256_planes(r["V"]), Z_sha=O.sha256_planes(r["Z"]),
               oracle_seconds=dt, oracle_threads=threads or os.cpu_count(),
               desc=O.NS_CONFIGS[name][1], **extra)
    np.savez_compressed(os.path.join(HERE, "ns_%s.npz" % name), **out)
    print("%s: %d sweeps, total %d, big %d, converged %s, %.0f s" % (name, r["sweeps"], r["total"], r["big"],
                                                                     r["converged"], dt), flush=True)


if __name__ == "__main__":
    for nm in sys.argv[1:] or ["config2", "config3", "config4"]:
        make(nm)
