"""Golden fixtures for the device accuracy report, from the REFERENCE itself
(build container only):  python tests/golden/make_accuracy_golden.py

For three golden pairs: the reference's solve result, its accuracy_report
(harness.py:436-465) and the complete-pivoting LU factors of Z
(_k_lu_complete, harness.py:323-371) with the permutations and X = Z^{-1}.
"""

import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))


def main():
    sys.path.insert(0, REF)
    import hzgsvd as hz
    from hzgsvd import harness as H
    for name in ("corpus64_real_w16", "corpus64_complex_w16", "gauss200_w16"):
        c = dict(np.load(os.path.join(HERE, name + ".npz")))
        F, G = c["F"], c["G"]
        cfg = hz.SolverConfig(block_width=16)
        r = hz.solve(F, G, cfg)
        p = hz.ProblemPair(hz.MatrixPlanePair.from_dense(F), hz.MatrixPlanePair.from_dense(G))
        rep = H.accuracy_report(p, r)
        Z = r.Z.to_dense()
        Ar, Ai, cplx = H._dense(np.array(Z))
        n = Ar.shape[0]
        rp = np.arange(n, dtype=np.int64)
        cp = np.arange(n, dtype=np.int64)
        assert H._k_lu_complete(Ar, Ai, cplx, rp, cp) == 0
        X = H.invert_via_lu(Z)
        np.savez_compressed(os.path.join(HERE, "acc_%s.npz" % name), F=F, G=G, U=r.U.to_dense(), V=r.V.to_dense(),
                            Z=Z, sigmaF=r.sigmaF, sigmaG=r.sigmaG, sigma=r.sigma, LUr=Ar, LUi=Ai, rp=rp, cp=cp, X=X,
                            report=np.array([rep.resF, rep.resG, rep.orthU, rep.orthV]))
        print(name, rep)


if __name__ == "__main__":
    main()
