"""Golden vectors for preprocess_tall, generated from the REFERENCE package.

Run in the build container only (needs /root/reference):
    python tests/golden/make_tall_golden.py
Each tall_*.npz holds the inputs F, G (re / im planes), the reference's
shortened pair F'', G'' and the permutation piv of hzgsvd.blocked.
preprocess_tall (blocked.py:405-428), or the RankError it raised
("error": "F" / "G").  tests/test_gpu_tall.py requires the device path to
reproduce them bitwise.
"""

import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))


def cases():
    sys.path.insert(0, REF)
    from hzgsvd.harness import gaussian_stream

    def g(seed, m, n, cplx=False):
        a = gaussian_stream(seed, m * n).reshape((m, n), order="F")
        if cplx:
            a = a + 1j * gaussian_stream(seed + 1, m * n).reshape((m, n), order="F")
        return a

    out = [("tall_real_40x24", g(1, 40, 24), g(3, 30, 24)),
           ("tall_complex_48x32", g(5, 48, 32, True), g(7, 40, 32, True)),
           ("tall_square_real_24", g(9, 24, 24), g(11, 24, 24)),
           ("tall_real_130x96", g(13, 130, 96), g(15, 100, 96))]
    # equal column norms everywhere: every pivot choice is a tie (lowest index)
    F = np.vstack([np.eye(8), np.zeros((4, 8))])
    out.append(("tall_ties_real", F, g(17, 10, 8)))
    # a zero column of F: the QR stops (RankError)
    F = g(19, 20, 12)
    F[:, 5] = 0.0
    out.append(("tall_zero_column", F, g(21, 16, 12)))
    # a nearly dependent column pair: a diagonal below n eps x its entry norm
    F = g(23, 20, 12)
    F[:, 7] = F[:, 2] * 3.0 + 1e-18
    out.append(("tall_dependent_columns", F, g(25, 16, 12)))
    # complex G nearly rank deficient
    G = g(27, 18, 10, True)
    G[:, 9] = G[:, 0] * (1 - 2j)
    out.append(("tall_complex_dependent_G", g(29, 24, 10, True), G))
    return out


def main():
    sys.path.insert(0, REF)
    from hzgsvd.blocked import preprocess_tall
    from hzgsvd.core import MatrixPlanePair
    from hzgsvd.errors import RankError

    for name, F, G in cases():
        data = dict(F_re=np.real(F), F_im=np.imag(F), G_re=np.real(G), G_im=np.imag(G),
                    cplx=np.array(int(np.iscomplexobj(F) or np.iscomplexobj(G))))
        try:
            Fpp, Gpp, piv = preprocess_tall(MatrixPlanePair.from_dense(F), MatrixPlanePair.from_dense(G))
            a, b = Fpp.to_dense(), Gpp.to_dense()
            data.update(Fpp_re=np.real(a), Fpp_im=np.imag(a), Gpp_re=np.real(b), Gpp_im=np.imag(b),
                        piv=np.asarray(piv, dtype=np.int64), error=np.array(""))
        except RankError as e:
            which = "F" if "of F" in str(e) or " F " in str(e) else "G"
            data.update(error=np.array(which))
        np.savez_compressed(os.path.join(HERE, name + ".npz"), **data)
        print(name, F.shape, G.shape, "error=" + str(data["error"]))


if __name__ == "__main__":
    main()
