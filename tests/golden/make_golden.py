"""Generate the golden fixtures from the REFERENCE package itself.

Run in the build container only (needs /root/reference):
    python tests/golden/make_golden.py
Each case stores the inputs (F, G), the configuration and the reference's
outputs of hzgsvd.solve (sigma vectors, counters, and for small cases the
full U, V, Z).  tests/test_oracle.py requires the C oracle to reproduce
them bitwise; the GPU parity tests use the oracle as the checker.
"""

import json
import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))


def cases(hz):
    out = []

    def add(name, F, G, full=True, **cfg):
        out.append((name, np.asarray(F), np.asarray(G), cfg, full))

    CORPUS_SEED = 20260808
    for field, base in (("real", 0), ("complex", 1000)):
        pair, _ = hz.gen_pair(hz.random_genspec(64, CORPUS_SEED + base, field))
        add("corpus64_%s_w8" % field, pair.F.to_dense(), pair.G.to_dense(), block_width=8)
        add("corpus64_%s_w16" % field, pair.F.to_dense(), pair.G.to_dense(), block_width=16)
    pair, _ = hz.gen_pair(hz.random_genspec(32, CORPUS_SEED + 77))
    add("small32_default", pair.F.to_dense(), pair.G.to_dense())
    F = np.triu(np.ones((4, 4)))
    G = np.triu(np.ones((4, 4)))
    G[0, 0] = 1e-10
    add("pitfall4x4_w2", F, G, block_width=2)
    add("pitfall4x4_w16", F, G, block_width=16)
    add("identity16_w4", np.eye(16), np.eye(16), block_width=4)
    add("diag16_w4", np.diag(np.arange(1.0, 17.0)), np.diag(np.roll(np.arange(1.0, 17.0), 1)), block_width=4)
    from hzgsvd.harness import gaussian_stream
    Fc = (gaussian_stream(11, 48 * 32) + 1j * gaussian_stream(12, 48 * 32)).reshape((48, 32), order="F")
    Gc = (gaussian_stream(13, 32 * 32) + 1j * gaussian_stream(14, 32 * 32)).reshape((32, 32), order="F")
    add("complex_tall48x32_w4", Fc, Gc, block_width=4)
    add("complex_tall48x32_w8", Fc, Gc, block_width=8)
    pair, _ = hz.gen_pair(hz.random_genspec(48, 99, "real"))
    for vid in (0, 2, 4, 6):
        add("real48_v%d_w4" % vid, pair.F.to_dense(), pair.G.to_dense(), block_width=4, variant_id=vid)
    add("real48_bo_w4", pair.F.to_dense(), pair.G.to_dense(), block_width=4, blocking="bo")
    add("real48_mm_w4", pair.F.to_dense(), pair.G.to_dense(), block_width=4, outer_kind="mm", inner_kind="mm")
    add("real48_nosort_w4", pair.F.to_dense(), pair.G.to_dense(), block_width=4, sorting=False)
    pairc, _ = hz.gen_pair(hz.random_genspec(40, 98, "complex"))
    add("complex40_v2_w4", pairc.F.to_dense(), pairc.G.to_dense(), block_width=4, variant_id=2)
    add("complex40_v4_w8", pairc.F.to_dense(), pairc.G.to_dense(), block_width=8, variant_id=4)
    g = gaussian_stream(2024, 2 * 200 * 200)
    add("gauss200_w16", g[:40000].reshape((200, 200), order="F"), g[40000:].reshape((200, 200), order="F"),
        full=False, block_width=16)
    # nearly dependent F columns: block Grammians fail Cholesky, the QR
    # shortening fallback takes over (blocked.py:450-462; test_blocked.py:213-230)
    def dependent(n, seed, eps=1e-9, cplx=False):
        rng = np.random.default_rng(seed)
        base = rng.standard_normal(n) + (1j * rng.standard_normal(n) if cplx else 0)
        F = np.empty((n, n), dtype=complex if cplx else float)
        for j in range(n):
            F[:, j] = base + eps * rng.standard_normal(n)
        G = np.eye(n) + 1e-3 * rng.standard_normal((n, n))
        if cplx:
            G = G + 1e-3j * rng.standard_normal((n, n))
        return F, G
    add("qrfallback8_w2", *dependent(8, 31), block_width=2)
    add("qrfallback64_w16", *dependent(64, 7), block_width=16)
    add("qrfallback64_w8", *dependent(64, 7), block_width=8)
    add("qrfallback48_complex_w8", *dependent(48, 11, cplx=True), block_width=8)
    pair, _ = hz.gen_pair(hz.random_genspec(256, 4242, "real"))
    add("genpair256_w16", pair.F.to_dense(), pair.G.to_dense(), full=False, block_width=16)
    # QR shortening instead of Grammian + Cholesky for every block pair
    # (cfg.shorten == "qr", blocked.py:445-447, :487-500)
    pair, _ = hz.gen_pair(hz.random_genspec(48, 99, "real"))
    add("real48_shortenqr_w4", pair.F.to_dense(), pair.G.to_dense(), block_width=4, shorten="qr")
    add("complex40_shortenqr_w4", pairc.F.to_dense(), pairc.G.to_dense(), block_width=4, shorten="qr")
    # compensated dot products (odd variant ids, pointwise.py:40-81, dotprod.py:125-252)
    for vid in (1, 3, 5, 7):
        add("real48_v%d_w4" % vid, pair.F.to_dense(), pair.G.to_dense(), block_width=4, variant_id=vid)
    add("complex40_v1_w4", pairc.F.to_dense(), pairc.G.to_dense(), block_width=4, variant_id=1)
    add("complex40_v7_w8", pairc.F.to_dense(), pairc.G.to_dense(), block_width=8, variant_id=7)
    return out


def main():
    sys.path.insert(0, REF)
    import hzgsvd as hz
    only = None
    if len(sys.argv) > 2 and sys.argv[1] == "--only":
        only = set(sys.argv[2].split(","))
    mpath = os.path.join(HERE, "manifest.json")
    manifest = {}
    if only and os.path.exists(mpath):
        with open(mpath) as fh:
            manifest = json.load(fh)
    for name, F, G, cfg, full in cases(hz):
        if only and name not in only:
            continue
        r = hz.solve(F, G, hz.SolverConfig(**cfg))
        data = dict(F=F, G=G, sigma=r.sigma, sigmaF=r.sigmaF, sigmaG=r.sigmaG,
                    counters=np.array([r.sweeps, r.total_transforms, r.big_transforms, int(r.converged)]))
        if full:
            data.update(U=r.U.to_dense(), V=r.V.to_dense(), Z=r.Z.to_dense())
        np.savez_compressed(os.path.join(HERE, name + ".npz"), **data)
        manifest[name] = dict(cfg=cfg, full=full, n=int(F.shape[1]), mF=int(F.shape[0]), mG=int(G.shape[0]),
                              complex=bool(np.iscomplexobj(F)), sweeps=int(r.sweeps))
        print(name, r.sweeps, r.total_transforms, r.big_transforms, r.converged, flush=True)
    with open(mpath, "w") as fh:
        json.dump(manifest, fh, indent=1, sort_keys=True)


if __name__ == "__main__":
    main()
