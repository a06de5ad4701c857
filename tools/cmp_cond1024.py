"""GPU vs oracle on the n=1024 config-4-style pair (oracle outputs made in
the build container: scratch/cond1024_*.npy)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_1909_00101_b200 as hz
F = np.load("scratch/cond1024_F.npy"); G = np.load("scratch/cond1024_G.npy"); s_ref = np.load("scratch/cond1024_sigma.npy")
for blocking in ("fb", "bo"):
    r = hz.solve(F, G, hz.SolverConfig(block_width=16, max_outer_sweeps=100, blocking=blocking))
    print(blocking, "sweeps", r.sweeps, "total", r.total_transforms, "big", r.big_transforms,
          "max rel sigma vs oracle(fb) %.2e" % np.max(np.abs(r.sigma - s_ref) / s_ref))
r = hz.solve(F, G, hz.SolverConfig(block_width=16, max_outer_sweeps=100, exact=True))
print("exact sweeps", r.sweeps, "total", r.total_transforms, "big", r.big_transforms, "bitwise", np.array_equal(r.sigma, s_ref))
