"""Isolated per-kernel times of one outer sweep at config 4 (real 4096^2,
sigma in [1e-8, 1e8], w = 16), early (sweep 2) and after convergence:
python tools/step_breakdown.py [n] [w]"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_1909_00101_b200 as hz  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
w = int(sys.argv[2]) if len(sys.argv) > 2 else 16


class A:
    pass


a = A()
a.n, a.kind, a.seed, a.w = n, "cond", 4096, w
F0, G0, _ = bench.gen_pair(a, torch, torch.device("cuda"))
dev = hz.DeviceGsvd({"Fr": F0, "Gr": G0, "Fi": None, "Gi": None}, hz.SolverConfig(block_width=w, max_outer_sweeps=100))
osteps = n // w - 1


def timed_sweep():
    dev.kernel_times(reset=True)
    dev.run_steps(0, osteps)
    kt = dev.kernel_times(reset=True)
    t, b = dev.collect()
    if b:
        dev.rescale_z()
    return kt, b


def show(label, kt):
    tot = sum(ms for ms, _ in kt.values())
    parts = "  ".join("%s %.1f us/step (%.0f%%)" % (k, ms * 1e3 / osteps, 100 * ms / tot) for k, (ms, c) in kt.items())
    print("%s: %.1f ms per sweep serialised; %s" % (label, tot, parts), flush=True)


dev.set_timing(True)
dev.init()
for sw in range(100):
    kt, b = timed_sweep()
    if sw < 3 or b == 0 or sw % 10 == 9:
        show("sweep %d" % (sw + 1), kt)
    if b == 0:
        break

# the converged regime: inner-step cycles of CTA 0 (hzg_debug_phases) over
# one more sweep, against the inner launch time
import ctypes  # noqa: E402

import numpy as np  # noqa: E402

ph = np.zeros(4, dtype=np.int64)
dev.lib.hzg_debug_phases(dev.ctx, 1, None)
kt, b = timed_sweep()
dev.lib.hzg_debug_phases(dev.ctx, 0, ph.ctypes.data_as(ctypes.c_void_p))
ph[0] -= (int(ph[0]) // 1000000000) * 1000000000
show("one more sweep (phase counters on)", kt)
steps = int(ph[3])
cyc = ph[:3].sum() / max(1, steps)
inner_us = kt["inner"][0] * 1e3 / osteps
loop_us = steps / osteps * cyc / 1.965e3
print("CTA 0: %.1f inner steps per outer step, %.0f cycles each (A %.0f B %.0f C %.0f): %.1f us of the %.1f us "
      "inner launch; the rest (fold, Cholesky, prescale, theta rescale, identity test, Z~ store, launch) %.1f us"
      % (steps / osteps, cyc, ph[0] / steps, ph[1] / steps, ph[2] / steps, loop_us, inner_us, inner_us - loop_us))
