"""In-tree build of libhzg.so (sm_100a) with nvcc.

Every translation unit is compiled with -fmad=false: products and sums stay
separately rounded unless the source writes fma(), the reference's rule
(pkg/src/hzgsvd/_fp.py:16-31), which is what makes the reference-order
kernels bit-compatible with the CPU reference.
"""

import os
import shutil
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
OUT_DIR = os.path.join(HERE, "_lib")
LIB = os.path.join(OUT_DIR, "libhzg.so")
PEAK_LIB = os.path.join(OUT_DIR, "libhzg_peak.so")
SOURCES = ["hzg_api.cu", "hzg_kernels.cu", "hzg_inner.cu", "hzg_dmma.cu", "hzg_tall.cu", "hzg_nccl.cu", "hzg_accuracy.cu"]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def nvcc():
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", shutil.which("nvcc")):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found")


def flags():
    return ARCH + ["-O3", "-lineinfo", "-std=c++17", "-fmad=false", "-Xcompiler", "-fPIC",
                   "-I", os.path.join(ROOT, "include"), "-Xptxas", "-warn-spills"]


def _stale(target, deps):
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def build(force=False, verbose=False):
    os.makedirs(OUT_DIR, exist_ok=True)
    headers = [os.path.join(CSRC, h) for h in os.listdir(CSRC) if h.endswith((".h", ".cuh"))]
    headers.append(os.path.join(ROOT, "include", "hzg.h"))
    objs = []
    jobs = []
    for src in SOURCES:
        s = os.path.join(CSRC, src)
        o = os.path.join(OUT_DIR, src.replace(".cu", ".o"))
        objs.append(o)
        if force or _stale(o, [s] + headers):
            jobs.append([nvcc()] + flags() + ["-c", s, "-o", o])

    def run(cmd):
        if verbose:
            print(" ".join(cmd), flush=True)
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError("nvcc failed:\n" + r.stdout + r.stderr)
        return r.stderr

    with ThreadPoolExecutor(max_workers=len(jobs) or 1) as ex:
        for msg in ex.map(run, jobs):
            if verbose and msg:
                sys.stderr.write(msg)
    if force or jobs or _stale(LIB, objs):
        run([nvcc()] + ARCH + ["-shared", "-o", LIB] + objs + ["-lcuda", "-ldl"])
    # the FP64 DMMA peak probe bench.py measures its roofline denominator
    # with (tools/hzg_peak.cu; measurement only, not on the solve path)
    src = os.path.join(ROOT, "tools", "hzg_peak.cu")
    if force or _stale(PEAK_LIB, [src]):
        run([nvcc()] + ARCH + ["-O3", "-std=c++17", "-Xcompiler", "-fPIC", "-shared", "-o", PEAK_LIB, src])
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True))
