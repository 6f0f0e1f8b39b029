"""Build libgmaf.so in-tree with nvcc for sm_100a (no GPU needed).

Translation units:
  geometry.cu  --fmad=false  (thickness / assembly / quadrature: bitwise reproducible)
  pcg.cu                      (two-phase Table-1 PCG-ASSOR kernels; FMA allowed)
  sr.cu                       (single-pass PCG-ASSOR kernel, TMA row streaming)
  gmaf_api.cu                 (host runtime, C ABI of include/gmaf.h)
  picard.cu                   (host Picard driver: general forces, FD Jacobians, update)
"""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
BUILD = os.path.join(HERE, "_build")
LIB = os.path.join(HERE, "libgmaf.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
COMMON = ["-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC,-ffp-contract=off,-fno-fast-math",
          "-I" + os.path.join(ROOT, "include"), "-Xptxas", "-v"]
UNITS = [("geometry.cu", ["--fmad=false"]), ("pcg.cu", []), ("sr.cu", []), ("gmaf_api.cu", []), ("picard.cu", [])]
# GMAF_NVCC_EXTRA: extra nvcc flags for timing-only experiments (e.g. -DGMAF_EXPERIMENT_NOBAR);
# never set for the product build
EXTRA = os.environ.get("GMAF_NVCC_EXTRA", "").split()


def _deps():
    files = [os.path.join(CSRC, f) for f in os.listdir(CSRC)]
    files.append(os.path.join(ROOT, "include", "gmaf.h"))
    files.append(os.path.abspath(__file__))
    return max(os.path.getmtime(f) for f in files)


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and os.path.exists(LIB) and os.path.getmtime(LIB) >= _deps():
        return LIB
    os.makedirs(BUILD, exist_ok=True)
    objs = []
    for src, extra in UNITS:
        obj = os.path.join(BUILD, src.replace(".cu", ".o"))
        cmd = [NVCC, *ARCH, *COMMON, *extra, *EXTRA, "-c", os.path.join(CSRC, src), "-o", obj]
        res = subprocess.run(cmd, capture_output=True, text=True)
        log = os.path.join(BUILD, src + ".log")
        with open(log, "w") as f:
            f.write(" ".join(cmd) + "\n" + res.stdout + res.stderr)
        if res.returncode != 0:
            sys.stderr.write(res.stdout + res.stderr)
            raise RuntimeError(f"nvcc failed for {src} (see {log})")
        if verbose:
            sys.stdout.write(res.stderr)
        objs.append(obj)
    tmp = LIB + ".tmp"
    cmd = [NVCC, *ARCH, "-shared", "-o", tmp, *objs, "-Xcompiler", "-fPIC"]
    subprocess.check_call(cmd)
    os.replace(tmp, LIB)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True))
