"""Build libchfsi.so in-tree with nvcc for sm_100a (no torch JIT, no cache).

    python -m paper_1206_3768_b200.csrc.build [--force] [-v]

Objects go to paper_1206_3768_b200/csrc/build/, the shared library to
paper_1206_3768_b200/libchfsi.so (git-ignored; it travels to the GPU box
with the gpurun snapshot).
"""

from __future__ import annotations

import argparse
import os
import subprocess
import sys

CSRC = os.path.dirname(os.path.abspath(__file__))
PKG = os.path.dirname(CSRC)
ROOT = os.path.dirname(PKG)
BUILD = os.path.join(CSRC, "build")
LIB = os.path.join(PKG, "libchfsi.so")
SOURCES = ["cheb_step.cu", "cheb_step_3m.cu", "lanczos.cu", "nd_eig.cu", "nd_persist.cu", "aux_kernels.cu", "panel_kernels.cu",
           "chfsi_abi.cu", "chfsi_loop.cu"]
HEADERS = ["common.cuh", "cheb_step_kernel.cuh", "chfsi_internal.h", "abi_internal.h"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
CFLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-Xcompiler", "-fvisibility=hidden",
          "--expt-relaxed-constexpr", "-Xptxas", "-warn-spills"]
LDFLAGS = ["-L/usr/local/cuda/lib64", "-lcublas", "-lcusolver", "-Xlinker", "-rpath=/usr/local/cuda/lib64"]


def _newer(target, deps):
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def _run(cmd, verbose):
    if verbose:
        print(" ".join(cmd), flush=True)
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        sys.stderr.write(res.stdout + res.stderr)
        raise RuntimeError(f"nvcc failed: {' '.join(cmd)}")
    if verbose and (res.stdout or res.stderr):
        print(res.stdout + res.stderr)
    return res


def build(force=False, verbose=False, ptxas_verbose=False):
    os.makedirs(BUILD, exist_ok=True)
    headers = [os.path.join(CSRC, h) for h in HEADERS] + [os.path.join(ROOT, "include", "chfsi.h")]
    objs, jobs = [], []
    for src in SOURCES:
        s = os.path.join(CSRC, src)
        o = os.path.join(BUILD, src.replace(".cu", ".o"))
        objs.append(o)
        if force or _newer(o, [s] + headers + [__file__]):
            extra = ["-Xptxas", "-v"] if ptxas_verbose else []
            jobs.append([NVCC, *ARCH, *CFLAGS, *extra, "-DCHFSI_BUILDING", "-c", s, "-o", o])
    if jobs:  # translation units compile in parallel (nvcc is single-threaded)
        import concurrent.futures

        with concurrent.futures.ThreadPoolExecutor(max_workers=min(len(jobs), os.cpu_count() or 1)) as ex:
            for f in [ex.submit(_run, cmd, verbose or ptxas_verbose) for cmd in jobs]:
                f.result()
    if force or _newer(LIB, objs):
        _run([NVCC, *ARCH, "-shared", *objs, "-o", LIB, *LDFLAGS], verbose)
    return LIB


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--force", action="store_true")
    ap.add_argument("-v", "--verbose", action="store_true")
    ap.add_argument("--ptxas", action="store_true", help="print registers/spills per kernel")
    a = ap.parse_args()
    print(build(a.force, a.verbose, a.ptxas))


if __name__ == "__main__":
    main()
