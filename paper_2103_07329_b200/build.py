"""Build libmrsolve_b200.so in-tree (sm_100a) from csrc/.

    python -m paper_2103_07329_b200.build        # or __graft_entry__.build()

CUDA sources: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo.
Host setup (amg_setup.cpp): g++ -O2 -ffp-contract=off (bitwise reference
arithmetic).  The CUDA runtime is linked statically so the library does not
depend on torch's runtime version.  Rebuilds only when a source is newer
than the library.
"""

from __future__ import annotations

import concurrent.futures as cf
import glob
import os
import shutil
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
ROOT = os.path.dirname(HERE)
# MRS_CHECKS=1: the checked variant (device asserts, see csrc/common.cuh)
CHECKED = os.environ.get("MRS_CHECKS", "0") == "1"
LIB = os.path.join(HERE, "libmrsolve_b200_checked.so" if CHECKED else "libmrsolve_b200.so")
BUILD = os.path.join(ROOT, "build", "mrsolve_b200_checked" if CHECKED else "mrsolve_b200")

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = (["-DMRS_CHECKS"] if os.environ.get("MRS_CHECKS", "0") == "1" else []) + [
              "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "--expt-relaxed-constexpr",
              "-Xptxas", "-warn-spills"]
CXX_FLAGS = ["-O2", "-ffp-contract=off", "-fno-fast-math", "-fPIC", "-std=c++17"]


def _nvcc():
    for c in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", shutil.which("nvcc")):
        if c and os.path.exists(c):
            return c
    raise RuntimeError("nvcc not found: the CUDA extension cannot be built")


def _sources():
    cu = sorted(glob.glob(os.path.join(CSRC, "*.cu")))
    cpp = sorted(glob.glob(os.path.join(CSRC, "*.cpp")))
    deps = sorted(glob.glob(os.path.join(CSRC, "*.cuh")) + glob.glob(os.path.join(CSRC, "*.h"))
                  + glob.glob(os.path.join(ROOT, "include", "*.h")))
    return cu, cpp, deps


def needs_build() -> bool:
    if not os.path.exists(LIB):
        return True
    cu, cpp, deps = _sources()
    t = os.path.getmtime(LIB)
    return any(os.path.getmtime(f) > t for f in cu + cpp + deps + [__file__])


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and not needs_build():
        return LIB
    nvcc = _nvcc()
    os.makedirs(BUILD, exist_ok=True)
    cu, cpp, _ = _sources()
    jobs = []
    for src in cu:
        if os.path.basename(src) == "spmm_inst.cu":
            # the SpMM template family: one object per (value type, op)
            for f32 in (0, 1):
                for op in range(4):
                    obj = os.path.join(BUILD, f"spmm_inst_{'f32' if f32 else 'f64'}_{op}.o")
                    jobs.append([nvcc, *ARCH, *NVCC_FLAGS, f"-DMRS_INST_F32={f32}",
                                 f"-DMRS_INST_OP={op}", "-c", src, "-o", obj])
            continue
        obj = os.path.join(BUILD, os.path.basename(src) + ".o")
        jobs.append([nvcc, *ARCH, *NVCC_FLAGS, "-c", src, "-o", obj])
    cxx = os.environ.get("CXX", "g++")
    for src in cpp:
        obj = os.path.join(BUILD, os.path.basename(src) + ".o")
        jobs.append([cxx, *CXX_FLAGS, "-c", src, "-o", obj])

    def run(cmd):
        r = subprocess.run(cmd, capture_output=True, text=True)
        return cmd, r

    with cf.ThreadPoolExecutor(max_workers=min(12, os.cpu_count() or 2)) as ex:
        for cmd, r in ex.map(run, jobs):
            if verbose or r.returncode != 0:
                sys.stderr.write(" ".join(cmd) + "\n" + r.stdout + r.stderr)
            if r.returncode != 0:
                raise RuntimeError(f"compile failed: {os.path.basename(cmd[-3])}")
    objs = [j[-1] for j in jobs]
    tmp = LIB + ".tmp"
    link = [nvcc, *ARCH, "-shared", "-o", tmp, *objs, "-cudart", "static", "-lnccl", "-lpthread",
            "-ldl", "-lrt"]
    r = subprocess.run(link, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(" ".join(link) + "\n" + r.stdout + r.stderr)
        raise RuntimeError("link failed")
    os.replace(tmp, LIB)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
