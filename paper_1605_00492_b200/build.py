"""Build the CUDA library libhmg.so in-tree (sm_100a, nvcc).

Flags: -fmad=false on device code and -ffp-contract=off on host code keep the
canonical operation order of DESIGN.md (no FMA contraction), so the V-cycle
path is bitwise comparable with the oracle.  Division and sqrt stay IEEE
round-to-nearest (nvcc defaults -prec-div=true -prec-sqrt=true).
"""
from __future__ import annotations

import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libhmg.so")
SOURCES = ["api.cu", "kernels.cu", "sweep_tc.cu", "sweep_st.cu", "apply_st.cu", "sweep_small.cu", "thomas_factor.cu",
           "coarse_coop.cu", "mesh.cpp", "dist.cpp", "nccl_dyn.cpp", "mixed.cu", "band.cu"]
# test-only in-process collective transport (HMG_TRANSPORT=local), its own library
TEST_SOURCES = ["local_transport.cu"]
TEST_LIB = os.path.join(HERE, "libhmg_localtx.so")
HEADERS = ["hmg_internal.h", "mf_ops.cuh", "small_tile.cuh", "mesh.h", "sm100_ptx.cuh", "dist.h", "nccl_dyn.h", os.path.join("..", "..", "include", "hmg.h")]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-fmad=false", "-Xcompiler", "-fPIC,-ffp-contract=off,-O2",
         "-Xptxas", "-v", "--expt-relaxed-constexpr"]


def _stale() -> bool:
    if not (os.path.exists(LIB) and os.path.exists(TEST_LIB)):
        return True
    t = min(os.path.getmtime(LIB), os.path.getmtime(TEST_LIB))
    deps = [os.path.join(CSRC, f) for f in SOURCES + TEST_SOURCES + HEADERS] + [__file__]
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and not _stale():
        return LIB
    tmp = LIB + f".tmp{os.getpid()}"
    objdir = os.path.join(HERE, "build")
    os.makedirs(objdir, exist_ok=True)
    # one nvcc per translation unit, in parallel, then one link
    jobs = []
    for src in SOURCES:
        obj = os.path.join(objdir, src + f".{os.getpid()}.o")
        jobs.append(([NVCC, *ARCH, *FLAGS, "-c", os.path.join(CSRC, src), "-o", obj], obj))
    with ThreadPoolExecutor(max_workers=min(len(jobs), os.cpu_count() or 1)) as ex:
        results = list(ex.map(lambda j: subprocess.run(j[0], capture_output=True, text=True), jobs))
    link = [NVCC, *ARCH, "-shared", *[o for _, o in jobs], "-o", tmp, "-ldl"]
    results.append(subprocess.run(link, capture_output=True, text=True) if all(r.returncode == 0 for r in results)
                   else subprocess.CompletedProcess(link, 1, "", "link skipped: compile failed\n"))
    # the test-only transport library (not linked into libhmg.so)
    tmp_test = TEST_LIB + f".tmp{os.getpid()}"
    test_cmd = [NVCC, *ARCH, *FLAGS, "-shared", *[os.path.join(CSRC, f) for f in TEST_SOURCES], "-o", tmp_test]
    results.append(subprocess.run(test_cmd, capture_output=True, text=True))
    log = "".join(" ".join(c) + "\n" + r.stdout + r.stderr
                  for c, r in zip([j[0] for j in jobs] + [link, test_cmd], results))
    with open(os.path.join(HERE, "build.log"), "w") as fh:
        fh.write(log)
    for _, o in jobs:
        if os.path.exists(o):
            os.remove(o)
    if any(r.returncode != 0 for r in results):
        sys.stderr.write(log)
        raise RuntimeError("nvcc failed building libhmg.so (see paper_1605_00492_b200/build.log)")
    if verbose:
        sys.stderr.write(log)
    os.replace(tmp, LIB)
    os.replace(tmp_test, TEST_LIB)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True))
