"""Build libmcf_b200.so in-tree: nvcc for sm_100a, g++ for the host runtime.

The library is the product: CUDA kernels + the C-ABI of include/mcf_gpu.h.
It is built in place (paper_2207_08867_b200/libmcf_b200.so) so that it
travels with the repository snapshot to the GPU box.

FP flags: -fmad=false (no contraction anywhere; FMAs are explicit
__fmaf_rn/__fma_rn), -ftz=false, -prec-div=true, -prec-sqrt=true -- the
error-free transforms need exactly rounded IEEE operations with subnormals.
"""
from __future__ import annotations

import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
BUILD = os.path.join(ROOT, "build", "mcf")
LIB = os.path.join(PKG, "libmcf_b200.so")
CUDA = os.environ.get("CUDA_HOME", "/usr/local/cuda")
NVCC = os.path.join(CUDA, "bin", "nvcc")

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVFLAGS = ARCH + [
    "-O3", "-lineinfo", "-std=c++17", "--expt-relaxed-constexpr",
    "-fmad=false", "-ftz=false", "-prec-div=true", "-prec-sqrt=true",
    "-Xcompiler", "-fPIC", "-Xptxas", "-warn-spills",
    "-I" + os.path.join(ROOT, "include"),
]
CXXFLAGS = ["-O2", "-fPIC", "-std=c++17", "-ffp-contract=off", "-I" + os.path.join(CUDA, "include"),
            "-I" + os.path.join(ROOT, "include")]

CU_SOURCES = ["elementwise.cu", "linalg.cu", "mm_fast.cu", "mm_ozaki.cu", "stream_fast.cu", "mlp.cu", "mlp_fast.cu", "mc_nn.cu",
              "hostapi.cu", "tc_gemm.cu", "mm_skinny.cu"]
CXX_SOURCES = ["runtime.cpp"]


def _sources():
    return [s for s in CU_SOURCES + CXX_SOURCES if os.path.exists(os.path.join(CSRC, s))]


def _deps():
    return [os.path.join(CSRC, f) for f in os.listdir(CSRC)] + [
        os.path.join(ROOT, "include", "mcf_gpu.h"), os.path.abspath(__file__)]


def _stale(target, deps):
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps if os.path.exists(d))


def _compile(src, verbose=False):
    obj = os.path.join(BUILD, src + ".o")
    path = os.path.join(CSRC, src)
    if src.endswith(".cu"):
        cmd = [NVCC] + NVFLAGS + (["-Xptxas", "-v"] if verbose else []) + ["-c", path, "-o", obj]
    else:
        cmd = ["g++"] + CXXFLAGS + ["-c", path, "-o", obj]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"compile failed: {' '.join(cmd)}\n{r.stdout}\n{r.stderr}")
    return obj, r.stderr


def build(force: bool = False, verbose: bool = False) -> str:
    os.makedirs(BUILD, exist_ok=True)
    deps = _deps()
    if not force and not _stale(LIB, deps):
        return LIB
    srcs = _sources()
    with ThreadPoolExecutor(max_workers=len(srcs)) as ex:
        results = list(ex.map(lambda s: _compile(s, verbose), srcs))
    objs = [o for o, _ in results]
    if verbose:
        for (_, log), s in zip(results, srcs):
            if log.strip():
                print(f"--- {s}\n{log}", file=sys.stderr)
    cmd = [NVCC] + ARCH + ["-shared", "-o", LIB] + objs + ["-lquadmath", "-lcudart", "-lcublasLt",
                                                     "-Xlinker", "-rpath=" + os.path.join(CUDA, "lib64")]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"link failed: {' '.join(cmd)}\n{r.stdout}\n{r.stderr}")
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
