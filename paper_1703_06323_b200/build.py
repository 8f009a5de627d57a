"""Build libcutbddc.so in-tree for sm_100a (nvcc cross-compiles without a GPU).

geometry.cu and element.cu are compiled with -fmad=false: phi,
classification and cut-cell quadrature keep the host op order (bit-exact
parity with the reference classification and the CPU restatement).
"""
from __future__ import annotations

import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
BUILD = os.path.join(HERE, "_build")
LIB = os.path.join(HERE, "libcutbddc.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NO_FMA = {"geometry.cu", "element.cu"}
CU = ["geometry.cu", "element.cu", "assembly.cu", "dist.cu", "factor.cu", "sweep.cu", "dense_dag.cu", "coarse_sparse.cu", "bddc.cu", "pcg.cu",
      "objects.cu", "peak.cu", "capi.cu"]
CPP = ["nd_template.cpp", "host_partition.cpp"]
def _nccl_dir() -> str:
    """NCCL of the torch wheel (the one torch itself loads: one libnccl per process)."""
    import importlib.util
    spec = importlib.util.find_spec("nvidia")
    for base in (list(spec.submodule_search_locations) if spec else []):
        d = os.path.join(base, "nccl")
        if os.path.exists(os.path.join(d, "include", "nccl.h")):
            return d
    raise RuntimeError("NCCL headers not found (nvidia-nccl wheel)")


NCCL = _nccl_dir()
HEADERS = [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".hpp", ".cuh"))] + [
    os.path.join(ROOT, "include", "cutbddc.h")]


def _stale(obj: str, src: str) -> bool:
    if not os.path.exists(obj):
        return True
    t = os.path.getmtime(obj)
    return any(os.path.getmtime(p) > t for p in [src] + HEADERS)


def _run(cmd):
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError("build failed:\n" + " ".join(cmd) + "\n" + r.stdout + r.stderr)
    return r.stdout + r.stderr


def build(verbose: bool = False, force: bool = False) -> str:
    os.makedirs(BUILD, exist_ok=True)
    inc = ["-I" + CSRC, "-I" + os.path.join(ROOT, "include"), "-I" + os.path.join(NCCL, "include")]
    jobs = []
    objs = []
    for f in CU:
        src, obj = os.path.join(CSRC, f), os.path.join(BUILD, f + ".o")
        objs.append(obj)
        if force or _stale(obj, src):
            flags = ["-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC", "-Xptxas", "-v" if verbose else "-O3",
                     "--expt-relaxed-constexpr"] + ARCH + inc
            flags.append("-fmad=false" if f in NO_FMA else "-fmad=true")
            flags += os.environ.get("CUTBDDC_NVCC_EXTRA", "").split()  # tuning macros (tools/tune_sweep.sh)
            jobs.append([NVCC] + flags + ["-c", src, "-o", obj])
    for f in CPP:
        src, obj = os.path.join(CSRC, f), os.path.join(BUILD, f + ".o")
        objs.append(obj)
        if force or _stale(obj, src):
            jobs.append(["g++", "-O3", "-std=c++20", "-fPIC", "-Wall", "-ffp-contract=off"] + inc +
                        ["-I/usr/local/cuda/include", "-c", src, "-o", obj])
    with ThreadPoolExecutor(max_workers=os.cpu_count() or 4) as ex:
        outs = list(ex.map(_run, jobs))
    if verbose:
        for o in outs:
            sys.stdout.write(o)
    if jobs or not os.path.exists(LIB):
        lib = os.path.join(NCCL, "lib")
        _run([NVCC] + ARCH + ["-shared", "-o", LIB] + objs +
             ["-lcudart", "-L" + lib, "-l:libnccl.so.2", "-Xlinker", "-rpath=" + lib])
    return LIB


if __name__ == "__main__":
    print(build(verbose="-v" in sys.argv, force="-f" in sys.argv))
