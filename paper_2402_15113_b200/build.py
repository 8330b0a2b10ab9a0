"""Build libmspipe.so (sm_100a) in-tree with nvcc.  No JIT, no torch extension:
the product is a plain C-ABI shared library (include/mspipe.h)."""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libmspipe.so")
SOURCES = ["api.cu", "sampler.cu", "memory.cu", "prep.cu", "gru_simt.cu", "gru_tc.cu", "shard.cu", "nccl_xchg.cu", "planner.cu",
           "stale.cu", "features.cu", "train.cu", "apan.cu"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")


def _nccl_dir():
    """NCCL ships with the torch wheel (nvidia/nccl): headers + libnccl.so.2."""
    import importlib.util
    spec = importlib.util.find_spec("nvidia")
    for base in (spec.submodule_search_locations if spec else []):
        d = os.path.join(base, "nccl")
        if os.path.exists(os.path.join(d, "include", "nccl.h")):
            return d
    raise RuntimeError("nccl.h not found (expected site-packages/nvidia/nccl)")


NCCL = _nccl_dir()


def _cublas_dir():
    """cuBLAS as torch loads it (nvidia/cublas): the F4 training stage's plain GEMMs."""
    import importlib.util
    spec = importlib.util.find_spec("nvidia")
    for base in (spec.submodule_search_locations if spec else []):
        d = os.path.join(base, "cublas")
        if os.path.exists(os.path.join(d, "lib", "libcublas.so.12")):
            return d
    raise RuntimeError("libcublas.so.12 not found (expected site-packages/nvidia/cublas)")


CUBLAS = _cublas_dir()
FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-rdc=true", "-O3", "-lineinfo", "-std=c++17",
         "-Xcompiler", "-fPIC,-fvisibility=hidden", "--expt-relaxed-constexpr",
         "-I", os.path.join(ROOT, "include"), "-I", CSRC, "-I", os.path.join(NCCL, "include"),
         "-I", os.path.join(_cublas_dir(), "include")]


def _stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = [os.path.join(CSRC, f) for f in os.listdir(CSRC)] + [os.path.join(ROOT, "include", "mspipe.h")]
    return any(os.path.getmtime(f) > t for f in deps)


def build(force: bool = False, verbose: bool = False, extra_flags=(), out: str | None = None) -> str:
    lib = out or LIB
    if not force and not extra_flags and out is None and not _stale():
        return LIB
    objdir = os.path.join(HERE, "build") if out is None else out + ".objs"
    os.makedirs(objdir, exist_ok=True)
    objs = []
    procs = []
    for src in SOURCES:
        obj = os.path.join(objdir, src.replace(".cu", ".o"))
        cmd = [NVCC, *FLAGS, *extra_flags, "-c", os.path.join(CSRC, src), "-o", obj]
        if verbose:
            cmd += ["-Xptxas", "-v"]
        procs.append((cmd, subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.STDOUT)))
        objs.append(obj)
    for cmd, p in procs:
        out, _ = p.communicate()
        if p.returncode != 0 or verbose:
            sys.stderr.write(out.decode())
        if p.returncode != 0:
            raise RuntimeError("nvcc failed: " + " ".join(cmd))
    tmp = lib + f".{os.getpid()}.tmp"
    subprocess.check_call([NVCC, "-gencode", "arch=compute_100a,code=sm_100a", "-rdc=true", "-shared", "-o", tmp, *objs,
                           "-Xcompiler", "-fPIC", "-L", os.path.join(NCCL, "lib"), "-l:libnccl.so.2",
                           "-Xlinker", "-rpath=" + os.path.join(NCCL, "lib"),
                           "-L", os.path.join(CUBLAS, "lib"), "-l:libcublas.so.12",
                           "-Xlinker", "-rpath=" + os.path.join(CUBLAS, "lib")])
    os.replace(tmp, lib)
    return lib


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
