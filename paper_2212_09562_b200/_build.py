"""Build the in-tree CUDA library ``paper_2212_09562_b200/lib/librecsplit_b200.so``.

nvcc for sm_100a only (``-gencode arch=compute_100a,code=sm_100a``), ``-lineinfo`` so
ncu's source page maps to the kernels; host C++ with g++ through nvcc.  The CUDA
runtime is linked statically with its symbols hidden, so the library coexists with
the runtime PyTorch loads.
"""
from __future__ import annotations

import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
OUT_DIR = os.environ.get("RS_BUILD_DIR", os.path.join(HERE, "lib"))
LIB = os.path.join(OUT_DIR, "librecsplit_b200.so")
EXTRA = os.environ.get("RS_NVCC_FLAGS", "").split()  # development experiments only
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")

SOURCES = ["scan.cu", "partition.cu", "search.cu", "encode.cu", "pipeline.cu", "query.cu", "tables.cpp", "format.cpp",
           "abi.cpp"]
HEADERS = ["device.cuh", "kernels.h", "pipeline.h", "tables.h", "format.h", "murmur3.h"]


def _stale(lib: str = LIB) -> bool:
    if not os.path.exists(lib):
        return True
    t = os.path.getmtime(lib)
    deps = [os.path.join(CSRC, f) for f in SOURCES + HEADERS]
    deps.append(os.path.join(HERE, "..", "include", "recsplit.h"))
    deps.append(__file__)
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = False, out_dir: str = OUT_DIR, extra=None) -> str:
    """Compile the library into out_dir (extra: additional nvcc flags; default RS_NVCC_FLAGS)."""
    extra = EXTRA if extra is None else extra
    lib = os.path.join(out_dir, "librecsplit_b200.so")
    if not force and not _stale(lib):
        return lib
    obj_dir = os.path.join(out_dir, "obj")
    os.makedirs(obj_dir, exist_ok=True)
    common = ["-O3", "-std=c++17", "-Xcompiler", "-fPIC", "-Xcompiler", "-fvisibility=hidden"]

    def compile_one(src):
        path = os.path.join(CSRC, src)
        obj = os.path.join(obj_dir, src + ".o")
        cmd = [NVCC, *ARCH, *common, *extra, "-c", path, "-o", obj]
        if src.endswith(".cu"):
            cmd[1:1] = ["-lineinfo", "-Xptxas", "-v" if verbose else "-O3", "--expt-relaxed-constexpr"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            sys.stderr.write(r.stdout + r.stderr)
            raise RuntimeError(f"nvcc failed on {src}")
        if verbose and (r.stdout or r.stderr):
            sys.stderr.write(r.stdout + r.stderr)
        return obj

    # the translation units are independent: compile them concurrently
    with ThreadPoolExecutor(max_workers=min(len(SOURCES), os.cpu_count() or 1)) as ex:
        objs = list(ex.map(compile_one, SOURCES))
    tmp = lib + f".tmp{os.getpid()}"
    cmd = [NVCC, *ARCH, "-shared", "-cudart", "static", "-o", tmp, *objs,
           "-Xlinker", "--exclude-libs,ALL", "-lpthread"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError("link failed")
    os.replace(tmp, lib)
    return lib


def build_count_variant(force: bool = False) -> str:
    """Diagnostic build with -DRS_COUNT_EVALS (every search kernel counts the key evaluations it
    executes): bench.py's executed-evaluation fraction loads it in a subprocess.
    Never the product path (paper_2212_09562_b200 loads lib/ only)."""
    return build(force=force, out_dir=os.path.join(HERE, "..", "build_var", "count"), extra=["-DRS_COUNT_EVALS"])


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
