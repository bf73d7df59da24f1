"""Build libmempool.so in-tree (sm_100a only).

    python paper_2406_17565_b200/build.py [--force] [-v]

nvcc cross-compiles on a CPU-only box; the .so travels to the GPU box with the
repo snapshot.  The library links the CUDA runtime statically, so it does not
depend on torch's copy of libcudart.
"""
import os
import subprocess
import sys
import sysconfig

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
LIBDIR = os.path.join(HERE, "_lib")
LIB = os.path.join(LIBDIR, "libmempool.so")
INCLUDE = os.path.join(os.path.dirname(HERE), "include")

SOURCES = ["pool.cpp", "api_memory_index.cpp", "api_transfer.cpp", "api_swap.cpp",
           "remote.cpp", "gs.cpp", "kernels.cu"]
HEADERS = ["kernels.cuh", "index.hpp", "pool.hpp", "bitmap_updates.hpp"]

NVCC_FLAGS = [
    "-O3", "-std=c++17", "-lineinfo",
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-Xcompiler", "-fPIC,-Wall,-Wno-unused-function",
    "-Xptxas", "-v",
    "-shared", "-lrt",
]


# CPython binding of the per-request calls (csrc/pyfast.c), linked against the
# library above (rpath $ORIGIN: both live in _lib/).
PYEXT_SRC = os.path.join(CSRC, "pyfast.c")
PYEXT = os.path.join(LIBDIR, "_mpfast" + sysconfig.get_config_var("EXT_SUFFIX"))


# The paper's NCCL send/recv transport as a comparison arm (csrc/nccl_arm.cpp,
# include/mempool_nccl.h), in its own library: libmempool.so stays NCCL-free.
# Linked against the NCCL that torch loads (same soname, one copy per process).
NCCL_SRC = os.path.join(CSRC, "nccl_arm.cpp")
NCCL_LIB = os.path.join(LIBDIR, "libmempool_nccl.so")


def _nccl_dirs():
    import importlib.util
    spec = importlib.util.find_spec("nvidia")
    for base in (list(spec.submodule_search_locations) if spec else []):
        inc, lib = os.path.join(base, "nccl", "include"), os.path.join(base, "nccl", "lib")
        if os.path.exists(os.path.join(inc, "nccl.h")) and os.path.isdir(lib):
            return inc, lib
    return "/usr/include", "/usr/lib/x86_64-linux-gnu"


def build_nccl_arm(verbose: bool = False) -> str:
    inc, lib = _nccl_dirs()
    cuda = os.environ.get("CUDA_HOME", "/usr/local/cuda")
    tmp = NCCL_LIB + ".tmp"
    cmd = ["g++", "-O2", "-std=c++17", "-shared", "-fPIC", "-Wall", "-I", inc,
           "-I", os.path.join(cuda, "include"), "-I", INCLUDE, NCCL_SRC, "-o", tmp,
           "-L", lib, "-l:libnccl.so.2", "-Wl,-rpath," + lib,
           "-L", os.path.join(cuda, "lib64"), "-lcudart"]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if verbose or res.returncode != 0:
        sys.stderr.write(res.stdout + res.stderr)
    if res.returncode != 0:
        raise RuntimeError("g++ failed building libmempool_nccl.so")
    os.replace(tmp, NCCL_LIB)
    return NCCL_LIB


def _build_nccl_arm_soft(verbose: bool = False):
    """The comparison arm must not fail the product's build."""
    try:
        build_nccl_arm(verbose)
    except Exception as e:  # reported, not fatal
        sys.stderr.write(f"warning: libmempool_nccl.so (NCCL comparison arm) not built: {e}\n")


def nccl_stale() -> bool:
    if not os.path.exists(NCCL_LIB):
        return True
    t = os.path.getmtime(NCCL_LIB)
    return any(os.path.getmtime(d) > t for d in (NCCL_SRC, os.path.join(INCLUDE, "mempool_nccl.h")))


def _nvcc():
    cand = os.path.join(os.environ.get("CUDA_HOME", "/usr/local/cuda"), "bin", "nvcc")
    return cand if os.path.exists(cand) else "nvcc"


def stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = [os.path.join(CSRC, s) for s in SOURCES + HEADERS]
    deps.append(os.path.join(INCLUDE, "mempool.h"))
    return any(os.path.getmtime(d) > t for d in deps)


def pyext_stale() -> bool:
    if not os.path.exists(PYEXT):
        return True
    t = os.path.getmtime(PYEXT)
    return any(os.path.getmtime(d) > t for d in (PYEXT_SRC, LIB, os.path.join(INCLUDE, "mempool.h")))


def build_pyext(verbose: bool = False) -> str:
    import numpy
    tmp = PYEXT + ".tmp"
    cmd = ["gcc", "-O2", "-shared", "-fPIC", "-Wall", "-Wno-missing-field-initializers",
           "-I", sysconfig.get_paths()["include"], "-I", numpy.get_include(), "-I", INCLUDE,
           PYEXT_SRC, "-o", tmp, "-L", LIBDIR, "-lmempool", "-Wl,-rpath,$ORIGIN"]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if verbose or res.returncode != 0:
        sys.stderr.write(res.stdout + res.stderr)
    if res.returncode != 0:
        raise RuntimeError("gcc failed building the _mpfast binding")
    os.replace(tmp, PYEXT)
    return PYEXT


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and not stale():
        if pyext_stale():
            build_pyext(verbose)
        if nccl_stale():
            _build_nccl_arm_soft(verbose)
        return LIB
    os.makedirs(LIBDIR, exist_ok=True)
    tmp = LIB + ".tmp"
    cmd = [_nvcc(), *NVCC_FLAGS, "-I", INCLUDE,
           *[os.path.join(CSRC, s) for s in SOURCES], "-o", tmp]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if verbose or res.returncode != 0:
        sys.stderr.write(res.stdout + res.stderr)
    if res.returncode != 0:
        raise RuntimeError("nvcc failed building libmempool.so")
    os.replace(tmp, LIB)
    with open(os.path.join(LIBDIR, "ptxas.log"), "w") as f:
        f.write(res.stderr)
    build_pyext(verbose)
    _build_nccl_arm_soft(verbose)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
