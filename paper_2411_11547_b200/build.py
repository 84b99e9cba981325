"""Build libphmm.so in-tree for sm_100a (nvcc, no JIT cache): the built library
travels with the repo snapshot to the GPU box.

The library is several translation units (csrc/*.cu: the host engine, the small kernels,
one file per stream-kernel mode) compiled in parallel to objects under _lib/obj and
linked with nvcc -shared.  No relocatable device code: kernels are only launched from
the translation unit that instantiates them (through the tables in phmm_registry.h)."""
from __future__ import annotations

import glob
import os
import subprocess
import sys
import sysconfig
from concurrent.futures import ThreadPoolExecutor

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
SOURCES = sorted(glob.glob(os.path.join(CSRC, "*.cu")))
HEADERS = sorted(glob.glob(os.path.join(CSRC, "*.h")) + glob.glob(os.path.join(CSRC, "*.cuh"))) + [
    os.path.join(ROOT, "include", "phmm.h")]
OUT = os.path.join(HERE, "_lib", "libphmm.so")
HOST_SRC = [os.path.join(CSRC, "datagen.cpp"), os.path.join(CSRC, "batchio.cpp"), os.path.join(CSRC, "gather.cpp")]
HOST_OUT = os.path.join(HERE, "_lib", "libphmm_host.so")   # host-only: input generator, batch text I/O
FLAT_SRC = os.path.join(CSRC, "flatten.cpp")                # CPython extension: Batch list -> flat arrays
FLAT_OUT = os.path.join(HERE, "_lib", "_phmm_flatten" + (sysconfig.get_config_var("EXT_SUFFIX") or ".so"))
OBJ = os.path.join(HERE, "_lib", "obj")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
         "-Xcompiler", "-fPIC", "-Xcompiler", "-pthread", "-Xptxas", "-warn-spills"] + \
    os.environ.get("PHMM_NVCC_EXTRA", "").split()          # experiments: e.g. -DPHMM_UNROLL4


def _obj(src: str) -> str:
    return os.path.join(OBJ, os.path.basename(src)[:-3] + ".o")


def _stale(target: str, deps) -> bool:
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(p) > t for p in deps)


def up_to_date() -> bool:
    return not _stale(OUT, SOURCES + HEADERS)


def build_host(force: bool = False, verbose: bool = False) -> str:
    """g++ -> libphmm_host.so (no CUDA: also used by the CPU tests)."""
    if not force and not _stale(HOST_OUT, HOST_SRC):
        return HOST_OUT
    os.makedirs(os.path.dirname(HOST_OUT), exist_ok=True)
    cmd = ["g++", "-O2", "-std=c++17", "-shared", "-fPIC", "-o", HOST_OUT + ".tmp"] + HOST_SRC
    if verbose:
        print(" ".join(cmd), file=sys.stderr)
    subprocess.run(cmd, check=True)
    os.replace(HOST_OUT + ".tmp", HOST_OUT)
    return HOST_OUT


def build_flatten(force: bool = False, verbose: bool = False) -> str:
    """g++ -> the _phmm_flatten CPython extension (Python.h of this interpreter)."""
    if not force and not _stale(FLAT_OUT, [FLAT_SRC]):
        return FLAT_OUT
    os.makedirs(os.path.dirname(FLAT_OUT), exist_ok=True)
    import numpy
    cmd = ["g++", "-O2", "-std=c++17", "-shared", "-fPIC", "-pthread", "-I", sysconfig.get_paths()["include"],
           "-I", numpy.get_include(), "-o", FLAT_OUT + ".tmp", FLAT_SRC]
    if verbose:
        print(" ".join(cmd), file=sys.stderr)
    subprocess.run(cmd, check=True)
    os.replace(FLAT_OUT + ".tmp", FLAT_OUT)
    return FLAT_OUT


def build_native(force: bool = False, verbose: bool = False) -> str:
    build_host(force, verbose)
    build_flatten(force, verbose)
    if not force and up_to_date():
        return OUT
    os.makedirs(OBJ, exist_ok=True)
    inc = ["-I", os.path.join(ROOT, "include")]

    def compile_one(src):
        obj = _obj(src)
        if not force and not _stale(obj, [src] + HEADERS):
            return obj
        cmd = [NVCC] + FLAGS + inc + ["-c", "-o", obj + ".tmp", src]
        if verbose:
            print(" ".join(cmd), file=sys.stderr)
        subprocess.run(cmd, check=True)
        os.replace(obj + ".tmp", obj)
        return obj

    with ThreadPoolExecutor(max_workers=max(1, min(len(SOURCES), os.cpu_count() or 1))) as ex:
        objs = list(ex.map(compile_one, SOURCES))
    cmd = [NVCC, "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-Xcompiler", "-pthread",
           "-o", OUT + ".tmp"] + objs
    if verbose:
        print(" ".join(cmd), file=sys.stderr)
    subprocess.run(cmd, check=True)
    os.replace(OUT + ".tmp", OUT)
    return OUT


if __name__ == "__main__":
    print(build_native(force="--force" in sys.argv, verbose=True))
