"""Build libsunfold.so (the C-ABI of include/sunfold.h) in-tree for sm_100a with nvcc.

Each .cu is compiled to its own object in parallel (the translation units share no device
symbols), then linked into one shared library."""
from __future__ import annotations

import os
import subprocess
from concurrent.futures import ThreadPoolExecutor

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
OBJDIR = os.path.join(HERE, "build")
LIB = os.path.join(HERE, "libsunfold.so")
SOURCES = [os.path.join(CSRC, "sunfold.cu"), os.path.join(CSRC, "sunfold_dense.cu"), os.path.join(CSRC, "sunfold_sc.cu"),
           os.path.join(CSRC, "sunfold_general.cu")]
HEADERS = [os.path.join(CSRC, "sunfold_kernels.cuh"), os.path.join(CSRC, "sunfold_general.cuh"),
           os.path.join(ROOT, "include", "sunfold.h")]
DEPS = SOURCES + HEADERS

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-Xcompiler", "-fPIC",
    "-I", os.path.join(ROOT, "include"),
]


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if cand and (os.path.sep not in cand or os.path.exists(cand)):
            return cand
    return "nvcc"


def _obj(src: str) -> str:
    return os.path.join(OBJDIR, os.path.basename(src)[:-3] + ".o")


def _obj_stale(src: str) -> bool:
    o = _obj(src)
    if not os.path.exists(o):
        return True
    t = os.path.getmtime(o)
    return any(os.path.getmtime(d) > t for d in [src] + HEADERS)


def stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    return any(os.path.getmtime(d) > t for d in DEPS)


def build(force: bool = False, verbose: bool = False, extra_flags: list[str] | None = None) -> str:
    if not force and not stale():
        return LIB
    os.makedirs(OBJDIR, exist_ok=True)
    flags = NVCC_FLAGS + list(extra_flags or [])
    todo = [s for s in SOURCES if force or _obj_stale(s)]

    def compile_one(src: str) -> None:
        o = _obj(src)
        tmp = o + f".tmp{os.getpid()}"
        cmd = [nvcc(), *flags, "-c", "-o", tmp, src]
        if verbose:
            print(" ".join(cmd), flush=True)
        subprocess.check_call(cmd)
        os.replace(tmp, o)

    with ThreadPoolExecutor(max_workers=max(1, len(todo))) as ex:
        for f in [ex.submit(compile_one, s) for s in todo]:
            f.result()
    tmp = LIB + f".tmp{os.getpid()}"
    cmd = [nvcc(), "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-Xcompiler", "-fPIC",
           "-o", tmp, *[_obj(s) for s in SOURCES]]
    if verbose:
        print(" ".join(cmd), flush=True)
    subprocess.check_call(cmd)
    os.replace(tmp, LIB)
    return LIB


if __name__ == "__main__":
    print(build(force=True, verbose=True))
