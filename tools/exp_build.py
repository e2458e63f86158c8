"""Experiment builds: libsunfold with extra nvcc flags on sunfold.cu (e.g. -DSUN_PB_WIDE=1), written to
paper_1812_11626_b200/exp/libsunfold_<name>.so for A/B runs through SUNFOLD_LIB (diagnostics only).
usage: python tools/exp_build.py NAME [FLAG ...]"""
import os
import subprocess
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1812_11626_b200 import _build as B  # noqa: E402


def main():
    name, flags = sys.argv[1], sys.argv[2:]
    B.build()
    exp = os.path.join(B.HERE, "exp")
    os.makedirs(exp, exist_ok=True)
    obj = os.path.join(exp, f"sunfold_{name}.o")
    src = B.SOURCES[0]
    subprocess.check_call([B.nvcc(), *B.NVCC_FLAGS, *flags, "-c", "-o", obj, src])
    lib = os.path.join(exp, f"libsunfold_{name}.so")
    objs = [obj] + [B._obj(s) for s in B.SOURCES[1:]]
    subprocess.check_call([B.nvcc(), "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-Xcompiler", "-fPIC",
                           "-o", lib, *objs])
    print(lib)


if __name__ == "__main__":
    main()
