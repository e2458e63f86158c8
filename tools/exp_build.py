"""Experiment builds: libsunfold with extra nvcc flags on sunfold.cu (e.g. -DSUN_PB_WIDE=1), written to
paper_1812_11626_b200/exp/libsunfold_<name>.so for A/B runs through SUNFOLD_LIB (diagnostics only).
usage: python tools/exp_build.py NAME [--rev GITREV] [FLAG ...]   (--rev: sunfold.cu and its headers as of GITREV)"""
import os
import subprocess
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1812_11626_b200 import _build as B  # noqa: E402


def main():
    name, flags = sys.argv[1], sys.argv[2:]
    rev = None
    if flags[:1] == ["--rev"]:
        rev, flags = flags[1], flags[2:]
    B.build()
    exp = os.path.join(B.HERE, "exp")
    os.makedirs(exp, exist_ok=True)
    obj = os.path.join(exp, f"sunfold_{name}.o")
    src = B.SOURCES[0]
    if rev:  # a copy of the source tree's csrc/ and include/ at that revision
        tmp = os.path.join(exp, f"src_{name}")
        for d in ("paper_1812_11626_b200/csrc", "include"):
            os.makedirs(os.path.join(tmp, d), exist_ok=True)
            for f in subprocess.check_output(["git", "ls-tree", "--name-only", rev, d + "/"], cwd=B.ROOT, text=True).split():
                with open(os.path.join(tmp, f), "w") as fh:
                    fh.write(subprocess.check_output(["git", "show", f"{rev}:{f}"], cwd=B.ROOT, text=True))
        src = os.path.join(tmp, "paper_1812_11626_b200/csrc/sunfold.cu")
        flags = ["-I", os.path.join(tmp, "include")] + flags
    subprocess.check_call([B.nvcc(), *B.NVCC_FLAGS, *flags, "-c", "-o", obj, src])
    lib = os.path.join(exp, f"libsunfold_{name}.so")
    objs = [obj] + [B._obj(s) for s in B.SOURCES[1:]]
    subprocess.check_call([B.nvcc(), "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-Xcompiler", "-fPIC",
                           "-o", lib, *objs])
    print(lib)


if __name__ == "__main__":
    main()
