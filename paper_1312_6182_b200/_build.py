"""Build libgpspca_b200.so in-tree with nvcc for sm_100a.

    python -m paper_1312_6182_b200._build          # incremental
    python -m paper_1312_6182_b200._build --force

The shared library is the C ABI declared in include/gpspca_b200.h; cudart is
linked statically so the .so is self-contained next to torch's own runtime.
"""

import hashlib
import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIB = os.path.join(PKG, "libgpspca_b200.so")
STAMP = LIB + ".srchash"
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def _sources():
    files = [os.path.join(ROOT, "include", "gpspca_b200.h")]
    for name in sorted(os.listdir(CSRC)):
        if name.endswith((".cu", ".cuh", ".h")):
            files.append(os.path.join(CSRC, name))
    return files


def _digest(extra):
    h = hashlib.sha256(" ".join(extra).encode())
    for f in _sources():
        with open(f, "rb") as fh:
            h.update(fh.read())
    return h.hexdigest()


def nvcc_command(out=LIB, verbose=False):
    cmd = [os.environ.get("NVCC", "nvcc"), *ARCH, "-O3", "-lineinfo", "-std=c++17",
           "-Xcompiler", "-fPIC", "-shared", "-cudart", "static",
           "-o", out, os.path.join(CSRC, "capi.cu")]
    if verbose:
        cmd.insert(1, "-Xptxas=-v")
    extra = os.environ.get("GPSPCA_NVCC_FLAGS", "").split()  # diagnostics builds, e.g. -DGPS_TC_PROFILE
    return cmd[:-1] + extra + cmd[-1:]


def build(force=False, verbose=False):
    cmd = nvcc_command(verbose=verbose)
    digest = _digest(cmd)
    if not force and os.path.exists(LIB) and os.path.exists(STAMP):
        with open(STAMP) as fh:
            if fh.read().strip() == digest:
                return LIB
    subprocess.run(cmd, check=True)
    with open(STAMP, "w") as fh:
        fh.write(digest)
    return LIB


if __name__ == "__main__":
    path = build(force="--force" in sys.argv, verbose="-v" in sys.argv)
    print(path)
