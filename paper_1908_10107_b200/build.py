"""Build liborca.so (the C-ABI library) in-tree with nvcc for sm_100a."""
from __future__ import annotations

import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIB = os.path.join(PKG, "liborca.so")
TEST_LIB = os.path.join(PKG, "liborca_test.so")  # + -DORCA_TEST_HOOKS (the fake-NCCL tests only)
SOURCES = [os.path.join(CSRC, "orca.cu")]
DEPS = SOURCES + [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".cuh", ".h"))] + \
    [os.path.join(ROOT, "include", "orca.h")]

NVCC_FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
              "-prec-div=false", "-prec-sqrt=false",
              "-Xcompiler", "-fPIC", "-shared", "-Xptxas", "-v", "-ldl"]


def nvcc() -> str:
    for c in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if c and (os.path.isabs(c) and os.path.exists(c) or not os.path.isabs(c)):
            return c
    return "nvcc"


def _flags(test_hooks: bool = False) -> list:
    return NVCC_FLAGS + os.environ.get("ORCA_NVCC_EXTRA", "").split() + (["-DORCA_TEST_HOOKS"] if test_hooks else [])


def stale(test_hooks: bool = False) -> bool:
    lib = TEST_LIB if test_hooks else LIB
    if not os.path.exists(lib):
        return True
    try:
        with open(lib + ".flags") as f:  # the nvcc flags the library was built with
            if f.read() != " ".join(_flags(test_hooks)):
                return True  # built with other flags (e.g. a sweep's ORCA_NVCC_EXTRA -D overrides)
    except OSError:
        return True
    t = os.path.getmtime(lib)
    return any(os.path.getmtime(d) > t for d in DEPS if os.path.exists(d))


def build(force: bool = False, verbose: bool = False, test_hooks: bool = False) -> str:
    """liborca.so (the product), or with test_hooks liborca_test.so: the same sources plus
    -DORCA_TEST_HOOKS (ORCA_NCCL_LIB honoured), loaded only by the multi-process tests."""
    lib = TEST_LIB if test_hooks else LIB
    if not force and not stale(test_hooks):
        return lib
    cmd = [nvcc()] + _flags(test_hooks) + ["-I", os.path.join(ROOT, "include"), "-o", lib] + SOURCES
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError("nvcc failed building liborca.so")
    if verbose:
        sys.stderr.write(r.stderr)
    with open(lib + ".flags", "w") as f:
        f.write(" ".join(_flags(test_hooks)))
    return lib


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True, test_hooks="--test-hooks" in sys.argv))
