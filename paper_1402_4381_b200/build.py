"""Build the sm_100a shared library in-tree (nvcc, no JIT cache).

``python -m paper_1402_4381_b200.build`` or ``__graft_entry__.build()``.
"""
from __future__ import annotations

import glob
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
LIB = os.path.join(HERE, "libct_oslalm.so")
SOURCES = sorted(glob.glob(os.path.join(HERE, "csrc", "*.cu")) + glob.glob(os.path.join(HERE, "csrc", "*.cuh"))
                 + [os.path.join(ROOT, "include", "ct_oslalm.h")])
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17", "-ftz=true",
         "-Xcompiler", "-fPIC", "-shared", "-Xptxas", "-v"]


def source_hash(extra=()) -> str:
    """sha256 (16 hex digits) of every source the library is built from and the nvcc flags;
    compiled into ct_build_info() as "src=<hash>" and checked by ctlib.load()."""
    import hashlib
    h = hashlib.sha256()
    for s in SOURCES:
        h.update(os.path.basename(s).encode())
        with open(s, "rb") as f:
            h.update(f.read())
    h.update(" ".join(FLAGS + list(extra)).encode())
    return h.hexdigest()[:16]


def needs_build() -> bool:
    if not os.path.exists(LIB) or not os.path.exists(LIB + ".srchash"):
        return True
    with open(LIB + ".srchash") as f:
        return f.read().strip() != source_hash()


def build(force: bool = False, verbose: bool = False, out: str = None, extra=()) -> str:
    """Build libct_oslalm.so (or a tuning variant at `out` with extra nvcc flags, e.g. -D...)."""
    lib = out or LIB
    if out is None and not force and not needs_build():
        return LIB
    tmp = lib + f".tmp{os.getpid()}"
    sh = source_hash(extra)
    cmd = [NVCC, *FLAGS, *extra, f"-DCT_SRC_HASH=\"{sh}\"", "-o", tmp, os.path.join(HERE, "csrc", "ct_abi.cu"), "-ldl"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError("nvcc failed building libct_oslalm.so")
    if out is None:
        with open(os.path.join(HERE, "csrc", "ptxas_info.txt"), "w") as f:
            f.write(r.stderr)
    if verbose:
        sys.stderr.write(r.stderr)
    os.replace(tmp, lib)
    if out is None:
        with open(LIB + ".srchash", "w") as f:
            f.write(sh)
    return lib


if __name__ == "__main__":
    # python -m paper_1402_4381_b200.build [--force] [--out PATH -DNAME=V ...]
    a = sys.argv[1:]
    out = a[a.index("--out") + 1] if "--out" in a else None
    extra = [x for x in a if x.startswith("-D")]
    print(build(force="--force" in a, verbose=out is None, out=out, extra=extra))
