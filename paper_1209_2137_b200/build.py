"""Build libintzip_b200.so in-tree with nvcc for sm_100a (no JIT cache).

    python -m paper_1209_2137_b200.build [--force]

The library holds the fused decode kernels, the GPU encoder and the C ABI of
include/intzip_b200.h — nothing else (the bench/test input generators and
host encoder live in harness/, a separate library).
cudart is linked statically so the .so is self-contained on the GPU box.
"""
from __future__ import annotations

import concurrent.futures
import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIBDIR = os.path.join(PKG, "_lib")
LIB = os.path.join(LIBDIR, "libintzip_b200.so")
OBJDIR = os.path.join(LIBDIR, "obj")

SOURCES = ["decode.cu", "decode_scalar.cu", "decode_probe.cu", "decode_split.cu",
           "decode_group.cu", "decode_cta.cu", "decode_team.cu", "decode_relay.cu", "intersect.cu", "host.cpp", "container.cpp"]
# per-source extra flags (none: decode_scalar.cu is built at -O3 again since
# round 2, see the comment at its top); IZG_SCALAR_O1=1 restores the old
# -Xptxas -O1 build of it for comparisons
SOURCE_FLAGS = {"decode_scalar.cu": ["-Xptxas", "-O1"]} if os.environ.get("IZG_SCALAR_O1") == "1" else {}
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-O3",
         "-Xptxas", "-v"]


def _deps():
    files = [os.path.join(CSRC, f) for f in os.listdir(CSRC)]
    files.append(os.path.join(ROOT, "include", "intzip_b200.h"))
    files.append(os.path.abspath(__file__))
    return files


def _stale(target, deps):
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = False) -> str:
    os.makedirs(LIBDIR, exist_ok=True)
    if not force and not _stale(LIB, _deps()):
        return LIB
    objdir = OBJDIR
    os.makedirs(objdir, exist_ok=True)
    extra = os.environ.get("IZG_NVCC_EXTRA", "").split()  # debug builds only

    def compile_one(src):
        obj = os.path.join(objdir, src + ".o")
        cmd = [NVCC, *ARCH, *FLAGS, *SOURCE_FLAGS.get(src, []), *extra, "-c",
               os.path.join(CSRC, src), "-o", obj]
        return src, obj, subprocess.run(cmd, capture_output=True, text=True)

    jobs = max(1, min(len(SOURCES), os.cpu_count() or 1))
    with concurrent.futures.ThreadPoolExecutor(jobs) as pool:
        results = list(pool.map(compile_one, SOURCES))
    objs = []
    for src, obj, res in results:
        if res.returncode != 0:
            raise RuntimeError(f"nvcc failed for {src}:\n{res.stderr}")
        if verbose:
            sys.stderr.write(res.stderr)
        objs.append(obj)
    tmp = LIB + ".tmp"
    cmd = [NVCC, *ARCH, "-shared", "-o", tmp, *objs, "-lpthread"]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError(f"link failed:\n{res.stderr}")
    os.replace(tmp, LIB)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
