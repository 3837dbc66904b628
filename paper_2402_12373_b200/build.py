"""Builds `csrc/libltlcore.so` (the C-ABI CUDA library, sm_100a only) in-tree with nvcc.

`python -m paper_2402_12373_b200.build` or `__graft_entry__.build()`.  One translation unit per row
width W (the hot kernels are fully unrolled over W), compiled in parallel, linked with the static CUDA
runtime so the shared object has no load-time dependency on libcuda / libcudart.
"""
from __future__ import annotations

import hashlib
import os
import shutil
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(CSRC, "libltlcore.so")
OBJ = os.path.join(CSRC, "build")
MAX_W = 16
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC", "-Xcompiler", "-fvisibility=hidden"]
FLAGS += os.environ.get("LTL_NVCC_DEFS", "").split()  # A/B switches, e.g. -DLTL_SEMANTICS_SCAN -DLTL_SHIFT_MADHI


def nvcc() -> str:
    exe = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"
    if not os.path.exists(exe):
        raise RuntimeError("nvcc not found: the CUDA library cannot be built")
    return exe


def _sources_digest() -> str:
    h = hashlib.sha256()
    for name in sorted(os.listdir(CSRC)):
        if name.endswith((".cu", ".cuh")):
            with open(os.path.join(CSRC, name), "rb") as fh:
                h.update(name.encode() + b"\0" + fh.read())
    with open(os.path.join(os.path.dirname(HERE), "include", "ltl_core.h"), "rb") as fh:
        h.update(fh.read())
    h.update(" ".join(ARCH + FLAGS).encode())
    return h.hexdigest()


def _compile(args):
    src, obj, defs = args
    cmd = [nvcc(), *ARCH, *FLAGS, *defs, "-c", src, "-o", obj]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode:
        raise RuntimeError(f"nvcc failed: {' '.join(cmd)}\n{res.stdout}\n{res.stderr}")
    return obj


def build(force: bool = False, verbose: bool = False) -> str:
    digest = _sources_digest()
    stamp = os.path.join(OBJ, "digest.txt")
    if not force and os.path.exists(LIB) and os.path.exists(stamp) and open(stamp).read() == digest:
        return LIB
    os.makedirs(OBJ, exist_ok=True)
    jobs = [(os.path.join(CSRC, "core.cu"), os.path.join(OBJ, "core.o"), []),
            (os.path.join(CSRC, "traces.cu"), os.path.join(OBJ, "traces.o"), [])]
    for w in range(1, MAX_W + 1):
        jobs.append((os.path.join(CSRC, "screen_inst.cu"), os.path.join(OBJ, f"screen_w{w}.o"), [f"-DLTL_W={w}"]))
    jobs.append((os.path.join(CSRC, "screen_inst.cu"), os.path.join(OBJ, "screen_w1p.o"), ["-DLTL_W=1", "-DLTL_PAIR"]))
    with ThreadPoolExecutor(max_workers=min(len(jobs), os.cpu_count() or 4)) as pool:
        objs = list(pool.map(_compile, jobs))
    cmd = [nvcc(), *ARCH, "-shared", "-cudart", "static", "-o", LIB, *objs]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode:
        raise RuntimeError(f"link failed: {' '.join(cmd)}\n{res.stdout}\n{res.stderr}")
    with open(stamp, "w") as fh:
        fh.write(digest)
    if verbose:
        print(f"built {LIB}", file=sys.stderr)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True))
