"""Build libsart.so (all CUDA kernels + the C-ABI) in-tree for sm_100a with nvcc."""
from __future__ import annotations

import glob
import hashlib
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
LIB = os.environ.get("SART_LIB_OUT", os.path.join(HERE, "libsart.so"))   # SART_LIB_OUT: A/B variants
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
         "--extended-lambda", "-Xcompiler", "-fPIC", "-Xptxas", "-warn-spills",
         "-cudart", "static"] + os.environ.get("SART_NVCC_EXTRA", "").split()


def sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")))


OBJDIR = os.path.join(HERE, "build") if "SART_LIB_OUT" not in os.environ else LIB + ".objs"
STAMP = os.path.join(OBJDIR, "flags.txt")


def fingerprint() -> str:
    """SHA-256 over the nvcc command line and the CONTENT of every source / header (not their
    mtimes: a checkout or a copied tree with uniform mtimes must not reuse a stale library)."""
    h = hashlib.sha256()
    h.update(" ".join([NVCC] + FLAGS).encode())
    deps = sorted(sources() + glob.glob(os.path.join(CSRC, "*.cuh")) + glob.glob(os.path.join(CSRC, "*.h")) +
                  [os.path.join(HERE, "..", "include", "sart.h")])
    for d in deps:
        h.update(os.path.basename(d).encode())
        with open(d, "rb") as f:
            h.update(hashlib.sha256(f.read()).digest())
    return h.hexdigest()


def up_to_date() -> bool:
    """The library exists and was built from exactly these sources and flags, and its own
    bytes are the ones that build wrote (stamp = source fingerprint + library hash)."""
    if not os.path.exists(LIB) or not os.path.exists(STAMP):
        return False
    try:
        fp, lib_hash = open(STAMP).read().split()
    except ValueError:
        return False
    if fp != fingerprint():
        return False
    with open(LIB, "rb") as f:
        return hashlib.sha256(f.read()).hexdigest() == lib_hash


def build(force: bool = False, verbose: bool = True, jobs: int = 8) -> str:
    if not force and up_to_date():
        return LIB
    objdir = OBJDIR
    os.makedirs(objdir, exist_ok=True)
    procs = []
    objs = []
    for src in sources():
        obj = os.path.join(objdir, os.path.basename(src) + ".o")
        objs.append(obj)
        cmd = [NVCC, *FLAGS, "-I", CSRC, "-I", os.path.join(HERE, "..", "include"), "-c", src, "-o", obj]
        procs.append((src, subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.STDOUT)))
        if len([p for _, p in procs if p.poll() is None]) >= jobs:
            procs[0][1].wait()
    failed = False
    for src, p in procs:
        out = p.communicate()[0].decode()
        if p.returncode != 0:
            failed = True
            sys.stderr.write(f"---- {src}\n{out}\n")
        elif verbose and out.strip():
            sys.stderr.write(f"---- {src}\n{out}\n")
    if failed:
        raise RuntimeError("nvcc failed")
    tmp = LIB + ".tmp"
    cmd = [NVCC, "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-cudart", "static", *objs,
           "-o", tmp, "-lcuda"]
    subprocess.check_call(cmd)
    os.replace(tmp, LIB)
    with open(LIB, "rb") as f:
        lib_hash = hashlib.sha256(f.read()).hexdigest()
    with open(STAMP, "w") as f:
        f.write(fingerprint() + " " + lib_hash)
    return LIB


if __name__ == "__main__":
    print(build(force="-f" in sys.argv))
