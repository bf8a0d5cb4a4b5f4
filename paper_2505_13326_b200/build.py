"""Build libsart.so (all CUDA kernels + the C-ABI) in-tree for sm_100a with nvcc."""
from __future__ import annotations

import glob
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


def up_to_date() -> bool:
    if not os.path.exists(LIB):
        return False
    if not os.path.exists(STAMP) or open(STAMP).read() != " ".join(FLAGS):
        return False
    t = os.path.getmtime(LIB)
    deps = sources() + glob.glob(os.path.join(CSRC, "*.cuh")) + glob.glob(os.path.join(CSRC, "*.h")) + \
        [os.path.join(HERE, "..", "include", "sart.h")]
    return all(os.path.getmtime(d) <= t for d in deps)


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
    with open(STAMP, "w") as f:
        f.write(" ".join(FLAGS))
    return LIB


if __name__ == "__main__":
    print(build(force="-f" in sys.argv))
