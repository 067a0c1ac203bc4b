"""Build liblrcnn.so in-tree: nvcc for sm_100a only (the product targets B200).

    python -m paper_2401_11471_b200.build [--force]
"""
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
OUT = os.path.join(HERE, "liblrcnn.so")
OBJ = os.path.join(HERE, "build")

NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-Xcompiler", "-fvisibility=hidden",
         "--expt-relaxed-constexpr", "-I", os.path.join(ROOT, "include")]
SOURCES = ["plan.cpp", "kernels_simt.cu", "conv_tc.cu", "bneck_tc.cu", "bn.cu", "comm.cu", "engine.cu"]
HEADERS = ["plan.hpp", "kernels.hpp", "tc.hpp", "tc_ptx.cuh", "comm.hpp"]


def _newer(src, dst):
    return not os.path.exists(dst) or os.path.getmtime(src) > os.path.getmtime(dst)


def build(force=False, verbose=False):
    os.makedirs(OBJ, exist_ok=True)
    hdr_mtime = max([os.path.getmtime(os.path.join(CSRC, h)) for h in HEADERS if os.path.exists(os.path.join(CSRC, h))]
                    + [os.path.getmtime(os.path.join(ROOT, "include", "lrcnn.h"))])
    objs = []
    for s in SOURCES:
        src = os.path.join(CSRC, s)
        obj = os.path.join(OBJ, s + ".o")
        objs.append(obj)
        if force or _newer(src, obj) or (os.path.exists(obj) and os.path.getmtime(obj) < hdr_mtime):
            cmd = [NVCC, *ARCH, *FLAGS, "-Xptxas", "-v" if verbose else "-O3", "-c", src, "-o", obj]
            if s.endswith(".cpp"):   # host-only planner
                cmd = ["g++", "-O2", "-std=c++17", "-fPIC", "-fvisibility=hidden", "-Wall",
                       "-I", os.path.join(ROOT, "include"), "-I", "/usr/local/cuda/include", "-c", src, "-o", obj]
            print(" ".join(cmd), flush=True)
            subprocess.check_call(cmd)
    if force or not os.path.exists(OUT) or any(os.path.getmtime(o) > os.path.getmtime(OUT) for o in objs):
        cmd = [NVCC, *ARCH, "-shared", "-o", OUT, *objs, "-cudart", "static", "-ldl"]
        print(" ".join(cmd), flush=True)
        subprocess.check_call(cmd)
    return OUT


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose="-v" in sys.argv)
