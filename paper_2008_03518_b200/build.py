"""Build libfmdp.so in-tree for sm_100a (nvcc cross-compiles without a GPU)."""
from __future__ import annotations

import os
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
SRCS = [os.path.join(HERE, "csrc", f) for f in ("fmdp_host.cu", "fmdp_walk.cu")]
DEPS = SRCS + [os.path.join(HERE, "csrc", "fmdp_dev.h"), os.path.join(ROOT, "include", "fmdp.h")]
LIB = os.path.join(HERE, "libfmdp.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
FLAGS = ["-std=c++17", "-O3", "-gencode", "arch=compute_100a,code=sm_100a", "-lineinfo",
         "-Xcompiler", "-fPIC", "-shared", "-I" + os.path.join(ROOT, "include")]


def build(force: bool = False, verbose: bool = False, out: str = LIB, defines=()) -> str:
    """Compile libfmdp.so; `out` / `defines` (-D flags) build A/B variants of the same sources."""
    if not force and os.path.exists(out) and os.path.getmtime(out) >= max(os.path.getmtime(p) for p in DEPS):
        return out
    cmd = [NVCC, *FLAGS, *(["-Xptxas", "-v"] if verbose else []), *[f"-D{d}" for d in defines], "-o", out + ".tmp",
           *SRCS]
    subprocess.run(cmd, check=True)
    os.replace(out + ".tmp", out)
    return out


if __name__ == "__main__":
    print(build(force=True, verbose=True))
