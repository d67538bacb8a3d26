"""Build libsfv.so in-tree with nvcc for sm_100a (no JIT cache, so the
built library travels with the repository snapshot to the GPU box)."""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libsfv.so")
SOURCES = [os.path.join(CSRC, f) for f in ("sfv_kernels.cu", "sfv_host.cu")]
DEPS = SOURCES + [os.path.join(CSRC, "sfv_internal.h"), os.path.join(ROOT, "include", "sfv.h")]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def nccl_include():
    import importlib.util
    spec = importlib.util.find_spec("nvidia")
    cands = []
    if spec and spec.submodule_search_locations:
        for loc in spec.submodule_search_locations:
            cands.append(os.path.join(loc, "nccl", "include"))
    cands.append("/usr/include")
    for c in cands:
        if os.path.exists(os.path.join(c, "nccl.h")):
            return c
    raise RuntimeError("nccl.h not found (torch's nvidia-nccl wheel expected)")


def up_to_date():
    if not os.path.exists(LIB):
        return False
    t = os.path.getmtime(LIB)
    return all(os.path.getmtime(d) <= t for d in DEPS)


def build(force=False, verbose=False, out=None, defines=(), extra=()):
    if out is None and not force and up_to_date():
        return LIB
    target = out or LIB
    cmd = ["nvcc", *ARCH, *[f"-D{d}" for d in defines], "-O3", "-lineinfo", "-std=c++17", "-Xptxas", "-v",
           "-Xcompiler", "-fPIC", "-shared", "-I", os.path.join(ROOT, "include"),
           "-I", CSRC, "-I", nccl_include(), *extra, *SOURCES, "-o", target + ".tmp", "-ldl"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    with open(os.path.join(HERE, "build.log" if out is None else os.path.basename(target) + ".log"), "w") as f:
        f.write(" ".join(cmd) + "\n" + r.stdout + r.stderr)
    if r.returncode != 0:
        sys.stderr.write(r.stderr)
        raise RuntimeError("nvcc failed building libsfv.so")
    os.replace(target + ".tmp", target)
    if verbose:
        print(r.stderr)
    return target


if __name__ == "__main__":
    if "--variant" in sys.argv:  # A/B experiment builds: --variant NAME DEF=V ... [-- NVCC FLAGS]
        k = sys.argv.index("--variant")
        rest = sys.argv[k + 2:]
        extra = rest[rest.index("--") + 1:] if "--" in rest else []
        defs = rest[:rest.index("--")] if "--" in rest else rest
        print(build(out=os.path.join(HERE, f"libsfv_{sys.argv[k + 1]}.so"), defines=defs, extra=extra))
    else:
        build(force="--force" in sys.argv, verbose=True)
