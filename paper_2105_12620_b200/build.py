"""Build the in-tree C-ABI library ``libbn.so`` for sm_100a with nvcc (no JIT cache)."""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
SRC = [os.path.join(HERE, "csrc", "bn_api.cu")]
DEPS = SRC + [os.path.join(HERE, "csrc", "bn_kernels.cuh"),
              os.path.join(os.path.dirname(HERE), "include", "bn.h")]
LIB = os.path.join(HERE, "libbn.so")

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17", "--fmad=false",
    "-Xcompiler", "-fPIC,-ffp-contract=off,-fno-fast-math",
    "-Xptxas", "-v",
    "-shared",
]


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if cand and (os.path.sep not in cand or os.path.exists(cand)):
            return cand
    return "nvcc"


def build(force: bool = False, verbose: bool = False, out: str = LIB, defines: tuple[str, ...] = ()) -> str:
    """Compile `out` (default: the in-tree libbn.so).  `defines` (-D...) build experiment variants
    under another name, loaded with BN_LIB=<path>."""
    stale = not os.path.exists(out) or any(os.path.getmtime(d) > os.path.getmtime(out) for d in DEPS)
    if force or stale or defines:
        cmd = [nvcc(), *NVCC_FLAGS, *[f"-D{d}" for d in defines], "-o", out, *SRC, "-ldl"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            sys.stderr.write(r.stdout + r.stderr)
            raise RuntimeError("nvcc failed building libbn.so")
        if verbose:
            sys.stderr.write(r.stderr)
        if out == LIB:
            with open(os.path.join(HERE, "build_ptxas.log"), "w") as f:
                f.write(r.stderr)
    return out


if __name__ == "__main__":
    args = sys.argv[1:]
    out = args[args.index("-o") + 1] if "-o" in args else LIB
    defs = tuple(a[2:] for a in args if a.startswith("-D"))
    print(build(force="--force" in args, verbose=True, out=out, defines=defs))
