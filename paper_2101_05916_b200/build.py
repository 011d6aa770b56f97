"""In-tree build of libhjb.so (the product) with nvcc for sm_100a.

The library is a plain shared object (static cudart, no torch dependency);
Python reaches it through ctypes (abi.py), C/C++ callers link it directly.
"""
from __future__ import annotations

import os
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
CSRC = PKG / "csrc"
OUT = PKG / "libhjb.so"

SOURCES = ["hjb_capi.cu", "hjb_kernels.cu", "hjb_fast4d.cu", "hjb_shard.cu", "hjb_ho.cu",
           "hjb_filter.cu", "hjb_gp.cu"]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = [
    "-O3", "-lineinfo", "-std=c++17",
    # bitwise parity with the reference: no a*b+c contraction, IEEE div/sqrt
    "-fmad=false", "-prec-div=true", "-prec-sqrt=true",
    "-Xcompiler", "-fPIC,-O3,-ffp-contract=off,-fno-fast-math",
    "-Xptxas", "-v", "--threads", "0",
]


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if cand and (Path(cand).exists() or cand == "nvcc"):
            return cand
    return "nvcc"


def needs_build() -> bool:
    if not OUT.exists():
        return True
    mtime = OUT.stat().st_mtime
    deps = list(CSRC.glob("*.cu")) + list(CSRC.glob("*.cuh")) + [PKG.parent / "include" / "hjb.h"]
    return any(p.stat().st_mtime > mtime for p in deps)


def build(force: bool = False, verbose: bool = False, out: Path = OUT,
          defines: tuple = ()) -> Path:
    """Compile the library.  ``out``/``defines`` build an experiment variant
    (e.g. _variants/libhjb_x.so with -DFOO=1) that abi.py loads when HJB_LIB
    names it; the product is OUT with no extra defines."""
    if out == OUT and not defines and not force and not needs_build():
        return OUT
    out.parent.mkdir(parents=True, exist_ok=True)
    cmd = [nvcc(), *ARCH, *NVCC_FLAGS, *[f"-D{d}" for d in defines], "-shared", "-o", str(out),
           *[str(CSRC / s) for s in SOURCES], "-lcudart_static", "-ldl", "-lrt", "-lpthread"]
    proc = subprocess.run(cmd, cwd=CSRC, capture_output=True, text=True)
    log = proc.stdout + proc.stderr
    (PKG / ("build.log" if out == OUT else f"build_{out.stem}.log")).write_text(
        " ".join(cmd) + "\n" + log)
    if proc.returncode != 0:
        sys.stderr.write(log)
        raise RuntimeError(f"nvcc failed ({proc.returncode}); see {PKG / 'build.log'}")
    if verbose:
        sys.stderr.write(log)
    return out


if __name__ == "__main__":
    # python build.py [--force] [--variant NAME -DX=1 ...]
    args = sys.argv[1:]
    if "--variant" in args:
        name = args[args.index("--variant") + 1]
        defs = tuple(a[2:] for a in args if a.startswith("-D"))
        print(build(out=PKG / "_variants" / f"libhjb_{name}.so", defines=defs))
    else:
        build(force="--force" in args, verbose=True)
