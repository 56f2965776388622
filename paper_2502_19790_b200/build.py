"""Build libmxb200.so (all CUDA sources, sm_100a) in-tree with nvcc.

`python -m paper_2502_19790_b200.build` or ``__graft_entry__.build()``.
Flags: -gencode arch=compute_100a,code=sm_100a, -O3, -lineinfo (ncu source
page), --fmad=false (the f64 planner/ADO math must not contract a*b+c so it
follows the reference's IEEE operation order), -Xptxas -v into build.log.
"""

from __future__ import annotations

import os
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
CSRC = PKG / "csrc"
LIB = PKG / "libmxb200.so"
SOURCES = ["capi.cu", "stage1.cu", "cursor.cu", "stage2.cu", "stage3.cu", "shard.cu", "serialize.cu", "register.cu", "tokenize.cu"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "--fmad=false", "-std=c++17",
    "-Xcompiler", "-fPIC", "-Xcompiler", "-O2",
    "-Xptxas", "-v",
]


def build(force: bool = False, verbose: bool = False) -> Path:
    srcs = [CSRC / s for s in SOURCES]
    deps = srcs + list(CSRC.glob("*.cuh")) + [PKG.parent / "include" / "mixtera_b200.h"]
    if LIB.exists() and not force and all(d.stat().st_mtime <= LIB.stat().st_mtime for d in deps):
        return LIB
    objs = []
    log = []
    for src in srcs:
        obj = CSRC / (src.stem + ".o")
        cmd = [NVCC, *FLAGS, "-I", str(PKG.parent / "include"), "-dc", str(src), "-o", str(obj)]
        r = subprocess.run(cmd, capture_output=True, text=True)
        log.append(" ".join(cmd) + "\n" + r.stdout + r.stderr)
        if r.returncode != 0:
            sys.stderr.write(r.stdout + r.stderr)
            raise RuntimeError(f"nvcc failed on {src.name}")
        objs.append(str(obj))
    tmp = LIB.with_suffix(".so.tmp")
    cmd = [NVCC, "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-Xcompiler", "-fPIC",
           *objs, "-o", str(tmp), "-lcudart"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    log.append(" ".join(cmd) + "\n" + r.stdout + r.stderr)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError("nvcc link failed")
    os.replace(tmp, LIB)
    (CSRC / "build.log").write_text("\n".join(log))
    for o in objs:
        os.remove(o)
    if verbose:
        print("\n".join(log))
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
