"""Build the in-tree C-ABI library ``libhexgen.so`` for sm_100a with nvcc.

    python -m paper_2311_11514_b200.build [--force]

Every ``csrc/*.cu`` is compiled with ``-gencode arch=compute_100a,code=sm_100a
-lineinfo -O3`` and linked into ``paper_2311_11514_b200/libhexgen.so`` (static
cudart; the driver entry point for TMA descriptors is resolved at run time).
The library lands next to this file so it travels to the GPU box with the
repo snapshot.
"""

from __future__ import annotations

import os
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
CSRC = PKG / "csrc"
INCLUDE = PKG.parent / "include"
LIB = PKG / "libhexgen.so"
BUILD = PKG.parent / "build" / "hexgen"

NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-Xptxas", "-v",
         f"-I{INCLUDE}"]


def sources() -> list[Path]:
    return sorted(CSRC.glob("*.cu"))


def _stale(target: Path, deps) -> bool:
    if not target.exists():
        return True
    t = target.stat().st_mtime
    return any(d.stat().st_mtime > t for d in deps)


def build(force: bool = False, verbose: bool = False) -> Path:
    deps = sources() + sorted(CSRC.glob("*.cuh")) + sorted(INCLUDE.glob("*.h"))
    BUILD.mkdir(parents=True, exist_ok=True)
    objs = []
    for src in sources():
        obj = BUILD / (src.stem + ".o")
        objs.append(obj)
        if force or _stale(obj, [src] + sorted(CSRC.glob("*.cuh")) + sorted(INCLUDE.glob("*.h"))):
            cmd = [NVCC, *ARCH, *FLAGS, "-c", str(src), "-o", str(obj)]
            res = subprocess.run(cmd, capture_output=True, text=True)
            if res.returncode != 0:
                sys.stderr.write(res.stdout + res.stderr)
                raise RuntimeError(f"nvcc failed on {src.name}")
            (BUILD / (src.stem + ".ptxas.txt")).write_text(res.stderr)
            if verbose:
                print(f"compiled {src.name}")
    if force or _stale(LIB, objs + deps):
        cmd = [NVCC, *ARCH, "-shared", "-o", str(LIB), *map(str, objs), "-cudart", "static"]
        res = subprocess.run(cmd, capture_output=True, text=True)
        if res.returncode != 0:
            sys.stderr.write(res.stdout + res.stderr)
            raise RuntimeError("nvcc link failed")
        if verbose:
            print(f"linked {LIB}")
    return LIB


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose=True)
