"""Build the in-tree CUDA library ``libdawn.so`` for sm_100a.

The library is compiled with nvcc straight into the package directory so the
built ``.so`` travels with the repository snapshot to the GPU box (a JIT cache
under ~/.cache would not).  ``python -m paper_2306_07872_b200.build`` or
``__graft_entry__.build()`` runs it; it is a no-op when the ``.so`` is newer
than every source.
"""

from __future__ import annotations

import os
import shutil
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
CSRC = PKG / "csrc"
INCLUDE = PKG.parent / "include"
LIB = PKG / "libdawn.so"

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-Xcompiler", "-fPIC",
]
CXX_FLAGS = ["-O2", "-std=c++17", "-fPIC", "-Wall"]
OBJ = PKG / "_build"  # per-unit objects, so a host-only edit does not recompile the kernels


def _nvcc() -> str:
    cand = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"
    if not os.path.exists(cand):
        raise RuntimeError("nvcc not found; cannot build libdawn.so")
    return cand


def _sources() -> list[Path]:
    return (sorted(CSRC.glob("*.cu")) + sorted(CSRC.glob("*.cpp")) + sorted(CSRC.glob("*.cuh"))
            + sorted(INCLUDE.glob("*.h")))


def needs_build() -> bool:
    if not LIB.exists():
        return True
    t = LIB.stat().st_mtime
    return any(p.stat().st_mtime > t for p in _sources())


def _units() -> list[tuple[Path, list[Path]]]:
    """(translation unit, files whose change makes it stale): the CUDA unit
    depends on every header; a host .cpp on itself and include/."""
    headers = sorted(CSRC.glob("*.cuh")) + sorted(INCLUDE.glob("*.h"))
    units = [(CSRC / "dawn.cu", [CSRC / "dawn.cu", *headers])]
    units += [(p, [p, *sorted(INCLUDE.glob("*.h"))]) for p in sorted(CSRC.glob("*.cpp"))]
    return units


def build(force: bool = False, verbose: bool = False) -> Path:
    if not force and not needs_build():
        return LIB
    OBJ.mkdir(exist_ok=True)
    objs = []
    for src, deps in _units():
        obj = OBJ / (src.name + ".o")
        objs.append(obj)
        if not force and obj.exists() and all(d.stat().st_mtime <= obj.stat().st_mtime for d in deps):
            continue
        if src.suffix == ".cu":
            cmd = [_nvcc(), *NVCC_FLAGS, "-c", "-o", str(obj), str(src)]
            if verbose:
                cmd.insert(1, "-Xptxas=-v")
        else:
            cmd = [shutil.which("g++") or "g++", *CXX_FLAGS, "-c", "-o", str(obj), str(src)]
        if verbose:
            print(" ".join(cmd), file=sys.stderr)
        subprocess.run(cmd, check=True)
    tmp = LIB.with_suffix(".so.tmp")
    subprocess.run([_nvcc(), "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-o", str(tmp),
                    *map(str, objs), "-lcudart"], check=True)
    os.replace(tmp, LIB)
    return LIB


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose="-v" in sys.argv)
    print(LIB)
