"""In-tree build of libksvd.so (sm_100a) with nvcc.

The shared library is built next to this file so it travels with the repo
snapshot to the GPU box.  NCCL comes from the torch-bundled wheel (the same
libnccl.so.2 torch loads), with an rpath so the library also loads without
torch.
"""

from __future__ import annotations

import os
import shutil
import subprocess
import sys
from pathlib import Path

HERE = Path(__file__).resolve().parent
ROOT = HERE.parent
CSRC = HERE / "csrc"
INCLUDE = ROOT / "include"
LIB = HERE / "libksvd.so"
SOURCES = [CSRC / "ksvd.cu", CSRC / "eig.cpp"]
HEADERS = sorted(CSRC.glob("*.cuh")) + [INCLUDE / "ksvd.h", INCLUDE / "ksvd_gen.h"]
ARCH = "-gencode=arch=compute_100a,code=sm_100a"


def _nccl_dirs() -> tuple[Path, Path]:
    try:
        import nvidia.nccl  # type: ignore

        base = Path(list(nvidia.nccl.__path__)[0])
        if (base / "include" / "nccl.h").exists():
            return base / "include", base / "lib"
    except ImportError:
        pass
    return Path("/usr/include"), Path("/usr/lib/x86_64-linux-gnu")


def _nvcc() -> str:
    for cand in (shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and Path(cand).exists():
            return cand
    raise RuntimeError("nvcc not found; the CUDA toolkit is required to build libksvd.so")


def needs_build() -> bool:
    if not LIB.exists():
        return True
    t = LIB.stat().st_mtime
    return any(p.stat().st_mtime > t for p in SOURCES + HEADERS + [Path(__file__)])


def build(force: bool = False, verbose: bool = False) -> Path:
    if not force and not needs_build():
        return LIB
    inc, lib = _nccl_dirs()
    tmp = LIB.with_suffix(".so.tmp")
    cmd = [
        _nvcc(), ARCH, "-O3", "-std=c++17", "-lineinfo", "-shared",
        "-Xcompiler", "-fPIC,-ffp-contract=off,-O3",
        "-Xptxas", "-v" if verbose else "-O3",
        f"-I{INCLUDE}", f"-I{CSRC}", f"-I{inc}",
        *[str(s) for s in SOURCES],
        "-o", str(tmp),
        f"-L{lib}", "-l:libnccl.so.2", "-lpthread", f"-Xlinker=-rpath,{lib}",
    ]
    if verbose:
        print(" ".join(cmd), file=sys.stderr)
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError(f"nvcc failed ({res.returncode}):\n{res.stdout}\n{res.stderr}")
    if verbose:
        print(res.stderr, file=sys.stderr)
    os.replace(tmp, LIB)
    return LIB


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose="-v" in sys.argv)
    print(LIB)
