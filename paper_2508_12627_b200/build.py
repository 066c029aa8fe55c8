"""Builds the native library ``libustats_b200.so`` in-tree.

Host C++ (planning, lattice, C-ABI) is compiled with g++ -std=c++20; the
sm_100a kernels with ``nvcc -gencode arch=compute_100a,code=sm_100a -lineinfo``;
the shared object is linked by nvcc (static cudart). Incremental: an object is
rebuilt when its source or any header under csrc/ is newer.
"""
from __future__ import annotations

import concurrent.futures as cf
import os
import shutil
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
CSRC = PKG / "csrc"
REPO = PKG.parent
OBJ = REPO / "build" / "obj"
LIB = PKG / "libustats_b200.so"

CUDA_HOME = Path(os.environ.get("CUDA_HOME", "/usr/local/cuda"))
NVCC = str(CUDA_HOME / "bin" / "nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
INCLUDES = [f"-I{CSRC / 'include'}", f"-I{CSRC}", f"-I{CSRC / 'device'}", f"-I{REPO / 'include'}"]

CXX_SOURCES = sorted((CSRC / "host").glob("*.cpp")) + sorted((CSRC / "device").glob("*.cpp")) + [CSRC / "capi.cpp"]
CU_SOURCES = sorted((CSRC / "device").glob("*.cu"))


def _headers_mtime() -> float:
    hs = list(CSRC.rglob("*.hpp")) + list(CSRC.rglob("*.cuh")) + list((REPO / "include").glob("*.h"))
    return max((h.stat().st_mtime for h in hs), default=0.0)


def _compile(src: Path, hdr_mtime: float, verbose: bool) -> Path:
    obj = OBJ / (src.relative_to(CSRC).as_posix().replace("/", "__") + ".o")
    if obj.exists() and obj.stat().st_mtime >= max(src.stat().st_mtime, hdr_mtime):
        return obj
    if src.suffix == ".cu":
        cmd = [NVCC, *ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC",
               "--expt-relaxed-constexpr", "-Xcompiler", "-fvisibility=hidden", *INCLUDES, "-c", str(src), "-o", str(obj)]
    else:
        cmd = ["g++", "-std=c++20", "-O2", "-fPIC", "-Wall", "-Wextra", "-Wno-unused-parameter", "-fvisibility=hidden",
               *INCLUDES, f"-I{CUDA_HOME / 'include'}", "-c", str(src), "-o", str(obj)]
    if verbose:
        print(" ".join(cmd), flush=True)
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"compile failed: {src}\n{r.stdout}\n{r.stderr}")
    if verbose and r.stderr.strip():
        print(r.stderr, file=sys.stderr)
    return obj


def build(verbose: bool = False) -> Path:
    if shutil.which(NVCC) is None and not Path(NVCC).exists():
        raise RuntimeError("nvcc not found; the B200 engine has no CPU fallback")
    OBJ.mkdir(parents=True, exist_ok=True)
    hdr = _headers_mtime()
    srcs = CXX_SOURCES + CU_SOURCES
    with cf.ThreadPoolExecutor(max_workers=os.cpu_count() or 4) as ex:
        objs = list(ex.map(lambda s: _compile(s, hdr, verbose), srcs))
    newest = max(o.stat().st_mtime for o in objs)
    if LIB.exists() and LIB.stat().st_mtime >= newest:
        return LIB
    cmd = [NVCC, *ARCH, "-shared", "-o", str(LIB), *map(str, objs), "-lpthread", "-Xlinker", "--no-undefined",
           "-Xlinker", "-Bsymbolic"]
    if verbose:
        print(" ".join(cmd), flush=True)
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"link failed\n{r.stdout}\n{r.stderr}")
    return LIB


if __name__ == "__main__":
    print(build(verbose="-v" in sys.argv))
