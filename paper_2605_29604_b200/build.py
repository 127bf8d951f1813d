"""Build the in-tree CUDA libraries for sm_100a.

* ``libtcmis_b200.so`` -- kernels + the C-ABI of ``include/tcmis_b200.h``;
* ``libtcmis.so``      -- the C++ drop-in API of ``include/tcmis/*.hpp``
  (namespace ``tcmis``) layered on the C-ABI.

Built in-tree so the ``.so`` files travel to the GPU box with the snapshot.
``python -m paper_2605_29604_b200.build`` or ``__graft_entry__.build()``.
"""
from __future__ import annotations

import concurrent.futures as cf
import os
import shutil
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
INC = os.path.join(ROOT, "include")
OBJ = os.path.join(PKG, "_obj")
LIB = os.path.join(PKG, "libtcmis_b200.so")
CXXLIB = os.path.join(PKG, "libtcmis.so")

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = ARCH + [
    "-O3", "-lineinfo", "-std=c++17", "--expt-relaxed-constexpr",
    "-Xcompiler", "-fPIC,-fvisibility=hidden,-ffp-contract=off",
    "-I", INC, "-I", CSRC,
] + os.environ.get("TCMIS_NVCC_EXTRA", "").split()
CU_SOURCES = ["capi.cu", "solver.cu", "tiles.cu", "gen.cu", "tiled_spmv.cu", "dist.cu",
              "partitioned.cu", "staging.cu", "order.cu", "tile_cand.cu", "validate.cu"]
CXX_SOURCES = ["engine.cpp"]


def nvcc() -> str:
    for cand in (shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found")


def _stale(out: str, deps: list[str]) -> bool:
    if not os.path.exists(out):
        return True
    t = os.path.getmtime(out)
    return any(os.path.getmtime(d) > t for d in deps if os.path.exists(d))


def _headers() -> list[str]:
    hs = [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".cuh", ".h"))]
    hs.append(os.path.join(INC, "tcmis_b200.h"))
    tdir = os.path.join(INC, "tcmis")
    if os.path.isdir(tdir):
        hs += [os.path.join(tdir, f) for f in os.listdir(tdir)]
    return hs


def _compile(src: str, verbose: bool) -> str:
    out = os.path.join(OBJ, os.path.basename(src) + ".o")
    if not _stale(out, [src] + _headers()):
        return out
    cmd = [nvcc()] + NVCC_FLAGS + ["-c", src, "-o", out]
    if src.endswith(".cpp"):  # host-only C++ (the drop-in API): plain g++
        cmd = ["g++", "-O2", "-std=c++20", "-fPIC", "-ffp-contract=off", "-I", INC, "-c", src,
               "-o", out]
    if verbose:
        print(" ".join(cmd), flush=True)
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"compile failed: {src}\n{r.stdout}\n{r.stderr}")
    if verbose and r.stderr.strip():
        print(r.stderr, file=sys.stderr)
    return out


def build(verbose: bool = False) -> str:
    os.makedirs(OBJ, exist_ok=True)
    srcs = [os.path.join(CSRC, s) for s in CU_SOURCES]
    with cf.ThreadPoolExecutor(max_workers=len(srcs)) as ex:
        objs = list(ex.map(lambda s: _compile(s, verbose), srcs))
    if _stale(LIB, objs):
        cmd = [nvcc()] + ARCH + ["-shared", "-o", LIB] + objs + ["-ldl", "-Xlinker", "-z,defs"]
        if verbose:
            print(" ".join(cmd), flush=True)
        subprocess.run(cmd, check=True)
    cxx = [os.path.join(CSRC, s) for s in CXX_SOURCES if os.path.exists(os.path.join(CSRC, s))]
    if cxx:
        cobjs = [_compile(s, verbose) for s in cxx]
        if _stale(CXXLIB, cobjs + [LIB]):
            cmd = ["g++", "-shared", "-o", CXXLIB] + cobjs + [
                "-L", PKG, "-ltcmis_b200", "-Wl,-rpath,$ORIGIN", "-Wl,-z,defs"]
            if verbose:
                print(" ".join(cmd), flush=True)
            subprocess.run(cmd, check=True)
    return LIB


if __name__ == "__main__":
    print(build(verbose="-v" in sys.argv))
