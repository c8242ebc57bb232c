"""Build libarfx.so in-tree (paper_2212_10550_b200/lib/) with nvcc for sm_100a.

No torch in the build: the library is plain CUDA runtime + host C++ behind the
C-ABI in include/arfx.h. Objects are rebuilt only when a source or header is
newer than the object (headers are global dependencies: any change rebuilds).
"""
from __future__ import annotations

import concurrent.futures as cf
import os
import shutil
import subprocess
import sys
from pathlib import Path

HERE = Path(__file__).resolve().parent
ROOT = HERE.parent
CSRC = HERE / "csrc"
# tuning variants (tools/build_variant.sh) build into their own object dir / library path
OBJ = Path(os.environ.get("ARFX_BUILD_DIR", ROOT / "build" / "obj"))
LIBNAME = Path(os.environ.get("ARFX_LIB_OUT", HERE / "lib" / "libarfx.so"))
LIB = LIBNAME.parent

NVCC = os.environ.get("NVCC", shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
# --fmad=false: no FMA contraction anywhere on the exact path (the kernels also use
# explicit __dadd_rn/__dmul_rn intrinsics); -ffp-contract=off for host C++.
NVCC_FLAGS = ARCH + [
    "-O3", "-lineinfo", "-std=c++17", "--fmad=false", "-Xptxas", "-O3",
    "-Xcompiler", "-fPIC", "-Xcompiler", "-ffp-contract=off", "-Xcompiler", "-O2",
    "-I", str(CSRC), "-I", str(ROOT / "include"),
] + os.environ.get("ARFX_NVCC_EXTRA", "").split()  # tuning experiments (e.g. -DARFX_DS_MIN_BLOCKS=6)
CXX = os.environ.get("CXX", "g++")
CXX_FLAGS = ["-std=c++17", "-O2", "-fPIC", "-ffp-contract=off", "-fno-fast-math", "-Wall",
             "-I", str(CSRC), "-I", str(ROOT / "include"), "-I", "/usr/local/cuda/include"]


def _sources():
    return sorted(CSRC.glob("*.cu")) + sorted(CSRC.glob("*.cpp"))


def _headers():
    return list(CSRC.glob("*.h")) + list(CSRC.glob("*.cuh")) + list((ROOT / "include").glob("*.h"))


def _compile(src: Path, verbose: bool) -> Path:
    obj = OBJ / (src.name + ".o")
    newest_dep = max([src.stat().st_mtime] + [h.stat().st_mtime for h in _headers()])
    if obj.exists() and obj.stat().st_mtime >= newest_dep:
        return obj
    if src.suffix == ".cu":
        cmd = [NVCC] + NVCC_FLAGS + ["-c", str(src), "-o", str(obj)]
    else:
        cmd = [CXX] + CXX_FLAGS + ["-c", str(src), "-o", str(obj)]
    if verbose:
        print(" ".join(cmd), flush=True)
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"compile failed: {src.name}\n{r.stdout}\n{r.stderr}")
    if verbose and r.stderr.strip():
        print(r.stderr, file=sys.stderr)
    return obj


def build(verbose: bool = False, force: bool = False) -> Path:
    OBJ.mkdir(parents=True, exist_ok=True)
    LIB.mkdir(parents=True, exist_ok=True)
    if force:
        for o in OBJ.glob("*.o"):
            o.unlink()
    srcs = _sources()
    with cf.ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 4)) as ex:
        objs = list(ex.map(lambda s: _compile(s, verbose), srcs))
    newest = max(o.stat().st_mtime for o in objs)
    if force or not LIBNAME.exists() or LIBNAME.stat().st_mtime < newest:
        cmd = [NVCC] + ARCH + ["-shared", "-o", str(LIBNAME)] + [str(o) for o in objs] + [
            "-cudart", "static", "-Xlinker", "--no-undefined", "-lpthread", "-ldl", "-lrt"]
        if verbose:
            print(" ".join(cmd), flush=True)
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"link failed\n{r.stdout}\n{r.stderr}")
    return LIBNAME


if __name__ == "__main__":
    print(build(verbose=True, force="--force" in sys.argv))
