"""In-tree build of the sm_100a extension: paper_2304_07338_b200/libpfgpu.so.

Plain nvcc (no torch extension machinery): the product is a C-ABI shared
library (include/pf_gpu.h) that any host -- C++, ctypes, cgo -- can load.
Translation units whose results must round exactly like the x86 reference
(binary64 tracking, KNN distances, Eq. 6) are compiled with --fmad=false.
"""
from __future__ import annotations

import concurrent.futures as cf
import os
import subprocess
import sys
from pathlib import Path

HERE = Path(__file__).resolve().parent
CSRC = HERE / "csrc"
BUILD = HERE / "_build"
LIB = HERE / "libpfgpu.so"
INCLUDE = HERE.parent / "include"

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
COMMON = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "--expt-relaxed-constexpr",
          "-Xptxas", "-warn-spills"]
SOURCES = {
    "pf_trace_parity.cu": ["--fmad=false"],
    "pf_trace_fast.cu": [],
    "pf_trace_fast_batch.cu": ["-Xptxas", "-O1"],  # ptxas -O3 miscompiles its DDA walk (see the file)
    "pf_pathtrace_parity.cu": ["--fmad=false"],
    "pf_pathtrace_fast.cu": [],
    "pf_field.cu": [],
    "pf_compose.cu": [],
    "pf_knn.cu": ["--fmad=false"],
    "pf_photon.cu": ["--fmad=false"],
    "pf_train.cu": [],
    "pf_capi.cu": [],
}


def _nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if cand and (Path(cand).exists() or cand == "nvcc"):
            return cand
    raise RuntimeError("nvcc not found")


def _newest_dep() -> float:
    files = list(CSRC.glob("*.cuh")) + list(CSRC.glob("*.h")) + list(INCLUDE.glob("*.h"))
    return max(f.stat().st_mtime for f in files)


def _compile(src: str, extra: list[str], force: bool) -> Path:
    obj = BUILD / (src.replace(".cu", ".o"))
    s = CSRC / src
    if not force and obj.exists() and obj.stat().st_mtime > max(s.stat().st_mtime, _newest_dep()):
        return obj
    cmd = [_nvcc(), *ARCH, *COMMON, *extra, "-I", str(INCLUDE), "-c", str(s), "-o", str(obj)]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed for {src}:\n{r.stdout}\n{r.stderr}")
    return obj


def build(force: bool = False, verbose: bool = False) -> Path:
    BUILD.mkdir(exist_ok=True)
    with cf.ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 2)) as ex:
        objs = list(ex.map(lambda kv: _compile(kv[0], kv[1], force), SOURCES.items()))
    if force or not LIB.exists() or LIB.stat().st_mtime < max(o.stat().st_mtime for o in objs):
        cmd = [_nvcc(), *ARCH, "-shared", "-cudart", "static", "-o", str(LIB), *map(str, objs)]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"link failed:\n{r.stdout}\n{r.stderr}")
    if verbose:
        print(f"built {LIB}")
    return LIB


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose=True)
