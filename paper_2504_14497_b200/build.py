"""Build libpcmm.so (the C-ABI library) for sm_100a with nvcc, in-tree.

Each translation unit in csrc/ is compiled in parallel (`nvcc -c`), then linked
into paper_2504_14497_b200/libpcmm.so with the static CUDA runtime.  Rebuilds
only when a source or header is newer than the library (or force=True).
"""
from __future__ import annotations

import concurrent.futures as cf
import os
import shutil
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
BUILD = os.path.join(HERE, "_build")
LIB = os.path.join(HERE, "libpcmm.so")
# checked variant (PCMM_CHECKED=1: device-side bounds checks, pcmm.py loads it when PCMM_LIB_VARIANT=checked)
LIB_CHECKED = os.path.join(HERE, "libpcmm_checked.so")
BUILD_CHECKED = os.path.join(HERE, "_build_checked")
INCLUDE = os.path.join(os.path.dirname(HERE), "include")
UNITS = ["hot.cu", "kernels.cu", "affine.cu", "taff.cu", "tgz.cu", "school.cu", "strassen.cu", "wide.cu", "next2.cu", "paillier.cu", "api.cu"]
# per-unit ptxas options (measured: k_affine 256^3 0.289 -> 0.261 ms at -O1; the other units want -O3)
UNIT_FLAGS = {"affine.cu": ["-Xptxas", "-O1"], "school.cu": ["-DPCMM_INLINE_ACCUM=0"]}
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC,-fvisibility=hidden", "-I", INCLUDE]


def _nvcc() -> str:
    for c in (shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if c and os.path.exists(c):
            return c
    raise RuntimeError("nvcc not found: cannot build libpcmm.so")


def _deps():
    out = [os.path.join(INCLUDE, "pcmm.h"), os.path.abspath(__file__)]
    for f in os.listdir(CSRC):
        if f.endswith((".cu", ".cuh", ".h")):
            out.append(os.path.join(CSRC, f))
    return out


def needs_build(checked: bool = False) -> bool:
    lib = LIB_CHECKED if checked else LIB
    if not os.path.exists(lib):
        return True
    t = os.path.getmtime(lib)
    return any(os.path.getmtime(d) > t for d in _deps())


def build(force: bool = False, verbose: bool = False, ptxas_v: bool = False, checked: bool = False) -> str:
    lib = LIB_CHECKED if checked else LIB
    bdir = BUILD_CHECKED if checked else BUILD
    if not force and not needs_build(checked):
        return lib
    nvcc = _nvcc()
    os.makedirs(bdir, exist_ok=True)
    extra = ["-DPCMM_CHECKED=1"] if checked else []

    def compile_unit(u):
        obj = os.path.join(bdir, u.replace(".cu", ".o"))
        cmd = [nvcc, *ARCH, *FLAGS, *UNIT_FLAGS.get(u, []), *extra,
               *os.environ.get("PCMM_EXTRA_NVCC_FLAGS", "").split(), "-c", os.path.join(CSRC, u), "-o", obj]
        if ptxas_v:
            cmd += ["-Xptxas", "-v"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"nvcc failed for {u}:\n{r.stdout}\n{r.stderr}")
        return obj, r.stderr

    with cf.ThreadPoolExecutor(max_workers=len(UNITS)) as ex:
        results = list(ex.map(compile_unit, UNITS))
    if verbose:
        for _, err in results:
            sys.stderr.write(err)
    tmp = lib + f".tmp{os.getpid()}"
    cmd = [nvcc, *ARCH, "-shared", "-cudart", "static", "-o", tmp] + [o for o, _ in results]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"link failed:\n{r.stdout}\n{r.stderr}")
    os.replace(tmp, lib)
    return lib


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True, ptxas_v="-v" in sys.argv, checked="--checked" in sys.argv))
