"""In-tree build of libcapsim_b200.so for sm_100a (nvcc, no JIT cache).

    python -m paper_2306_12247_b200.build [--force] [-v]

The shared library lands in paper_2306_12247_b200/_lib/ so it travels with the repo snapshot
to the GPU box (it is git-ignored, not gpurun-ignored).
"""

from __future__ import annotations

import os
import shutil
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
CSRC = PKG / "csrc"
LIBDIR = PKG / "_lib"
LIB = LIBDIR / "libcapsim_b200.so"
INCLUDE = PKG.parent / "include"

SOURCES = ["staging.cpp", "capi.cpp", "eval.cu", "aux_kernels.cu", "replay.cu", "sampling.cu", "sweep.cu", "ingest.cpp",
           "comm.cpp"]
HEADERS = ["cs_internal.h", "cs_mt.cuh"]

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = [
    "-O3",
    "-std=c++17",
    "-lineinfo",
    "-fmad=false",  # the fp64 epilogue relies on explicit FMAs only (error-free transforms)
    "-Xcompiler", "-fPIC,-ffp-contract=off,-O2",
    "-Xptxas", "-v",
    "--expt-relaxed-constexpr",
    "-cudart=static",
]


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", shutil.which("nvcc")):
        if cand and Path(cand).exists():
            return cand
    raise RuntimeError("nvcc not found: the CUDA toolkit is required to build libcapsim_b200.so")


def stale() -> bool:
    if not LIB.exists():
        return True
    t = LIB.stat().st_mtime
    deps = [CSRC / s for s in SOURCES + HEADERS] + [INCLUDE / "capsim_b200.h"]
    return any(p.stat().st_mtime > t for p in deps)


def build(force: bool = False, verbose: bool = False, out: Path | None = None, defines: tuple = ()) -> Path:
    """Compile the library (``out``/``defines`` build experiment variants next to it)."""
    lib = out or LIB
    if not force and out is None and not stale():
        return LIB
    LIBDIR.mkdir(exist_ok=True)
    from concurrent.futures import ThreadPoolExecutor

    def compile_one(src):  # the sources compile independently: the nvcc processes run in parallel
        obj = LIBDIR / (lib.stem + "." + src + ".o")
        dflags = [f"-D{d}" for d in defines]
        cmd = [nvcc(), *ARCH, *NVCC_FLAGS, *dflags, "-I", str(INCLUDE), "-c", str(CSRC / src), "-o", str(obj)]
        if src.endswith(".cpp"):
            cmd = [nvcc(), "-x", "cu", *ARCH, *NVCC_FLAGS, *dflags, "-I", str(INCLUDE), "-c", str(CSRC / src), "-o",
                   str(obj)]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"nvcc failed on {src}:\n{r.stdout}\n{r.stderr}")
        return str(obj), r.stdout + r.stderr

    with ThreadPoolExecutor(max(1, min(len(SOURCES), os.cpu_count() or 1))) as ex:
        done = list(ex.map(compile_one, SOURCES))
    objs = [o for o, _ in done]
    log = [g for _, g in done]
    tmp = lib.with_suffix(".so.tmp")
    cmd = [nvcc(), *ARCH, "-shared", "-cudart=static", "-o", str(tmp), *objs, "-lpthread", "-ldl"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"link failed:\n{r.stdout}\n{r.stderr}")
    os.replace(tmp, lib)
    for o in objs:  # objects are scratch: keep the GPU snapshot small
        Path(o).unlink(missing_ok=True)
    (LIBDIR / (lib.stem + ".ptxas.log")).write_text("\n".join(log))
    if verbose:
        print("\n".join(log))
    return lib


if __name__ == "__main__":
    p = build(force="--force" in sys.argv, verbose="-v" in sys.argv)
    print(p)
