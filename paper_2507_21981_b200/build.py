"""In-tree build of libgsim_gpu.so (sm_100a only) with nvcc.

The shared library holds the CUDA kernels, the host orchestration and the C ABI declared in
include/gsim_gpu.h. It is built next to this file so it travels with the repository snapshot.
preprocess.cu is compiled with -fmad=false: its double-precision geometry must not contract
multiply-adds, to stay bit-identical with the reference (see csrc/common.cuh).
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
BUILD = ROOT / "build" / "gsim_gpu"
LIB = HERE / "libgsim_gpu.so"

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
COMMON = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-Xcompiler", "-O3",
          "--expt-relaxed-constexpr", f"-I{ROOT / 'include'}"]
SOURCES = {
    "preprocess.cu": ["-fmad=false"],
    "sort.cu": [],
    "bin.cu": [],
    "raster.cu": [],
    "encode.cu": [],
    "tracks.cu": ["-fmad=false"],
    "ply.cu": ["-fmad=false"],
    "transfer.cu": ["-fmad=false"],
    "lidar.cu": ["-fmad=false"],
    "bvh.cu": ["-fmad=false"],
    "host.cu": [],
}
DEPS = ["common.cuh", "kernels.hpp", "encode.cuh"]


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and Path(cand).exists():
            return cand
    raise RuntimeError("nvcc not found: the CUDA toolkit is required to build libgsim_gpu.so")


def _stale(target: Path, inputs: list[Path]) -> bool:
    if not target.exists():
        return True
    t = target.stat().st_mtime
    return any(p.stat().st_mtime > t for p in inputs)


def build(verbose: bool = False, ptxas_info: bool = False, force: bool = False,
          debug: bool = False) -> Path:
    """libgsim_gpu.so, or with debug=True libgsim_gpu_debug.so: the same sources with the
    GSIM_DCHECK bounds checks compiled in (common.cuh; select it with GSIM_GPU_LIB)."""
    build_dir = BUILD.with_name(BUILD.name + "_debug") if debug else BUILD
    lib = LIB.with_name("libgsim_gpu_debug.so") if debug else LIB
    flags = ["-DGSIM_DEBUG_CHECKS"] if debug else []
    build_dir.mkdir(parents=True, exist_ok=True)
    cc = nvcc()
    header_deps = [CSRC / d for d in DEPS] + [ROOT / "include" / "gsim_gpu.h", Path(__file__)]
    objs = []
    for src, extra in SOURCES.items():
        obj = build_dir / (src + ".o")
        objs.append(obj)
        if not force and not ptxas_info and not _stale(obj, [CSRC / src] + header_deps):
            continue
        cmd = [cc, *ARCH, *COMMON, *flags, *extra, "-c", str(CSRC / src), "-o", str(obj)]
        if ptxas_info:
            cmd += ["-Xptxas", "-v"]
        if verbose:
            print(" ".join(cmd), flush=True)
        res = subprocess.run(cmd, capture_output=True, text=True)
        if res.returncode != 0:
            raise RuntimeError(f"nvcc failed on {src}:\n{res.stdout}\n{res.stderr}")
        if ptxas_info or verbose:
            sys.stdout.write(res.stderr)
    if force or _stale(lib, objs):
        tmp = lib.with_suffix(".so.tmp")
        # static CUDA runtime: the library needs only the driver, whoever loads it
        cmd = [cc, *ARCH, "-shared", "-cudart", "static", "-o", str(tmp), *map(str, objs)]
        if verbose:
            print(" ".join(cmd), flush=True)
        res = subprocess.run(cmd, capture_output=True, text=True)
        if res.returncode != 0:
            raise RuntimeError(f"link failed:\n{res.stdout}\n{res.stderr}")
        os.replace(tmp, lib)
    return lib


if __name__ == "__main__":
    build(verbose=True, ptxas_info="--ptxas" in sys.argv, force="--force" in sys.argv,
          debug="--debug" in sys.argv)
