"""In-tree build of the native libraries (explicit nvcc / g++ commands, no JIT cache).

  _lib/libtsdd_cuda.so   the sm_100a kernels + host driver + C ABI (include/tsdd_cuda.h)
  _lib/libtsdd_gen.so    the seeded workload generators (host-only C++)

The built files are git-ignored but travel to the GPU box with the snapshot.
``python -m paper_1901_00155_b200.build`` rebuilds what is out of date.
"""
from __future__ import annotations

import os
import shutil
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "_lib")
OBJ = os.path.join(HERE, "_lib", "obj")
INCLUDE = os.path.join(ROOT, "include")

CUDA_SOURCES = ["prep_kernels.cu", "search_kernels.cu", "tc_kernels.cu", "probe_kernels.cu", "engine.cu"]
CUDA_HEADERS = ["common.cuh", "kernels.hpp", os.path.join(INCLUDE, "tsdd_cuda.h")]
NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a", "-lineinfo", "-O3", "-std=c++17",
    "-Xcompiler", "-fPIC", "-I", INCLUDE, "-I", CSRC,
] + os.environ.get("TSDD_NVCC_EXTRA", "").split()  # e.g. "-DTSDD_SCAN_CHUNK=32 -DTSDD_SCAN_STAGES=4"
HOST_CXX = "/usr/bin/g++"


def _nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", shutil.which("nvcc")):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found")


def _stale(target: str, deps: list[str]) -> bool:
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def _run(cmd: list[str]) -> None:
    proc = subprocess.run(cmd, capture_output=True, text=True)
    if proc.returncode != 0:
        raise RuntimeError("build failed:\n  " + " ".join(cmd) + "\n" + proc.stdout + proc.stderr)


def build_cuda(force: bool = False, verbose: bool = False, debug_bounds: bool = False) -> str:
    """libtsdd_cuda.so; with debug_bounds the checked build libtsdd_cuda_dbg.so (-DTSDD_DEBUG_BOUNDS:
    in-kernel index checks, csrc/common.cuh) that the GPU tests run the randomised edge shapes on."""
    OBJ = os.path.join(LIB, "obj_dbg" if debug_bounds else "obj")
    NVCC_FLAGS = globals()["NVCC_FLAGS"] + (["-DTSDD_DEBUG_BOUNDS"] if debug_bounds else [])
    os.makedirs(OBJ, exist_ok=True)
    target = os.path.join(LIB, "libtsdd_cuda_dbg.so" if debug_bounds else "libtsdd_cuda.so")
    # objects built with other flags (TSDD_NVCC_EXTRA) are stale whatever their age
    stamp = os.path.join(OBJ, "flags.txt")
    flags = " ".join(NVCC_FLAGS)
    if not os.path.exists(stamp) or open(stamp).read() != flags:
        force = True
        with open(stamp, "w") as f:
            f.write(flags)
    headers = [h if os.path.isabs(h) else os.path.join(CSRC, h) for h in CUDA_HEADERS]
    objects, jobs = [], []
    for src in CUDA_SOURCES:
        path = os.path.join(CSRC, src)
        obj = os.path.join(OBJ, src.replace(".cu", ".o"))
        objects.append(obj)
        if force or _stale(obj, [path] + headers):
            if verbose:
                print("nvcc", src, flush=True)
            jobs.append([_nvcc(), *NVCC_FLAGS, "-c", path, "-o", obj])
    if jobs:  # the translation units compile side by side (search_kernels.cu alone takes about a minute)
        from concurrent.futures import ThreadPoolExecutor
        with ThreadPoolExecutor(max_workers=len(jobs)) as pool:
            list(pool.map(_run, jobs))
    if force or _stale(target, objects):
        _run([_nvcc(), "-shared", "-gencode", "arch=compute_100a,code=sm_100a", "-Xcompiler", "-fPIC",
              "-o", target, *objects, "-ldl", "-lpthread"])
    return target


def build_gen(force: bool = False) -> str:
    os.makedirs(LIB, exist_ok=True)
    target = os.path.join(LIB, "libtsdd_gen.so")
    src = os.path.join(CSRC, "series_gen.cpp")
    if force or _stale(target, [src]):
        cxx = HOST_CXX if os.path.exists(HOST_CXX) else "g++"
        _run([cxx, "-std=c++17", "-O2", "-ffp-contract=off", "-fPIC", "-shared", "-o", target, src])
    return target


def build_tools(force: bool = False) -> str:
    """tools/tsdd_cuda (find | bench | generate): the C++ host layer (include/tsdd/cuda_engine.hpp) end to end."""
    target = os.path.join(LIB, "tsdd_cuda")
    src = os.path.join(ROOT, "tools", "tsdd_cuda.cpp")
    deps = [src, os.path.join(INCLUDE, "tsdd", "cuda_engine.hpp"), os.path.join(INCLUDE, "tsdd_cuda.h"),
            os.path.join(LIB, "libtsdd_cuda.so")]
    if force or _stale(target, deps):
        cxx = HOST_CXX if os.path.exists(HOST_CXX) else "g++"
        _run([cxx, "-std=c++17", "-O2", "-Wall", "-Wextra", "-I", INCLUDE, "-o", target, src, "-L", LIB,
              "-ltsdd_cuda", "-ldl", "-lpthread", "-Wl,-rpath,$ORIGIN"])
    return target


def build_test_programs(force: bool = False) -> str:
    """tests/cpp/mirror_check: the reference-shaped C++ entry points (SubsequenceMatrix::build ->
    DiscordIndexes::build -> phidd_discord) of include/tsdd/cuda_engine.hpp, driven by the GPU tests."""
    target = os.path.join(LIB, "mirror_check")
    src = os.path.join(ROOT, "tests", "cpp", "mirror_check.cpp")
    deps = [src, os.path.join(INCLUDE, "tsdd", "cuda_engine.hpp"), os.path.join(INCLUDE, "tsdd_cuda.h"),
            os.path.join(LIB, "libtsdd_cuda.so")]
    if force or _stale(target, deps):
        cxx = HOST_CXX if os.path.exists(HOST_CXX) else "g++"
        _run([cxx, "-std=c++17", "-O2", "-Wall", "-Wextra", "-I", INCLUDE, "-o", target, src, "-L", LIB,
              "-ltsdd_cuda", "-ldl", "-lpthread", "-Wl,-rpath,$ORIGIN"])
    return target


def build_all(force: bool = False, verbose: bool = False) -> dict:
    out = {"gen": build_gen(force), "cuda": build_cuda(force, verbose)}
    out["cli"] = build_tools(force)
    out["mirror_check"] = build_test_programs(force)
    out["cuda_dbg"] = build_cuda(force, verbose, debug_bounds=True)
    return out


if __name__ == "__main__":
    out = build_all(force="--force" in sys.argv, verbose=True)
    for k, v in out.items():
        print(k, v)
