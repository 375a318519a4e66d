"""Build liblancet_moe.so (the C-ABI library) in-tree with nvcc for sm_100a.

    python -m paper_2404_19429_b200.build [--force] [--jobs N]

Each .cu/.cpp under csrc/ is compiled to an object in build/ (in parallel, skipped when up to
date), then linked into paper_2404_19429_b200/liblancet_moe.so against the NCCL shipped with
the torch wheel (nvidia/nccl, 2.28), with an rpath to it.
"""
from __future__ import annotations

import argparse
import concurrent.futures as cf
import glob
import os
import shutil
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
INCLUDE = os.path.join(os.path.dirname(HERE), "include")
# experiment variants (A/B builds): LANCET_BUILD_OUT=<lib path> LANCET_BUILD_DEFS="-DX -DY"
LIB = os.environ.get("LANCET_BUILD_OUT") or os.path.join(HERE, "liblancet_moe.so")
BUILD = os.path.join(HERE, "build") if LIB == os.path.join(HERE, "liblancet_moe.so") else LIB + ".objs"
DEFS = os.environ.get("LANCET_BUILD_DEFS", "").split()
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def nvcc() -> str:
    for p in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", shutil.which("nvcc")):
        if p and os.path.exists(p):
            return p
    raise RuntimeError("nvcc not found")


def nccl_dirs() -> tuple[str, str]:
    import importlib.util
    spec = importlib.util.find_spec("nvidia.nccl")
    if spec is not None and spec.submodule_search_locations:
        root = list(spec.submodule_search_locations)[0]
        inc, lib = os.path.join(root, "include"), os.path.join(root, "lib")
        if os.path.exists(os.path.join(inc, "nccl.h")):
            return inc, lib
    return "/usr/include", "/usr/lib/x86_64-linux-gnu"


def _deps_newer(obj: str, src: str) -> bool:
    if not os.path.exists(obj):
        return True
    t = os.path.getmtime(obj)
    deps = [src] + glob.glob(os.path.join(CSRC, "*.h")) + glob.glob(os.path.join(CSRC, "*.cuh")) \
        + glob.glob(os.path.join(INCLUDE, "*.h"))
    return any(os.path.getmtime(d) > t for d in deps)


def compile_one(src: str, force: bool, verbose: bool) -> str:
    nccl_inc, _ = nccl_dirs()
    obj = os.path.join(BUILD, os.path.basename(src) + ".o")
    if not force and not _deps_newer(obj, src):
        return obj
    cmd = [nvcc(), *ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-fvisibility=hidden",
           "-I", CSRC, "-I", INCLUDE, "-I", nccl_inc, "--expt-relaxed-constexpr", *DEFS,
           "-Xptxas", "-v" if verbose else "-O3", "-c", src, "-o", obj + ".tmp"]
    if src.endswith(".cpp"):
        cmd = [c for c in cmd if c not in ("--expt-relaxed-constexpr",)]
        cmd[cmd.index("-c"):cmd.index("-c")] = ["-x", "cu"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed for {src}:\n{' '.join(cmd)}\n{r.stdout}\n{r.stderr}")
    if verbose and r.stderr:
        sys.stderr.write(r.stderr)
    os.replace(obj + ".tmp", obj)
    return obj


def build(force: bool = False, jobs: int = 8, verbose: bool = False) -> str:
    os.makedirs(BUILD, exist_ok=True)
    srcs = sorted(glob.glob(os.path.join(CSRC, "*.cu")) + glob.glob(os.path.join(CSRC, "*.cpp")))
    with cf.ThreadPoolExecutor(max_workers=jobs) as ex:
        objs = list(ex.map(lambda s: compile_one(s, force, verbose), srcs))
    if not force and os.path.exists(LIB) and all(os.path.getmtime(o) <= os.path.getmtime(LIB) for o in objs):
        return LIB
    _, nccl_lib = nccl_dirs()
    tmp = LIB + f".tmp{os.getpid()}"
    cmd = [nvcc(), *ARCH, "-shared", "-o", tmp, *objs, "-L", nccl_lib, "-l:libnccl.so.2",
           "-Xlinker", f"-rpath={nccl_lib}", "-lcuda" if os.path.exists("/usr/lib/x86_64-linux-gnu/libcuda.so") else "",
           "-Xcompiler", "-fvisibility=hidden"]
    cmd = [c for c in cmd if c]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"link failed:\n{' '.join(cmd)}\n{r.stdout}\n{r.stderr}")
    os.replace(tmp, LIB)
    return LIB


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--force", action="store_true")
    ap.add_argument("--jobs", type=int, default=8)
    ap.add_argument("-v", "--verbose", action="store_true")
    a = ap.parse_args()
    print(build(a.force, a.jobs, a.verbose))
