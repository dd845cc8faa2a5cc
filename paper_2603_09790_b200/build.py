"""Build libchebstep_gpu.so in-tree for sm_100a (nvcc cross-compiles; no GPU needed).

    python paper_2603_09790_b200/build.py [--force] [--jobs N]

(run as a script: importing the package needs the built library)

Every .cu/.cpp under csrc/ is compiled with
``-gencode arch=compute_100a,code=sm_100a -O3 -lineinfo`` into build/ and
linked into paper_2603_09790_b200/lib/libchebstep_gpu.so together with NCCL:
the torch-bundled libnccl.so.2 (nvidia/nccl in site-packages, rpath'd), so the
library and torch share ONE NCCL whichever is imported first (the older
system libnccl.so.2 loaded first would shadow torch's by soname).
"""
from __future__ import annotations

import argparse
import concurrent.futures as cf
import glob
import os
import shutil
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
OBJ = os.path.join(ROOT, "build", "obj")
LIB = os.path.join(PKG, "lib", "libchebstep_gpu.so")
CLI_SRC = os.path.join(PKG, "cli", "main.cpp")
CLI_BIN = os.path.join(PKG, "bin", "chebstep")
NVCC = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
_NCCL = sorted(glob.glob(os.path.join(sys.prefix, "lib", "python3*", "site-packages", "nvidia",
                                      "nccl")))
NCCL_DIR = _NCCL[0] if _NCCL and os.path.exists(os.path.join(_NCCL[0], "lib", "libnccl.so.2")) \
    else None
NCCL_INC = ["-I" + os.path.join(NCCL_DIR, "include")] if NCCL_DIR else []
NCCL_LINK = (["-L" + os.path.join(NCCL_DIR, "lib"), "-l:libnccl.so.2", "-Xlinker",
              "-rpath," + os.path.join(NCCL_DIR, "lib")] if NCCL_DIR else
             ["-lnccl", "-Xlinker", "-rpath,/usr/lib/x86_64-linux-gnu"])
COMMON = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-Xcompiler", "-Wall",
          "-Xcompiler", "-ffp-contract=off",
          "-I" + os.path.join(ROOT, "include"), "--expt-relaxed-constexpr", *NCCL_INC]


def _sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")) + glob.glob(os.path.join(CSRC, "*.cpp")))


def _headers():
    return (glob.glob(os.path.join(CSRC, "*.cuh")) + glob.glob(os.path.join(ROOT, "include", "*.h"))
            + glob.glob(os.path.join(ROOT, "include", "chebstep", "*.hpp")))


def _stale(target, deps):
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


CXX = shutil.which("g++") or "g++"
CUDA_INC = os.path.join(os.path.dirname(os.path.dirname(NVCC)), "include")
CXXFLAGS = ["-std=c++20", "-O3", "-fPIC", "-Wall", "-Wextra", "-ffp-contract=off",
            "-I" + os.path.join(ROOT, "include"),
            "-I" + CUDA_INC, *NCCL_INC]


EXTRA = [f"-D{d}" for d in os.environ.get("CS_DEFINES", "").split() if d]
if EXTRA:  # experiment builds go to their own object dir / library
    OBJ = OBJ + "_" + "_".join(d[2:] for d in EXTRA)
    LIB = os.environ.get("CS_LIB_OUT", LIB)


def _compile(src, force):
    obj = os.path.join(OBJ, os.path.basename(src) + ".o")
    if not force and not _stale(obj, [src] + _headers()):
        return obj, None
    if src.endswith(".cpp"):  # host-only C++ (C++20 for the std::span drop-in API)
        cmd = [CXX, *CXXFLAGS, "-c", src, "-o", obj]
    else:
        cmd = [NVCC, *ARCH, *COMMON, *EXTRA,
               "-Xptxas", "-v" if os.environ.get("CS_PTXAS_V") else "-O3", "-c", src, "-o", obj]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        return obj, f"{' '.join(cmd)}\n{r.stdout}\n{r.stderr}"
    if os.environ.get("CS_PTXAS_V"):
        sys.stderr.write(r.stderr)
    return obj, None


def build(force: bool = False, jobs: int = 8, verbose: bool = True) -> str:
    os.makedirs(OBJ, exist_ok=True)
    os.makedirs(os.path.dirname(LIB), exist_ok=True)
    srcs = _sources()
    objs, errors = [], []
    with cf.ThreadPoolExecutor(max_workers=jobs) as ex:
        for obj, err in ex.map(lambda s: _compile(s, force), srcs):
            objs.append(obj)
            if err:
                errors.append(err)
    if errors:
        raise RuntimeError("nvcc failed:\n" + "\n".join(errors))
    if force or _stale(LIB, objs):
        cmd = [NVCC, *ARCH, "-shared", "-o", LIB, *objs, *NCCL_LINK, "-Xlinker", "--no-undefined"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"link failed: {' '.join(cmd)}\n{r.stdout}\n{r.stderr}")
        if verbose:
            print(f"built {LIB}")
    if not EXTRA and (force or _stale(CLI_BIN, [LIB, CLI_SRC])):
        os.makedirs(os.path.dirname(CLI_BIN), exist_ok=True)
        cmd = [CXX, *CXXFLAGS, CLI_SRC, "-o", CLI_BIN, "-L" + os.path.dirname(LIB),
               "-lchebstep_gpu", "-Wl,-rpath,$ORIGIN/../lib"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"CLI link failed: {' '.join(cmd)}\n{r.stdout}\n{r.stderr}")
        if verbose:
            print(f"built {CLI_BIN}")
    return LIB


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--force", action="store_true")
    ap.add_argument("--jobs", type=int, default=8)
    a = ap.parse_args()
    build(a.force, a.jobs)
