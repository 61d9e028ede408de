# SPDX-License-Identifier: Apache-2.0
"""In-tree build of the native library (no JIT cache: the .so files travel with the repo).

    python -m paper_1902_06855_b200.build [--force] [--verbose]

Produces
  paper_1902_06855_b200/libgflow_b200.so          C-ABI (include/gflow_b200.h) + the C++ API
                                                  (csrc/include/gflow/*.hpp) + sm_100a kernels
  paper_1902_06855_b200/gflowpy*.so               pybind11 module mirroring the reference's
                                                  gflowpy (bindings/module.cpp) plus the GPU engine
Kernels are compiled for sm_100a only (-gencode arch=compute_100a,code=sm_100a) with
-lineinfo for ncu source correlation.
"""
from __future__ import annotations

import argparse
import concurrent.futures as cf
import glob
import os
import subprocess
import sys
import sysconfig

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
BUILD = os.path.join(PKG, "_build")
LIB = os.path.join(PKG, "libgflow_b200.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
CXX = os.environ.get("CXX", "g++")
CUDA_HOME = os.environ.get("CUDA_HOME", "/usr/local/cuda")

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
INCLUDES = ["-I" + os.path.join(ROOT, "include"), "-I" + os.path.join(CSRC, "include"), "-I" + CSRC]
NVCC_FLAGS = ARCH + ["-O3", "-lineinfo", "-std=c++20", "-Xcompiler", "-fPIC,-O2",
                     "-Xptxas", "-O3", "--expt-relaxed-constexpr"] + INCLUDES
CXX_FLAGS = ["-std=c++20", "-O2", "-fPIC", "-pthread", "-Wall", "-Wextra",
             "-I" + os.path.join(CUDA_HOME, "include")] + INCLUDES


def _srcs():
    cu = sorted(glob.glob(os.path.join(CSRC, "*.cu")))
    cpp = sorted(glob.glob(os.path.join(CSRC, "host", "*.cpp")))
    return cu, cpp


def _headers():
    hs = glob.glob(os.path.join(CSRC, "*.cuh")) + glob.glob(os.path.join(CSRC, "include", "gflow", "*.hpp"))
    hs.append(os.path.join(ROOT, "include", "gflow_b200.h"))
    return hs


def _mtime(p):
    return os.path.getmtime(p) if os.path.exists(p) else -1.0


def _obj(src):
    rel = os.path.relpath(src, CSRC).replace(os.sep, "_")
    return os.path.join(BUILD, rel + ".o")


def _run(cmd, verbose):
    if verbose:
        print(" ".join(cmd), flush=True)
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError("build failed:\n" + " ".join(cmd) + "\n" + r.stdout + r.stderr)
    return r.stdout + r.stderr


def pybind_module_path():
    suffix = sysconfig.get_config_var("EXT_SUFFIX") or ".so"
    return os.path.join(PKG, "gflowpy" + suffix)


def build(force: bool = False, verbose: bool = False, jobs: int | None = None) -> list[str]:
    os.makedirs(BUILD, exist_ok=True)
    cu, cpp = _srcs()
    newest_hdr = max((_mtime(h) for h in _headers()), default=0)
    jobs_list = []
    for s in cu:
        o = _obj(s)
        if force or _mtime(o) < max(_mtime(s), newest_hdr):
            jobs_list.append([NVCC] + NVCC_FLAGS + ["-c", s, "-o", o])
    for s in cpp:
        o = _obj(s)
        if force or _mtime(o) < max(_mtime(s), newest_hdr):
            jobs_list.append([CXX] + CXX_FLAGS + ["-c", s, "-o", o])
    with cf.ThreadPoolExecutor(max_workers=jobs or os.cpu_count() or 4) as ex:
        list(ex.map(lambda c: _run(c, verbose), jobs_list))
    objs = [_obj(s) for s in cu + cpp]
    if force or jobs_list or _mtime(LIB) < max(_mtime(o) for o in objs):
        _run([NVCC] + ARCH + ["-shared", "-o", LIB] + objs +
             ["-lcudart", "-Xlinker", "-rpath," + os.path.join(CUDA_HOME, "lib64")], verbose)
    out = [LIB]
    bind = os.path.join(CSRC, "bindings", "module.cpp")
    if os.path.exists(bind):
        mod = pybind_module_path()
        if force or _mtime(mod) < max(_mtime(LIB), _mtime(bind), newest_hdr):
            import pybind11
            pyinc = sysconfig.get_paths()["include"]
            _run([CXX] + CXX_FLAGS + ["-shared", "-I" + pybind11.get_include(), "-I" + pyinc,
                                      bind, "-o", mod, "-L" + PKG, "-lgflow_b200",
                                      "-L" + os.path.join(CUDA_HOME, "lib64"), "-lcudart",
                                      "-Wl,-rpath,$ORIGIN",
                                      "-Wl,-rpath," + os.path.join(CUDA_HOME, "lib64")], verbose)
        out.append(mod)
    return out


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--force", action="store_true")
    ap.add_argument("--verbose", action="store_true")
    args = ap.parse_args()
    for p in build(force=args.force, verbose=args.verbose):
        print(p)
    sys.exit(0)
