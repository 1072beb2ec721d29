"""In-tree build of the native libraries (sm_100a only).

    python -m paper_2506_02006_b200.build

produces paper_2506_02006_b200/lib/libmorphserve.so (CUDA kernels + C ABI,
include/morphserve.h).  The .so files are git-ignored but travel to the GPU
box with the gpurun snapshot.
"""
from __future__ import annotations

import concurrent.futures as cf
import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIB = os.environ.get("MS_LIB_DIR", os.path.join(PKG, "lib"))  # MS_LIB_DIR: experiment variants only
OBJ = os.path.join(LIB, "obj")

NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVFLAGS = ["-std=c++17", "-O3", "-lineinfo", "-Xcompiler", "-fPIC,-O3", "--expt-relaxed-constexpr",
           "-I" + os.path.join(ROOT, "include")]
NVFLAGS += os.environ.get("MS_NVCC_EXTRA", "").split()  # experiments only
CU_SOURCES = ["gemm.cu", "attention.cu", "prefill_attention.cu", "prefill_attention_tc.cu", "elementwise.cu",
              "runtime.cu"]


def _run(cmd):
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError("build failed:\n" + " ".join(cmd) + "\n" + r.stdout + r.stderr)
    return r


def _stale(out, deps):
    if not os.path.exists(out):
        return True
    t = os.path.getmtime(out)
    return any(os.path.getmtime(d) > t for d in deps)


def build_device_lib(verbose: bool = False) -> str:
    os.makedirs(OBJ, exist_ok=True)
    headers = [os.path.join(CSRC, h) for h in os.listdir(CSRC) if h.endswith((".h", ".cuh"))]
    headers.append(os.path.join(ROOT, "include", "morphserve.h"))
    jobs = []
    objs = []
    for src in CU_SOURCES:
        s = os.path.join(CSRC, src)
        o = os.path.join(OBJ, src + ".o")
        objs.append(o)
        if _stale(o, [s] + headers):
            jobs.append([NVCC, *ARCH, *NVFLAGS, "-c", s, "-o", o])
    with cf.ThreadPoolExecutor(max_workers=min(8, max(1, len(jobs)))) as ex:
        for r in ex.map(_run, jobs):
            if verbose and r.stderr:
                print(r.stderr, file=sys.stderr)
    out = os.path.join(LIB, "libmorphserve.so")
    if _stale(out, objs):
        _run([NVCC, *ARCH, "-shared", "-cudart", "static", "-o", out, *objs])
    return out


HOST_SOURCES = ["core.cpp", "engine.cpp", "device_backend.cpp"]
CXXFLAGS = ["-std=c++20", "-O2", "-fPIC", "-Wall", "-Wextra", "-Wno-unused-parameter"]


def build_host_lib(verbose: bool = False) -> str:
    """libmorphserve_host.so: the C++ engine / KV pool / controller (links libmorphserve.so)."""
    host = os.path.join(CSRC, "host")
    srcs = [os.path.join(host, s) for s in HOST_SOURCES]
    deps = srcs + [os.path.join(host, h) for h in os.listdir(host) if h.endswith(".hpp")]
    deps.append(os.path.join(ROOT, "include", "morphserve.h"))
    out = os.path.join(LIB, "libmorphserve_host.so")
    if _stale(out, deps + [os.path.join(LIB, "libmorphserve.so")]):
        r = _run(["g++", *CXXFLAGS, "-shared", "-o", out, *srcs, "-L" + LIB, "-lmorphserve",
                  "-Wl,-rpath,$ORIGIN"])
        if verbose and r.stderr:
            print(r.stderr, file=sys.stderr)
    return out


def build_pymodule(verbose: bool = False) -> str:
    import sysconfig

    import pybind11
    host = os.path.join(CSRC, "host")
    src = os.path.join(host, "bindings.cpp")
    out = os.path.join(PKG, "_core" + sysconfig.get_config_var("EXT_SUFFIX"))
    deps = [src] + [os.path.join(host, h) for h in os.listdir(host) if h.endswith(".hpp")]
    if _stale(out, deps + [os.path.join(LIB, "libmorphserve_host.so")]):
        r = _run(["g++", *CXXFLAGS, "-shared", "-o", out, src, "-I" + pybind11.get_include(),
                  "-I" + sysconfig.get_paths()["include"], "-L" + LIB, "-lmorphserve_host", "-lmorphserve",
                  "-Wl,-rpath,$ORIGIN/lib"])
        if verbose and r.stderr:
            print(r.stderr, file=sys.stderr)
    return out


def build_all(verbose: bool = False) -> None:
    build_device_lib(verbose)
    build_host_lib(verbose)
    build_pymodule(verbose)


if __name__ == "__main__":
    build_all(verbose=True)
    print("built", os.path.join(LIB, "libmorphserve.so"))
