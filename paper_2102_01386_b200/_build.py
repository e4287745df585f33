"""Build libautofreeze.so in-tree with nvcc for sm_100a (no JIT cache).

`python paper_2102_01386_b200/_build.py [--force] [-v] [--ptxas]` (run by path:
importing the package loads the library this script builds).
"""
import os
import subprocess
import sys
import sysconfig

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
SOURCES = ["af_host.cpp", "af_ctx.cpp", "af_cache_api.cpp", "af_norms.cu", "af_decide.cu", "af_cache.cu", "af_gemm.cu"]
HEADERS = ["af_internal.h", "af_host.h", "af_decide.cuh", "af_ptx.cuh"]
LIB = os.path.join(PKG, "libautofreeze.so")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def _nvcc():
    for c in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc"):
        if c and os.path.exists(c):
            return c
    return "nvcc"


def nccl_dirs():
    """Headers + library of the NCCL that torch loads (nvidia-nccl wheel), so one
    NCCL lives in the process; falls back to the system copy."""
    purelib = sysconfig.get_paths()["purelib"]
    base = os.path.join(purelib, "nvidia", "nccl")
    inc, lib = os.path.join(base, "include"), os.path.join(base, "lib")
    if os.path.exists(os.path.join(inc, "nccl.h")) and os.path.exists(os.path.join(lib, "libnccl.so.2")):
        return inc, lib
    return "/usr/include", "/usr/lib/x86_64-linux-gnu"


STAMP = LIB + ".flags"   # the AF_NVCC_EXTRA the library was built with (git-ignored)


def _extra():
    return os.environ.get("AF_NVCC_EXTRA", "").strip()


def _stale():
    if not os.path.exists(LIB):
        return True
    built = open(STAMP).read() if os.path.exists(STAMP) else ""
    if built != _extra():
        return True
    t = os.path.getmtime(LIB)
    deps = [os.path.join(CSRC, s) for s in SOURCES + HEADERS] + [os.path.join(ROOT, "include", "af.h"),
                                                                   os.path.abspath(__file__)]
    return any(os.path.getmtime(d) > t for d in deps)


def build(force=False, verbose=False, ptxas_verbose=False):
    if not force and not _stale():
        return LIB
    inc, lib = nccl_dirs()
    cmd = [_nvcc(), "-O3", "-std=c++17", *ARCH, "-lineinfo", "-shared",
           "-Xcompiler", "-fPIC,-fvisibility=hidden",
           "-I", os.path.join(ROOT, "include"), "-I", inc,
           *[os.path.join(CSRC, s) for s in SOURCES],
           "-o", LIB + ".tmp",
           "-L", lib, "-l:libnccl.so.2", "-Xlinker", f"-rpath,{lib}",
           "-cudart", "static"]
    if ptxas_verbose:
        cmd += ["-Xptxas", "-v"]
    cmd += _extra().split()
    if verbose:
        print(" ".join(cmd), flush=True)
    r = subprocess.run(cmd, cwd=CSRC, capture_output=True, text=True)
    if verbose or r.returncode != 0:
        sys.stdout.write(r.stdout)
        sys.stderr.write(r.stderr)
    if r.returncode != 0:
        raise RuntimeError("nvcc failed building libautofreeze.so")
    os.replace(LIB + ".tmp", LIB)
    with open(STAMP, "w") as fh:
        fh.write(_extra())
    return LIB


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose="-v" in sys.argv, ptxas_verbose="--ptxas" in sys.argv)
