"""Build libmsort.so (sm_100a) in-tree with nvcc; no JIT, no torch extension.

    python paper_2211_16479_b200/build.py [--force]

Objects go to paper_2211_16479_b200/build/, the shared library to
paper_2211_16479_b200/lib/libmsort.so (git-ignored; it travels to the GPU box
with the gpurun snapshot).  NCCL headers and libnccl.so.2 come from the
torch wheel's nvidia-nccl package, the same library torch itself loads.
"""
from __future__ import annotations

import glob
import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
BUILD = os.path.join(PKG, "build")
LIB = os.path.join(PKG, "lib", "libmsort.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = ARCH + ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC",
                     "-Xcompiler", "-Wall", "--expt-relaxed-constexpr", "-Xptxas", "-v"]


def nccl_dirs():
    import importlib.util

    spec = importlib.util.find_spec("nvidia")
    for base in list(spec.submodule_search_locations or []):
        inc = os.path.join(base, "nccl", "include")
        lib = os.path.join(base, "nccl", "lib")
        if os.path.exists(os.path.join(inc, "nccl.h")):
            return inc, lib
    raise RuntimeError("NCCL headers not found in the nvidia wheel")


def _sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")))


def _deps():
    return _sources() + glob.glob(os.path.join(CSRC, "*.cuh")) + glob.glob(
        os.path.join(CSRC, "*.h")) + [os.path.join(ROOT, "include", "msort.h"), __file__]


def up_to_date() -> bool:
    if not os.path.exists(LIB):
        return False
    t = os.path.getmtime(LIB)
    return all(os.path.getmtime(d) <= t for d in _deps())


def build(force: bool = False, verbose: bool = False, defines=(), out: str | None = None) -> str:
    """Build the library.  `defines` (e.g. ["MSORT_K3_NC=256"]) and `out`
    produce tuning variants at another path (loaded via MSORT_LIB)."""
    lib_path = out or LIB
    if not force and not defines and out is None and up_to_date():
        return LIB
    bdir = BUILD if not defines else os.path.join(BUILD, "v_" + "_".join(defines).replace("=", ""))
    os.makedirs(bdir, exist_ok=True)
    os.makedirs(os.path.dirname(lib_path), exist_ok=True)
    inc, libdir = nccl_dirs()
    incs = ["-I", os.path.join(ROOT, "include"), "-I", inc]
    dflags = [f"-D{d}" for d in defines]

    def compile_one(src):
        obj = os.path.join(bdir, os.path.basename(src) + ".o")
        cmd = [NVCC, *NVCC_FLAGS, *dflags, *incs, "-c", src, "-o", obj]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"nvcc failed on {src}:\n{r.stderr}")
        with open(obj + ".log", "w") as f:
            f.write(r.stderr)
        if verbose:
            print(r.stderr, file=sys.stderr)
        return obj

    with ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 1)) as ex:
        objs = list(ex.map(compile_one, _sources()))
    tmp = lib_path + ".tmp"
    cmd = [NVCC, *ARCH, "-shared", "-o", tmp, *objs, "-L", libdir, "-l:libnccl.so.2",
           "-Xlinker", f"-rpath={libdir}", "-cudart", "static"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"link failed:\n{r.stderr}")
    os.replace(tmp, lib_path)
    return lib_path


if __name__ == "__main__":
    import argparse

    ap = argparse.ArgumentParser()
    ap.add_argument("--force", action="store_true")
    ap.add_argument("-v", action="store_true")
    ap.add_argument("-D", action="append", default=[], help="NAME=VALUE define (variant build)")
    ap.add_argument("--out", default=None, help="output .so for a variant build")
    a = ap.parse_args()
    print(build(force=a.force, verbose=a.v, defines=tuple(a.D), out=a.out))
