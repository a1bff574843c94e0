"""Build libretina.so (all kernels + the C ABI) in-tree for sm_100a with nvcc."""
from __future__ import annotations

import glob
import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIB = os.path.join(PKG, "libretina.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-Xptxas", "-v",
         f"-I{os.path.join(ROOT, 'include')}"]


def sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")))


def _deps():
    return sources() + glob.glob(os.path.join(CSRC, "*.cuh")) + [os.path.join(ROOT, "include", "retina.h")]


def stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    return any(os.path.getmtime(p) > t for p in _deps())


def build(force: bool = False, verbose: bool = False, out: str = LIB, defines=()) -> str:
    """Compile every csrc/*.cu (one nvcc process per file, in parallel) and link them into one
    shared library (`defines` only for experiments)."""
    if out == LIB and not defines and not force and not stale():
        return LIB
    import concurrent.futures
    import tempfile
    dflags = [f"-D{d}" for d in defines]
    with tempfile.TemporaryDirectory(prefix="retina_build_") as tmp:
        objs = [os.path.join(tmp, os.path.basename(src) + ".o") for src in sources()]

        def compile_one(src_obj):
            src, obj = src_obj
            return subprocess.run([NVCC, *ARCH, *FLAGS, *dflags, "-c", "-o", obj, src], capture_output=True,
                                  text=True)

        with concurrent.futures.ThreadPoolExecutor(max_workers=min(8, len(objs))) as pool:
            results = list(pool.map(compile_one, zip(sources(), objs)))
        log = "".join(r.stderr for r in results)
        if any(r.returncode != 0 for r in results):
            sys.stderr.write("".join(r.stdout + r.stderr for r in results if r.returncode != 0))
            raise RuntimeError("nvcc failed building libretina.so")
        res = subprocess.run([NVCC, *ARCH, "-shared", "-Xcompiler", "-fPIC", "-o", out, *objs], capture_output=True,
                             text=True)
        if res.returncode != 0:
            sys.stderr.write(res.stdout + res.stderr)
            raise RuntimeError("nvcc failed linking libretina.so")
    if out == LIB:
        with open(os.path.join(PKG, "ptxas.log"), "w") as f:
            f.write(log)
    if verbose:
        sys.stderr.write(log)
    return out


if __name__ == "__main__":
    import argparse
    ap = argparse.ArgumentParser()
    ap.add_argument("--force", action="store_true")
    ap.add_argument("--out", default=LIB)
    ap.add_argument("-D", dest="defines", action="append", default=[])
    a = ap.parse_args()
    print(build(force=a.force, verbose=True, out=a.out, defines=a.defines))
