"""Build libmerf.so in-tree for sm_100a (nvcc; one object per translation unit, compiled in
parallel, then linked).  No torch, no JIT cache: the .so lives next to this file so it
travels with the repo snapshot to the GPU box."""
from __future__ import annotations

import glob
import os
import subprocess
from concurrent.futures import ThreadPoolExecutor

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
ROOT = os.path.dirname(HERE)
LIB = os.path.join(HERE, "libmerf.so")
OBJ = os.path.join(HERE, "build")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-Xptxas", "-v",
         "-I", os.path.join(ROOT, "include")]


def _sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")))


def _deps():
    return (_sources() + glob.glob(os.path.join(CSRC, "*.cuh")) + glob.glob(os.path.join(CSRC, "*.h"))
            + [os.path.join(ROOT, "include", "merf.h"), __file__])


def source_hash() -> str:
    """16-hex digest of the library sources (csrc + include/merf.h): stamps profile captures so
    that bench.py can tell whether a committed ncu capture still describes the built kernels."""
    import hashlib
    h = hashlib.sha256()
    for p in sorted(glob.glob(os.path.join(CSRC, "*.cu")) + glob.glob(os.path.join(CSRC, "*.cuh"))
                    + glob.glob(os.path.join(CSRC, "*.h")) + [os.path.join(ROOT, "include", "merf.h")]):
        h.update(os.path.basename(p).encode())
        with open(p, "rb") as f:
            h.update(f.read())
    return h.hexdigest()[:16]


def needs_build() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    return any(os.path.getmtime(p) > t for p in _deps())


def build(force: bool = False, verbose: bool = False, lib: str = LIB, extra=(), obj_dir: str = OBJ) -> str:
    """Build the library (default: in-tree libmerf.so).  `lib`/`extra`/`obj_dir` build a variant
    with extra nvcc flags elsewhere (e.g. scratch/ for A/B timing through MERF_LIB)."""
    if not force and lib == LIB and not needs_build():
        return LIB
    os.makedirs(obj_dir, exist_ok=True)

    def compile_one(src):
        obj = os.path.join(obj_dir, os.path.basename(src) + ".o")
        cmd = [NVCC, *ARCH, *FLAGS, *extra, "-c", src, "-o", obj]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"nvcc failed for {src}:\n{r.stderr}")
        return obj, r.stderr

    with ThreadPoolExecutor(max_workers=8) as ex:
        results = list(ex.map(compile_one, _sources()))
    if verbose:
        for _, log in results:
            print(log)
    with open(os.path.join(obj_dir, "ptxas.log"), "w") as f:
        for _, log in results:
            f.write(log)
    tmp = lib + ".tmp"
    cmd = [NVCC, *ARCH, "-shared", "-o", tmp, *[o for o, _ in results], "-lcudart", "-lz"]
    subprocess.check_call(cmd)
    os.replace(tmp, lib)
    return lib


if __name__ == "__main__":
    import sys
    build(force="-f" in sys.argv, verbose="-v" in sys.argv)
    print(LIB)
