"""Build libmcinv.so (the C-ABI library) in-tree with nvcc for sm_100a.

The library is the product: kernels (sweep3.cu, sweep5.cu, sweep.cu, contract.cu, reduce.cu) and
the C ABI / host preprocessing (mcinv_host.cu). ``--fmad=false`` so that
only explicit fma() calls fuse (reading R10); cudart is linked
statically so the library does not depend on the CUDA runtime torch ships.
"""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
SO = os.path.join(HERE, "libmcinv.so")
SOURCES = ["mcinv_host.cu", "levels.cu", "sweep.cu", "sweep3.cu", "sweep5.cu", "sweep6.cu", "contract.cu", "contract_ozaki.cu", "reduce.cu"]
HEADERS = ["mcinv_internal.cuh", "noise.cuh", "scalar.cuh", "levels.h", "sweep_common.cuh"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-std=c++17", "-lineinfo", "--fmad=false", "-Xcompiler", "-fPIC,-O2",
         "-Xptxas", "-v", "-cudart", "static", "-I", os.path.join(ROOT, "include")]
FLAGS += os.environ.get("MCINV_NVCC_EXTRA", "").split()  # experiments (e.g. -DMCINV_NOISE_FMA); force=True


def _stale() -> bool:
    if not os.path.exists(SO):
        return True
    t = os.path.getmtime(SO)
    deps = [os.path.join(CSRC, f) for f in SOURCES + HEADERS] + [os.path.join(ROOT, "include", "mcinv.h")]
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = False) -> str:
    """Compile every source to an object in parallel (relocatable device code is not
    needed: no kernel crosses a file), then link the shared library."""
    if not force and not _stale():
        return SO
    from concurrent.futures import ThreadPoolExecutor
    tmp = SO + ".tmp"
    objdir = os.path.join(HERE, "build_obj")
    os.makedirs(objdir, exist_ok=True)

    def compile_one(f):
        obj = os.path.join(objdir, f.replace(".cu", ".o"))
        cmd = [NVCC, *ARCH, *FLAGS, "-c", "-o", obj, os.path.join(CSRC, f)]
        r = subprocess.run(cmd, capture_output=True, text=True)
        return obj, cmd, r

    with ThreadPoolExecutor(max_workers=min(len(SOURCES), os.cpu_count() or 1)) as ex:
        results = list(ex.map(compile_one, SOURCES))
    link = [NVCC, *ARCH, "-shared", "-cudart", "static", "-o", tmp] + [o for o, _, _ in results] + ["-lpthread"]
    lr = subprocess.run(link, capture_output=True, text=True)
    log = os.path.join(HERE, "build.log")
    with open(log, "w") as f:
        for _, cmd, r in results:
            f.write(" ".join(cmd) + "\n" + r.stdout + r.stderr)
        f.write(" ".join(link) + "\n" + lr.stdout + lr.stderr)
    bad = [r for _, _, r in results if r.returncode != 0] + ([lr] if lr.returncode != 0 else [])
    if bad:
        for r in bad:
            sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError(f"nvcc failed (see {log})")
    if verbose:
        sys.stderr.write("".join(r.stderr for _, _, r in results))
    os.replace(tmp, SO)
    return SO


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True))
