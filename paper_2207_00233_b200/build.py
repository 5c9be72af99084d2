"""Build libfse_b200.so in-tree for sm_100a (nvcc; no GPU needed).

    python -m paper_2207_00233_b200.build [--force]

Translation units are compiled in parallel into objects under build/ and linked
into paper_2207_00233_b200/libfse_b200.so (static cudart), which travels to
the GPU box with the repo snapshot.
"""

from __future__ import annotations

import argparse
import os
import shutil
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

PKG = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
OBJ = os.path.join(REPO, "build", "fse_b200")
LIB = os.path.join(PKG, "libfse_b200.so")
# dev A/B builds: FSE_BUILD_TAG=x FSE_NVCC_DEFS="-DFOO" builds variants/libfse_b200_x.so
# (own object dir); load one with FSE_LIB=<path>.  The product build ignores both.
_TAG = os.environ.get("FSE_BUILD_TAG", "")
if _TAG:
    OBJ = os.path.join(REPO, "build", "fse_b200_" + _TAG)
    LIB = os.path.join(PKG, "variants", f"libfse_b200_{_TAG}.so")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-Xcompiler", "-O3",
              "--expt-relaxed-constexpr"]
HEADERS = ["fse_fit.cuh", "fse_common.h", "fse_kernel.cuh", "fse_fast.cuh", "fse_gen.cuh", "fse_wcache.h"]


def _nvcc() -> str:
    for cand in (shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found")


def sources():
    return sorted(f for f in os.listdir(CSRC) if f.endswith((".cu", ".cpp")))


def _stale(target, deps):
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = False) -> str:
    nvcc = _nvcc()
    os.makedirs(OBJ, exist_ok=True)
    hdrs = [os.path.join(CSRC, h) for h in HEADERS] + [os.path.join(REPO, "include", "fse_b200.h")]
    jobs = []
    objs = []
    for src in sources():
        s = os.path.join(CSRC, src)
        o = os.path.join(OBJ, src + ".o")
        objs.append(o)
        if force or _stale(o, [s] + hdrs):
            cmd = [nvcc, *ARCH, *NVCC_FLAGS, "-I", os.path.join(REPO, "include"), "-c", s, "-o", o]
            if _TAG:
                cmd += os.environ.get("FSE_NVCC_DEFS", "").split()
            if src.endswith(".cu"):
                cmd += ["-Xptxas", "-v"] if verbose else []
            jobs.append(cmd)

    def run(cmd):
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"{' '.join(cmd)}\n{r.stdout}\n{r.stderr}")
        if verbose:
            sys.stderr.write(r.stderr)
        return cmd

    with ThreadPoolExecutor(max_workers=max(1, min(len(jobs), os.cpu_count() or 1))) as ex:
        list(ex.map(run, jobs))
    os.makedirs(os.path.dirname(LIB), exist_ok=True)
    if force or jobs or _stale(LIB, objs):
        run([nvcc, *ARCH, "-shared", "-cudart", "static", "-o", LIB, *objs])
    return LIB


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--force", action="store_true")
    ap.add_argument("-v", "--verbose", action="store_true")
    a = ap.parse_args()
    print(build(force=a.force, verbose=a.verbose))
