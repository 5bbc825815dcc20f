"""In-tree build of the CUDA C-ABI library (sm_100a only).

    python -m paper_1805_12498_b200.build [--force] [-v]

Compiles csrc/hafb200.cu (ABI, shared-memory kernels, reductions) and one
object per register-kernel size (csrc/fast_inst.cu, mirror_inst.cu, modp_inst.cu
with -DHAFB_S=S) in
parallel, then links ``paper_1805_12498_b200/libhafb200.so``.  The .so is
git-ignored but travels to the GPU box with the repo snapshot.
"""

from __future__ import annotations

import os
import shutil
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

PKG = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
# objects live under the repo (git-ignored build/), one directory per flag set, so two
# checkouts or two flag variants never overwrite each other's objects
BUILD_ROOT = os.environ.get("HAFB200_BUILD_DIR", os.path.join(REPO, "build"))
# HAFB200_LIB sends a variant build elsewhere (the in-tree library stays the default build)
LIB = os.environ.get("HAFB200_LIB") or os.path.join(PKG, "libhafb200.so")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FAST_SIZES = list(range(2, 49, 2))  # kFastSMax = 48 (csrc/fast_launch.h)
MIRROR_SIZES = list(range(2, 65, 2))  # n <= 64 (D <= 32: 32-bit masks)


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found")


def _deps():
    out = [os.path.join(REPO, "include", "hafb200.h"), os.path.abspath(__file__)]
    for f in os.listdir(CSRC):
        if f.endswith((".cu", ".cuh", ".h")):
            out.append(os.path.join(CSRC, f))
    return out


def _stamp(flags) -> str:
    """Identity of a build: the compile flags (environment-selected variants included)."""
    import hashlib

    return hashlib.sha256(" ".join(flags).encode()).hexdigest()[:16]


def up_to_date(flags=None) -> bool:
    if not os.path.exists(LIB):
        return False
    stamp_path = LIB + ".stamp"
    want = _stamp(flags if flags is not None else _flags(False))
    if not os.path.exists(stamp_path) or open(stamp_path).read().strip() != want:
        return False
    t = os.path.getmtime(LIB)
    return all(os.path.getmtime(d) <= t for d in _deps())


def _flags(verbose):
    f = [*ARCH, "-O3", "-lineinfo", "-std=c++17", "--expt-relaxed-constexpr", "-Xcompiler", "-fPIC", "-Xcompiler", "-O2",
         "-I", os.path.join(REPO, "include")] + ([f"-DHAFB_STAGGER={os.environ['HAFB_STAGGER']}"] if os.environ.get("HAFB_STAGGER") else []) \
        + ([f"-DHAFB_SMEM_HI={os.environ['HAFB_SMEM_HI']}"] if os.environ.get("HAFB_SMEM_HI") else []) \
        + ([f"-DHAFB_REG_THREADS={os.environ['HAFB_REG_THREADS']}"] if os.environ.get("HAFB_REG_THREADS") else []) \
        + (os.environ["HAFB_EXTRA_FLAGS"].split() if os.environ.get("HAFB_EXTRA_FLAGS") else [])
    if verbose:
        f.append("-Xptxas=-v")
    return f


def _units():
    units = [("hafb200.o", os.path.join(CSRC, "hafb200.cu"), [])]
    for s in FAST_SIZES:
        units.append((f"fast_{s:02d}.o", os.path.join(CSRC, "fast_inst.cu"), [f"-DHAFB_S={s}"]))
    for s in MIRROR_SIZES:
        units.append((f"mirror_{s:02d}.o", os.path.join(CSRC, "mirror_inst.cu"), [f"-DHAFB_S={s}"]))
    for s in MIRROR_SIZES:
        units.append((f"modp_{s:02d}.o", os.path.join(CSRC, "modp_inst.cu"), [f"-DHAFB_S={s}"]))
    return units


def build(force: bool = False, verbose: bool = False, jobs: int | None = None) -> str:
    flags = _flags(verbose)
    stamp_flags = [f for f in flags if f != "-Xptxas=-v"]
    if not force and up_to_date(stamp_flags):
        return LIB
    OBJ = os.path.join(BUILD_ROOT, "obj-" + _stamp(stamp_flags))
    os.makedirs(OBJ, exist_ok=True)
    cc = nvcc()

    def compile_one(u):
        obj, src, extra = u
        out = os.path.join(OBJ, obj)
        r = subprocess.run([cc, *flags, *extra, "-c", src, "-o", out], capture_output=True, text=True)
        return obj, r

    jobs = jobs or max(1, (os.cpu_count() or 2))
    failed = []
    with ThreadPoolExecutor(max_workers=jobs) as ex:
        for obj, r in ex.map(compile_one, _units()):
            if verbose and (r.stdout or r.stderr):
                sys.stderr.write(f"== {obj}\n{r.stdout}{r.stderr}")
            if r.returncode != 0:
                failed.append((obj, r.stderr))
    if failed:
        for obj, err in failed:
            sys.stderr.write(f"== {obj} FAILED\n{err}\n")
        raise RuntimeError(f"nvcc failed for {[f[0] for f in failed]}")
    objs = [os.path.join(OBJ, u[0]) for u in _units()]
    subprocess.run([cc, *ARCH, "--shared", "-o", LIB + ".tmp", *objs], check=True)
    os.replace(LIB + ".tmp", LIB)
    with open(LIB + ".stamp", "w") as f:
        f.write(_stamp(stamp_flags) + "\n")
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
