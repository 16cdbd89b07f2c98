"""In-tree build of the CUDA extension (libsplatnav_b200.so) for sm_100a.

nvcc compiles csrc/*.cu with -fmad=false (no implicit FMA contraction: the float64 geometry
reproduces the reference's rounding, see csrc/sn_common.cuh) and -lineinfo for ncu source views.
Translation units compile in parallel into build/ objects, then link into the shared library.
"""

import concurrent.futures as cf
import glob
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
OBJ = os.path.join(os.path.dirname(HERE), "build", "obj")
LIB = os.path.join(HERE, "libsplatnav_b200.so")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = ARCH + ["-O3", "-lineinfo", "-fmad=false", "-std=c++17", "-Xcompiler", "-fPIC,-O2",
                     "--expt-relaxed-constexpr"]


def sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")))


def headers():
    return sorted(glob.glob(os.path.join(CSRC, "*.cuh")) + glob.glob(os.path.join(CSRC, "*.h")) +
                  [os.path.join(os.path.dirname(HERE), "include", "splatnav_b200.h")])


def up_to_date():
    if not os.path.exists(LIB):
        return False
    t = os.path.getmtime(LIB)
    return all(os.path.getmtime(f) <= t for f in sources() + headers())


def build(force=False, verbose=False, extra_flags=(), lib=LIB, obj_dir=OBJ):
    """Compile csrc/*.cu into `lib`; `extra_flags` / `lib` / `obj_dir` build a variant (e.g. the
    bounds-checked -DSN_CHECKS library under build_variants/) without touching the product library."""
    if not force and not extra_flags and lib == LIB and up_to_date():
        return LIB
    nvcc = os.environ.get("NVCC", "nvcc")
    os.makedirs(obj_dir, exist_ok=True)
    os.makedirs(os.path.dirname(lib), exist_ok=True)
    flags = NVCC_FLAGS + list(extra_flags)

    def compile_one(src):
        obj = os.path.join(obj_dir, os.path.basename(src) + ".o")
        cmd = [nvcc] + flags + ["-c", "-o", obj, src]
        if verbose:
            print(" ".join(cmd), file=sys.stderr)
        subprocess.run(cmd, check=True, cwd=CSRC)
        return obj

    with cf.ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 1)) as ex:
        objs = list(ex.map(compile_one, sources()))
    cmd = [nvcc] + ARCH + ["-shared", "-o", lib] + objs
    if verbose:
        print(" ".join(cmd), file=sys.stderr)
    subprocess.run(cmd, check=True, cwd=CSRC)
    return lib


def build_checks(verbose=False):
    """The bounds-checked variant (SN_ASSERT on every shared-memory queue, gather and pair write)."""
    root = os.path.dirname(HERE)
    return build(force=True, verbose=verbose, extra_flags=["-DSN_CHECKS"],
                 lib=os.path.join(root, "build_variants", "libsn_checks.so"),
                 obj_dir=os.path.join(root, "build", "obj_checks"))


if __name__ == "__main__":
    if "--checks" in sys.argv:
        build_checks(verbose=True)
    else:
        build(force="--force" in sys.argv, verbose=True)
