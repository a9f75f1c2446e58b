"""Build libarv_b200.so (sm_100a) in-tree with nvcc.

    python paper_2012_09715_b200/_build.py [--verbose-ptxas]

The library is a plain C-ABI shared object (include/approxrv_b200.h); no
torch headers are involved.  It is written next to this file so that it
travels to the GPU box with the repository snapshot.
"""

from __future__ import annotations

import glob
import hashlib
import os
import shutil
import subprocess
import tempfile
import sys

PKG_DIR = os.path.dirname(os.path.abspath(__file__))
REPO_DIR = os.path.dirname(PKG_DIR)
CSRC = os.path.join(PKG_DIR, "csrc")
INCLUDE = os.path.join(REPO_DIR, "include")
LIB_NAME = "libarv_b200.so"
LIB_PATH = os.path.join(PKG_DIR, LIB_NAME)

ARCH_FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a"]
# The MLMC level kernels instantiate the same ncchi2 quantile code in several
# kernels (with / without the CTA sort, one-kernel / segmented); with implicit
# mul+add contraction ptxas may fuse differently per instantiation, so per-path
# results would depend on the launch form.  Every intended FMA there is
# written explicitly (fma()), so contraction is switched off for that file.
PER_FILE_FLAGS = {"arv_mlmc.cu": ["-fmad=false"]}


def nvcc_path() -> str:
    for cand in (os.environ.get("NVCC"), shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found: cannot build libarv_b200.so")


def sources() -> list[str]:
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")))


def _deps() -> list[str]:
    return sorted(sources() + glob.glob(os.path.join(CSRC, "*.cuh")) + glob.glob(os.path.join(INCLUDE, "*.h")))


def source_hash() -> str:
    """sha256 over the library's sources and build flags (embedded in the
    library as arv_source_hash(); a mismatch at load time = stale library)."""
    h = hashlib.sha256()
    for p in _deps():
        h.update(os.path.basename(p).encode())
        with open(p, "rb") as fh:
            h.update(fh.read())
    h.update(repr((ARCH_FLAGS, PER_FILE_FLAGS)).encode())
    return h.hexdigest()


def needs_build() -> bool:
    if not os.path.exists(LIB_PATH):
        return True
    t = os.path.getmtime(LIB_PATH)
    return any(os.path.getmtime(p) > t for p in _deps())


def build(verbose_ptxas: bool = False, force: bool = False, defines=(), out: str | None = None) -> str:
    """Compile every csrc/*.cu and link libarv_b200.so (or `out` with extra -D defines)."""
    target = out or LIB_PATH
    if not force and not defines and out is None and not needs_build():
        return LIB_PATH
    nvcc = nvcc_path()
    objdir = os.path.join(PKG_DIR, "build")
    os.makedirs(objdir, exist_ok=True)
    common = ARCH_FLAGS + [
        "-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC", "-Xcompiler", "-fvisibility=hidden",
        "-I", INCLUDE, "-I", CSRC, "--expt-relaxed-constexpr",
        # a misplaced `#pragma unroll` (warning 609-D) once silently dropped the
        # tuned unroll of the generators: every nvcc / ptxas warning fails the build
        "-Werror", "all-warnings",
    ]
    if verbose_ptxas:
        common += ["-Xptxas", "-v"]
    common += [f"-D{d}" for d in defines]
    common += [f'-DARV_SOURCE_HASH="{source_hash()}"']
    if defines or out is not None:  # experiment variants: objects outside the repo
        objdir = os.path.join(tempfile.gettempdir(), "arv_variant_build", os.path.basename(target))
        os.makedirs(objdir, exist_ok=True)
    objs = []
    procs = []
    for src in sources():
        obj = os.path.join(objdir, os.path.basename(src) + ".o")
        objs.append(obj)
        procs.append(subprocess.Popen([nvcc, *common, *PER_FILE_FLAGS.get(os.path.basename(src), []), "-c", src, "-o", obj]))
    bad = [p.args[-3] for p in procs if p.wait() != 0]
    if bad:
        raise RuntimeError(f"nvcc failed for {bad}")
    tmp = target + ".tmp"
    subprocess.run([nvcc, *ARCH_FLAGS, "-shared", "-o", tmp, *objs], check=True)
    os.replace(tmp, target)
    return target


if __name__ == "__main__":
    print(build(verbose_ptxas="--verbose-ptxas" in sys.argv, force=True))
