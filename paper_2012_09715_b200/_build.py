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


def built_hash(path: str) -> str | None:
    """arv_source_hash() of a built library, read from the file (the string is
    tagged "ARV_SOURCE_HASH=<hex>" in .rodata) without loading it."""
    import re

    with open(path, "rb") as fh:
        m = re.search(rb"ARV_SOURCE_HASH=([0-9a-f]{64}|unknown)", fh.read())
    return m.group(1).decode() if m else None


def needs_build() -> bool:
    """Missing, or built from other sources.  Content-based (the embedded
    source hash), not mtime-based: a snapshot copied to another machine may
    not keep file times, and a library whose sources are unchanged must not
    be rebuilt there."""
    if not os.path.exists(LIB_PATH):
        return True
    return built_hash(LIB_PATH) != source_hash()


def build(verbose_ptxas: bool = False, force: bool = False, defines=(), out: str | None = None) -> str:
    """Compile csrc/*.cu and link libarv_b200.so (or `out` with extra -D defines).

    Objects whose source, headers and command line are unchanged are reused
    unless ``force``."""
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
    if defines or out is not None:  # experiment variants: objects outside the repo
        objdir = os.path.join(tempfile.gettempdir(), "arv_variant_build", os.path.basename(target))
        os.makedirs(objdir, exist_ok=True)
    headers = sorted(glob.glob(os.path.join(CSRC, "*.cuh")) + glob.glob(os.path.join(INCLUDE, "*.h")))
    objs = []
    procs = []
    for src in sources():
        base = os.path.basename(src)
        obj = os.path.join(objdir, base + ".o")
        objs.append(obj)
        cmd = [nvcc, *common, *PER_FILE_FLAGS.get(base, [])]
        if base == "arv_runtime.cu":  # the only unit that embeds the source hash
            cmd += [f'-DARV_SOURCE_HASH="{source_hash()}"']
        cmd += ["-c", src, "-o", obj]
        # incremental: an object is reused when it is newer than its source and
        # every header and was built with the same command line
        stamp = obj + ".cmd"
        key = hashlib.sha256(repr(cmd).encode()).hexdigest()
        fresh = (not force and os.path.exists(obj) and os.path.exists(stamp)
                 and open(stamp).read() == key
                 and all(os.path.getmtime(d) <= os.path.getmtime(obj) for d in [src, *headers]))
        if fresh:
            continue
        p = subprocess.Popen(cmd)
        p.stamp, p.key = stamp, key
        procs.append(p)
    bad = [p.args[-3] for p in procs if p.wait() != 0]
    for p in procs:
        if p.returncode == 0:
            with open(p.stamp, "w") as fh:
                fh.write(p.key)
    if bad:
        raise RuntimeError(f"nvcc failed for {bad}")
    tmp = target + ".tmp"
    subprocess.run([nvcc, *ARCH_FLAGS, "-shared", "-o", tmp, *objs], check=True)
    os.replace(tmp, target)
    return target


if __name__ == "__main__":
    print(build(verbose_ptxas="--verbose-ptxas" in sys.argv, force=True))
