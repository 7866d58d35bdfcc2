"""Build libtlrb200.so in-tree with nvcc for sm_100a (no JIT cache)."""
from __future__ import annotations

import os
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
SRC = sorted((PKG / "csrc").glob("*.cu"))
OUT = PKG / "libtlrb200.so"
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
         "-Xcompiler", "-fPIC", "-shared", "--expt-relaxed-constexpr"]
if os.environ.get("TLRB_CLOCK_PROF") == "1":   # clock64 phase counters (rebuild with --force)
    FLAGS.append("-DTLRB_CLOCK_PROF")


def needs_build() -> bool:
    if not OUT.exists():
        return True
    t = OUT.stat().st_mtime
    deps = SRC + sorted((PKG / "csrc").glob("*.cuh")) + [PKG.parent / "include" / "tlrb200.h"]
    return any(p.stat().st_mtime > t for p in deps)


OBJ = PKG.parent / "build" / "obj"


def _compile(src: Path, force: bool, verbose: bool) -> Path:
    """One translation unit -> build/obj/<name>.o (rebuilt when the source or
    any shared header is newer)."""
    obj = OBJ / (src.stem + ".o")
    hdrs = sorted((PKG / "csrc").glob("*.cuh")) + [PKG.parent / "include" / "tlrb200.h"]
    if not force and obj.exists() and all(p.stat().st_mtime <= obj.stat().st_mtime for p in [src, *hdrs]):
        return obj
    flags = [f for f in FLAGS if f != "-shared"]
    cmd = [NVCC, *flags, "-c", str(src), "-o", str(obj)]
    if verbose:
        print(" ".join(cmd), file=sys.stderr)
    subprocess.run(cmd, check=True)
    return obj


def build(force: bool = False, verbose: bool = False) -> Path:
    if not force and not needs_build():
        return OUT
    from concurrent.futures import ThreadPoolExecutor
    OBJ.mkdir(parents=True, exist_ok=True)
    with ThreadPoolExecutor(max_workers=min(len(SRC), os.cpu_count() or 4)) as ex:
        objs = list(ex.map(lambda s: _compile(s, force, verbose), SRC))
    cmd = [NVCC, "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-Xcompiler", "-fPIC",
           *map(str, objs), "-o", str(OUT), "-lnccl"]
    if verbose:
        print(" ".join(cmd), file=sys.stderr)
    subprocess.run(cmd, check=True)
    return OUT


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose=True)
    print(OUT)
