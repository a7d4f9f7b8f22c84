"""Build the C-ABI shared library in-tree with nvcc (sm_100a only).

    python -m paper_2506_15556_b200.build [--force]

Output: paper_2506_15556_b200/libpredgen_b200.so (git-ignored, travels to the
GPU box with the gpurun snapshot). No torch extension machinery: the library
exports plain `extern "C"` symbols (include/predgen_b200.h) loaded via ctypes.
"""

from __future__ import annotations

import hashlib
import os
import shutil
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
INCLUDE = ROOT / "include"
LIB = PKG / "libpredgen_b200.so"
OBJ = PKG / "_build"
SOURCES = ["init.cu", "layers.cu", "gemm_simt.cu", "tma.cu", "megakernel.cu", "runtime.cu"]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", shutil.which("nvcc")):
        if cand and Path(cand).exists():
            return cand
    raise RuntimeError("nvcc not found")


def _flags() -> list[str]:
    # PS_DEBUG=1: bounded spin waits that trap instead of hanging (tc_common.cuh)
    debug = ["-DPS_DEBUG_SPIN"] if os.environ.get("PS_DEBUG") == "1" else []
    return ARCH + ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "--expt-relaxed-constexpr",
                   f"-I{INCLUDE}", f"-I{CSRC}"] + debug


def _digest() -> str:
    h = hashlib.sha256()
    for p in sorted(CSRC.glob("*")) + sorted(INCLUDE.glob("*.h")):
        h.update(p.name.encode())
        h.update(p.read_bytes())
    # flags without the checkout's absolute paths: a copy of the tree elsewhere (the
    # GPU box's snapshot) reuses the library built from the same sources
    h.update(" ".join(_flags()).replace(str(ROOT), "<root>").encode())
    return h.hexdigest()


LAST = {"compiled": False, "digest": ""}


def build(force: bool = False, verbose: bool = False) -> Path:
    """Compile when the sources, headers or flags changed (sha256 stamp); LAST records
    whether this call compiled or reused a library built from identical sources."""
    stamp = PKG / "_build" / "stamp"
    digest = _digest()
    LAST.update(compiled=False, digest=digest[:16])
    if LIB.exists() and stamp.exists() and stamp.read_text() == digest and not force:
        return LIB
    LAST["compiled"] = True
    OBJ.mkdir(exist_ok=True)
    cc = nvcc()

    def compile_one(src: str) -> Path:
        obj = OBJ / (src + ".o")
        cmd = [cc, *_flags(), "-c", str(CSRC / src), "-o", str(obj)]
        if verbose:
            print(" ".join(cmd), flush=True)
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"nvcc failed on {src}:\n{r.stderr}")
        if verbose and r.stderr:
            print(r.stderr, file=sys.stderr)
        return obj

    with ThreadPoolExecutor(max_workers=len(SOURCES)) as ex:
        objs = list(ex.map(compile_one, SOURCES))
    tmp = LIB.with_suffix(".so.tmp")
    cmd = [cc, *ARCH, "-shared", "-o", str(tmp), *map(str, objs), "-lcudart"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"link failed:\n{r.stderr}")
    os.replace(tmp, LIB)
    stamp.write_text(digest)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
