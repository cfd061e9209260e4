"""Build the in-tree CUDA library (sm_100a) -- ``python -m paper_2410_17375_b200.build``."""
from __future__ import annotations

import os
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
CSRC = PKG / "csrc"
LIB = PKG / "libamusd.so"
SOURCES = ["api.cu", "protocol.cu", "transformer.cu", "gemm_tc.cu", "forward_tc.cu", "prefill.cu", "decode_gv.cu", "decode_cl.cu"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC,-O2", "--expt-relaxed-constexpr",
]
OBJ = PKG / "build"


def sources():
    return [CSRC / s for s in SOURCES if (CSRC / s).exists()]


def needs_build() -> bool:
    if not LIB.exists():
        return True
    t = LIB.stat().st_mtime
    deps = list(CSRC.glob("*.cu")) + list(CSRC.glob("*.cuh")) + list(CSRC.glob("*.h")) + [PKG.parent / "include" / "amusd.h"]
    return any(p.stat().st_mtime > t for p in deps)


def build(force: bool = False, verbose: bool = False) -> Path:
    if not force and not needs_build():
        return LIB
    # one nvcc per translation unit, in parallel (no cross-TU device code: no -rdc), then link
    from concurrent.futures import ThreadPoolExecutor
    OBJ.mkdir(exist_ok=True)
    cmds = [[NVCC, *FLAGS, "-c", str(src), "-o", str(OBJ / (src.stem + ".o"))] for src in sources()]
    if verbose:
        for c in cmds:
            print(" ".join(c), file=sys.stderr)
    with ThreadPoolExecutor(len(cmds)) as ex:
        rcs = list(ex.map(lambda c: subprocess.run(c).returncode, cmds))
    if any(rcs):
        raise subprocess.CalledProcessError(max(rcs), "nvcc")
    tmp = LIB.with_suffix(".so.tmp")
    subprocess.run([NVCC, "-gencode", "arch=compute_100a,code=sm_100a", "-shared",
                    *[str(OBJ / (s.stem + ".o")) for s in sources()], "-o", str(tmp)], check=True)
    os.replace(tmp, LIB)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True))
