"""Builds the sm_100a CUDA library in-tree (no JIT cache): libwt_gpu.so.

`python -m paper_1711_07999_b200.build` or `build()` from __graft_entry__.
The tracking kernels use the default fp contraction; the synthetic renderer
(wt_render.cu) is compiled with -fmad=false so its fp64 arithmetic rounds
like the reference's unfused C++.
"""
from __future__ import annotations

import os
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
LIB = PKG / "libwt_gpu.so"
BUILD = PKG / "_build"
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
COMMON = ARCH + ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC",
                 "-I", str(ROOT / "include"), "-I", str(CSRC), "--expt-relaxed-constexpr"]
COMMON += os.environ.get("WT_NVCC_FLAGS", "").split()  # experiments only (e.g. -DWT_...)

UNITS = [
    ("wt_gpu.cu", []),
    ("wt_exact.cu", ["-fmad=false"]),
    ("wt_render.cu", ["-fmad=false"]),
    ("wt_model.cu", ["-fmad=false"]),
]


def _run(cmd: list[str], echo: bool = False) -> None:
    proc = subprocess.run(cmd, capture_output=True, text=True)
    if proc.returncode != 0:
        sys.stderr.write(proc.stdout + proc.stderr)
        raise RuntimeError(f"command failed: {' '.join(cmd)}")
    if echo:
        sys.stderr.write(proc.stdout + proc.stderr)


def build(force: bool = False, verbose: bool = False) -> Path:
    BUILD.mkdir(exist_ok=True)
    sources = [CSRC / u for u, _ in UNITS]
    headers = list(CSRC.glob("*.cuh")) + [ROOT / "include" / "wt_gpu.h"]
    newest = max(p.stat().st_mtime for p in sources + headers + [Path(__file__)])
    if LIB.exists() and not force and LIB.stat().st_mtime >= newest:
        return LIB
    objs = []
    for unit, extra in UNITS:
        obj = BUILD / (Path(unit).stem + ".o")
        cmd = [NVCC] + COMMON + extra + ["-c", str(CSRC / unit), "-o", str(obj)]
        if verbose:
            cmd += ["-Xptxas", "-v"]
        _run(cmd, echo=verbose)
        objs.append(str(obj))
    tmp = LIB.with_suffix(".so.tmp")
    _run([NVCC] + ARCH + ["-shared", "-o", str(tmp)] + objs + ["-lcudart"])
    os.replace(tmp, LIB)
    return LIB


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose="-v" in sys.argv)
    print(LIB)
