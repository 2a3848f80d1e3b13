"""Build libinpc_raster.so in-tree with nvcc for sm_100a (no JIT cache)."""
from __future__ import annotations

import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIB = os.path.join(PKG, "libinpc_raster.so")
SOURCES = [os.path.join(CSRC, "inpc_raster.cu")]
DEPS = SOURCES + [os.path.join(CSRC, f) for f in ("kernels.cuh", "raster_math.cuh", "single_sort.cuh", "spatial_order.cuh")] + [
    os.path.join(ROOT, "include", "inpc_raster.h")]

NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17", "-shared", "-Xcompiler", "-fPIC",
    "-Xcompiler", "-fvisibility=hidden",
    "--expt-relaxed-constexpr",
    "-Xptxas", "-v",
    # no --use_fast_math: the pinned op order must hold
]


FLAGS_FILE = LIB + ".flags"


def _extra():
    # diagnostics only, e.g. -DINPC_PHASE_TIMES
    return os.environ.get("INPC_NVCC_EXTRA", "").split()


def _flag_line(extra) -> str:
    return " ".join(FLAGS + list(extra))


def stale() -> bool:
    """Library missing, older than a source, or built with other flags."""
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    if any(os.path.getmtime(d) > t for d in DEPS):
        return True
    return built_flags() != _flag_line(_extra())


def built_flags():
    try:
        with open(FLAGS_FILE) as f:
            return f.read().strip()
    except OSError:
        return None


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and not stale():
        return LIB
    tmp = LIB + f".tmp{os.getpid()}"
    extra = _extra()
    cmd = [NVCC, *FLAGS, *extra, "-I", os.path.join(ROOT, "include"), "-I", CSRC, *SOURCES, "-o", tmp]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError("nvcc failed building libinpc_raster.so")
    if verbose:
        sys.stderr.write(r.stderr)
    with open(os.path.join(PKG, "ptxas_info.txt"), "w") as f:
        f.write(r.stderr)
    os.replace(tmp, LIB)
    with open(FLAGS_FILE, "w") as f:
        f.write(_flag_line(extra) + "\n")
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True))
