"""In-tree build of the CUDA library (nvcc, sm_100a only).

``build()`` compiles ``csrc/rmx_capi.cu`` (which includes every kernel) into
``librmx_b200.so`` next to this file.  Cross-compiles without a GPU.
"""
from __future__ import annotations

import glob
import os
import shutil
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
SOURCES = [os.path.join(HERE, "csrc", "rmx_capi.cu")]
DEPENDS = SOURCES + sorted(glob.glob(os.path.join(HERE, "csrc", "*.cu*"))) + [
    os.path.join(ROOT, "include", "remesh_b200.h"), os.path.abspath(__file__)]
OUTPUT = os.path.join(HERE, "librmx_b200.so")

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-Xcompiler", "-fPIC", "-shared",
    "--expt-relaxed-constexpr",
]


def nvcc() -> str:
    for cand in (shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found")


def up_to_date() -> bool:
    if not os.path.exists(OUTPUT):
        return False
    t = os.path.getmtime(OUTPUT)
    return all(os.path.getmtime(p) <= t for p in DEPENDS)


def build(force: bool = False, verbose: bool = False, defines=(), output: str | None = None) -> str:
    """Compile the library; ``defines`` (e.g. ("RMX_PHASES",)) build a tuning variant into ``output``."""
    out = output or OUTPUT
    if not force and not defines and out == OUTPUT and up_to_date():
        return OUTPUT
    tmp = out + ".tmp"
    cmd = [nvcc(), *NVCC_FLAGS, *[f"-D{d}" for d in defines], "-o", tmp, *SOURCES]
    if verbose:
        cmd.insert(1, "-Xptxas=-v")
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError(f"nvcc failed ({res.returncode}):\n{res.stderr}")
    if verbose:
        print(res.stderr)
    os.replace(tmp, out)
    return out


if __name__ == "__main__":
    import sys
    if "--phases" in sys.argv:
        print(build(defines=("RMX_PHASES",), output=os.path.join(HERE, "librmx_b200_phases.so")))
    elif "--checked" in sys.argv:  # bounds-counting build for tools/sanitize_probe.py (RMX_LIB=...)
        print(build(defines=("RMX_CHECKED",), output=os.path.join(HERE, "librmx_b200_checked.so")))
    else:
        print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
