"""Per-phase cycle shares of the packed sort passes (needs the -DRMX_PHASES build):

    RMX_LIB=paper_2109_09812_b200/librmx_b200_phases.so python tools/phase_step.py --config C2
"""
import ctypes
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2109_09812_b200 import _native  # noqa: E402

NAMES = ["acquire+TMA wait", "digits+rank", "counts+publish+scan", "reorder+lookback", "write-out"]

if __name__ == "__main__":
    out = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "profile_step.py")] + sys.argv[1:] + ["--steps", "1"],
                         capture_output=True, text=True)
    print(out.stdout)
