"""Host-to-host latency of reindex(mesh) on small/medium meshes vs the CPU oracle port.

    python tools/host_latency.py
"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import paper_2109_09812_b200 as rmx  # noqa: E402
from oracle import remesh_oracle as O  # noqa: E402


def best(fn, reps):
    fn()
    ts = []
    for _ in range(reps):
        t = time.perf_counter()
        fn()
        ts.append(time.perf_counter() - t)
    return min(ts) * 1e3


for n in (8, 64, 256, 1024):
    m = rmx.gen.grid_quads(n)
    v, e = m.vertices, m.elements
    gpu = best(lambda: rmx.reindex(m), 20)
    cpu = best(lambda: O.reindex(v, e), 3 if n >= 1024 else 10)
    print(f"grid_quads({n}): V={v.shape[0]:>9} gpu reindex {gpu:8.3f} ms   cpu oracle {cpu:9.3f} ms")
