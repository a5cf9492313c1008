"""Small-mesh latency: direct launches vs the captured graph (grid_quads(N), device-resident).

    python tools/tiny_latency.py
"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import time, torch
from paper_2109_09812_b200 import gen, pipeline
for n in (8, 64, 256):
    vtx, idx = gen.grid_quads_tensors(n)
    V, E = vtx.shape[0], idx.shape[0]
    ov, oe = torch.empty_like(vtx), torch.empty_like(idx)
    info = torch.zeros(2, dtype=torch.int64, device="cuda")
    ws = torch.empty(pipeline.workspace_bytes(V, 2, E, 4), dtype=torch.uint8, device="cuda")
    s = torch.cuda.current_stream()
    g = pipeline.PipelineGraph(vtx, V, 2, idx, E, 4, ov, oe, info, ws)
    for name, fn in (("direct", lambda: pipeline.launch(vtx, V, 2, idx, E, 4, ov, oe, info, ws, None, s)), ("graph", lambda: g.launch(s))):
        for _ in range(20): fn()
        torch.cuda.synchronize()
        t = time.perf_counter()
        for _ in range(200): fn()
        torch.cuda.synchronize()
        wall = (time.perf_counter() - t) / 200 * 1e3
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s); fn(); e1.record(s); torch.cuda.synchronize()
        print(f"n={n} V={V} {name}: wall {wall:.3f} ms/step, single device {e0.elapsed_time(e1):.3f} ms, count {int(info[0])}")
