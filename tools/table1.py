"""The paper's Table 1 workload on one B200: grid_quads(N) re-indexed on the device.

    python tools/table1.py [--sizes 8 64 1024 4096 8192] [--reps 10] [--out profiles/r01_table1.json]

grid_quads(N) (reference bench.py:42-68) is generated on the device; the timed
region is one rmx_reindex (CUDA events on its stream, median of --reps after a
warm-up).  Printed beside the paper's RTX 3090 thrust+CUDA times
(BASELINE.md section 1).
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2109_09812_b200 import gen, pipeline  # noqa: E402

PAPER_3090_MS = {1024: 9.2, 4096: 92.0, 8192: 338.0}
TABLE1_OUT = {8: 81, 64: 4225, 1024: 1050625, 4096: 16785409, 8192: 67125249}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--sizes", type=int, nargs="+", default=[8, 64, 1024, 4096, 8192])
    ap.add_argument("--reps", type=int, default=10)
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    dev = torch.device("cuda", 0)
    s = torch.cuda.current_stream(dev)
    rows = []
    for n in a.sizes:
        vtx, idx = gen.grid_quads_tensors(n, dev)
        V, E = vtx.shape[0], idx.shape[0]
        out_v, out_e = torch.empty_like(vtx), torch.empty_like(idx)
        info = torch.zeros(2, dtype=torch.int64, device=dev)
        ws = torch.empty(pipeline.workspace_bytes(V, 2, E, 4), dtype=torch.uint8, device=dev)
        pipeline.launch(vtx, V, 2, idx, E, 4, out_v, out_e, info, ws, None, s)
        times = []
        for _ in range(a.reps):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            e0.record(s)
            pipeline.launch(vtx, V, 2, idx, E, 4, out_v, out_e, info, ws, None, s)
            e1.record(s)
            torch.cuda.synchronize()
            times.append(e0.elapsed_time(e1))
        times.sort()
        ms = times[len(times) // 2]
        count = int(info[0].item())
        row = {"n": n, "vertices_in": V, "vertices_out": count, "ms": ms, "verts_per_s": V / (ms * 1e-3)}
        if n in TABLE1_OUT:
            row["table1_out_ok"] = count == TABLE1_OUT[n]
        if n in PAPER_3090_MS:
            row["rtx3090_ms"] = PAPER_3090_MS[n]
            row["speedup_vs_rtx3090"] = PAPER_3090_MS[n] / ms
        rows.append(row)
        print(json.dumps(row))
        del vtx, idx, out_v, out_e, ws
        torch.cuda.empty_cache()
    if a.out:
        with open(a.out, "w") as f:
            json.dump({"workload": "grid_quads(N): float2, 4-index quads, 5 rows per quad (1 unused centre)",
                       "timing": "device (CUDA events), median of reps, inputs resident", "rows": rows}, f, indent=1)


if __name__ == "__main__":
    main()
