"""C4 (BASELINE configs[3]) on one B200: merge of 8 welded 5000 x 5000 tiles with 500 shared rows.

    python tools/merge_bench.py [--steps 5] [--out profiles/r01_c4.json]

Tiles are generated on the device (bit-identical to oracle/lattice.py:welded_tile) before the
timed region; one step = ``merge_tensors`` = concatenation of the vertex blocks (copy engine),
``rmx_offset_indices`` per tile, and the full re-index (210,084,008 vertex slots in, 182,541,501
out).  Device-timed with CUDA events, median of --steps after a warm-up.  The multi-GPU form of
the same merge is ``bench.py --gpus N`` through ``dist.reindex_distributed`` (merge semantics).
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2109_09812_b200 as rmx  # noqa: E402

COLS, STEP, TILES = 5000, 4500, 8


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    pieces = [rmx.gen.welded_tile_tensors(COLS, STEP * k, k) for k in range(TILES)]
    V = sum(p[0].shape[0] for p in pieces)
    I = sum(p[1].numel() for p in pieces)
    s = torch.cuda.current_stream()
    res = rmx.merge_tensors(pieces)
    U = res.vertices.shape[0]
    assert U == 182_541_501, U
    del res
    times = []
    for _ in range(a.steps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record(s)
        res = rmx.merge_tensors(pieces)
        e1.record(s)
        torch.cuda.synchronize()
        times.append(e0.elapsed_time(e1))
        del res
    times.sort()
    ms = times[len(times) // 2]
    line = {"workload": "C4: merge of 8 welded 5000x5000-quad tiles, 500 shared rows (1xB200)",
            "n_vertices": V, "n_index_slots": I, "unique": U, "ms": ms, "verts_per_s": V / (ms * 1e-3),
            "steps": a.steps, "timing": "device (CUDA events), median; merge_tensors = concat + offsets + re-index",
            "note": "the reindex_tensors call inside allocates its outputs and workspace per call"}
    print(json.dumps(line))
    if a.out:
        with open(a.out, "w") as f:
            json.dump(line, f, indent=1)


if __name__ == "__main__":
    main()
