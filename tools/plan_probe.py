"""Key plan and device time of grid_quads(N) (the paper's Table 1 inputs, row-major grids).

For each N: rmx_plan_info {packed, key words, key bits, passes}, rmx_plan_key_info {field-ranked,
value-ranked components, bits before value ranks, bits}, rmx_plan_guess_info {bits of the plan
guessed from the sample, value sets worth collecting, candidates, check state}, device ms/call.
Run with RMX_VALUE_RANK=0 to compare without value ranks.

    python tools/plan_probe.py [--sizes 1024 4096 8192] [--reps 5]
"""
import argparse
import ctypes
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2109_09812_b200 import _native, gen, pipeline  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--sizes", type=int, nargs="+", default=[1024, 4096, 8192])
    ap.add_argument("--reps", type=int, default=5)
    a = ap.parse_args()
    lib = _native.lib()
    for n in a.sizes:
        vtx, idx = gen.grid_quads_tensors(n)
        V, D = vtx.shape
        E, K = idx.shape
        ov, oe = torch.empty_like(vtx), torch.empty_like(idx)
        info = torch.zeros(2, dtype=torch.int64, device=vtx.device)
        ws = torch.empty(pipeline.workspace_bytes(V, D, E, K), dtype=torch.uint8, device=vtx.device)
        s = torch.cuda.current_stream()
        for _ in range(3):
            pipeline.launch(vtx, V, D, idx, E, K, ov, oe, info, ws, None, s)
        t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t0.record()
        for _ in range(a.reps):
            pipeline.launch(vtx, V, D, idx, E, K, ov, oe, info, ws, None, s)
        t1.record()
        torch.cuda.synchronize()
        p, k, g = ((ctypes.c_uint32 * 4)() for _ in range(3))
        _native.check(lib.rmx_plan_info(ws.data_ptr(), V, D, s.cuda_stream, p))
        _native.check(lib.rmx_plan_key_info(ws.data_ptr(), V, D, s.cuda_stream, k))
        _native.check(lib.rmx_plan_guess_info(ws.data_ptr(), V, D, s.cuda_stream, g))
        print(f"grid_quads({n}): V={V:,} D={D} plan={list(p)} keys={list(k)} guess={list(g)} "
              f"{t0.elapsed_time(t1) / a.reps:.3f} ms, {int(info[0]):,} unique")


if __name__ == "__main__":
    main()
