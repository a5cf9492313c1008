"""Device time of the wide-key (AoS rows) path: the C2 soup with every coordinate's low
mantissa bits scrambled by a function of the value (duplicates stay duplicates, but 23
mantissa bits vary per component -> > 64 key bits, like scanned geometry).

    python tools/aos_probe.py [--config C2] [--steps 3]
"""
import argparse
import ctypes
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2109_09812_b200 import _native, gen, pipeline  # noqa: E402
from oracle import lattice  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="C2")
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--bits", type=int, default=11, help="low mantissa bits scrambled")
    a = ap.parse_args()
    kind, cells = lattice.CONFIGS[a.config]
    vtx, idx = gen.lattice_soup_tensors(kind, cells)
    w = vtx.to(torch.int64) & 0xFFFFFFFF
    h = ((w * 2654435761) & 0xFFFFFFFF) >> (32 - a.bits)
    vtx = (w ^ h).to(torch.int64)
    vtx = torch.where(vtx >= 2**31, vtx - 2**32, vtx).to(torch.int32).contiguous()
    V, D = vtx.shape
    E, K = idx.shape
    dev = vtx.device
    s = torch.cuda.current_stream()
    out_v, out_e = torch.empty_like(vtx), torch.empty_like(idx)
    info = torch.zeros(2, dtype=torch.int64, device=dev)
    ws = torch.empty(pipeline.workspace_bytes(V, D, E, K), dtype=torch.uint8, device=dev)
    lib = _native.lib()
    n_ev = lib.rmx_stage_count(D)
    names = [lib.rmx_stage_name(D, k).decode() for k in range(n_ev)]
    pipeline.launch(vtx, V, D, idx, E, K, out_v, out_e, info, ws, None, s)
    evs = [torch.cuda.Event(enable_timing=True) for _ in range(n_ev)]
    for e in evs:  # torch only measures events it has recorded once itself
        e.record(s)
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    t0.record(s)
    for _ in range(a.steps):
        pipeline.launch(vtx, V, D, idx, E, K, out_v, out_e, info, ws, None, s, [e.cuda_event for e in evs])
    t1.record(s)
    torch.cuda.synchronize()
    pinfo = (ctypes.c_uint32 * 4)()
    _native.check(lib.rmx_plan_info(ws.data_ptr(), V, D, s.cuda_stream, pinfo))
    print(f"{a.config} scrambled {a.bits} bits: count {int(info[0])} status {int(info[1])} plan {list(pinfo)}")
    for k in range(1, n_ev):
        ms = evs[k - 1].elapsed_time(evs[k])
        if ms > 0.02:
            print(f"{names[k]:>14s} {ms:8.3f} ms")
    print(f"{'step':>14s} {t0.elapsed_time(t1) / a.steps:8.3f} ms  ({V / (t0.elapsed_time(t1) / a.steps) / 1e6:.2f} G verts/s)")


if __name__ == "__main__":
    main()
