"""Device time of meshes with wide vertices (position + normal + uv, D = 8) on the packed / AoS
paths: a lattice soup of (nx x ny) quads whose vertices carry x, y, z (lattice), a normal from 6
axis directions and uv = lattice coordinates / extent.

    python tools/wide_probe.py [--nx 2000] [--ny 2000] [--steps 3]
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
    ap.add_argument("--nx", type=int, default=2000)
    ap.add_argument("--ny", type=int, default=2000)
    ap.add_argument("--steps", type=int, default=3)
    a = ap.parse_args()
    vtx3, idx = gen.lattice_soup_tensors("tri", (a.nx, a.ny))
    V = vtx3.shape[0]
    f = vtx3.view(torch.float32)
    normals = torch.tensor([[1, 0, 0], [-1, 0, 0], [0, 1, 0], [0, -1, 0], [0, 0, 1], [0, 0, -1]],
                           dtype=torch.float32, device=f.device)
    n = normals[(f[:, 0] * 2 + f[:, 1] * 6).to(torch.int64) % 6]
    uv = torch.stack([f[:, 0] / (0.5 * a.nx), f[:, 1] / (0.5 * a.ny)], 1)
    vtx = torch.cat([f, n, uv], 1).contiguous().view(torch.int32)
    D = vtx.shape[1]
    E, K = idx.shape
    out_v, out_e = torch.empty_like(vtx), torch.empty_like(idx)
    info = torch.zeros(2, dtype=torch.int64, device=vtx.device)
    ws = torch.empty(pipeline.workspace_bytes(V, D, E, K), dtype=torch.uint8, device=vtx.device)
    s = torch.cuda.current_stream()
    lib = _native.lib()
    for _ in range(2):
        pipeline.launch(vtx, V, D, idx, E, K, out_v, out_e, info, ws, None, s)
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0.record()
    for _ in range(a.steps):
        pipeline.launch(vtx, V, D, idx, E, K, out_v, out_e, info, ws, None, s)
    t1.record()
    torch.cuda.synchronize()
    ms = t0.elapsed_time(t1) / a.steps
    pinfo = (ctypes.c_uint32 * 4)()
    _native.check(lib.rmx_plan_info(ws.data_ptr(), V, D, s.cuda_stream, pinfo))
    print(f"D={D} V={V:,} unique={int(info[0]):,} plan(packed, words, bits, passes)={list(pinfo)} "
          f"{ms:.3f} ms ({V / ms / 1e6:.2f} G verts/s)")


if __name__ == "__main__":
    main()
