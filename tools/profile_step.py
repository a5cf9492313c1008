"""One generated config + N re-indexing steps on cuda:0 (the command ncu wraps).

    python tools/profile_step.py --config C2 --steps 2
"""
import argparse
import ctypes
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2109_09812_b200 import _native, pipeline  # noqa: E402

CFG = {"C1": (0, 625, 800, 0, 3), "C2": (0, 5000, 5000, 0, 3), "C3": (1, 150, 150, 148, 4)}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="C2")
    ap.add_argument("--steps", type=int, default=2)
    ap.add_argument("--no-compare", action="store_true", help="skip the direct-vs-graph timing (ncu launch lists)")
    a = ap.parse_args()
    lib = _native.lib()
    dev = torch.device("cuda", 0)
    s = torch.cuda.current_stream(dev)
    if a.config in ("C4", "C4S"):  # 8 welded tiles concatenated with index offsets (the merge input)
        from paper_2109_09812_b200 import gen
        pieces = [gen.welded_tile_tensors(5000, 4500 * k, k, a.config == "C4S") for k in range(8)]
        D = 3
        V = sum(p[0].shape[0] for p in pieces)
        E = sum(p[1].shape[0] for p in pieces)
        vtx = torch.cat([p[0] for p in pieces])
        offs, o = [], 0
        for p in pieces:
            offs.append(o)
            o += p[0].shape[0]
        idx = torch.cat([(p[1].to(torch.int64) + off).to(torch.int32) for p, off in zip(pieces, offs)])
        del pieces
    elif a.config == "C5s":  # one GPU's shard of C5 at 8 GPUs: the first 1/8 of the 1B-triangle soup
        from paper_2109_09812_b200 import gen
        E_all, _ = gen.lattice_sizes("tri", (20000, 25000))
        vtx, idx = gen.lattice_soup_tensors("tri", (20000, 25000), seed=0, n_elem_take=E_all // 8)
        V, D = vtx.shape
        E = idx.shape[0]
    elif a.config == "C2s":  # C2 with real-valued coordinates (oracle/lattice.py:scramble_words): hash mode
        from paper_2109_09812_b200 import gen
        vtx, idx = gen.lattice_soup_tensors("tri", (5000, 5000))
        vtx = gen.scramble_tensor(vtx)
        V, D = vtx.shape
        E = idx.shape[0]
    else:
        kid, nx, ny, nz, D = CFG[a.config]
        E, V = ctypes.c_uint64(), ctypes.c_uint64()
        lib.rmx_lattice_sizes(kid, nx, ny, nz, 1 << 63, ctypes.byref(E), ctypes.byref(V))
        E, V = E.value, V.value
        vtx = torch.empty((V, D), dtype=torch.int32, device=dev)
        idx = torch.empty((E, D), dtype=torch.int32, device=dev)
        _native.check(lib.rmx_gen_lattice_soup(kid, nx, ny, nz, 0, 1 << 63, vtx.data_ptr(), idx.data_ptr(),
                                               s.cuda_stream))
    out_v = torch.empty_like(vtx)
    out_e = torch.empty_like(idx)
    info = torch.zeros(2, dtype=torch.int64, device=dev)
    ws = torch.empty(pipeline.workspace_bytes(V, D, E, D), dtype=torch.uint8, device=dev)
    n_ev = lib.rmx_stage_count(D)
    names = [lib.rmx_stage_name(D, k).decode() for k in range(n_ev)]
    evs = [torch.cuda.Event(enable_timing=True) for _ in range(n_ev)]
    for e in evs:
        e.record(s)
    for _ in range(a.steps):
        pipeline.launch(vtx, V, D, idx, E, D, out_v, out_e, info, ws, None, s, [e.cuda_event for e in evs])
    torch.cuda.synchronize()
    print("count", int(info[0]), "status", int(info[1]))
    tot = 0.0
    for k in range(1, n_ev):
        ms = evs[k - 1].elapsed_time(evs[k])
        tot += ms
        print(f"{names[k]:>14s} {ms:8.3f} ms")
    print(f"{'total':>14s} {tot:8.3f} ms")
    hi = (ctypes.c_uint32 * 4)()
    _native.check(lib.rmx_hash_info(ws.data_ptr(), V, D, s.cuda_stream, hi))
    gi = (ctypes.c_uint32 * 4)()
    _native.check(lib.rmx_plan_guess_info(ws.data_ptr(), V, D, s.cuda_stream, gi))
    si = (ctypes.c_uint32 * 2)()
    _native.check(lib.rmx_soup_info(ws.data_ptr(), V, D, s.cuda_stream, si))
    wi = (ctypes.c_uint32 * 4)()
    _native.check(lib.rmx_window_info(ws.data_ptr(), V, D, s.cuda_stream, wi))
    print(f"window mode {wi[0] & 1}, fallback {(wi[0] >> 1) & 1}, used rows {wi[1]:,}, non-empty windows "
          f"{wi[2]:,}, largest {wi[3]:,} rows")
    print(f"value sets wanted {gi[1]}, check state {gi[3] & 0xFF:#x}, speculative {(gi[3] >> 8) & 1}, "
          f"check failed {(gi[3] >> 9) & 1}; soup rows {si[0]:,}, strictly increasing {si[1]}")
    if hi[0]:
        print(f"hash mode: {hi[1]:,} candidate rows ({hi[1] / int(info[0]):.2f} per distinct key), "
              f"{hi[2]} AoS passes over them, {hi[3]}-row dedup tiles")
    # whole-step time: direct launches vs the captured graph (conditional nodes)
    g = pipeline.PipelineGraph(vtx, V, D, idx, E, D, out_v, out_e, info, ws) if not a.no_compare else None
    for name, fn in [] if a.no_compare else (("direct", lambda: pipeline.launch(vtx, V, D, idx, E, D, out_v, out_e, info, ws, None, s)),
                     ("graph", lambda: g.launch(s))):
        fn()
        t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        t0.record(s)
        for _ in range(a.steps):
            fn()
        t1.record(s)
        torch.cuda.synchronize()
        print(f"{name + ' step':>14s} {t0.elapsed_time(t1) / a.steps:8.3f} ms   count {int(info[0])}")
    ph = (ctypes.c_ulonglong * 4)()
    if lib.rmx_debug_phase_cycles(ph, 4, 1) and ph[2]:
        print(f"  look-back (digit 0): {ph[0] / ph[2]:.2f} windows, {ph[1] / ph[2]:.2f} spins per tile")


if __name__ == "__main__":
    main()
