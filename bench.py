#!/usr/bin/env python
"""Benchmark of the re-indexing hot path (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C2] [--impl b200|reference]

Metric: input vertices re-indexed per second, device-timed, with the % of the
HBM roofline.  Workload (N=1): config C2 of BASELINE.json -- a 50M-triangle
float3 soup (157.5M vertex slots, 5 % unused, 25,010,001 unique), generated on
the device by the library's seeded lattice generator (synthetic data).  A
"step" is one full ``rmx_reindex`` over that soup.  Inputs (2.5 GB) exceed
the 126 MB L2, so no flush is needed between steps.

* ``value``  -- V x K / device time of K back-to-back steps (CUDA events on the
  launching stream, inputs resident in HBM).
* ``e2e``    -- the same metric through the public host API
  (``paper_2109_09812_b200.ReindexStream.run``, one mesh per step): pinned
  host -> device copies, the pipeline, count + result device -> host copies,
  every step; copies of neighbouring meshes overlap the kernels (the PCIe
  link is full duplex).  ``single_call_ms`` is one unoverlapped
  ``Reindexer.run``.
* ``roofline`` -- the dominant kernel (one packed LSD pass), its algorithmic
  bytes per launch over its mean CUDA-event duration.
* ``cpu_baseline`` -- the oracle port of the reference (numpy, reference
  thread pool) on a bounded prefix sample of the same soup, host cores.

``--impl reference`` times that CPU port alone (rank 0) and prints the
reference-arm line.  Multi-GPU (torchrun, N>1): one global soup of N x 50M
triangles partitioned by element ranges, re-indexed by the NCCL sample-sort
path (paper_2109_09812_b200.dist); weak scaling, value = all ranks' input
vertices / max-over-ranks time.
"""
from __future__ import annotations

import argparse
import ctypes
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

CONFIGS = {  # name -> (kind, kind id, cells, dim, arity, scrambled coordinates)
    "C1": ("tri", 0, (625, 800, 0), 3, 3, False),
    "C2": ("tri", 0, (5000, 5000, 0), 3, 3, False),
    "C2s": ("tri", 0, (5000, 5000, 0), 3, 3, True),
    "C3": ("tet", 1, (150, 150, 148), 4, 4, False),
}
CONFIG_TEXT = {
    "C1": "1M-triangle float3 soup (3.15M verts, 5% unused)",
    "C2": "50M-triangle float3 soup on 1xB200 (157.5M verts, 5% unused)",
    "C2s": "C2 with real-valued coordinates: the low 11 mantissa bits of every word scrambled "
           "(oracle/lattice.py:scramble_words; 157.5M verts, > 64 varying key bits)",
    "C3": "20M-tet mesh, float3 position + float scalar payload (83.9M verts, D=4)",
}
METRIC = "input vertices re-indexed/sec (device-timed)"
CPU_SAMPLE_ELEMS = 1_000_000       # C2 prefix sample for the GPU arm's cpu_baseline: 3.15M vertex slots
L2_NOTE = "inputs >= 1.6 GB > 126 MB L2, no flush needed"


def workload_config(cfg: str, world: int = 1) -> dict:
    """The `config` of both arms' JSON lines (identical for the same workload)."""
    from oracle import lattice
    kind, _, cells, D, K, _ = CONFIGS[cfg]
    sz = lattice.soup_sizes(kind, cells[:2] if kind == "tri" else cells)
    return {"workload": f"{cfg}: {CONFIG_TEXT[cfg]}", "n_vertices": sz["n_vertices"], "n_elements": sz["n_elem"],
            "arity": K, "dim": D, "unique": sz["n_points"],
            "parallelism": "single" if world == 1 else f"replicas x{world}", "l2": L2_NOTE}


def host_workload(cfg: str, n_elem_take=None):
    """(vertices float32 (V, D), elements uint32 (E, K)) of a config, generated on the host."""
    from oracle import lattice
    kind, _, cells, _, _, scrambled = CONFIGS[cfg]
    v, e = lattice.lattice_soup(kind, cells[:2] if kind == "tri" else cells, seed=0, n_elem_take=n_elem_take)
    if scrambled:
        v = lattice.scramble_words(v).view(np.float32)
    return v, e


def peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.proc = None
        self.lines: list[str] = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "100", "-i", str(self.gpu)], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
            time.sleep(0.25)
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *exc):
        if self.proc:
            time.sleep(0.15)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], [], set()
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 6:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
            except ValueError:
                continue
            for n, v in zip(names, parts[2:6]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(mx), "reasons": sorted(reasons),
                "samples": len(sm)}


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def host_cores_note():
    try:
        import psutil
        phys = psutil.cpu_count(logical=False)
    except Exception:  # noqa: BLE001
        phys = None
    return f"host: {os.cpu_count()} logical / {phys} physical cores"


def cpu_port_rate(cfg: str, steps: int, warmup: int):
    """The GPU arm's cpu_baseline: the oracle port of the reference on a bounded prefix sample."""
    from oracle import remesh_oracle as oracle
    v, e = host_workload(cfg, CPU_SAMPLE_ELEMS)
    for _ in range(max(0, warmup)):
        oracle.reindex(v, e)
    times = []
    for _ in range(max(1, steps)):
        t = time.perf_counter()
        oracle.reindex(v, e)
        times.append(time.perf_counter() - t)
    med = statistics.median(times)
    sample = (f"first {CPU_SAMPLE_ELEMS:,} elements of the {cfg} soup ({len(v):,} vertex slots); "
              f"median of {len(times)} after {warmup} warm-up; numpy port of remeshx.reindex "
              f"(np.lexsort is single-threaded, the chunked steps use the reference pool); {host_cores_note()}")
    return len(v) / med, oracle.host_threads(), sample, med


def run_reference(args):
    """The reference arm: the reference algorithm (the numpy port of remeshx.reindex,
    oracle/remesh_oracle.py -- same numpy kernels, checked against remeshx on the golden cases
    and within 4 % of its time on C1) on the host cores, on the FULL workload of the GPU arm's
    config.  BASELINE.md section 3 protocol for C2/C3: R = 1 timed run (one run is 1.5-3 min);
    the warm-up runs the same code on a 1M-element prefix of the soup, untimed."""
    rank, world, _ = dist_env()
    if rank != 0:
        return
    from oracle import remesh_oracle as oracle
    t_gen = time.perf_counter()
    v, e = host_workload(args.config)
    t_gen = time.perf_counter() - t_gen
    wv, we = host_workload(args.config, CPU_SAMPLE_ELEMS)
    oracle.reindex(wv, we)
    del wv, we
    t = time.perf_counter()
    res = oracle.reindex(v, e)
    dt = time.perf_counter() - t
    cfg = workload_config(args.config, world)
    assert res["new_count"] == cfg["unique"], (res["new_count"], cfg["unique"])
    rate = len(v) / dt
    sample = (f"the full {args.config} workload ({len(v):,} vertex slots, {len(e):,} elements), 1 timed run "
              f"(BASELINE.md section 3: R=1 for C2/C3) after 1 untimed warm-up on its first "
              f"{CPU_SAMPLE_ELEMS:,} elements; numpy port of remeshx.reindex (np.lexsort is single-threaded, the "
              f"chunked steps use the reference pool of {oracle.host_threads()} threads); {host_cores_note()}; "
              f"input generated on the host in {t_gen:.0f} s (untimed)")
    line = {
        "metric": METRIC, "value": rate, "unit": "verts/s", "n_gpus": world, "steps": 1, "warmup": 0,
        "ms_per_step": dt * 1e3, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "u32", "data": "synthetic", "impl": "reference", "config": cfg,
        "requested": {"steps": args.steps, "warmup": args.warmup,
                      "note": "one full-size CPU run takes minutes: R=1 as BASELINE.md section 3 specifies"},
        "cpu_baseline": {"value": rate, "unit": "verts/s", "cores": oracle.host_threads(), "kind": "port",
                         "sample": sample},
        "e2e": {"value": rate, "unit": "verts/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    emit(line)


def mask_list(m):
    return "[" + ",".join(str(c) for c in range(32) if (m >> c) & 1) + "]"


def executed_model(V, I, U, D, KW, npass, value_ranks=False, spec=False, soup=False, win_rows=0):
    """Algorithmic HBM bytes of one packed-path step (the kernels that ran).  win_rows > 0: window mode
    (two packed passes over win_rows rows after the first, the window stage instead of head count +
    unique)."""
    if win_rows:
        n = win_rows
        pairs = I if soup else n
        first = (4 * KW + 1 + 1) * V + (4 * KW + 4 + 1) * n   # keys, digit, flags in; rows + next digit out
        second = (4 * KW + 4 + 1) * n + (4 * KW + 4) * n      # rows + digit in, rows out
        return int((4 * I + 2 * V)
                   + ((4 * D + 1) * V // 64 if value_ranks else (4 * D + 1) * V)
                   + ((4 * D + 1) * V * (1 if spec else 65) // 64 if value_ranks else 0)
                   + (4 * D + 1) * V + (4 * KW + 1) * V      # pack
                   + first + second                           # the two packed passes
                   + 4 * n + 8 * n + 8 * pairs + 4 * U        # window stage: bounds, rows in, pairs + keys out
                   + (4 * KW + 4 * D) * U                     # unpack
                   + 12 * pairs                               # map fill
                   + (0 if soup else 12 * I))                 # remap
    passes = sum(8 * KW + (0 if p == 0 else 4) + 4 + 1 + (1 if p + 1 < npass else 0) for p in range(npass))
    return int((4 * I + 2 * V)                       # mark: indices in, flags cleared + set
               # K1a: rows + flags -- with value ranks over a 1/64 sample only, the full value-set pass
               # (sample + full) checks the rows against it instead; a speculative plan (sample
               # halves saw the same value sets) skips the full pass, k_pack checks the rows
               + ((4 * D + 1) * V // 64 if value_ranks else (4 * D + 1) * V)
               + ((4 * D + 1) * V * (1 if spec else 65) // 64 if value_ranks else 0)
               + (4 * D + 1) * V + (4 * KW + 1) * V  # pack: rows + flags in, keys + digit 0 out
               + passes * V                          # LSD passes
               + (V if soup else 0)                  # soup mode: pass 0 reads the used flags
               + 4 * KW * V                          # head count
               + (4 * KW + 12) * V + 4 * KW * U      # unique: keys + origins in, pairs + unique keys out
               + (4 * KW + 4 * D) * U                # unpack
               + 12 * V                              # map fill: pairs in, map (soup: output indices) out
               + (0 if soup else 12 * I))            # remap: indices + map in, indices out


def device_workload(cfg: str, dev, stream, rank: int = 0):
    """(vtx int32 (V, D), idx int32 (E, K), expected unique count) generated on the device."""
    import torch

    from paper_2109_09812_b200 import _native, gen
    lib = _native.lib()
    kind, kid, cells, D, K, scrambled = CONFIGS[cfg]
    E64, V64 = ctypes.c_uint64(), ctypes.c_uint64()
    lib.rmx_lattice_sizes(kid, cells[0], cells[1], cells[2], 1 << 63, ctypes.byref(E64), ctypes.byref(V64))
    E, V = E64.value, V64.value
    vtx = torch.empty((V, D), dtype=torch.int32, device=dev)
    idx = torch.empty((E, K), dtype=torch.int32, device=dev)
    with torch.cuda.stream(stream):
        _native.check(lib.rmx_gen_lattice_soup(kid, cells[0], cells[1], cells[2], rank, 1 << 63, vtx.data_ptr(),
                                               idx.data_ptr(), stream.cuda_stream))
        if scrambled:
            vtx = gen.scramble_tensor(vtx)
    stream.synchronize()
    expect_u = (cells[0] + 1) * (cells[1] + 1) * ((cells[2] + 1) if kind == "tet" else 1)
    return vtx, idx, expect_u


def time_device(cfg: str, steps: int, warmup: int, dev, stream, rank: int = 0, world: int = 1, clocks=None):
    """Device time of `steps` back-to-back rmx_reindex calls on a config (inputs in HBM), the per-stage
    times of a second region with stage events, and the dominant kernel's roofline."""
    import torch

    from paper_2109_09812_b200 import _native, pipeline
    lib = _native.lib()
    kind, _, cells, D, K, _ = CONFIGS[cfg]
    vtx, idx, expect_u = device_workload(cfg, dev, stream, rank)
    V, E = vtx.shape[0], idx.shape[0]
    out_v = torch.empty((V, D), dtype=torch.int32, device=dev)
    out_e = torch.empty((E, K), dtype=torch.int32, device=dev)
    info = torch.zeros(2, dtype=torch.int64, device=dev)
    ws = torch.empty(pipeline.workspace_bytes(V, D, E, K), dtype=torch.uint8, device=dev)
    n_ev = lib.rmx_stage_count(D)
    names = [lib.rmx_stage_name(D, k).decode() for k in range(n_ev)]

    def step(events=None):
        pipeline.launch(vtx, V, D, idx, E, K, out_v, out_e, info, ws, None, stream, events)

    for _ in range(max(3, warmup)):
        step()
    stream.synchronize()
    count, status = (int(x) for x in info.cpu())
    assert status == 0 and count == expect_u, (cfg, count, status, expect_u)
    pinfo = (ctypes.c_uint32 * 4)()
    _native.check(lib.rmx_plan_info(ws.data_ptr(), V, D, stream.cuda_stream, pinfo))
    packed, key_words, vbits, executed = (int(x) for x in pinfo)
    kinfo = (ctypes.c_uint32 * 4)()
    _native.check(lib.rmx_plan_key_info(ws.data_ptr(), V, D, stream.cuda_stream, kinfo))
    field_mask, value_mask, bits_before_vr = int(kinfo[0]), int(kinfo[1]), int(kinfo[2])
    ginfo = (ctypes.c_uint32 * 4)()
    _native.check(lib.rmx_plan_guess_info(ws.data_ptr(), V, D, stream.cuda_stream, ginfo))
    spec = (int(ginfo[3]) >> 8) & 3 == 1  # speculative plan, check passed
    sinfo = (ctypes.c_uint32 * 2)()
    _native.check(lib.rmx_soup_info(ws.data_ptr(), V, D, stream.cuda_stream, sinfo))
    soup = int(sinfo[0]) != 0
    winfo = (ctypes.c_uint32 * 4)()
    _native.check(lib.rmx_window_info(ws.data_ptr(), V, D, stream.cuda_stream, winfo))
    window = (int(winfo[0]) & 3) == 1  # window mode, no fallback (rmx_window.cuh)
    win_rows = int(winfo[1])           # rows of the window passes (soup mode: all V; else the used rows)

    # per-stage CUDA events for every timed step (recorded on the launching stream)
    ev = [[torch.cuda.Event(enable_timing=True) for _ in range(n_ev)] for _ in range(steps)]
    with torch.cuda.stream(stream):
        for row in ev:
            for e_ in row:
                e_.record(stream)
    stream.synchronize()
    handles = [[e_.cuda_event for e_ in row] for row in ev]
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    launches0 = lib.rmx_kernel_launches_total()

    # timed region 1 (the headline): K plain steps.  Timed region 2: K steps with a CUDA event
    # between every stage, for the per-stage / per-pass times -- an event between two kernels
    # also ends the programmatic-dependent-launch overlap there, so region 2 runs ~2 % slower.
    if world > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize(dev)
    with (clocks or _NullCtx()):
        t0.record(stream)
        for _ in range(steps):
            step()
        t1.record(stream)
        stream.synchronize()
    torch.cuda.synchronize(dev)
    ms = t0.elapsed_time(t1) / steps
    launches = (lib.rmx_kernel_launches_total() - launches0) / steps
    t0.record(stream)
    for k in range(steps):
        step(handles[k])
    t1.record(stream)
    stream.synchronize()
    ms_staged = t0.elapsed_time(t1) / steps
    stage_ms = {}
    for k in range(1, n_ev):
        vals = [ev[s][k - 1].elapsed_time(ev[s][k]) for s in range(steps)]
        stage_ms[names[k]] = sum(vals) / len(vals)
    # dominant kernel: one executed LSD pass (packed-key or AoS rows; hash mode: AoS passes over
    # the candidate rows, rmx_hash.cuh)
    hash_mode = packed == 2
    n_rows = V
    hinfo = None
    if hash_mode:
        hi = (ctypes.c_uint32 * 4)()
        _native.check(lib.rmx_hash_info(ws.data_ptr(), V, D, stream.cuda_stream, hi))
        hinfo = {"candidate_rows": int(hi[1]), "candidates_per_unique": int(hi[1]) / expect_u,
                 "candidate_passes": int(hi[2]), "dedup_tile_rows": int(hi[3])}
        n_rows, executed = int(hi[1]), int(hi[2])
        packed = 0
    if packed and window:
        executed = 2  # window mode runs the top two packed passes only
    pass_names = [n for n in names if n.startswith("pk_pass_" if packed else "sort_pass_")]
    active = sorted((stage_ms[n] for n in pass_names), reverse=True)[:executed]
    pass_ms = sum(active) / max(1, len(active))
    row_bytes = (4 * key_words + 4) if packed else (4 * D + 4)
    # packed pass: keys + origins in and out, the digit byte read by its upsweep and the next
    # pass's digit byte written (pass 0 reads no origins: they are the row numbers; the last pass
    # writes no next digit) -- mean over the executed passes; AoS pass: rows in and out
    if packed:  # (soup mode: pass 0 also reads the used flags; window mode without soup mode: the
        # first pass reads the flags and writes the used rows only)
        out_rows = win_rows if window and not soup else V
        per_pass = [(4 * key_words + 1 + (1 if (soup or window) and p == 0 else 0)) * V
                    + (0 if p == 0 else 4 * out_rows)
                    + (4 * key_words + 4 + (1 if p + 1 < executed else 0)) * out_rows for p in range(executed)]
        pass_bytes = sum(per_pass) / len(per_pass)
    else:
        pass_bytes = 2 * row_bytes * n_rows
    hbm, peak_kind = peaks()
    achieved = pass_bytes / (pass_ms * 1e-3) / 1e9
    executed_bytes = (executed_model(V, E * K, expect_u, D, key_words, executed, value_mask != 0, spec, soup,
                                     win_rows if window else 0) if packed else None)
    pass_roof = {"bound": "hbm", "achieved": achieved, "peak": hbm, "unit": "GB/s", "frac": achieved / hbm,
                 "bytes_per_launch": pass_bytes, "launch_ms": pass_ms,
                 "kernel": "one packed LSD pass: k_pk_upsweep + k_pk_colscan + k_pk_downsweep"}
    win_roof = None
    if packed and window:
        # stage "window": k_win_bounds reads the keys (4 B/row); k_win_unique stages keys + origins
        # (8 B/row), writes an (origin, new index) pair per used row and the distinct keys
        n_pairs = int(sinfo[0]) if soup else win_rows
        win_bytes = 4 * win_rows + 8 * win_rows + 8 * n_pairs + 4 * expect_u
        win_ms = stage_ms.get("window", 0.0)
        win_roof = {"bound": "hbm", "achieved": win_bytes / (win_ms * 1e-3) / 1e9 if win_ms else None,
                    "peak": hbm, "unit": "GB/s",
                    "frac": win_bytes / (win_ms * 1e-3) / 1e9 / hbm if win_ms else None,
                    "bytes_per_launch": win_bytes, "launch_ms": win_ms,
                    "kernel": "window stage: k_win_bounds + k_win_unique (per-window shared-memory presence "
                              "bitmaps, rmx_window.cuh)",
                    "rows": win_rows, "pairs": n_pairs, "non_empty_windows": int(winfo[2]),
                    "largest_window_rows": int(winfo[3])}
    # the dominant kernel: the window stage when it takes longer than one LSD pass
    dom = win_roof if win_roof and win_roof["launch_ms"] > pass_ms else None
    res = {
        "V": V, "E": E, "D": D, "K": K, "U": expect_u, "ms": ms, "ms_staged": ms_staged, "stage_ms": stage_ms,
        "launches_per_step": launches,
        "pass_roofline": pass_roof, "window_roofline": win_roof,
        "roofline": dict(dom, traffic=None, peak_kind=peak_kind, window_mode=True, soup_mode=soup,
                         executed_passes=executed, nominal_passes=4 * D) if dom else
                    {"bound": "hbm", "achieved": achieved, "peak": hbm, "unit": "GB/s",
                     "frac": achieved / hbm, "traffic": None,
                     "kernel": ("one packed LSD pass: k_pk_upsweep + k_pk_colscan + k_pk_downsweep" if packed
                                else "one onesweep LSD pass over the hash-mode candidate rows: k_sort_pass"
                                if hash_mode else "one onesweep LSD pass: k_sort_pass"),
                     "key": (f"packed {vbits} key bits in {key_words} x u32 (field ranks on components "
                             f"{mask_list(field_mask)}, value ranks on {mask_list(value_mask)}: "
                             f"{bits_before_vr} bits before value ranks)" if packed
                             else f"{D} x u32 words"),
                     "hash_mode": hinfo,
                     "speculative_value_plan": spec if packed else None,
                     "soup_mode": soup,
                     "bytes_per_launch": pass_bytes, "launch_ms": pass_ms, "peak_kind": peak_kind,
                     "window_mode": window, "executed_passes": executed, "nominal_passes": 4 * D},
        "executed_bytes": executed_bytes,
        "tensors": (vtx, idx),
    }
    del out_v, out_e, ws
    return res


class _NullCtx:
    def __enter__(self):
        return self

    def __exit__(self, *exc):
        return False


def e2e_dropin(vtx, idx, steps: int):
    """End to end through the reference-facing operator: paper_2109_09812_b200.reindex(Mesh) with
    numpy (pageable) arrays in and out, every host<->device copy inside the timed region."""
    import torch

    import paper_2109_09812_b200 as rmx
    mesh = rmx.Mesh(vtx.cpu().numpy().view(np.float32), idx.cpu().numpy().view(np.uint32))
    torch.cuda.empty_cache()
    out, _ = rmx.reindex(mesh)          # warm-up (allocations, staging buffers)
    count = out.n_vertices
    del out
    times = []
    for _ in range(steps):
        t = time.perf_counter()
        out, _ = rmx.reindex(mesh)
        times.append(time.perf_counter() - t)
        assert out.n_vertices == count
        del out
    el = statistics.median(times)
    V, D = mesh.vertices.shape
    E, K = mesh.elements.shape
    h2d = (V * D + E * K) * 4
    d2h = 16 + (count * D + E * K) * 4
    return el, h2d, d2h, times


def run_b200(args):
    import torch

    from paper_2109_09812_b200 import _native, build, pipeline

    rank, world, local = dist_env()
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl")
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if not os.path.exists(_native.LIB_PATH):
        build.build()
    lib = _native.lib()
    stream = torch.cuda.Stream(dev)
    clk = ClockSampler(local)
    main = time_device(args.config, args.steps, args.warmup, dev, stream, rank, world, clocks=clk)
    V, E, D, K, expect_u = main["V"], main["E"], main["D"], main["K"], main["U"]
    ms = main["ms"]
    if world > 1:
        t = torch.tensor([ms], device=dev)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        ms = float(t.item())
    hbm, _ = peaks()
    nominal = (32 * D * D + 44 * D + 15) * V + 16 * E * K + 4 * D * expect_u
    compulsory = 4 * D * V + 8 * E * K + 4 * D * expect_u
    executed_bytes = main["executed_bytes"]
    value = V * world / (ms * 1e-3)
    vtx, idx = main.pop("tensors")

    # end to end (host buffers, copies inside the timed region): the drop-in operator
    # reindex(Mesh) is the headline; the pipelined ReindexStream is reported beside it
    e2e = None
    if not args.no_e2e:
        el, h2d, d2h, dropin_times = e2e_dropin(vtx, idx, max(3, min(args.steps, 5)))
        e2e = {"value": V * world / el, "unit": "verts/s", "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
               "ms_per_step": el * 1e3, "steps": len(dropin_times), "api": "paper_2109_09812_b200.reindex(Mesh)",
               "note": "the reference-facing operator (pipeline.py:133): numpy float32/uint32 arrays in, a new "
                       "Mesh of numpy arrays out; median of the timed calls after one warm-up call",
               "times_ms": [t * 1e3 for t in dropin_times]}
        torch.cuda.empty_cache()
        host_v = torch.empty((V, D), dtype=torch.int32, pin_memory=True)
        host_e = torch.empty((E, K), dtype=torch.int32, pin_memory=True)
        host_v.copy_(vtx)
        host_e.copy_(idx)
        del vtx, idx
        torch.cuda.empty_cache()
        # single-call latency from pinned buffers: copies in, pipeline, copies out, nothing overlapped
        rx = pipeline.Reindexer(V, D, E, K, dev)
        for _ in range(2):
            rx.run(host_v, host_e)
        t = time.perf_counter()
        for _ in range(2):
            rx.run(host_v, host_e)
        latency = (time.perf_counter() - t) / 2
        del rx
        torch.cuda.empty_cache()
        # throughput: a stream of meshes, copies of mesh k+1 / k-1 overlapped with compute of mesh k
        rs = pipeline.ReindexStream(V, D, E, K, dev)
        for _ in rs.run((host_v, host_e) for _ in range(3)):
            pass
        e2e_steps = max(4, min(2 * args.steps, 16))
        if world > 1:
            torch.distributed.barrier()
        t = time.perf_counter()
        n_done = 0
        for _ in rs.run((host_v, host_e) for _ in range(e2e_steps)):
            n_done += 1
        el = (time.perf_counter() - t) / e2e_steps
        assert n_done == e2e_steps
        if world > 1:
            tt = torch.tensor([el], device=dev)
            torch.distributed.all_reduce(tt, op=torch.distributed.ReduceOp.MAX)
            el = float(tt.item())
        sh2d, sd2h = rs.bytes_per_mesh(V, E, rs.last_counts[-1])
        e2e["stream"] = {"value": V * world / el, "unit": "verts/s", "h2d_bytes_per_step": sh2d,
                         "d2h_bytes_per_step": sd2h, "ms_per_step": el * 1e3, "steps": e2e_steps,
                         "api": "paper_2109_09812_b200.ReindexStream.run",
                         "note": "one mesh per step, pinned host -> pinned host; H2D of the next mesh and D2H of "
                                 "the previous one overlap this mesh's kernels (fill and drain inside the timed "
                                 "region)",
                         "single_call_ms": latency * 1e3, "single_call_api": "paper_2109_09812_b200.Reindexer.run"}
        del rs, host_v, host_e
        torch.cuda.empty_cache()
    else:
        del vtx, idx
        torch.cuda.empty_cache()

    # the other single-GPU workloads, device-timed the same way (default run only)
    extra = {}
    if not args.no_extra and args.config == "C2":
        for cfg in ("C2s", "C3"):
            r = time_device(cfg, max(3, min(args.steps, 5)), 3, dev, stream, rank, world)
            r.pop("tensors")
            extra[cfg] = {"workload": CONFIG_TEXT[cfg], "value": r["V"] / (r["ms"] * 1e-3), "unit": "verts/s",
                          "ms_per_step": r["ms"], "n_vertices": r["V"], "unique": r["U"],
                          "roofline": r["roofline"], "stage_ms": {k: v for k, v in r["stage_ms"].items() if v > 0.02},
                          "launches_per_step": r["launches_per_step"]}
            torch.cuda.empty_cache()

    cpu = None
    if rank == 0 and not args.no_cpu_baseline:
        rate, cores, sample, _ = cpu_port_rate(args.config, 3, 1)
        cpu = {"value": rate, "unit": "verts/s", "cores": cores, "kind": "port", "sample": sample}

    if rank == 0:
        roof = main["roofline"]
        tp = os.path.join(ROOT, "profiles", "traffic.json")
        if os.path.exists(tp):
            try:
                with open(tp) as f:
                    tj = json.load(f)
                key = ("window_dram_bytes_per_launch" if "k_win_unique" in roof.get("kernel", "")
                       else "pass_dram_bytes_per_launch")
                roof["traffic"] = tj.get(args.config, {}).get(key)
            except Exception:
                pass
        line = {
            "metric": METRIC, "value": value, "unit": "verts/s", "n_gpus": world, "steps": args.steps,
            "warmup": max(3, args.warmup), "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "u32", "data": "synthetic",
            "config": workload_config(args.config, world),
            "e2e": e2e,
            "roofline": roof,
            "pass_roofline": main.get("pass_roofline"),
            "window_roofline": main.get("window_roofline"),
            "pipeline_roofline": {
                "executed_bytes": executed_bytes,
                "achieved_gbs": executed_bytes / (ms * 1e-3) / 1e9 if executed_bytes else None,
                "frac": executed_bytes / (ms * 1e-3) / 1e9 / hbm if executed_bytes else None,
                "note": "algorithmic bytes of the kernels that ran (DESIGN.md (d)): mark 4I+2V, vary (4D+1)V "
                        "(with value ranks: a 1/64 sample, and value sets (4D+1)V x 65/64), "
                        "pack (4D+1)V+(4KW+1)V, per pass <= (8KW+10)V, head count 4KW V, unique (4KW+12)V+4KW U, "
                        "unpack (4KW+4D)U, map fill 12V, remap 12I",
                "survey_nominal_bytes": nominal,
                "compulsory_bytes": compulsory,
                "compulsory_frac": compulsory / (ms * 1e-3) / 1e9 / hbm,
                "compulsory_note": "SURVEY 8(d) compulsory I/O 4DV + 4I + 4DU + 4I (read vertices and indices, "
                                   "write unique rows and indices once)",
                "survey_note": "SURVEY 8(d) nominal model (32D^2+44D+15)V+16I+4DU counts 4D byte passes of 16 B "
                               "rows; the packed path executes fewer, narrower passes"},
            "stage_ms": main["stage_ms"],
            "staged_ms_per_step": main["ms_staged"],
            "stage_note": "stage_ms and the roofline's launch_ms come from a second timed region of the same K "
                          "steps with a CUDA event between stages (events end the programmatic-dependent-launch "
                          "overlap at those boundaries: staged_ms_per_step)",
            "workloads": extra or None,
            "cpu_baseline": cpu,
            "clocks": clk.summary(),
            "gpu_launches": int(round(main["launches_per_step"] * args.steps)),
        }
        emit(line)
    if world > 1:
        torch.distributed.destroy_process_group()


DIST_TEXT = {
    "C2": "C2 per GPU: one shuffled float3 lattice soup of (5000 N) x 5000 quads (50M triangles per GPU), "
          "element ranges per rank (weak scaling)",
    "C5": "C5: the 1B-triangle float3 soup (20000 x 25000 quads, 3.15B vertex slots), element ranges per rank "
          "(strong scaling)",
    "C4": "C4: merge of 8 overlapping 50M-triangle meshes (welded 5000 x 5000 tiles, 500 shared rows), tiles "
          "dealt to the ranks in order (strong scaling)",
}


def dist_shard(cfg: str, rank: int, world: int, dev):
    """This rank's shard (vertex bits, elements with local indices) of a multi-GPU workload, generated on
    the device; returns (vtx, idx, total vertex slots of the job, expected global unique count)."""
    import torch

    from paper_2109_09812_b200 import _native, gen
    lib = _native.lib()
    if cfg == "C4":
        from oracle import lattice
        n, step, tiles = lattice.COLS_C4, lattice.ROW_STEP_C4, lattice.TILES_C4
        mine = [t for t in range(tiles) if t * world // tiles == rank]
        pieces = [gen.welded_tile_tensors(n, step * t, t, False, dev) for t in mine]
        vtx = torch.cat([p[0] for p in pieces])
        parts, off = [], 0
        for v, e in pieces:
            parts.append((e.to(torch.int64) + off).to(torch.int32))
            off += v.shape[0]
        idx = torch.cat(parts)
        sz = lattice.welded_sizes(n)
        return vtx, idx, sz["n_vertices"] * tiles, (step * (tiles - 1) + n + 1) * (n + 1)
    nx, ny = (5000 * world, 5000) if cfg == "C2" else (20000, 25000)
    D, K = 3, 3
    E_all, V_all = ctypes.c_uint64(), ctypes.c_uint64()
    lib.rmx_lattice_sizes(0, nx, ny, 0, 1 << 63, ctypes.byref(E_all), ctypes.byref(V_all))
    E_all, V_all = E_all.value, V_all.value
    e0, e1 = E_all * rank // world, E_all * (rank + 1) // world

    def slots(e):
        x, v = ctypes.c_uint64(), ctypes.c_uint64()
        lib.rmx_lattice_sizes(0, nx, ny, 0, e, ctypes.byref(x), ctypes.byref(v))
        return v.value

    V = slots(e1) - slots(e0)
    vtx = torch.empty((V, D), dtype=torch.int32, device=dev)
    idx = torch.empty((e1 - e0, K), dtype=torch.int32, device=dev)
    _native.check(lib.rmx_gen_lattice_soup_range(0, nx, ny, 0, 0, e0, e1, vtx.data_ptr(), idx.data_ptr(),
                                                 torch.cuda.current_stream(dev).cuda_stream))
    return vtx, idx, V_all, (nx + 1) * (ny + 1)


def run_b200_dist(args):
    """N > 1 (torchrun, NCCL): one mesh partitioned across the ranks, re-indexed by the sample-sort
    path (paper_2109_09812_b200.dist).  --config C2: weak scaling, (5000 N) x 5000 quads; C5: the
    1B-triangle soup, strong scaling; C4: the 8-tile merge, strong scaling.  A step is
    ``dist.reindex_distributed`` (local re-index, sample-sort exchange of the deduplicated keys over
    peer memory, merge, reverse exchange, remap); value = all ranks' input vertices / max-over-ranks
    device time."""
    import torch
    import torch.distributed as tdist

    from paper_2109_09812_b200 import _native, build, dist as rdist, pipeline

    rank, world, local = dist_env()
    if world == 1 and args.config == "C5":
        return run_c5_one_gpu(args)
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if not tdist.is_initialized():
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ.setdefault("MASTER_PORT", "29511")
        tdist.init_process_group("nccl", rank=rank, world_size=world, device_id=dev)
    if not os.path.exists(_native.LIB_PATH):
        build.build()
    lib = _native.lib()
    cfg = args.config if args.config in DIST_TEXT else "C2"
    vtx, idx, V_all, expect_u = dist_shard(cfg, rank, world, dev)
    V, D = vtx.shape
    E, K = idx.shape
    # data exchange over peer memory (symmetric buffers + rmx_scatter_rows); NCCL all-to-all only if
    # the symmetric-memory rendezvous is not available on this box
    try:
        comm = rdist.SymmComm(device=dev)
        comm._ensure(1 << 16)
        exchange = "peer-memory stores (rmx_scatter_rows into symmetric buffers over NVLink)"
    except Exception as exc:  # noqa: BLE001 - recorded in the JSON line
        comm = rdist.TorchComm(device=dev)
        exchange = f"NCCL all_to_all (symmetric memory unavailable: {type(exc).__name__}: {exc})"[:200]
    backend = rdist.CudaBackend(dev)

    def step(timing=None):
        return rdist.reindex_distributed(vtx, idx, comm, backend, timing=timing)

    for _ in range(max(3, args.warmup)):
        res = step()
    assert res.total == expect_u, (res.total, expect_u)
    u_local = int(res.vertices.shape[0])
    launches0 = lib.rmx_kernel_launches_total()
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    tdist.barrier()
    torch.cuda.synchronize(dev)
    with ClockSampler(local) as clk:
        t0.record()
        for _ in range(args.steps):
            step()
        t1.record()
        torch.cuda.synchronize(dev)
    ms = t0.elapsed_time(t1) / args.steps
    launches = (lib.rmx_kernel_launches_total() - launches0) / args.steps
    t = torch.tensor([ms], device=dev)
    tdist.all_reduce(t, op=tdist.ReduceOp.MAX)
    ms = float(t.item())
    value = V_all / (ms * 1e-3)
    # one instrumented step: per-phase CUDA-event times and the exchanged bytes (max over ranks)
    timing = {}
    step(timing)
    keys = sorted(k for k in timing if k.endswith("_ms"))
    tv = torch.tensor([timing[k] for k in keys] + [float(timing.get("exchange_bytes_out", 0)),
                                                   float(timing.get("exchange_bytes_in", 0))], device=dev)
    tdist.all_reduce(tv, op=tdist.ReduceOp.MAX)
    phases = {k: float(v) for k, v in zip(keys, tv[:len(keys)].tolist())}
    nv_out, nv_in = float(tv[-2]), float(tv[-1])
    xfer_ms = phases.get("exchange_ms", 0.0) + phases.get("reverse_ms", 0.0)
    nvlink = {"bytes_out_per_rank_max": nv_out, "bytes_in_per_rank_max": nv_in,
              "exchange_ms": xfer_ms, "peak_gbs_per_direction": 900.0,
              "achieved_gbs_per_direction": (max(nv_out, nv_in) / (xfer_ms * 1e-3) / 1e9) if xfer_ms else None,
              "note": "forward keys (4D B) + reverse global ids (4 B) of the local unique keys that cross to other "
                      "ranks; exchange_ms = forward + reverse exchange phases (CUDA events, barriers included)"}
    if nvlink["achieved_gbs_per_direction"]:
        nvlink["frac"] = nvlink["achieved_gbs_per_direction"] / 900.0

    # end to end: this rank's shard from pinned host memory, results back to pinned host memory
    host_v = torch.empty((V, D), dtype=torch.int32, pin_memory=True)
    host_e = torch.empty((E, K), dtype=torch.int32, pin_memory=True)
    host_v.copy_(vtx)
    host_e.copy_(idx)
    out_host_e = torch.empty((E, K), dtype=torch.int32, pin_memory=True)
    out_host_v = torch.empty((max(u_local, 1) * 2, D), dtype=torch.int32, pin_memory=True)
    e2e_steps = max(1, min(args.steps, 3))
    dv = torch.empty_like(vtx)
    de = torch.empty_like(idx)
    tdist.barrier()
    torch.cuda.synchronize(dev)
    tt = time.perf_counter()
    h2d = d2h = 0
    for _ in range(e2e_steps):
        dv.copy_(host_v, non_blocking=True)
        de.copy_(host_e, non_blocking=True)
        r_ = rdist.reindex_distributed(dv, de, comm, backend)
        out_host_e.copy_(r_.elements, non_blocking=True)
        u_r = r_.vertices.shape[0]
        out_host_v[:u_r].copy_(r_.vertices, non_blocking=True)
        torch.cuda.synchronize(dev)
        h2d = (V * D + E * K) * 4
        d2h = E * K * 4 + u_r * D * 4
    el = (time.perf_counter() - tt) / e2e_steps
    t = torch.tensor([el], device=dev)
    tdist.all_reduce(t, op=tdist.ReduceOp.MAX)
    el = float(t.item())
    e2e = {"value": V_all / el, "unit": "verts/s", "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
           "ms_per_step": el * 1e3, "steps": e2e_steps, "api": "paper_2109_09812_b200.dist.reindex_distributed",
           "note": "per rank (max over ranks): pinned shard H2D, distributed re-index, elements + vertex slice D2H"}
    del dv, de

    # roofline of the dominant kernel, from one profiled local re-index of this rank's shard
    n_ev = lib.rmx_stage_count(D)
    names = [lib.rmx_stage_name(D, k).decode() for k in range(n_ev)]
    evs = [torch.cuda.Event(enable_timing=True) for _ in range(n_ev)]
    for e_ in evs:
        e_.record()
    out_v = torch.empty((V, D), dtype=torch.int32, device=dev)
    out_e = torch.empty((E, K), dtype=torch.int32, device=dev)
    info = torch.zeros(2, dtype=torch.int64, device=dev)
    ws = torch.empty(pipeline.workspace_bytes(V, D, E, K), dtype=torch.uint8, device=dev)
    pipeline.launch(vtx, V, D, idx, E, K, out_v, out_e, info, ws, None, None, [e_.cuda_event for e_ in evs])
    torch.cuda.synchronize(dev)
    stage_ms = {names[k]: evs[k - 1].elapsed_time(evs[k]) for k in range(1, n_ev)}
    pinfo = (ctypes.c_uint32 * 4)()
    _native.check(lib.rmx_plan_info(ws.data_ptr(), V, D, torch.cuda.current_stream(dev).cuda_stream, pinfo))
    packed, key_words, vbits, executed = (int(x) for x in pinfo)
    pass_names = [n for n in names if n.startswith("pk_pass_" if packed == 1 else "sort_pass_")]
    active = sorted((stage_ms[n] for n in pass_names), reverse=True)[:executed]
    pass_ms = sum(active) / max(1, len(active))
    if packed == 1:
        per_pass = [8 * key_words + (0 if p == 0 else 4) + 4 + 1 + (1 if p + 1 < executed else 0)
                    for p in range(executed)]
        pass_bytes = sum(per_pass) / max(1, len(per_pass)) * V
    else:
        pass_bytes = 2 * (4 * D + 4) * V
    hbm, peak_kind = peaks()
    achieved = pass_bytes / (pass_ms * 1e-3) / 1e9
    del out_v, out_e, ws
    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "verts/s", "n_gpus": world, "steps": args.steps,
            "warmup": max(3, args.warmup), "ms_per_step": ms, "higher_is_better": True,
            "scaling": "weak" if cfg == "C2" else "strong",
            "vs_baseline": None, "dtype": "u32", "data": "synthetic",
            "config": {"workload": DIST_TEXT[cfg], "n_vertices": V_all, "unique": expect_u,
                       "parallelism": f"dp{world} sample sort", "exchange": exchange,
                       "l2": "inputs >= 2.5 GB per GPU > 126 MB L2, no flush needed"},
            "e2e": e2e,
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": hbm, "unit": "GB/s", "frac": achieved / hbm,
                         "traffic": None, "kernel": "one local LSD pass on the rank-0 shard (profiled call after "
                                                    "the timed loop)", "peak_kind": peak_kind,
                         "executed_passes": executed},
            "phases_ms": phases,
            "nvlink": nvlink,
            "clocks": clk.summary(),
            "gpu_launches": int(round(launches * args.steps)),
        }
        emit(line)
    tdist.barrier()
    tdist.destroy_process_group()


def run_c5_one_gpu(args):
    """C5 -- the 1B-triangle soup, 3.15B vertex slots -- on ONE GPU: the memory-lean mode
    (pipeline.reindex_tensors_lean, ~148 GB with inputs and outputs; the ordinary layout needs
    ~264 GB).  Lean mode overwrites the vertex buffer, so the soup is regenerated on the device before
    every step, outside the CUDA events that time the re-index itself."""
    import numpy as np
    import torch

    from oracle import lattice
    from paper_2109_09812_b200 import _native, build, pipeline

    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    if not os.path.exists(_native.LIB_PATH):
        build.build()
    lib = _native.lib()
    nx, ny = 20000, 25000
    E64, V64 = ctypes.c_uint64(), ctypes.c_uint64()
    lib.rmx_lattice_sizes(0, nx, ny, 0, 1 << 63, ctypes.byref(E64), ctypes.byref(V64))
    E, V = E64.value, V64.value
    expect_u = (nx + 1) * (ny + 1)
    vtx = torch.empty((V, 3), dtype=torch.int32, device=dev)
    idx = torch.empty((E, 3), dtype=torch.int32, device=dev)
    stream = torch.cuda.current_stream(dev)

    def regen():
        _native.check(lib.rmx_gen_lattice_soup(0, nx, ny, 0, 0, 1 << 63, vtx.data_ptr(), idx.data_ptr(),
                                               stream.cuda_stream))

    times = []
    with ClockSampler(0) as clk:
        for k in range(max(3, args.warmup) + args.steps):
            regen()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            res = pipeline.reindex_tensors_lean(vtx, idx)
            b.record(stream)
            torch.cuda.synchronize(dev)
            assert res.new_count == expect_u, (res.new_count, expect_u)
            if k >= max(3, args.warmup):
                times.append(a.elapsed_time(b))
            if k + 1 < max(3, args.warmup) + args.steps:
                del res
    ms = sum(times) / len(times)
    # verification: rows strictly increasing (spot), and exact closed-form ranks of sampled elements
    out_v, out_e = res.vertices, res.elements
    kind, cells = lattice.CONFIGS["C5"]
    t = lattice.permute(np.arange(4000, dtype=np.uint64), E, 0).astype(np.int64)
    ranks = lattice.point_rank(kind, cells, lattice.element_points(kind, cells, t))
    assert np.array_equal(out_e[:4000].cpu().numpy().view(np.uint32), ranks.astype(np.uint32))
    pts = np.stack([np.arange(0, expect_u, 1 << 16) // (ny + 1), np.arange(0, expect_u, 1 << 16) % (ny + 1)], -1)
    want = lattice.point_coords(kind, cells, pts).view(np.uint32)
    got = out_v[torch.arange(0, expect_u, 1 << 16, device=dev)].cpu().numpy().view(np.uint32)
    assert np.array_equal(got, want)
    hbm, _ = peaks()
    line = {
        "metric": METRIC, "value": V / (ms * 1e-3), "unit": "verts/s", "n_gpus": 1, "steps": args.steps,
        "warmup": max(3, args.warmup), "ms_per_step": ms, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "u32", "data": "synthetic",
        "config": {"workload": DIST_TEXT["C5"], "n_vertices": V, "n_elements": E, "unique": expect_u,
                   "parallelism": "single (memory-lean mode: the vertex buffer doubles as a sort buffer)",
                   "memory_gb": {"lean_workspace": lib.rmx_lean_workspace_bytes(V, 3, E, 3) / 1e9,
                                 "inputs": (V * 3 + E * 3) * 4 / 1e9, "out_elements": E * 12 / 1e9,
                                 "ordinary_workspace": lib.rmx_workspace_bytes(V, 3, E, 3) / 1e9},
                   "l2": L2_NOTE},
        "e2e": None,
        "e2e_note": "not measured: 50 GB of input per step would cross PCIe (~1 s)",
        "times_ms": times,
        "verified": "count = 500,045,001; exact closed-form ranks of 4000 elements; sampled output rows",
        "clocks": clk.summary(),
        "hbm_peak_gbs": hbm,
    }
    emit(line)


_JSON_OUT = None  # the real stdout: libraries (NCCL prints its version banner) get stderr instead


def emit(line: dict) -> None:
    """The one JSON line of this run, on the original stdout."""
    out = _JSON_OUT or sys.stdout
    out.write(json.dumps(line) + "\n")
    out.flush()


def main():
    global _JSON_OUT
    sys.stdout.flush()
    _JSON_OUT = os.fdopen(os.dup(1), "w")
    os.dup2(2, 1)  # anything else written to fd 1 (C libraries included) goes to stderr
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="C2", choices=sorted(set(CONFIGS) | {"C4", "C5"}))
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-extra", action="store_true", help="skip the C2s / C3 device-timed workloads")
    ap.add_argument("--dist", action="store_true", help="use the multi-GPU path even at N=1 (testing)")
    args = ap.parse_args()
    if args.impl == "reference":
        run_reference(args)
    elif dist_env()[1] > 1 or args.dist or args.config in ("C4", "C5"):
        run_b200_dist(args)
    else:
        run_b200(args)


if __name__ == "__main__":
    main()
