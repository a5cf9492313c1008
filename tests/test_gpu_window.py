"""GPU: window mode (rmx_window.cuh) against the oracle.

Packed u32 keys of 25..32 bits are sorted by their top 16 bits only (two LSD passes; the first
drops the unused rows) and every 2^16-key "window" is resolved by a shared-memory presence bitmap:
a key's new index is the number of distinct keys below it (reference pipeline.py:72-113).  These
cases engage the mode (rmx_window_info), cover windows staged in shared memory and windows streamed
from global memory, soup and indexed meshes with unused rows, 32-bit keys (the last window
non-empty), and the fallback to the full packed path when one window holds more than
kWinMaxRows rows.  Every case is checked against the oracle, and against RMX_WINDOW=0.
"""
import ctypes

import numpy as np
import pytest
import torch

from oracle import remesh_oracle as O

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def rmx(cuda_ok):
    import paper_2109_09812_b200 as p
    return p


def run(words, idx):
    """reindex through the tensor pipeline; returns (vertices, elements, window_info)."""
    from paper_2109_09812_b200 import _native, pipeline
    V, D = words.shape
    E, K = idx.shape
    dev = torch.device("cuda")
    vt = torch.from_numpy(np.ascontiguousarray(words).view(np.int32)).to(dev)
    it = torch.from_numpy(np.ascontiguousarray(idx).view(np.int32)).to(dev)
    ov, oe = torch.empty_like(vt), torch.empty_like(it)
    info = torch.zeros(2, dtype=torch.int64, device=dev)
    ws = torch.empty(pipeline.workspace_bytes(V, D, E, K), dtype=torch.uint8, device=dev)
    s = torch.cuda.current_stream()
    pipeline.launch(vt, V, D, it, E, K, ov, oe, info, ws, None, s)
    winfo = (ctypes.c_uint32 * 4)()
    _native.check(_native.lib().rmx_window_info(ws.data_ptr(), V, D, s.cuda_stream, winfo))
    torch.cuda.synchronize()
    assert int(info[1]) == 0
    u = int(info[0].item())
    return ov[:u].cpu().numpy().view(np.uint32), oe.cpu().numpy().view(np.uint32), [int(x) for x in winfo]


def check(words, idx, monkeypatch=None):
    ref = O.reindex(words, idx)
    v, e, winfo = run(words, idx)
    assert np.array_equal(v, ref["vertices"].view(np.uint32))
    assert np.array_equal(e, ref["elements"])
    if monkeypatch is not None:  # the same through the full packed path
        monkeypatch.setenv("RMX_WINDOW", "0")
        v0, e0, w0 = run(words, idx)
        monkeypatch.delenv("RMX_WINDOW")
        assert w0[0] == 0
        assert np.array_equal(v0, v) and np.array_equal(e0, e)
    return winfo


def test_indexed_mesh_with_unused_rows(rmx, monkeypatch):
    """28 random bits, random indices over 90 % of the rows: unused rows drop out of the first pass."""
    rng = np.random.default_rng(1)
    V = 300_000
    words = rng.integers(0, 1 << 28, size=(V, 1), dtype=np.uint64).astype(np.uint32)
    idx = rng.integers(0, 270_000, size=(200_000, 3)).astype(np.uint32)
    winfo = check(words, idx, monkeypatch)
    used = np.zeros(V, bool)
    used[idx.reshape(-1)] = True
    assert winfo[0] == 1 and winfo[1] == int(used.sum())


def test_soup_with_gaps(rmx, monkeypatch):
    """Strictly increasing indices (soup mode: index-position origins) with unused rows between."""
    rng = np.random.default_rng(2)
    V = 400_000
    words = rng.integers(0, 1 << 14, size=(V, 2), dtype=np.uint64).astype(np.uint32)
    keep = np.flatnonzero(rng.random(V) < 0.8)
    keep = keep[: (len(keep) // 3) * 3]
    idx = keep.astype(np.uint32).reshape(-1, 3)
    winfo = check(words, idx, monkeypatch)
    assert winfo[0] == 1 and winfo[1] == V  # soup mode keeps the unused rows (skipped by origin)


def test_soup_with_unused_tail(rmx, monkeypatch):
    """Soup with 30 % spare slots at the end (whole 4-row groups unused): their keys are spread by
    a hash, not set to the replacement key -- no giant window, no fallback."""
    rng = np.random.default_rng(7)
    V = 600_000
    words = rng.integers(0, 1 << 14, size=(V, 2), dtype=np.uint64).astype(np.uint32)
    idx = np.arange(420_000, dtype=np.uint32).reshape(-1, 3)
    winfo = check(words, idx, monkeypatch)
    assert winfo[0] == 1 and winfo[3] < 20_000


def test_full_32_bit_keys(rmx, monkeypatch):
    """All 32 bits vary: windows 0 and 65535 both hold rows; duplicates across the whole range."""
    rng = np.random.default_rng(3)
    pool = rng.integers(0, 1 << 32, size=60_000, dtype=np.uint64).astype(np.uint32)
    pool[:2] = [0, 0xFFFFFFFF]
    V = 250_000
    words = pool[rng.integers(0, pool.size, size=V)].reshape(-1, 1)
    idx = rng.integers(0, V, size=(120_000, 2)).astype(np.uint32)
    idx[0] = [np.flatnonzero(words[:, 0] == 0)[0], np.flatnonzero(words[:, 0] == 0xFFFFFFFF)[0]]
    winfo = check(words, idx, monkeypatch)
    assert winfo[0] == 1


def test_streamed_windows(rmx, monkeypatch):
    """25 varying bits whose top nine take 16 patterns in nearly every row: windows of ~15K rows
    (more than kWinCap) stream from global memory."""
    rng = np.random.default_rng(4)
    V = 240_000
    hi = rng.integers(0, 16, size=V).astype(np.uint32) << np.uint32(20)
    words = (hi | rng.integers(0, 1 << 16, size=V).astype(np.uint32)).reshape(-1, 1)
    words[:7, 0] |= np.uint32(0x010F0000)  # bits 16..19 and 24 vary in a few rows (B = 25)
    idx = rng.integers(0, V, size=(100_000, 3)).astype(np.uint32)
    winfo = check(words, idx, monkeypatch)
    assert winfo[0] == 1 and winfo[3] > 6144


def test_one_huge_window_falls_back(rmx, monkeypatch):
    """One window of more than kWinMaxRows rows would serialise on one CTA: the full packed path
    runs after the first two passes (window-grouped rows, digit 0 re-extracted)."""
    rng = np.random.default_rng(5)
    V = 2_400_000
    words = (np.uint32(0x0AB0000) | rng.integers(0, 1 << 16, size=V).astype(np.uint32)).reshape(-1, 1)
    spread = rng.integers(0, V, size=50_000)
    words[spread, 0] = rng.integers(0, 1 << 28, size=spread.size).astype(np.uint32)
    idx = rng.permutation(V).astype(np.uint32).reshape(-1, 3)  # every row used
    winfo = check(words, idx)
    assert winfo[0] == 3  # window mode decided, its fallback ran


def test_scratch_request_keeps_the_full_path(rmx):
    """Scratch arrays (org_id, nodup, new_idx, perm) come from the sorted rows: no window mode."""
    rng = np.random.default_rng(6)
    words = rng.integers(0, 1 << 28, size=(50_000, 1), dtype=np.uint64).astype(np.uint32)
    idx = rng.integers(0, 50_000, size=(40_000, 3)).astype(np.uint32)
    ref = O.reindex(words, idx)
    out, sc = rmx.reindex(rmx.Mesh(words.view(np.float32), idx))
    assert np.array_equal(out.elements, ref["elements"])
    for f in ("org_id", "nodup", "new_idx", "perm"):
        assert np.array_equal(np.asarray(getattr(sc, f)), ref[f]), f


def test_four_components_keep_the_full_path(rmx):
    """Window mode is used for D <= 3 (C3's D = 4 tets measured faster without it)."""
    rng = np.random.default_rng(8)
    words = rng.integers(0, 1 << 7, size=(200_000, 4), dtype=np.uint64).astype(np.uint32)
    idx = rng.integers(0, 200_000, size=(100_000, 4)).astype(np.uint32)
    assert check(words, idx)[0] == 0


def test_full_window(rmx, monkeypatch):
    """One window holds all 2^16 low values (the distinct count fills its 17-bit field) next to
    windows holding one key each."""
    rng = np.random.default_rng(9)
    full = (np.uint32(0x0123) << np.uint32(16)) | np.arange(1 << 16, dtype=np.uint32)
    other = rng.integers(0, 1 << 28, size=40_000, dtype=np.uint64).astype(np.uint32)
    words = np.concatenate([full, full[::-1], other]).reshape(-1, 1)
    perm = rng.permutation(words.shape[0])
    words = words[perm]
    idx = rng.integers(0, words.shape[0], size=(90_000, 2)).astype(np.uint32)
    idx[: words.shape[0] // 2] = np.arange(words.shape[0], dtype=np.uint32)[: (words.shape[0] // 2) * 2].reshape(-1, 2)
    winfo = check(words, idx, monkeypatch)
    assert winfo[0] == 1


def test_lean_mode(rmx, monkeypatch):
    """Memory-lean mode (the vertex buffer is the second sort buffer) with window mode: 30-bit keys,
    unused rows dropped by the first window pass, pairs written into the caller's vertex buffer."""
    from paper_2109_09812_b200 import pipeline
    rng = np.random.default_rng(10)
    V = 300_000
    words = (rng.integers(0, 1 << 10, size=(V, 3), dtype=np.uint64) << np.uint64(8)).astype(np.uint32)
    idx = rng.integers(0, 280_000, size=(150_000, 3)).astype(np.uint32)
    ref = O.reindex(words, idx)
    for win in ("1", "0"):
        monkeypatch.setenv("RMX_WINDOW", win)
        vt = torch.from_numpy(words.view(np.int32)).cuda()
        it = torch.from_numpy(idx.view(np.int32)).cuda()
        r = pipeline.reindex_tensors_lean(vt, it)
        assert np.array_equal(r.vertices[:r.new_count].cpu().numpy().view(np.uint32), ref["vertices"].view(np.uint32))
        assert np.array_equal(r.elements.cpu().numpy().view(np.uint32), ref["elements"])


def test_soup_huge_window_falls_back(rmx, monkeypatch):
    """Soup mode (unused rows kept with spread keys) and one window of more than kWinMaxRows rows:
    the fallback's full passes must not count the unused rows' spread keys as distinct keys."""
    rng = np.random.default_rng(11)
    V = 2_700_000
    words = (np.uint32(0x0AB0000) | rng.integers(0, 1 << 16, size=V).astype(np.uint32)).reshape(-1, 1)
    spread = rng.integers(0, V, size=50_000)
    words[spread, 0] = rng.integers(0, 1 << 28, size=spread.size).astype(np.uint32)
    keep = np.ones(V, bool)
    keep[100_000:160_000] = False            # whole 4-row groups unused (hash-spread keys)
    keep[rng.integers(0, V, size=20_000)] = False
    keep = np.flatnonzero(keep)
    keep = keep[: (keep.size // 3) * 3]
    idx = keep.astype(np.uint32).reshape(-1, 3)
    winfo = check(words, idx, monkeypatch)
    assert winfo[0] == 3  # window mode decided, its fallback ran


def test_dropped_rows_huge_window_falls_back(rmx, monkeypatch):
    """Indexed mesh (the first window pass drops the unused rows) with one window of more than
    kWinMaxRows used rows: the fallback's full passes run over the kept rows only."""
    rng = np.random.default_rng(12)
    V = 3_000_000
    words = (np.uint32(0x0AB0000) | rng.integers(0, 1 << 16, size=V).astype(np.uint32)).reshape(-1, 1)
    spread = rng.integers(0, V, size=50_000)
    words[spread, 0] = rng.integers(0, 1 << 28, size=spread.size).astype(np.uint32)
    idx = rng.permutation(V)[: 2_700_000].astype(np.uint32).reshape(-1, 3)  # 10 % unused
    winfo = check(words, idx, monkeypatch)
    assert winfo[0] == 3 and winfo[1] == 2_700_000
