"""GPU: soup mode (rmx_packed.cuh k_soup_decide) against the oracle.

Strictly increasing indices -- triangle soups and their shards: every used row referenced once, in
row order -- with a packed plan give each used vertex slot the origin "used slots before it",
which is its index position: the map fill then writes the output indices directly (no map, no
remap; unused slots get origins >= I and are skipped).  k_mark decides "strictly increasing" on
the device, including across its 4-index groups, the warp's last lane and the scalar tail; these
tests put single violations at those places.  Every case is checked against the oracle, with
rmx_soup_info telling whether the mode engaged.
"""
import ctypes

import numpy as np
import pytest
import torch

from oracle import lattice as LAT
from oracle import remesh_oracle as O

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def rmx(cuda_ok):
    import paper_2109_09812_b200 as p
    return p


def run(rmx, words, idx):
    """reindex through the tensor pipeline; returns (vertices, elements, soup_info)."""
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
    sinfo = (ctypes.c_uint32 * 2)()
    _native.check(_native.lib().rmx_soup_info(ws.data_ptr(), V, D, s.cuda_stream, sinfo))
    torch.cuda.synchronize()
    u = int(info[0].item())
    return ov[:u].cpu().numpy().view(np.uint32), oe.cpu().numpy().view(np.uint32), [int(x) for x in sinfo]


def check(rmx, words, idx):
    ref = O.reindex(words, idx)
    v, e, sinfo = run(rmx, words, idx)
    assert np.array_equal(v, ref["vertices"].view(np.uint32))
    assert np.array_equal(e, ref["elements"])
    return sinfo


def lattice(cells, seed=0):
    w, i = LAT.lattice_soup("tri", cells, seed=seed)
    return w.view(np.uint32).reshape(-1, 3), i.astype(np.uint32).reshape(-1, 3)


def test_lattice_soup_engages(rmx, monkeypatch):
    words, idx = lattice((120, 90))
    sinfo = check(rmx, words, idx)
    assert sinfo == [idx.size, 1]
    monkeypatch.setenv("RMX_SOUP", "0")
    assert check(rmx, words, idx) == [0, 1]


def test_indexed_mesh_does_not_engage(rmx):
    rng = np.random.default_rng(3)
    words = rng.integers(0, 1 << 12, size=(50_000, 3)).astype(np.uint32) << np.uint32(8)
    idx = rng.integers(0, 50_000, size=(60_000, 3)).astype(np.uint32)
    assert check(rmx, words, idx) == [0, 0]


@pytest.mark.parametrize("D", [1, 2, 3, 4, 5])
def test_sorted_subset_with_gaps(rmx, D):
    """Strictly increasing with gaps (unused rows hold other values): the unused rows drop out."""
    rng = np.random.default_rng(10 + D)
    V = 40_000
    words = (rng.integers(0, 64, size=(V, D)).astype(np.uint32) << np.uint32(11)) | np.uint32(0x3F800000)
    keep = np.sort(rng.choice(V, size=3 * 9_001, replace=False)).astype(np.uint32)
    words[np.setdiff1d(np.arange(V), keep)] = np.uint32(0x7F7FFFFF)  # unused rows: values no used row has
    sinfo = check(rmx, words, keep.reshape(-1, 3))
    assert sinfo == [keep.size, 1]  # (<= 64 varying bits: a packed plan)


def _violate(idx, p, how):
    f = idx.reshape(-1).copy()
    if how == "equal":
        f[p + 1] = f[p]
    else:  # swap: f[p] > f[p + 1]
        f[p], f[p + 1] = f[p + 1], f[p]
    return f.reshape(idx.shape)


# positions of idx[p] vs idx[p + 1]: inside a 4-index group, between groups of neighbouring
# lanes, across the warp's last lane (group 31 -> 32), into the scalar tail, the very end
POSITIONS = [1, 3, 4 * 31 + 3, None, -2]


@pytest.mark.parametrize("pos", POSITIONS, ids=["in_group", "lane_to_lane", "warp_edge", "into_tail", "last"])
@pytest.mark.parametrize("how", ["equal", "swap"])
def test_single_violation_is_seen(rmx, pos, how):
    words, idx = lattice((60, 50), seed=1)
    n = idx.size
    if n % 4 == 0:  # a scalar tail needs I % 4 != 0
        idx = idx[:-1]
        n = idx.size
    p = {None: (n // 4) * 4 - 1, -2: n - 2}.get(pos, pos)
    bad = _violate(idx, p, how)
    sinfo = check(rmx, words, bad)
    assert sinfo == [0, 0]
    assert check(rmx, words, idx) == [n, 1]


def test_two_indices_past_the_small_path(rmx):
    """V above the one-CTA path, I = 2: no 4-index group at all, the scalar loop decides."""
    rng = np.random.default_rng(5)
    words = rng.integers(0, 1 << 10, size=(10_000, 2)).astype(np.uint32) << np.uint32(3)
    assert check(rmx, words, np.array([[17, 9_000]], np.uint32)) == [2, 1]
    assert check(rmx, words, np.array([[9_000, 17]], np.uint32)) == [0, 0]


def hash_info(V, D, ws_ptr, stream):
    from paper_2109_09812_b200 import _native
    hi = (ctypes.c_uint32 * 4)()
    _native.check(_native.lib().rmx_hash_info(ws_ptr, V, D, stream, hi))
    return [int(x) for x in hi]


@pytest.mark.parametrize("violate", [False, True])
def test_hash_mode_soup(rmx, violate):
    """Real-valued (scrambled) coordinates: hash mode, whose raw first hashed pass makes the soup
    origins (used masks per 32 rows folded into its digit loop and scan)."""
    words, idx = lattice((90, 70), seed=3)
    words = LAT.scramble_words(words, 16).reshape(words.shape)  # > 64 varying bits: hash mode
    if violate:
        idx = _violate(idx, 4 * 31 + 3, "swap")
    ref = O.reindex(words, idx)
    from paper_2109_09812_b200 import _native, pipeline
    V, D = words.shape
    E, K = idx.shape
    dev = torch.device("cuda")
    vt = torch.from_numpy(words.view(np.int32)).to(dev)
    it = torch.from_numpy(idx.view(np.int32)).to(dev)
    ov, oe = torch.empty_like(vt), torch.empty_like(it)
    info = torch.zeros(2, dtype=torch.int64, device=dev)
    ws = torch.empty(pipeline.workspace_bytes(V, D, E, K), dtype=torch.uint8, device=dev)
    s = torch.cuda.current_stream()
    pipeline.launch(vt, V, D, it, E, K, ov, oe, info, ws, None, s)
    sinfo = (ctypes.c_uint32 * 2)()
    _native.check(_native.lib().rmx_soup_info(ws.data_ptr(), V, D, s.cuda_stream, sinfo))
    assert hash_info(V, D, ws.data_ptr(), s.cuda_stream)[0] == 1
    assert [int(x) for x in sinfo] == ([0, 0] if violate else [idx.size, 1])
    u = int(info[0].item())
    assert np.array_equal(ov[:u].cpu().numpy().view(np.uint32), ref["vertices"].view(np.uint32))
    assert np.array_equal(oe.cpu().numpy().view(np.uint32), ref["elements"])
