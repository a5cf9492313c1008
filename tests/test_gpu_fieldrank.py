"""GPU: packed keys with field ranks (rmx_base.cuh) against the oracle.

Each component draws its sign+exponent field from a small set (both signs,
binades far apart -- outside the 32-exponent window K1a keeps in registers --
zero, denormals, inf/NaN fields) and a few mantissa bits, so the plan must
rank the fields; rmx_plan_info confirms packed mode with fewer key bits than
the raw varying bits.  Results are bit-exact against the oracle incl. scratch.
"""
import ctypes

import numpy as np
import pytest
import torch

from conftest import FIELDS
from oracle import remesh_oracle as O

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def rmx(cuda_ok):
    import paper_2109_09812_b200 as p
    return p


def field_mesh(seed, V, D, E, K, fields, mant_bits):
    rng = np.random.default_rng(seed)
    f = np.asarray(fields, np.uint32)
    fld = f[rng.integers(0, len(f), size=(V, D))]
    mant = rng.integers(0, 1 << mant_bits, size=(V, D)).astype(np.uint32) << np.uint32(23 - mant_bits)
    words = (fld << np.uint32(23)) | mant
    idx = rng.integers(0, max(1, V - V // 8), size=(E, K)).astype(np.uint32)
    return words, idx


def raw_varying_bits(words, idx):
    used = np.zeros(words.shape[0], bool)
    used[idx.reshape(-1)] = True
    ref = words[idx[0, 0]]
    x = np.bitwise_or.reduce(words[used] ^ ref, axis=0)
    return int(sum(bin(int(v)).count("1") for v in x))


def plan_info(rmx, words, idx, guess=None):
    """rmx_plan_info of a fresh call; with ``guess`` (a list) also rmx_plan_guess_info into it."""
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
    pinfo = (ctypes.c_uint32 * 4)()
    _native.check(_native.lib().rmx_plan_info(ws.data_ptr(), V, D, s.cuda_stream, pinfo))
    if guess is not None:
        g = (ctypes.c_uint32 * 4)()
        _native.check(_native.lib().rmx_plan_guess_info(ws.data_ptr(), V, D, s.cuda_stream, g))
        guess[:] = [int(x) for x in g]
    return [int(x) for x in pinfo]


CASES = [
    # seed, V, D, E, K, fields, mantissa bits
    (1, 200_000, 3, 80_000, 3, [0x7F, 0x80, 0x17F, 0x180, 0x20, 0xE0, 0x120, 0x1E0], 12),
    (2, 150_000, 2, 60_000, 4, [0x00, 0x100, 0x01, 0xFF, 0x1FF], 20),          # zero/denormal/inf/NaN fields
    (3, 300_000, 4, 90_000, 4, [0x7E, 0x7F, 0x80, 0x81, 0x82], 9),
    (4, 100_000, 1, 50_000, 2, list(range(0x60, 0xA0, 4)) + [0x180], 18),
    (5, 120_000, 2, 50_000, 3, [0x83], 22),                                     # one field: no rank bits
    (6, 90_000, 4, 40_000, 3, [0x10, 0x40, 0x70, 0xA0, 0xD0, 0x110, 0x140, 0x170, 0x1A0, 0x1D0], 10),
]


@pytest.mark.parametrize("seed,V,D,E,K,fields,mb", CASES, ids=[f"case{c[0]}" for c in CASES])
def test_field_rank_parity(rmx, seed, V, D, E, K, fields, mb):
    words, idx = field_mesh(seed, V, D, E, K, fields, mb)
    ref = O.reindex(words, idx)
    out, sc = rmx.reindex(rmx.Mesh(words.view(np.float32), idx))
    assert np.array_equal(out.vertices.view(np.uint32), ref["vertices"].view(np.uint32))
    assert np.array_equal(out.elements, ref["elements"])
    for f in FIELDS:
        assert np.array_equal(np.asarray(getattr(sc, f)), ref[f]), f
    packed, kw, bits, _ = plan_info(rmx, words, idx)
    assert packed == 1
    raw = raw_varying_bits(words, idx)
    if len(fields) > 1 and D <= 4:
        assert bits < raw, (bits, raw)
    else:
        assert bits == raw


def test_field_rank_with_unused_rows_outside_the_set(rmx):
    """Unused rows carry fields that never occur in used rows: they are replaced before ranking."""
    words, idx = field_mesh(11, 50_000, 3, 20_000, 3, [0x7F, 0x80, 0x81], 8)
    used = np.zeros(words.shape[0], bool)
    used[idx.reshape(-1)] = True
    words[~used] = np.uint32(0xFF7FFFFF)                 # -max float: a field no used row has
    ref = O.reindex(words, idx)
    out, _ = rmx.reindex(rmx.Mesh(words.view(np.float32), idx))
    assert np.array_equal(out.vertices.view(np.uint32), ref["vertices"].view(np.uint32))
    assert np.array_equal(out.elements, ref["elements"])


def _masked_mesh(seed, V, D, E, K, masks):
    """Vertex words whose varying bits are exactly `masks[c]` (per component) around a base row."""
    rng = np.random.default_rng(seed)
    base = rng.integers(0, 1 << 32, size=D, dtype=np.uint64).astype(np.uint32)
    noise = rng.integers(0, 1 << 32, size=(V, D), dtype=np.uint64).astype(np.uint32)
    words = (base & ~np.array(masks, np.uint32)) | (noise & np.array(masks, np.uint32))
    words[: V // 3] = words[V // 3: 2 * (V // 3)]            # duplicates
    idx = rng.integers(0, V - V // 10, size=(E, K)).astype(np.uint32)
    return words, idx


@pytest.mark.parametrize("D,masks", [
    (2, [0x55555555, 0x55555555]),                      # 32 one-bit runs, u32 key
    (4, [0x55550000, 0x00005555, 0x0000AAAA, 0xAAAA0000]),  # 32 runs, u32 key
    (4, [0x55555555, 0xAAAAAAAA, 0x00000001, 0x00000000]),  # 65 bits: AoS rows
    (3, [0x0F0F0F0F, 0xF0F0F0F0, 0x00FF00FF]),          # 64 bits in 12 runs, u64 key
    (2, [0xFFFFFFFF, 0xFFFFFFFF]),                      # exactly 64 bits
    (4, [0x5555AAAA, 0x5555AAAA, 0x00000003, 0x0]), ])  # 34 runs
def test_many_runs_and_width_edges(rmx, D, masks):
    V, E, K = 60_000, 25_000, 3
    words, idx = _masked_mesh(D * 13 + len(masks), V, D, E, K, masks)
    ref = O.reindex(words, idx)
    out, sc = rmx.reindex(rmx.Mesh(words.view(np.float32), idx))
    assert np.array_equal(out.vertices.view(np.uint32), ref["vertices"].view(np.uint32))
    assert np.array_equal(out.elements, ref["elements"])
    for f in FIELDS:
        assert np.array_equal(np.asarray(getattr(sc, f)), ref[f]), f
