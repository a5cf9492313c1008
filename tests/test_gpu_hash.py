"""GPU: hash mode (rmx_hash.cuh) -- keys wider than 64 bits deduplicated by a 32-bit hash, then
only the distinct rows sorted exactly -- against the oracle, including forced hash collisions.

Exactness must not depend on the hash: two different keys with the same 32-bit hash interleave
in the hash-sorted order; the candidate groups split there and the exact sort of the candidates
gives both keys their right ranks.  The collisions are found by a birthday search with a numpy
mirror of the device hash (``hash_key`` below must equal rmx_hash.cuh's).
"""
import numpy as np
import pytest

from conftest import FIELDS
from oracle import remesh_oracle as O

pytestmark = pytest.mark.gpu
M32 = np.uint64(0xFFFFFFFF)


def hash_key(words: np.ndarray) -> np.ndarray:
    """Mirror of rmx_hashfn.cuh:hash_key over rows of uint32 words."""
    w = words.astype(np.uint64)
    h = np.full(w.shape[0], 0x9747B28C, np.uint64)
    for c in range(w.shape[1]):
        h = ((h ^ w[:, c]) * np.uint64(0x9E3779B1)) & M32
    h ^= h >> np.uint64(15)
    h = (h * np.uint64(0x85EBCA77)) & M32
    h ^= h >> np.uint64(13)
    return h.astype(np.uint32)


def colliding_pairs(rng, D, want=3):
    """`want` pairs of distinct D-word keys with equal hashes (birthday search)."""
    out = []
    while len(out) < want:
        keys = rng.integers(0, 2**32, size=(1 << 18, D), dtype=np.uint64).astype(np.uint32)
        h = hash_key(keys)
        order = np.argsort(h, kind="stable")
        hs = h[order]
        dup = np.flatnonzero(hs[1:] == hs[:-1])
        for i in dup:
            a, b = keys[order[i]], keys[order[i + 1]]
            if not np.array_equal(a, b):
                out.append((a, b))
    return out[:want]


@pytest.fixture(scope="module")
def rmx(cuda_ok):
    import paper_2109_09812_b200 as p
    return p


@pytest.fixture(autouse=True)
def large_path(monkeypatch):
    monkeypatch.setenv("RMX_SMALL", "0")
    monkeypatch.delenv("RMX_HASH", raising=False)


def plan_mode(rmx, words, idx):
    from test_gpu_fieldrank import plan_info
    return plan_info(rmx, words, idx)


def check(rmx, words, idx):
    ref = O.reindex(words, idx)
    out, sc = rmx.reindex(rmx.Mesh(words.view(np.float32), idx))
    assert np.array_equal(out.vertices.view(np.uint32), ref["vertices"].view(np.uint32))
    assert np.array_equal(out.elements, ref["elements"])
    for f in FIELDS:   # scratch: the AoS path of the lazily re-run call
        assert np.array_equal(np.asarray(getattr(sc, f)), ref[f]), f


def test_mirror_hash_is_the_device_hash(rmx):
    """Rows built to collide under the numpy mirror really share a hash run on the device: a mesh of
    two colliding keys only, interleaved, must come out as exactly two vertices."""
    rng = np.random.default_rng(1)
    (a, b), = colliding_pairs(rng, 3, 1)
    assert hash_key(a[None])[0] == hash_key(b[None])[0]
    V = 20_000
    words = np.where((np.arange(V) % 2 == 0)[:, None], a, b).astype(np.uint32)
    words[::97] = rng.integers(0, 2**32, size=(len(words[::97]), 3), dtype=np.uint64).astype(np.uint32)
    idx = np.arange(V, dtype=np.uint32).reshape(-1, 4)
    check(rmx, words, idx)
    assert plan_mode(rmx, words, idx)[0] == 2   # > 64 varying bits, no scratch: hash mode
    out, _ = rmx.reindex(rmx.Mesh(words.view(np.float32), idx))
    assert out.n_vertices == len(np.unique(words, axis=0))


@pytest.mark.parametrize("D", [3, 4, 5, 8])
def test_collisions_interleaved_with_random_rows(rmx, D):
    rng = np.random.default_rng(10 + D)
    pairs = colliding_pairs(rng, D, 3)
    V = 60_000
    words = rng.integers(0, 2**32, size=(V, D), dtype=np.uint64).astype(np.uint32)
    # every colliding key many times, interleaved at random positions (runs of one hash, two keys)
    for a, b in pairs:
        pos = rng.choice(V, size=400, replace=False)
        words[pos[:200]] = a
        words[pos[200:]] = b
    # ordinary duplicates too
    dup = rng.integers(0, V, size=(8000, 2))
    words[dup[:, 0]] = words[dup[:, 1]]
    idx = rng.integers(0, V, size=(V // 3, 3)).astype(np.uint32)
    check(rmx, words, idx)
    assert plan_mode(rmx, words, idx)[0] == 2


def test_collision_with_the_replacement_row(rmx):
    """A used row whose hash equals the replacement row's (unused rows hash as the replacement):
    the unused check must read its flag and keep its own key."""
    rng = np.random.default_rng(3)
    (a, b), = colliding_pairs(rng, 3, 1)
    V = 40_000
    words = rng.integers(0, 2**32, size=(V, 3), dtype=np.uint64).astype(np.uint32)
    words[0] = a                                  # the replacement row (idx[0, 0] = 0)
    words[rng.choice(np.arange(1, V), 300, replace=False)] = b
    idx = rng.integers(0, V, size=(V // 4, 3)).astype(np.uint32)
    idx[0, 0] = 0
    check(rmx, words, idx)


def test_tile_boundaries_and_long_runs(rmx):
    """Runs of one key across many hash tiles (2048 rows), keys that differ only in the last word,
    every row used or the replacement's duplicates spread."""
    rng = np.random.default_rng(4)
    V = 50_000
    base = rng.integers(0, 2**32, size=(40, 3), dtype=np.uint64).astype(np.uint32)
    words = base[rng.integers(0, 40, size=V)]
    words[:, 2] ^= rng.integers(0, 2, size=V).astype(np.uint32)   # pairs differing in one bit
    words[: V // 2] = base[0]                                      # one key on ~25K rows
    idx = np.arange(V, dtype=np.uint32).reshape(-1, 5)
    check(rmx, words, idx)


def test_hash_off_matches(rmx, monkeypatch):
    rng = np.random.default_rng(5)
    V = 30_000
    words = rng.integers(0, 2**32, size=(V, 4), dtype=np.uint64).astype(np.uint32)
    words[rng.integers(0, V, 9000)] = words[rng.integers(0, V, 9000)]
    idx = rng.integers(0, V, size=(V // 3, 3)).astype(np.uint32)
    assert plan_mode(rmx, words, idx)[0] == 2
    monkeypatch.setenv("RMX_HASH", "0")
    check(rmx, words, idx)
    assert plan_mode(rmx, words, idx)[0] == 0


def test_constant_last_component(rmx):
    """The last component is constant: the candidates' first executed AoS pass is pass 4, whose
    histogram k_first_hist builds from the candidate buffer."""
    rng = np.random.default_rng(6)
    V = 40_000
    words = rng.integers(0, 2**32, size=(V, 4), dtype=np.uint64).astype(np.uint32)
    words[:, 3] = np.uint32(0x3F800000)
    words[rng.integers(0, V, 12000)] = words[rng.integers(0, V, 12000)]
    idx = rng.integers(0, V, size=(V // 3, 3)).astype(np.uint32)
    check(rmx, words, idx)
    assert plan_mode(rmx, words, idx)[0] == 2
