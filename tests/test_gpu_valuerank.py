"""GPU: packed keys with value ranks (rmx_base.cuh) against the oracle.

Each component takes its values from a small set of words whose varying
bits span 4..17 bits, so a component's packed value cv can be replaced by
its rank among the occurring values.  Results must be bit-exact against the
oracle (incl. scratch) with value ranks on and off (RMX_VALUE_RANK=0), and
rmx_plan_info must report the key width a Python model of the plan predicts.
Meshes of >= 2^22 rows take the sampled decision first (the first 256 rows of
every 16384); one of them is built so that the sample promises a gain the
full set does not deliver -- the plan must fall back to the plain packed key.
"""

import numpy as np
import pytest

from conftest import FIELDS
from oracle import remesh_oracle as O
from test_gpu_fieldrank import plan_info

pytestmark = pytest.mark.gpu

BASE = np.uint32(0x3F800000)  # 1.0f: sign and exponent field constant, no field rank


@pytest.fixture(scope="module")
def rmx(cuda_ok):
    import paper_2109_09812_b200 as p
    return p


@pytest.fixture(autouse=True)
def value_rank_default(monkeypatch):
    """Width assertions need value ranks on, whatever the suite runs under, and on the small
    meshes of these tests (by default only meshes of >= 2^25 rows use them)."""
    monkeypatch.delenv("RMX_VALUE_RANK", raising=False)
    monkeypatch.setenv("RMX_VALUE_RANK_MIN", "0")


@pytest.fixture
def value_rank_off(monkeypatch):
    monkeypatch.setenv("RMX_VALUE_RANK", "0")


def value_set(rng, m, b):
    """m distinct values in [0, 2^b) including 0 and 2^b - 1 (so all b bits vary)."""
    if m <= 2:
        return np.array([0, (1 << b) - 1][:m], np.uint32)
    mid = rng.choice(np.arange(1, (1 << b) - 1, dtype=np.uint32), size=m - 2, replace=False)
    return np.concatenate([[0, (1 << b) - 1], mid]).astype(np.uint32)


def set_mesh(seed, V, E, K, comps):
    """comps: per component (m distinct values, b varying bits, mantissa shift)."""
    rng = np.random.default_rng(seed)
    D = len(comps)
    words = np.empty((V, D), np.uint32)
    for c, (m, b, sh) in enumerate(comps):
        vals = value_set(rng, m, b)
        words[:, c] = BASE | (vals[rng.integers(0, len(vals), size=V)] << np.uint32(sh))
    idx = rng.integers(0, V, size=(E, K)).astype(np.uint32)
    idx[0, 0] = 0
    return words, idx


def bits_for(n):
    return 0 if n <= 1 else int(n - 1).bit_length()


def model_bits(words, idx):
    """(plain packed bits, bits with value ranks) of the plan for `set_mesh` data (< 2^22 rows)."""
    used = np.zeros(words.shape[0], bool)
    used[idx.reshape(-1)] = True
    u = words[used]
    ref = words[idx[0, 0]]
    w = [bin(int(np.bitwise_or.reduce(u[:, c] ^ ref[c]))).count("1") for c in range(words.shape[1])]
    m = [len(np.unique(u[:, c])) for c in range(words.shape[1])]
    bits = sum(w)
    npass, kw = (bits + 7) // 8, 2 if bits > 32 else 1
    if words.shape[1] > 4:
        return bits, bits
    cand = [4 <= wc <= 16 for wc in w]
    while sum(1 << wc for cd, wc in zip(cand, w) if cd) > 192 * 1024:   # byte maps of one CTA
        widest = max((wc, -c) for c, (cd, wc) in enumerate(zip(cand, w)) if cd)
        cand[-widest[1]] = False

    def gain(nb):
        return (nb + 7) // 8 < npass or (kw == 2 and nb <= 32)

    if not any(cand) or not gain(sum(0 if cd else wc for cd, wc in zip(cand, w))):
        return bits, bits
    ranked = [cd and bits_for(mc) < wc for cd, wc, mc in zip(cand, w, m)]
    nb = sum(bits_for(mc) if r else wc for r, wc, mc in zip(ranked, w, m))
    return bits, (nb if gain(nb) else bits)


def check(rmx, words, idx):
    ref = O.reindex(words, idx)
    out, sc = rmx.reindex(rmx.Mesh(words.view(np.float32), idx))
    assert np.array_equal(out.vertices.view(np.uint32), ref["vertices"].view(np.uint32))
    assert np.array_equal(out.elements, ref["elements"])
    for f in FIELDS:
        assert np.array_equal(np.asarray(getattr(sc, f)), ref[f]), f


CASES = [
    # seed, V, E, K, [(m, b, shift) per component]
    (1, 200_000, 90_000, 3, [(5001, 16, 7), (5001, 16, 7), (64, 8, 15)]),   # C2-like: 40 -> 32 bits
    (2, 150_000, 60_000, 4, [(151, 12, 11), (151, 12, 11), (149, 12, 3), (97, 10, 0)]),  # C3-like
    (3, 120_000, 50_000, 3, [(3, 16, 0), (2, 16, 7), (17, 16, 4)]),         # few values, wide spans
    (4, 100_000, 40_000, 2, [(300, 17, 6), (300, 14, 0)]),                  # 17 bits: not a candidate
    (5, 100_000, 40_000, 1, [(9, 4, 19)]),                                  # 4 bits, too few to gain
    (6, 100_000, 40_000, 1, [(1000, 16, 0)]),                               # 16 -> 10 bits, 2 -> 2 passes
    (7, 100_000, 40_000, 4, [(16, 16, 0), (16, 16, 0), (16, 16, 0), (16, 16, 0)]),  # 64 -> 28 bits (3 maps fit)
    (8, 100_000, 40_000, 2, [(40_000, 16, 7), (2, 5, 0)]),                  # ~30K used values: 21 -> 16 bits
    (9, 30_000, 10_000, 6, [(7, 9, 0), (7, 9, 0), (7, 9, 0), (7, 9, 0), (7, 9, 0)]),  # D = 5: no value ranks
]


@pytest.mark.parametrize("seed,V,E,K,comps", CASES, ids=[f"case{c[0]}" for c in CASES])
def test_value_rank_parity_and_width(rmx, seed, V, E, K, comps):
    words, idx = set_mesh(seed, V, E, K, comps)
    check(rmx, words, idx)
    plain, ranked = model_bits(words, idx)
    packed, kw, bits, passes = plan_info(rmx, words, idx)
    assert packed == 1
    assert bits == ranked, (bits, ranked, plain)
    assert kw == (2 if bits > 32 else 1)
    assert passes == (bits + 7) // 8


@pytest.mark.parametrize("seed", [1, 2, 3, 7])
def test_value_rank_off_matches(rmx, value_rank_off, seed):
    case = next(c for c in CASES if c[0] == seed)
    words, idx = set_mesh(*case)
    check(rmx, words, idx)
    plain, _ = model_bits(words, idx)
    assert plan_info(rmx, words, idx)[2] == plain


def test_value_rank_with_unused_rows_outside_the_set(rmx):
    """Unused rows hold values no used row has: they take the replacement row before ranking."""
    words, idx = set_mesh(21, 80_000, 30_000, 3, [(300, 16, 7), (300, 16, 7), (5, 8, 0)])
    used = np.zeros(words.shape[0], bool)
    used[idx.reshape(-1)] = True
    words[~used, 0] = BASE | np.uint32(0x7FFF80)
    words[~used, 2] = np.uint32(0xC2000000)
    check(rmx, words, idx)


def test_sampled_decision_large(rmx):
    """>= 2^22 rows: the strided sample decides, the full set confirms (C2-like sets)."""
    V = (1 << 22) + 4099
    words, idx = set_mesh(31, V, V // 3, 3, [(3001, 16, 7), (3001, 16, 7), (64, 8, 15)])
    check(rmx, words, idx)
    assert plan_info(rmx, words, idx)[2] == 12 + 12 + 6


def test_sampled_decision_misled(rmx):
    """The sample (the first 256 rows of every 16384) sees 16 values per axis, the other rows
    ~all 2^16: the full pass must find no gain and keep the plain packed key."""
    V = 1 << 22
    rng = np.random.default_rng(41)
    words = np.empty((V, 2), np.uint32)
    in_sample = (np.arange(V) % 16384) < 256
    for c in range(2):
        words[:, c] = BASE | (rng.integers(0, 1 << 16, size=V).astype(np.uint32) << np.uint32(7))
        small = rng.integers(0, 16, size=int(in_sample.sum())).astype(np.uint32) << np.uint32(7 + 12)
        words[in_sample, c] = BASE | small
    idx = np.arange(V, dtype=np.uint32).reshape(-1, 4)
    check(rmx, words, idx)
    assert plan_info(rmx, words, idx)[2] == 32


def _sample_mask(V, shift=6, run=256):
    """The rows the guess is made from (mirror of rmx_packed.cuh:sample_row, meshes >= 2^22 rows)."""
    period = run << shift
    mask = np.zeros(V, bool)
    for b in range((V >> shift) // run + 1):
        jitter = (((b * 0x9E3779B1) & 0xFFFFFFFF) >> 8) % (period - run + 1)
        lo = b * period + jitter
        mask[lo:min(lo + run, V)] = True
    return mask


@pytest.mark.parametrize("what", ["bits", "fields", "both"])
def test_guess_from_the_sample_is_wrong(rmx, monkeypatch, what):
    """Rows outside the sampled runs carry varying bits / sign+exponent fields the sample never
    saw: the value-set pass flags the miss, K1a is recomputed, the decision is taken again and the
    second chance collects the values with the exact packing -- the components whose packing grew
    past 16 bits lose their ranks, the others keep them, and the result stays exact."""
    V = 1 << 22
    rng = np.random.default_rng(71)
    words = np.empty((V, 3), np.uint32)
    for c in range(3):
        vals = value_set(rng, 300, 16)
        words[:, c] = BASE | (vals[rng.integers(0, 300, size=V)] << np.uint32(7))
    out = ~_sample_mask(V)
    pick = np.flatnonzero(out)[rng.integers(0, int(out.sum()), size=50)]
    if what in ("bits", "both"):
        words[pick[:25], 0] |= np.uint32(1 << 2)                 # a mantissa bit the sample lacks
    if what in ("fields", "both"):
        words[pick[25:], 1] = np.uint32(0x40A00000)              # 5.0f: a binade the sample lacks
    idx = np.arange(V, dtype=np.uint32).reshape(-1, 4)
    check(rmx, words, idx)
    guess = []
    packed, kw, bits, passes = plan_info(rmx, words, idx, guess)
    assert packed == 1 and passes == (bits + 7) // 8
    assert guess[3] & 3 == 3  # the full pass checked the rows and found some outside the sample
    assert guess[1] == 1      # ... and value ranks still paid
    monkeypatch.setenv("RMX_VALUE_RANK", "0")
    assert bits < plan_info(rmx, words, idx)[2]


def test_guess_from_the_sample_is_right(rmx):
    """The common case: the sample sees every value's bits, the full pass only checks."""
    V = (1 << 22) + 77
    words, idx = set_mesh(72, V, V // 4, 4, [(700, 14, 9), (700, 14, 9), (9, 6, 0)])
    check(rmx, words, idx)
    guess = []
    assert plan_info(rmx, words, idx, guess)[2] == 10 + 10 + 4
    # worth collecting; the sample halves saw the same value sets, so the plan was speculative (bit
    # 8: no full value-set pass, the check state copied as clean) and k_pack's check passed (no bit 9)
    assert guess[1] == 1 and guess[3] == 1 | 256


def test_small_meshes_skip_value_ranks(rmx, monkeypatch):
    """Below RMX_VALUE_RANK_MIN rows (default 2^25) the sample kernels and the value-set pass would
    cost more than a saved pass: the plain packed key is used."""
    monkeypatch.delenv("RMX_VALUE_RANK_MIN")
    case = next(c for c in CASES if c[0] == 1)
    words, idx = set_mesh(*case)
    check(rmx, words, idx)
    plain, _ = model_bits(words, idx)
    assert plan_info(rmx, words, idx)[2] == plain


def test_sample_sees_no_used_row(rmx):
    """Every sampled row is unused: the guess is built from nothing (all components constant), the
    full pass finds every used row outside it, K1a is recomputed -- the result stays exact."""
    V = 1 << 22
    rng = np.random.default_rng(91)
    words = np.empty((V, 3), np.uint32)
    for c in range(3):
        vals = value_set(rng, 200, 16)
        words[:, c] = BASE | (vals[rng.integers(0, 200, size=V)] << np.uint32(7))
    outside = np.flatnonzero(~_sample_mask(V))
    idx = outside[rng.integers(0, len(outside), size=(V // 8, 3))].astype(np.uint32)
    check(rmx, words, idx)
    packed, kw, bits, passes = plan_info(rmx, words, idx)
    assert packed == 1 and passes == (bits + 7) // 8


def test_outlier_field_in_the_last_full_width_candidate(rmx):
    """three 16-bit candidates fill the value-set byte maps (3 x 2^16 = kValueSetBytes);
    the last one's field is ranked among 4 sampled fields (2 bits).  Rows outside the sample carry a
    field above every sampled one: under the guessed packing it ranks to 4 (3 bits), a value past
    the component's map.  The value-set pass must keep the store inside the map (and flag the
    miss); the result stays exact."""
    V = 1 << 22
    rng = np.random.default_rng(97)
    fields = np.array([0x7F, 0x80, 0x81, 0x82], np.uint32)
    words = np.empty((V, 3), np.uint32)
    for c in range(3):
        combos = np.stack([fields[rng.integers(0, 4, 300)],
                           rng.integers(0, 1 << 14, 300).astype(np.uint32)], 1)
        combos[:2] = [[0x7F, 0], [0x82, (1 << 14) - 1]]       # every field and mantissa bit varies
        pick = combos[rng.integers(0, 300, size=V)]
        words[:, c] = (pick[:, 0] << np.uint32(23)) | (pick[:, 1] << np.uint32(9))
    out = np.flatnonzero(~_sample_mask(V))
    far = out[rng.integers(0, len(out), size=50)]
    words[far, 2] = (np.uint32(0x83) << np.uint32(23)) | (rng.integers(0, 1 << 14, 50).astype(np.uint32) << 9)
    idx = np.arange(V, dtype=np.uint32).reshape(-1, 4)
    check(rmx, words, idx)
    guess = []
    packed, kw, bits, passes = plan_info(rmx, words, idx, guess)
    assert packed == 1 and passes == (bits + 7) // 8
    assert guess[3] & 3 == 3  # checked, and rows outside the sample were found


@pytest.mark.parametrize("what", ["value", "bits", "field"])
def test_speculative_plan_fails_the_check(rmx, monkeypatch, what):
    """The sample's two halves see the same 300 values per axis, so the plan is made from the sample
    alone (speculative: no full value-set pass).  Rows outside the sample carry a value the sample
    never saw (same varying bits and fields), a varying bit it never saw, or a field it never saw:
    k_pack's check of every row fails, the skipped path runs (full value-set pass, K1a, plan, rank
    tables) and the keys are made again.  Exact either way; a new value keeps the value ranks."""
    V = 3 * 1_400_000  # >= 2^22 rows: the sampled decision
    rng = np.random.default_rng(113)
    words = np.empty((V, 3), np.uint32)
    sets = []
    for c in range(3):
        vals = value_set(rng, 300, 16)
        sets.append(vals)
        words[:, c] = BASE | (vals[rng.integers(0, 300, size=V)] << np.uint32(7))
    out = np.flatnonzero(~_sample_mask(V))
    far = out[rng.integers(0, len(out), size=20)]
    if what == "value":
        fresh = np.setdiff1d(np.arange(1, (1 << 16) - 1, dtype=np.uint32), sets[1])[:1]
        words[far, 1] = BASE | (fresh[0] << np.uint32(7))
    elif what == "bits":
        words[far, 2] |= np.uint32(1 << 3)
    else:
        words[far, 0] = np.uint32(0x41200000) | (sets[0][5] << np.uint32(7))   # 10.0f's binade
    idx = np.arange(V, dtype=np.uint32).reshape(-1, 3)
    check(rmx, words, idx)
    guess = []
    packed, kw, bits, passes = plan_info(rmx, words, idx, guess)
    assert packed == 1 and passes == (bits + 7) // 8
    assert guess[3] & 0x300 == 0x300  # speculative, and the check failed
    if what == "value":
        assert guess[3] & 3 == 1      # the re-run's full pass: no row outside the sample's bits/fields
        assert bits == 3 * bits_for(301)  # 300 / 301 values per axis: 9 bits each
    monkeypatch.setenv("RMX_SPEC", "0")
    plain_guess = []
    assert plan_info(rmx, words, idx, plain_guess)[2] == bits  # the same plan without speculation
    assert plain_guess[3] & 0x300 == 0
