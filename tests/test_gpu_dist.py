"""GPU: the multi-rank path with the CUDA backend, G ranks as threads on one GPU
(no rank waits on another inside a kernel), against reindex(merge(shards))."""
import numpy as np
import pytest
import torch

from dist_helpers import as_tensors, check, random_shards

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("G", [1, 2, 4, 8])
@pytest.mark.parametrize("seed", [0, 1])
def test_cuda_thread_ranks_match_merge(cuda_ok, G, seed):
    from paper_2109_09812_b200.dist import CudaBackend, run_threads
    shards = random_shards(seed * 97 + G, G)
    res = run_threads(as_tensors(shards, "cuda"), lambda r: CudaBackend(torch.device("cuda", 0)),
                      samples_per_rank=16)
    check(res, shards)


def test_cuda_thread_ranks_random_bits_and_empty(cuda_ok):
    from paper_2109_09812_b200.dist import CudaBackend, run_threads
    rng = np.random.default_rng(5)
    shards = []
    for g in range(6):
        V = 0 if g == 2 else 20000
        words = rng.integers(0, 1 << 32, size=(V, 3), dtype=np.uint64).astype(np.uint32)
        words[rng.random(words.shape) < 0.7] &= 0xFFF00000      # cross-shard duplicates, > 64 varying bits
        E = 0 if V == 0 else 9000
        shards.append((words, rng.integers(0, max(V, 1), size=(E, 3)).astype(np.uint32)))
    res = run_threads(as_tensors(shards, "cuda"), lambda r: CudaBackend(torch.device("cuda", 0)))
    check(res, shards)


def test_cuda_lattice_shards_8(cuda_ok):
    """A C1-size lattice soup split into 8 element ranges (the C5 sharding, scaled down)."""
    from oracle import lattice
    from paper_2109_09812_b200.dist import CudaBackend, run_threads
    kind, cells = "tri", (125, 160)
    v, e = lattice.lattice_soup(kind, cells, seed=0)
    E, bits = len(e), v.view(np.uint32)
    cuts = [E * g // 8 for g in range(9)]
    # element e owns vertex slots from e[e, 0]; shard g = its elements + the slots up to the next shard
    starts = [int(e[c, 0]) for c in cuts[:8]] + [len(bits)]
    shards = [(bits[starts[g]:starts[g + 1]], (e[cuts[g]:cuts[g + 1]] - starts[g]).astype(np.uint32))
              for g in range(8)]
    res = run_threads(as_tensors(shards, "cuda"), lambda r: CudaBackend(torch.device("cuda", 0)))
    check(res, shards)
    assert res[0].total == (cells[0] + 1) * (cells[1] + 1)


@pytest.mark.parametrize("e0,e1", [(0, 700), (333, 1501), (1999, 2000), (1500, 1500)])
def test_range_generator_is_a_shard_of_the_soup(cuda_ok, e0, e1):
    import ctypes
    from oracle import lattice
    from paper_2109_09812_b200 import _native
    lib = _native.lib()
    kind, cells = "tri", (40, 25)
    v, e = lattice.lattice_soup(kind, cells, seed=4)
    bits = v.view(np.uint32)
    E = len(e)

    def slots(x):
        a, b = ctypes.c_uint64(), ctypes.c_uint64()
        lib.rmx_lattice_sizes(0, cells[0], cells[1], 0, x, ctypes.byref(a), ctypes.byref(b))
        return b.value

    s0, s1 = slots(e0), slots(e1)
    dv = torch.empty((max(s1 - s0, 1), 3), dtype=torch.int32, device="cuda")
    de = torch.empty((max(e1 - e0, 1), 3), dtype=torch.int32, device="cuda")
    assert lib.rmx_gen_lattice_soup_range(0, cells[0], cells[1], 0, 4, e0, e1, dv.data_ptr(), de.data_ptr(),
                                          torch.cuda.current_stream().cuda_stream) == 0
    assert E == 2 * cells[0] * cells[1]
    if e1 > e0:
        assert np.array_equal(dv[: s1 - s0].cpu().numpy().view(np.uint32), bits[s0:s1])
        assert np.array_equal(de[: e1 - e0].cpu().numpy().view(np.uint32), (e[e0:e1] - s0).astype(np.uint32))
