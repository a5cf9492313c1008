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


@pytest.mark.parametrize("G,words", [(1, 3), (2, 1), (5, 4), (8, 3), (16, 2)])
def test_scatter_rows_into_peer_buffers(cuda_ok, G, words):
    """rmx_scatter_rows with G 'peer' buffers on one GPU: rows [bounds[g], bounds[g+1]) land in
    buffer g from row dst_off[g] (the layout SymmComm relies on)."""
    from paper_2109_09812_b200 import _native
    rng = np.random.default_rng(G * 10 + words)
    counts = rng.integers(0, 500, size=G)
    counts[G // 2] = 0
    n = int(counts.sum())
    src = torch.from_numpy(rng.integers(-2**31, 2**31 - 1, size=(n, words), dtype=np.int64).astype(np.int32)).cuda()
    offs = rng.integers(0, 300, size=G)
    peers = [torch.full((int(offs[g] + counts[g] + 10), words), -1, dtype=torch.int32, device="cuda")
             for g in range(G)]
    bounds = np.concatenate([[0], np.cumsum(counts)]).astype(np.int64)
    meta = torch.tensor(np.concatenate([bounds, offs]).astype(np.int64), device="cuda")
    ptrs = torch.tensor([p.data_ptr() for p in peers], dtype=torch.int64, device="cuda")
    _native.check(_native.lib().rmx_scatter_rows(src.data_ptr(), n, words, meta.data_ptr(), G, ptrs.data_ptr(),
                                                 meta.data_ptr() + 8 * (G + 1),
                                                 torch.cuda.current_stream().cuda_stream))
    torch.cuda.synchronize()
    for g in range(G):
        got = peers[g].cpu()
        assert torch.equal(got[offs[g]:offs[g] + counts[g]], src[bounds[g]:bounds[g + 1]].cpu())
        assert bool((got[:offs[g]] == -1).all()) and bool((got[offs[g] + counts[g]:] == -1).all())


def test_symm_comm_world_of_one(cuda_ok):
    """SymmComm (symmetric memory + rmx_scatter_rows) in a one-rank NCCL group: the exchange is the
    identity, and reindex_distributed through it equals the single-GPU re-index."""
    import socket

    import torch.distributed as tdist

    import paper_2109_09812_b200 as rmx
    from paper_2109_09812_b200.dist import CudaBackend, SymmComm, reindex_distributed
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    dev = torch.device("cuda", 0)
    tdist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", rank=0, world_size=1, device_id=dev)
    try:
        comm = SymmComm(device=dev)
        rows = torch.randint(-2**31, 2**31 - 1, (12345, 3), dtype=torch.int32, device=dev)
        out, rc = comm.all_to_all(rows, [12345])
        assert rc == [12345] and torch.equal(out, rows)
        shards = random_shards(3, 1)
        (v, e), = as_tensors(shards, "cuda")
        res = reindex_distributed(v, e, comm, CudaBackend(dev))
        ref = rmx.reindex_tensors(v, e)
        assert torch.equal(res.vertices, ref.vertices) and torch.equal(res.elements, ref.elements)
    finally:
        tdist.destroy_process_group()


@pytest.mark.parametrize("G,D,n", [(1, 3, 5000), (2, 1, 100_000), (3, 4, 7777), (8, 3, 300_000), (5, 8, 20_000),
                                   (16, 2, 60_000)])
def test_merge_unique_runs_vs_numpy(cuda_ok, G, D, n):
    """rmx_merge_unique_runs: G sorted duplicate-free runs (keys shared across runs, empty runs)
    -> sorted unique keys and the rank of every row, against numpy."""
    from paper_2109_09812_b200.dist import CudaBackend
    rng = np.random.default_rng(G * 100 + D)
    pool = rng.integers(0, 1 << 32, size=(max(4, n // 2), D), dtype=np.uint64).astype(np.uint32)
    pool[: len(pool) // 3, 0] = pool[0, 0]                  # long shared prefixes on word 0
    runs = []
    for g in range(G):
        m = 0 if (g == 1 and G > 2) else int(rng.integers(1, max(2, 2 * n // G)))
        pick = np.unique(rng.integers(0, len(pool), size=m))
        run = pool[pick]
        order = np.lexsort(run.T[::-1])
        run = run[order]
        keep = np.ones(len(run), bool)
        keep[1:] = np.any(run[1:] != run[:-1], axis=1)
        runs.append(run[keep])
    keys = np.concatenate(runs) if runs else np.empty((0, D), np.uint32)
    counts = [len(r) for r in runs]
    uniq, inv = np.unique(keys, axis=0, return_inverse=True)      # numpy sorts rows lexicographically
    be = CudaBackend(torch.device("cuda", 0))
    buf, rank_of, cnt = be.merge_unique(torch.from_numpy(keys.view(np.int32)).cuda(), counts)
    mine = buf[:int(cnt.item())]
    assert np.array_equal(mine.cpu().numpy().view(np.uint32), uniq)
    assert np.array_equal(rank_of.view(-1).cpu().numpy().view(np.uint32), inv.reshape(-1).astype(np.uint32))
