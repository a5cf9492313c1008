"""CPU: multi-rank host logic of dist.reindex_distributed (thread ranks and gloo ranks)
against reindex(merge(shards)) from the oracle."""
import os
import socket

import numpy as np
import pytest
import torch

from dist_helpers import NumpyBackend, as_tensors, check, random_shards
from paper_2109_09812_b200.dist import run_threads


@pytest.mark.parametrize("G", [1, 2, 3, 4, 8])
@pytest.mark.parametrize("seed", [0, 1, 2])
def test_thread_ranks_match_merge(G, seed):
    shards = random_shards(seed * 31 + G, G)
    res = run_threads(as_tensors(shards), lambda r: NumpyBackend(), samples_per_rank=7)
    check(res, shards)


def test_thread_ranks_with_empty_shards_and_arity4():
    shards = random_shards(7, 5, D=2, K=4, empty=(0, 3))
    res = run_threads(as_tensors(shards), lambda r: NumpyBackend(), samples_per_rank=3)
    check(res, shards)


def test_all_shards_without_elements():
    rng = np.random.default_rng(3)
    shards = [(rng.integers(0, 5, size=(4, 3)).astype(np.uint32), np.empty((0, 3), np.uint32)) for _ in range(3)]
    res = run_threads(as_tensors(shards), lambda r: NumpyBackend())
    assert all(r.total == 0 and r.vertices.shape[0] == 0 for r in res)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _gloo_rank(rank, world, port, out_dir):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2109_09812_b200.dist import TorchComm, reindex_distributed
    shards = random_shards(11, world)
    v, e = as_tensors(shards)[rank]
    r = reindex_distributed(v, e, TorchComm(), NumpyBackend(), samples_per_rank=5)
    torch.save({"vertices": r.vertices, "elements": r.elements, "offset": r.offset, "total": r.total},
               os.path.join(out_dir, f"r{rank}.pt"))
    dist.barrier()
    dist.destroy_process_group()


def test_gloo_world_size_2(tmp_path):
    import torch.multiprocessing as mp
    mp.spawn(_gloo_rank, args=(2, _free_port(), str(tmp_path)), nprocs=2, join=True)

    class R:
        pass

    res = []
    for r in range(2):
        d = torch.load(tmp_path / f"r{r}.pt")
        x = R()
        x.vertices, x.elements, x.offset, x.total = d["vertices"], d["elements"], d["offset"], d["total"]
        res.append(x)
    check(res, random_shards(11, 2))
