"""Test-only helpers for the multi-rank path: a CPU backend built on the oracle,
shard generators, and the merged-mesh expectation (reference ops.py:10-35)."""
import bisect

import numpy as np
import torch

from oracle import remesh_oracle as O


class NumpyBackend:
    """Local steps on CPU tensors via the oracle (test infrastructure only)."""

    def reindex(self, vertex_bits, elements):
        r = O.reindex(vertex_bits.numpy().view(np.uint32), elements.numpy().view(np.uint32))
        return (torch.from_numpy(np.ascontiguousarray(r["vertices"]).view(np.int32)),
                torch.from_numpy(np.ascontiguousarray(r["elements"]).view(np.int32)))

    def lower_bound(self, rows, queries):
        keys = [tuple(r) for r in rows.numpy().view(np.uint32).tolist()]
        return [bisect.bisect_left(keys, tuple(q)) for q in queries.numpy().view(np.uint32).tolist()]

    def gather(self, table, idx):
        t = table.numpy().view(np.uint32)
        i = idx.numpy().view(np.uint32).astype(np.int64)
        return torch.from_numpy(t[i].view(np.int32))


def random_shards(seed, G, D=3, K=3, pool=6, empty=()):
    """G shards of one mesh; coordinates from a small pool so keys repeat across shards."""
    rng = np.random.default_rng(seed)
    shards = []
    for g in range(G):
        V = 0 if g in empty else int(rng.integers(1, 400))
        words = (rng.integers(0, pool, size=(V, D)).astype(np.uint32) * np.uint32(0x00810001)) ^ np.uint32(
            0x80000000 * (g % 2))
        E = 0 if V == 0 else int(rng.integers(0, 300))
        idx = rng.integers(0, max(V, 1), size=(E, K)).astype(np.uint32)
        shards.append((words, idx))
    return shards


def merged_expectation(shards):
    """reindex(merge(shards)): vertices stacked, indices offset (ops.py:28-35)."""
    D = shards[0][0].shape[1]
    K = shards[0][1].shape[1]
    verts = np.vstack([s[0].reshape(-1, D) for s in shards]).astype(np.uint32)
    parts, off = [], 0
    for v, e in shards:
        parts.append(e.astype(np.uint64) + off)
        off += len(v)
    elems = np.vstack(parts).astype(np.uint32).reshape(-1, K) if parts else np.empty((0, K), np.uint32)
    r = O.reindex(verts, elems)
    return r["vertices"].view(np.uint32), r["elements"]


def as_tensors(shards, device="cpu"):
    return [(torch.from_numpy(v.view(np.int32).copy()).to(device), torch.from_numpy(e.view(np.int32).copy()).to(device))
            for v, e in shards]


def check(results, shards):
    exp_v, exp_e = merged_expectation(shards)
    got_v = np.vstack([r.vertices.cpu().numpy().view(np.uint32).reshape(-1, exp_v.shape[1]) for r in results])
    got_e = np.vstack([r.elements.cpu().numpy().view(np.uint32).reshape(-1, exp_e.shape[1]) for r in results])
    assert np.array_equal(got_v, exp_v)
    assert np.array_equal(got_e, exp_e)
    offs = np.cumsum([0] + [r.vertices.shape[0] for r in results])
    for r, o in zip(results, offs):
        assert r.offset == o and r.total == len(exp_v)
