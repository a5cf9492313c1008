"""Small inputs through every kernel family -- for compute-sanitizer (memcheck / racecheck /
synccheck) where it runs, and with the bounds-counting build where it does not:

    compute-sanitizer --tool memcheck python tools/sanitize_probe.py
    python -m paper_2109_09812_b200.build --checked
    RMX_LIB=paper_2109_09812_b200/librmx_b200_checked.so python tools/sanitize_probe.py

* the one-CTA small path (k_small) and the large pipeline (RMX_SMALL=0) on packed keys (value and
  field ranks), AoS rows with scratch (onesweep look-back, mbarrier staging), hash mode (hashed
  passes, per-tile dedup, candidate sort), D = 1..5;
* merge_tensors / subset_tensors (offset and selection kernels), the multi-rank merge of sorted runs
  (k_merge_path), rmx_scatter_rows into peer buffers, rmx_lower_bound_rows, rmx_gather_u32.
Exits non-zero on any mismatch with the oracle.
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import torch  # noqa: E402

import paper_2109_09812_b200 as rmx  # noqa: E402
from oracle import remesh_oracle as O  # noqa: E402


def check(words, idx, scratch=True):
    ref = O.reindex(words, idx)
    out, sc = rmx.reindex(rmx.Mesh(words.view(np.float32), idx))
    assert np.array_equal(out.vertices.view(np.uint32), ref["vertices"].view(np.uint32))
    assert np.array_equal(out.elements, ref["elements"])
    if scratch:
        for f in ("is_used", "org_id", "nodup", "new_idx", "perm"):
            assert np.array_equal(np.asarray(getattr(sc, f)), ref[f]), f


def main():
    rng = np.random.default_rng(0)
    for small in ("1", "0"):
        os.environ["RMX_SMALL"] = small
        for D in (1, 2, 3, 4, 5):
            V = 3000 if small == "1" else 20_000
            lattice = (rng.integers(0, 40, size=(V, D)).astype(np.uint32) << np.uint32(12)) | np.uint32(0x3F800000)
            rand = rng.integers(0, 2**32, size=(V, D), dtype=np.uint64).astype(np.uint32)
            rand[rng.integers(0, V, V // 3)] = rand[rng.integers(0, V, V // 3)]
            for words in (lattice, rand):
                idx = rng.integers(0, V, size=(V // 3, 3)).astype(np.uint32)
                check(words, idx)
        print("reindex ok (small path)" if small == "1" else "reindex ok (pipeline)", flush=True)
    os.environ["RMX_SMALL"] = "0"
    os.environ["RMX_VALUE_RANK_MIN"] = "0"
    V = 40_000
    words = (rng.integers(0, 300, size=(V, 3)).astype(np.uint32) << np.uint32(7)) | np.uint32(0x3F800000)
    check(words, rng.integers(0, V, size=(V // 4, 3)).astype(np.uint32))
    print("value ranks ok", flush=True)
    dev = torch.device("cuda", 0)
    from paper_2109_09812_b200 import gen, ops
    pieces = [gen.welded_tile_tensors(20, 15 * k, k, k % 2 == 1, dev) for k in range(3)]
    res = ops.merge_tensors(pieces)
    keep = torch.zeros(pieces[0][1].shape[0], dtype=torch.bool, device=dev)
    keep[::3] = True
    ops.subset_tensors(pieces[0][0], pieces[0][1], keep)
    torch.cuda.synchronize()
    assert res.new_count == (15 * 2 + 21) * 21
    print("merge / subset ok", flush=True)
    from dist_helpers import as_tensors, check as dcheck, random_shards
    from paper_2109_09812_b200.dist import CudaBackend, run_threads
    shards = random_shards(5, 3)
    out = run_threads(as_tensors(shards, "cuda"), lambda r: CudaBackend(dev), samples_per_rank=16)
    dcheck(out, shards)
    print("distributed (thread ranks: merge runs, lower bound, gather) ok", flush=True)
    from paper_2109_09812_b200 import _native
    G, n, words_per_row = 3, 5000, 3
    src = torch.randint(-2**31, 2**31 - 1, (n, words_per_row), dtype=torch.int32, device=dev)
    counts = [1700, 1300, 2000]
    bounds = [0, 1700, 3000, 5000]
    offs = [5, 0, 11]
    peers = [torch.full((counts[g] + offs[g] + 7, words_per_row), -1, dtype=torch.int32, device=dev) for g in range(G)]
    meta = torch.tensor(bounds + offs, dtype=torch.int64, device=dev)
    ptrs = torch.tensor([p.data_ptr() for p in peers], dtype=torch.int64, device=dev)
    _native.check(_native.lib().rmx_scatter_rows(src.data_ptr(), n, words_per_row, meta.data_ptr(), G,
                                                 ptrs.data_ptr(), meta.data_ptr() + 8 * (G + 1),
                                                 torch.cuda.current_stream().cuda_stream))
    torch.cuda.synchronize()
    for g in range(G):
        assert torch.equal(peers[g][offs[g]:offs[g] + counts[g]], src[bounds[g]:bounds[g + 1]])
    print("scatter rows ok", flush=True)
    import ctypes
    oob = ctypes.c_ulonglong(0)
    if _native.lib().rmx_debug_oob_count(ctypes.byref(oob)) == 0:
        print(f"checked build: {oob.value} out-of-bounds scattered stores", flush=True)
        assert oob.value == 0


if __name__ == "__main__":
    main()
