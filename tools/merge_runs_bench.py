"""Multi-GPU step 4 on one GPU: merge of G sorted unique runs (rmx_merge_unique_runs) vs the
full re-index of their concatenation (the previous step 4).

    python tools/merge_runs_bench.py [--rows 110000000] [--runs 8]
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2109_09812_b200 as rmx  # noqa: E402
from paper_2109_09812_b200.dist import CudaBackend  # noqa: E402


def timed(fn, reps=3):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--rows", type=int, default=110_000_000)
    ap.add_argument("--runs", type=int, default=8)
    a = ap.parse_args()
    dev = torch.device("cuda", 0)
    g = torch.Generator(device=dev).manual_seed(0)
    runs = []
    per = a.rows // a.runs
    for r in range(a.runs):
        # lattice-like float3 keys: x = 0.5 i, y = 0.5 j, z in [0, 16) on a 1/4 grid (shared across runs)
        i = torch.randint(0, 40000, (per,), device=dev, generator=g)
        j = torch.randint(0, 5001, (per,), device=dev, generator=g)
        x = (i.float() * 0.5).view(torch.int32)
        y = (j.float() * 0.5).view(torch.int32)
        z = (((7 * i + 13 * j) % 64).float() * 0.25).view(torch.int32)
        k = torch.stack([x, y, z], 1).contiguous()
        ident = torch.arange(per, dtype=torch.int32, device=dev).view(per, 1)
        runs.append(rmx.reindex_tensors(k, ident).vertices.clone())
    keys = torch.cat(runs)
    counts = [r.shape[0] for r in runs]
    n = keys.shape[0]
    be = CudaBackend(dev)
    ident = torch.arange(n, dtype=torch.int32, device=dev).view(n, 1)
    t_merge = timed(lambda: be.merge_unique(keys, counts))
    t_sort = timed(lambda: rmx.reindex_tensors(keys, ident))
    buf, rank_of, cnt = be.merge_unique(keys, counts)
    mine = buf[:int(cnt.item())]
    ref = rmx.reindex_tensors(keys, ident)
    assert torch.equal(mine, ref.vertices) and torch.equal(rank_of, ref.elements)
    print(f"{a.runs} runs, {n:,} rows -> {mine.shape[0]:,} unique: merge {t_merge:.2f} ms, "
          f"re-index {t_sort:.2f} ms")


if __name__ == "__main__":
    main()
