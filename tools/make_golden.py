"""Generate tests/golden/*.npz by running the REFERENCE implementation.

Run in the build container (where /root/reference exists):

    python tools/make_golden.py

It imports ``remeshx`` read-only from /root/reference/pkg/src and records,
for every case, the input arrays and everything ``remeshx.reindex`` returns
(output mesh + all ReindexScratch fields).  The fixtures travel with the repo;
nothing at test time reads /root/reference.

Cases:
  worked      -- the paper's worked example (reference tests/conftest.py:8-19)
  reftests    -- hand cases from the reference tests (test_pipeline.py:149-192,
                 test_ops.py quads, test_mesh.py:67-74 special bit patterns)
  torture     -- raw bit patterns: +-0, +-inf, quiet/signalling NaNs with
                 payloads, denormals, negatives; dims 1..5,7; arities 1..8;
                 V=1, all-equal, all-distinct, zero-element meshes
  random      -- remeshx.random_mesh seeds sweeping dup/unused fraction, arity
  grid        -- remeshx.grid_quads(N) for N = 1, 2, 8, 64 (paper Table 1 counts)
  lattice     -- small oracle/lattice.py soups (pins the lattice closed form)
  ops         -- merge / soup_to_mesh / subset results
  rmx1/*.rmx  -- RMX1 files written by the reference write_bin
"""
from __future__ import annotations

import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF_SRC = "/root/reference/pkg/src"
OUT = os.path.join(ROOT, "tests", "golden")

sys.path.insert(0, ROOT)
sys.path.insert(0, REF_SRC)

import remeshx  # noqa: E402  (reference, read-only)
from oracle import lattice  # noqa: E402

FIELDS = ("is_used", "org_id", "nodup", "new_idx", "perm")


def record(cases: dict, name: str, vertices: np.ndarray, elements: np.ndarray) -> None:
    v = np.ascontiguousarray(vertices)
    if v.dtype == np.uint32:
        v = v.view(np.float32)
    mesh = remeshx.Mesh(v, elements)
    out, sc = remeshx.reindex(mesh)
    k = f"{name}"
    cases[f"{k}/in_vtx"] = mesh.vertices.view(np.uint32)
    cases[f"{k}/in_idx"] = mesh.elements
    cases[f"{k}/out_vtx"] = out.vertices.view(np.uint32)
    cases[f"{k}/out_idx"] = out.elements
    for f in FIELDS:
        cases[f"{k}/{f}"] = np.asarray(getattr(sc, f))
    cases[f"{k}/new_count"] = np.array(sc.new_count, np.int64)


def worked(cases):
    A, B, C, D, E, F = (0, 0), (0, 1), (0, 2), (0, 3), (0, 4), (0, 5)
    X, Y = (9, 9), (8, 8)
    v = np.array([A, B, C, X, D, C, E, F, Y, D], np.float32)
    e = np.array([(0, 1, 2), (0, 2, 4), (5, 6, 7), (5, 7, 9)], np.uint32)
    record(cases, "worked", v, e)


def f32(*vals):
    return np.array(vals, np.float32)


def bits(*words):
    return np.array(words, np.uint32).view(np.float32)


def reftests(cases):
    A, B, C = (0, 0), (0, 1), (0, 2)
    record(cases, "already_compact", np.array([B, A, C], np.float32), np.array([(0, 1, 2), (2, 1, 0)], np.uint32))
    record(cases, "neg_zero", np.array([(0.0, 1.0), (-0.0, 1.0)], np.float32), np.array([(0, 1, 0)], np.uint32))
    nan1 = np.uint32(0x7FC00001).view(np.float32)
    record(cases, "nan_weld", np.array([(nan1, 1.0), (nan1, 1.0), (2.0, 2.0)], np.float32),
           np.array([(0, 1, 2)], np.uint32))
    nan2 = np.uint32(0x7FC00002).view(np.float32)
    record(cases, "nan_payloads", np.array([(nan1, 1.0), (nan2, 1.0), (nan1, 1.0)], np.float32),
           np.array([(0, 1, 2)], np.uint32))
    record(cases, "zero_elements", np.array([A, B, C], np.float32), np.empty((0, 4), np.uint32))
    record(cases, "repeated_index", np.array([(2, 7)], np.float32), np.array([(0, 0, 0)], np.uint32))
    order_rows = np.array([(0.0, 0.0), (-0.0, 0.0), (np.nan, 1.0), (1.0, np.nan)], np.float32)
    record(cases, "total_order", order_rows, np.array([(0, 1, 2, 3)], np.uint32))
    quad = lambda x0, y0: np.array([(x0, y0), (x0 + 1, y0), (x0 + 1, y0 + 1), (x0, y0 + 1)], np.float32)
    record(cases, "two_quads", np.vstack([quad(0, 0), quad(1, 0)]), np.array([(0, 1, 2, 3), (4, 5, 6, 7)], np.uint32))


SPECIAL = np.array([0x00000000, 0x80000000, 0x7F800000, 0xFF800000, 0x7FC00000, 0x7FC00001,
                    0xFFC00000, 0x7F800001, 0xFF800001, 0x7FBFFFFF, 0x00000001, 0x807FFFFF,
                    0x3F800000, 0xBF800000, 0x40000000, 0xC0000000, 0x00800000, 0x80800000,
                    0x3F800001, 0x4F000000, 0xFFFFFFFF, 0x7FFFFFFF, 0x12345678, 0x87654321], np.uint32)


def torture(cases):
    rng = np.random.default_rng(2109)
    n = 0
    for dim in (1, 2, 3, 4, 5, 7):
        for arity in (1, 2, 3, 4, 8):
            for mode in ("pool", "raw", "equal", "distinct"):
                V = int(rng.integers(1, 300))
                if mode == "pool":
                    words = SPECIAL[rng.integers(0, len(SPECIAL), size=(V, dim))]
                elif mode == "raw":
                    words = rng.integers(0, 1 << 32, size=(V, dim), dtype=np.uint64).astype(np.uint32)
                elif mode == "equal":
                    words = np.tile(SPECIAL[rng.integers(0, len(SPECIAL), size=(1, dim))], (V, 1))
                else:
                    words = rng.integers(0, 1 << 32, size=(V, dim), dtype=np.uint64).astype(np.uint32)
                    words[:, 0] = rng.permutation(V).astype(np.uint32) * 7919 + 11
                m = int(rng.integers(1, 80))
                # leave some vertices unused: indices only from the first ~80 %
                hi = max(1, (V * 4) // 5)
                e = rng.integers(0, hi, size=(m, arity)).astype(np.uint32)
                record(cases, f"torture_{n:03d}_d{dim}_k{arity}_{mode}", words.view(np.float32), e)
                n += 1
    # V = 1 and an element-free mesh per dim
    for dim in (1, 3):
        record(cases, f"torture_single_d{dim}", SPECIAL[:dim].reshape(1, dim).view(np.float32),
               np.zeros((3, 2), np.uint32))
        record(cases, f"torture_noelem_d{dim}", SPECIAL[:4 * dim].reshape(4, dim).view(np.float32),
               np.empty((0, 3), np.uint32))
    # one mid-size raw case that spans several sort / scan tiles
    V = 20000
    words = SPECIAL[rng.integers(0, len(SPECIAL), size=(V, 3))]
    words[::3, 1] = rng.integers(0, 1 << 32, size=(V + 2) // 3, dtype=np.uint64).astype(np.uint32)
    e = rng.integers(0, V - 500, size=(9000, 3)).astype(np.uint32)
    record(cases, "torture_multitile", words.view(np.float32), e)


def random_meshes(cases):
    fr = [0.0, 0.25, 0.5]
    for seed in range(36):
        spec = remeshx.RandomMeshSpec(seed=seed, dup_fraction=fr[seed % 3], unused_fraction=fr[(seed // 3) % 3],
                                      arity=[3, 4][(seed // 9) % 2], dim=[2, 3][(seed // 18) % 2])
        m = remeshx.random_mesh(spec)
        record(cases, f"random_{seed:03d}", m.vertices, m.elements)
    big = remeshx.random_mesh(remeshx.RandomMeshSpec(seed=777, n_base_vertices=6000, n_elements=9000,
                                                     arity=4, coord_pool_size=40, dim=3))
    record(cases, "random_big", big.vertices, big.elements)


def grids(cases):
    for n in (1, 2, 8, 64):
        g = remeshx.grid_quads(n)
        record(cases, f"grid_{n}", g.vertices, g.elements)


def lattices(cases):
    for kind, cells in (("tri", (7, 5)), ("tet", (3, 4, 2)), ("tri", (37, 23)), ("tet", (5, 4, 6))):
        for take in (None, 40):
            v, e = lattice.lattice_soup(kind, cells, seed=3, n_elem_take=take)
            name = f"lattice_{kind}_{'x'.join(map(str, cells))}_{'all' if take is None else take}"
            record(cases, name, v, e)


def record_mesh(cases, name, mesh):
    cases[f"{name}/out_vtx"] = np.asarray(mesh.vertices).view(np.uint32)
    cases[f"{name}/out_idx"] = np.asarray(mesh.elements)


def ops(cases):
    """remeshx.merge / soup_to_mesh / subset (ops.py:10-87) on seeded inputs."""
    for seed in range(12):
        arity = [3, 4][seed % 2]
        parts = [remeshx.random_mesh(remeshx.RandomMeshSpec(seed=seed * 10 + k, arity=arity,
                                                            dim=[2, 3][(seed // 2) % 2])) for k in range(1 + seed % 4)]
        name = f"merge_{seed:02d}"
        for k, p in enumerate(parts):
            cases[f"{name}/piece_vtx_{k}"] = p.vertices.view(np.uint32)
            cases[f"{name}/piece_idx_{k}"] = p.elements
        cases[f"{name}/n_pieces"] = np.array(len(parts))
        record_mesh(cases, name, remeshx.merge(parts))
        soup = remeshx.dereference(parts[0])
        cases[f"soup_{seed:02d}/soup"] = soup.view(np.uint32)
        record_mesh(cases, f"soup_{seed:02d}", remeshx.soup_to_mesh(soup))
        m = parts[-1]
        keep = [e for e in range(m.n_elements) if (e + seed) % 3]
        cases[f"subset_{seed:02d}/in_vtx"] = m.vertices.view(np.uint32)
        cases[f"subset_{seed:02d}/in_idx"] = m.elements
        cases[f"subset_{seed:02d}/keep"] = np.array(keep, np.int64)
        record_mesh(cases, f"subset_{seed:02d}", remeshx.subset(m, keep))
    q = lambda x0, y0: remeshx.Mesh(np.array([(x0, y0), (x0 + 1, y0), (x0 + 1, y0 + 1), (x0, y0 + 1)], np.float32),
                                    np.array([(0, 1, 2, 3)], np.uint32))
    parts = [q(0, 0), q(1, 0)]
    for k, p in enumerate(parts):
        cases[f"merge_quads/piece_vtx_{k}"] = p.vertices.view(np.uint32)
        cases[f"merge_quads/piece_idx_{k}"] = p.elements
    cases["merge_quads/n_pieces"] = np.array(2)
    record_mesh(cases, "merge_quads", remeshx.merge(parts))


def files():
    """RMX1 containers written by the reference write_bin (fileio.py:125-133)."""
    d = os.path.join(OUT, "rmx1")
    os.makedirs(d, exist_ok=True)
    A, B, C, D, E, F = (0, 0), (0, 1), (0, 2), (0, 3), (0, 4), (0, 5)
    X, Y = (9, 9), (8, 8)
    meshes = {
        "worked": remeshx.Mesh(np.array([A, B, C, X, D, C, E, F, Y, D], np.float32),
                               np.array([(0, 1, 2), (0, 2, 4), (5, 6, 7), (5, 7, 9)], np.uint32)),
        "empty": remeshx.Mesh.empty(),
        "nan_bits": remeshx.Mesh(np.array([(np.uint32(0x7FC00123).view(np.float32), -0.0)], np.float32),
                                 np.array([(0, 0, 0)], np.uint32)),
        "random_quads3d": remeshx.random_mesh(remeshx.RandomMeshSpec(seed=5, arity=4, dim=3)),
    }
    for name, m in meshes.items():
        remeshx.write_bin(m, os.path.join(d, f"{name}.rmx"))
        print(f"{d}/{name}.rmx")


def main():
    os.makedirs(OUT, exist_ok=True)
    files()
    groups = {"worked": worked, "reftests": reftests, "torture": torture, "random": random_meshes,
              "grid": grids, "lattice": lattices, "ops": ops}
    for gname, fn in groups.items():
        cases: dict = {}
        fn(cases)
        path = os.path.join(OUT, f"{gname}.npz")
        np.savez_compressed(path, **cases)
        print(f"{path}: {len([k for k in cases if k.endswith('/in_vtx')])} cases, {os.path.getsize(path)} bytes")


if __name__ == "__main__":
    main()
