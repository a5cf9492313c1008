"""Seeded lattice soups and their closed-form re-indexing -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU legs may
import this module.  The product package has its own CUDA generator
(``rmx_gen_lattice_soup`` in the C-ABI) that must reproduce
:func:`lattice_soup` bit for bit; ``tests/test_gpu_parity.py`` checks that.

Workload recipe; the
counter-based hashing below is this repo's own definition, chosen so the host
and device generators agree exactly:

* ``tri`` (float3, K=3): lattice points ``(i, j)``, ``0<=i<=nx, 0<=j<=ny`` at
  ``(0.5 i, 0.5 j, 0.25 ((7i + 13j) mod 64))``; quad ``(qi, qj)`` splits into
  triangles ``(a, b, c)`` and ``(a, c, d)``.
* ``tet`` (float3 + scalar, D=4, K=4): points ``(i, j, k)`` at
  ``(0.5 i, 0.5 j, 0.5 k, 0.125 ((3i + 5j + 7k) mod 97))``; each cube splits
  into the 6 Kuhn tetrahedra around its main diagonal.
* Soup: element ``e`` holds lattice element ``pi(e)`` for a seeded Feistel
  bijection ``pi``; its K vertices are stored by value at consecutive slots.
* Unused rows: ``I // 20`` (5 % of the index slots) spread evenly between
  elements, holding random finite floats in ``+-[1, 1024)``.

All coordinates are non-negative, so the reference's raw-bit order equals the
numeric order and the re-indexed output is known in closed form: output
vertex ``r`` is lattice point ``r`` (row-major) and every index becomes the
rank of its lattice point.  ``tests/test_oracle.py`` pins this closed form
against ``remesh_oracle.reindex`` and against golden vectors made by the
reference ``remeshx.reindex`` (``tools/make_golden.py``).
"""
from __future__ import annotations

import numpy as np

M64 = np.uint64(0xFFFFFFFFFFFFFFFF)

# (kind, cells) per config of BASELINE.json; seed 0 everywhere
CONFIGS = {
    "C1": ("tri", (625, 800)),
    "C2": ("tri", (5000, 5000)),
    "C3": ("tet", (150, 150, 148)),
    "C5": ("tri", (20000, 25000)),
}

KUHN = np.array([(0, 1, 2), (0, 2, 1), (1, 0, 2), (1, 2, 0), (2, 0, 1), (2, 1, 0)], np.int64)


def splitmix64(x):
    """splitmix64 finaliser on uint64 arrays/scalars (wrapping arithmetic)."""
    with np.errstate(over="ignore"):
        z = (np.asarray(x, dtype=np.uint64) + np.uint64(0x9E3779B97F4A7C15))
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        return z ^ (z >> np.uint64(31))


def shape_of(kind: str, cells) -> dict:
    if kind == "tri":
        nx, ny = cells
        n_elem = 2 * nx * ny
        return dict(dim=3, arity=3, n_elem=n_elem, n_points=(nx + 1) * (ny + 1))
    if kind == "tet":
        nx, ny, nz = cells
        n_elem = 6 * nx * ny * nz
        return dict(dim=4, arity=4, n_elem=n_elem, n_points=(nx + 1) * (ny + 1) * (nz + 1))
    raise ValueError(kind)


def feistel_keys(seed: int) -> np.ndarray:
    return splitmix64(np.arange(4, dtype=np.uint64) + np.uint64(seed * 4 + 1))


def permute(x: np.ndarray, n: int, seed: int) -> np.ndarray:
    """Seeded bijection on [0, n): 4-round Feistel on an even bit width, cycle-walked."""
    bits = max(2, int(n - 1).bit_length())
    bits += bits & 1
    half = np.uint64(bits // 2)
    mask = np.uint64((1 << (bits // 2)) - 1)
    keys = feistel_keys(seed)

    def rounds(v):
        left = v >> half
        right = v & mask
        for r in range(4):
            f = (splitmix64(right ^ keys[r]) >> np.uint64(7)) & mask
            left, right = right, left ^ f
        return (left << half) | right

    y = rounds(np.asarray(x, dtype=np.uint64))
    bad = y >= np.uint64(n)
    while bad.any():
        y[bad] = rounds(y[bad])
        bad = y >= np.uint64(n)
    return y


def point_coords(kind: str, cells, pts: np.ndarray) -> np.ndarray:
    """float32 coordinates of lattice points given as (..., 2|3) integer arrays."""
    if kind == "tri":
        i, j = pts[..., 0], pts[..., 1]
        z = (7 * i + 13 * j) % 64
        out = np.stack([i.astype(np.float32) * np.float32(0.5),
                        j.astype(np.float32) * np.float32(0.5),
                        z.astype(np.float32) * np.float32(0.25)], axis=-1)
    else:
        i, j, k = pts[..., 0], pts[..., 1], pts[..., 2]
        s = (3 * i + 5 * j + 7 * k) % 97
        out = np.stack([i.astype(np.float32) * np.float32(0.5),
                        j.astype(np.float32) * np.float32(0.5),
                        k.astype(np.float32) * np.float32(0.5),
                        s.astype(np.float32) * np.float32(0.125)], axis=-1)
    return out.astype(np.float32)


def element_points(kind: str, cells, t: np.ndarray) -> np.ndarray:
    """Lattice points (E, K, 2|3) int64 of lattice elements ``t``."""
    t = np.asarray(t, dtype=np.int64)
    if kind == "tri":
        nx, ny = cells
        q, half = t >> 1, t & 1
        qi, qj = q // ny, q % ny
        a = np.stack([qi, qj], -1)
        b = np.stack([qi + 1, qj], -1)
        c = np.stack([qi + 1, qj + 1], -1)
        d = np.stack([qi, qj + 1], -1)
        second = np.where(half[:, None] == 1, c, b)
        third = np.where(half[:, None] == 1, d, c)
        return np.stack([a, second, third], axis=1)
    nx, ny, nz = cells
    c, s = t // 6, t % 6
    ci, cj, ck = c // (ny * nz), (c // nz) % ny, c % nz
    v0 = np.stack([ci, cj, ck], -1)
    perm = KUHN[s]
    eye = np.eye(3, dtype=np.int64)
    v1 = v0 + eye[perm[:, 0]]
    v2 = v1 + eye[perm[:, 1]]
    v3 = v0 + 1
    return np.stack([v0, v1, v2, v3], axis=1)


def point_rank(kind: str, cells, pts: np.ndarray) -> np.ndarray:
    if kind == "tri":
        nx, ny = cells
        return pts[..., 0] * (ny + 1) + pts[..., 1]
    nx, ny, nz = cells
    return (pts[..., 0] * (ny + 1) + pts[..., 1]) * (nz + 1) + pts[..., 2]


def unused_words(seed: int, ordinals: np.ndarray, dim: int) -> np.ndarray:
    """Random finite float words +-[1, 1024) for unused rows (pure integer ops)."""
    useed = splitmix64(np.uint64(seed) + np.uint64(0x5555))
    lin = ordinals.astype(np.uint64)[:, None] * np.uint64(dim) + np.arange(dim, dtype=np.uint64)
    h = splitmix64(lin ^ useed)
    expo = (np.uint64(0x7F) + ((h >> np.uint64(32)) % np.uint64(10))) << np.uint64(23)
    return ((h & np.uint64(0x807FFFFF)) | expo).astype(np.uint32)


def soup_sizes(kind: str, cells) -> dict:
    s = shape_of(kind, cells)
    n_idx = s["n_elem"] * s["arity"]
    s["n_unused"] = n_idx // 20
    s["n_vertices"] = n_idx + s["n_unused"]
    return s


def lattice_soup(kind: str, cells, seed: int = 0, n_elem_take: int | None = None):
    """(vertices float32 (V, D), elements uint32 (E, K)) of the seeded soup.

    ``n_elem_take`` keeps only the first elements (and the vertex slots before
    the next element) -- a bounded sample of the same workload.
    """
    s = soup_sizes(kind, cells)
    E, K, D = s["n_elem"], s["arity"], s["dim"]
    n_unused = s["n_unused"]
    take = E if n_elem_take is None else min(int(n_elem_take), E)
    e = np.arange(take + 1, dtype=np.int64)
    u = (e.astype(np.uint64) * np.uint64(n_unused)) // np.uint64(E)   # unused before e
    base = e * K + u.astype(np.int64)
    n_vtx = int(base[take])
    verts = np.empty((n_vtx, D), dtype=np.uint32)
    t = permute(np.arange(take, dtype=np.uint64), E, seed).astype(np.int64)
    pts = element_points(kind, cells, t)                      # (take, K, d)
    coords = point_coords(kind, cells, pts).view(np.uint32)    # (take, K, D)
    slots = base[:take, None] + np.arange(K)
    verts[slots.ravel()] = coords.reshape(-1, D)
    # unused rows: ordinals u(e) .. u(e+1)-1 sit right after element e's K rows
    n_u = int(u[take])
    if n_u:
        ords = np.arange(n_u, dtype=np.int64)
        owner = np.searchsorted(u[1:take + 1].astype(np.int64), ords, side="right")
        pos = base[owner] + K + (ords - u[owner].astype(np.int64))
        verts[pos] = unused_words(seed, ords, D)
    elements = slots.astype(np.uint32)
    return verts.view(np.float32), elements


def lattice_expected(kind: str, cells, seed: int = 0, n_elem_take: int | None = None):
    """Closed-form re-indexing result of :func:`lattice_soup` (full soups only
    have every lattice point used; for samples the used subset is ranked)."""
    s = soup_sizes(kind, cells)
    E = s["n_elem"]
    take = E if n_elem_take is None else min(int(n_elem_take), E)
    t = permute(np.arange(take, dtype=np.uint64), E, seed).astype(np.int64)
    pts = element_points(kind, cells, t)
    ranks = point_rank(kind, cells, pts)                    # (take, K) global lattice rank
    if take == E:
        n_pts = s["n_points"]
        if kind == "tri":
            nx, ny = cells
            grid = np.stack(np.meshgrid(np.arange(nx + 1), np.arange(ny + 1), indexing="ij"), -1)
        else:
            nx, ny, nz = cells
            grid = np.stack(np.meshgrid(np.arange(nx + 1), np.arange(ny + 1), np.arange(nz + 1),
                                        indexing="ij"), -1)
        out_v = point_coords(kind, cells, grid.reshape(n_pts, -1))
        return out_v, ranks.astype(np.uint32)
    used, inv = np.unique(ranks.ravel(), return_inverse=True)
    # rank -> point: invert the row-major rank
    if kind == "tri":
        nx, ny = cells
        p = np.stack([used // (ny + 1), used % (ny + 1)], -1)
    else:
        nx, ny, nz = cells
        p = np.stack([used // ((ny + 1) * (nz + 1)), (used // (nz + 1)) % (ny + 1), used % (nz + 1)], -1)
    out_v = point_coords(kind, cells, p)
    return out_v, inv.reshape(ranks.shape).astype(np.uint32)


# ---------------------------------------------------------------------------
# C2s: the C2 soup with real-valued coordinates.  Every float word w keeps its
# sign, exponent and high mantissa bits and gets its low ``bits`` mantissa bits
# XOR-ed with a hash of the whole word:
#     w' = w ^ ((w * 2654435761 mod 2^32) >> (32 - bits))
# Equal words stay equal (duplicates still weld) but >= 23 bits vary per
# component, like scanned geometry: the key no longer packs into 64 bits.
SCRAMBLE_BITS = 11


def scramble_words(words: np.ndarray, bits: int = SCRAMBLE_BITS) -> np.ndarray:
    """The C2s transform on uint32 words (any shape); returns a new uint32 array."""
    w = np.asarray(words).view(np.uint32).astype(np.uint64)
    h = ((w * np.uint64(2654435761)) & np.uint64(0xFFFFFFFF)) >> np.uint64(32 - bits)
    return (w ^ h).astype(np.uint32)


# ---------------------------------------------------------------------------
# C4: welded (indexed) tiles for merge (BASELINE configs[3]):
# tile k = the triangulated n x n quad grid whose lattice rows start at
# ``row0`` (C4: n = 5000, row0 = 4500 k -> 500 shared rows between
# neighbours), every lattice point stored ONCE (welded), + 5 % unused rows.
#
# * point p = i (n+1) + j (local, 0 <= i, j <= n) sits at position
#   q = p (row-major, like a grid generator writes it) or, with shuffle,
#   q = permute(p, n_pts, seed); position q owns slot q + u(q) with
#   u(q) = q n_unused // n_pts, and the u(q+1) - u(q) following slots hold
#   unused rows (ordinals u(q) ..), like the soup generator;
# * coordinates are those of the global lattice point (row0 + i, j);
# * element e = triangle e of the grid (row-major quads, same split as the
#   soup) or, with shuffle, triangle permute(e, E, seed + 1); indices = slots
#   of its corner points.  C4 uses the row-major tiles (SURVEY 8(d) models
#   mark/remap as streams); shuffled tiles are the random-access stress case.
#
# Merging tiles k = 0..T-1 (concatenated, indices offset) re-indexes to the
# closed form: the (row0_max + n + 1) x (n + 1) lattice points row-major.
COLS_C4 = 5000
ROW_STEP_C4 = 4500
TILES_C4 = 8


def welded_sizes(n: int) -> dict:
    n_pts = (n + 1) * (n + 1)
    n_unused = n_pts // 20
    return dict(n_points=n_pts, n_unused=n_unused, n_vertices=n_pts + n_unused, n_elem=2 * n * n)


def welded_tile(n: int, row0: int, seed: int = 0, shuffle: bool = False):
    """(vertices float32 (V, 3), elements uint32 (2 n^2, 3)) of one welded tile."""
    s = welded_sizes(n)
    n_pts, n_unused, V, E = s["n_points"], s["n_unused"], s["n_vertices"], s["n_elem"]
    p = np.arange(n_pts, dtype=np.int64)
    q = permute(p.astype(np.uint64), n_pts, seed).astype(np.int64) if shuffle else p
    uq = (q.astype(np.uint64) * np.uint64(n_unused) // np.uint64(n_pts)).astype(np.int64)
    slot_of_point = q + uq
    verts = np.empty((V, 3), dtype=np.uint32)
    pts = np.stack([row0 + p // (n + 1), p % (n + 1)], -1)
    verts[slot_of_point] = point_coords("tri", None, pts).view(np.uint32)
    # unused rows: after position q's slot, ordinals u(q) .. u(q+1)-1
    qa = np.arange(n_pts + 1, dtype=np.uint64)
    u = (qa * np.uint64(n_unused) // np.uint64(n_pts)).astype(np.int64)
    cnt = u[1:] - u[:-1]
    owners = np.repeat(np.arange(n_pts, dtype=np.int64), cnt)
    ords = np.arange(int(u[-1]), dtype=np.int64)
    if ords.size:
        verts[owners + u[owners] + 1 + (ords - u[owners])] = unused_words(seed, ords, 3)
    t = np.arange(E, dtype=np.int64)
    if shuffle:
        t = permute(t.astype(np.uint64), E, seed + 1).astype(np.int64)
    corners = element_points("tri", (n, n), t)                     # local (i, j)
    cp = corners[..., 0] * (n + 1) + corners[..., 1]
    elements = slot_of_point[cp].astype(np.uint32)
    return verts.view(np.float32), elements


def welded_merge_expected(n: int, row0s, seed: int = 0, shuffle: bool = False):
    """Closed-form merge + re-index of welded tiles at ``row0s`` (each with ``seed + k``)."""
    rows = max(row0s) + n + 1
    grid = np.stack(np.meshgrid(np.arange(rows), np.arange(n + 1), indexing="ij"), -1).reshape(-1, 2)
    out_v = point_coords("tri", None, grid)
    idx = []
    for k, r0 in enumerate(row0s):
        E = 2 * n * n
        t = np.arange(E, dtype=np.int64)
        if shuffle:
            t = permute(t.astype(np.uint64), E, seed + k + 1).astype(np.int64)
        corners = element_points("tri", (n, n), t)
        idx.append(((corners[..., 0] + r0) * (n + 1) + corners[..., 1]).astype(np.uint32))
    return out_v, np.concatenate(idx)
