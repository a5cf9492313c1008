"""GPU parity: the CUDA path against the reference's golden vectors and the CPU oracle.

Bit-exact everywhere (integer/byte work): output vertex words, output indices,
new_count and every ReindexScratch field.  Full-size configs are checked
through size-independent properties that determine the output uniquely
(strictly increasing unique rows + soup preservation + no unused vertex).
"""
import ctypes
import time

import numpy as np
import pytest

from conftest import FIELDS, all_golden, load_group
from oracle import lattice, remesh_oracle as O

pytestmark = pytest.mark.gpu

CASES = all_golden()


@pytest.fixture(scope="module")
def rmx(cuda_ok):
    import paper_2109_09812_b200 as p
    return p


def as_mesh(p, in_vtx, in_idx):
    return p.Mesh(np.asarray(in_vtx, np.uint32).view(np.float32), in_idx)


@pytest.fixture(params=["small", "large"])
def mesh_path(request, monkeypatch):
    """Run a test through the one-CTA small-mesh path and through the large-mesh pipeline."""
    monkeypatch.setenv("RMX_SMALL", "1" if request.param == "small" else "0")
    return request.param


@pytest.mark.parametrize("name,case", CASES, ids=[c[0] for c in CASES])
def test_reindex_matches_reference_golden(rmx, name, case, mesh_path):
    out, sc = rmx.reindex(as_mesh(rmx, case["in_vtx"], case["in_idx"]))
    assert np.array_equal(out.vertices.view(np.uint32), case["out_vtx"])
    assert np.array_equal(out.elements, case["out_idx"])
    assert sc.new_count == int(case["new_count"])
    for f in FIELDS:
        got = np.asarray(getattr(sc, f))
        assert got.dtype == case[f].dtype, f
        assert np.array_equal(got, case[f]), f


def test_worked_example_criterion_1(rmx):
    # reference test_acceptance.py:28-39: exact intermediates and best-of-20 < 1 ms
    c = load_group("worked")["worked"]
    mesh = as_mesh(rmx, c["in_vtx"], c["in_idx"])
    out, sc = rmx.reindex(mesh)
    assert out.n_vertices == 6
    assert out.elements.tolist() == [[0, 1, 2], [0, 2, 3], [2, 4, 5], [2, 5, 3]]
    assert sc.is_used.astype(int).tolist() == [1, 1, 1, 0, 1, 1, 1, 1, 0, 1]
    assert sc.nodup.astype(int).tolist() == [1, 0, 0, 1, 1, 0, 1, 0, 1, 1]
    assert sc.new_idx.tolist() == [0, 0, 0, 1, 2, 2, 3, 3, 4, 5]
    best = 1.0
    for _ in range(20):
        t = time.perf_counter()
        rmx.reindex(mesh)
        best = min(best, time.perf_counter() - t)
    assert best < 1e-3, best


def test_out_of_range_raises_with_issue_list(rmx, mesh_path):
    with pytest.raises(rmx.InvalidMeshError) as err:
        rmx.reindex(rmx.Mesh(np.array([(0, 0), (1, 1)], np.float32), np.array([(0, 1, 2)], np.uint32)))
    assert err.value.issues == [rmx.Issue(element=0, slot=2, index=2)]
    with pytest.raises(rmx.InvalidMeshError) as err:
        rmx.reindex(rmx.Mesh(np.zeros((1, 2), np.float32), np.array([(0, 5, 7), (9, 0, 0)], np.uint32)))
    assert len(err.value.issues) == 3 and err.value.issues[0] == rmx.Issue(0, 1, 5)
    # the pipeline keeps working afterwards (status is per call)
    out, _ = rmx.reindex(rmx.Mesh(np.array([(0, 0), (1, 1)], np.float32), np.array([(0, 1, 1)], np.uint32)))
    assert out.n_vertices == 2


def test_zero_elements(rmx):
    out, sc = rmx.reindex(rmx.Mesh(np.zeros((3, 2), np.float32), np.empty((0, 4), np.uint32)))
    assert out.n_vertices == 0 and out.n_elements == 0 and out.dim == 2 and out.arity == 4
    assert sc.is_used.tolist() == [False] * 3 and sc.new_count == 0
    assert len(sc.org_id) == 0 and len(sc.perm) == 0


def test_dim_limit_is_a_mesh_error(rmx):
    with pytest.raises(rmx.MeshError):
        rmx.reindex(rmx.Mesh(np.zeros((2, 33), np.float32), np.array([(0, 1)], np.uint32)))


def test_idempotent_and_tensor_api(rmx, mesh_path):
    import torch
    c = load_group("random")["random_big"]
    mesh = as_mesh(rmx, c["in_vtx"], c["in_idx"])
    once, _ = rmx.reindex(mesh)
    twice, _ = rmx.reindex(once)
    assert rmx.bitwise_equal(once, twice)
    dv = torch.from_numpy(mesh.vertices.view(np.int32).copy()).cuda()
    de = torch.from_numpy(mesh.elements.view(np.int32).copy()).cuda()
    res = rmx.reindex_tensors(dv, de)
    assert np.array_equal(res.vertices.cpu().numpy().view(np.uint32), once.vertices.view(np.uint32))
    assert np.array_equal(res.elements.cpu().numpy().view(np.uint32), once.elements)


def random_bits_mesh(seed, V, D, E, K, pool=None):
    rng = np.random.default_rng(seed)
    if pool is None:
        words = rng.integers(0, 1 << 32, size=(V, D), dtype=np.uint64).astype(np.uint32)
        words[rng.random((V, D)) < 0.5] &= 0xFF00FF00       # plenty of equal bytes / rows
    else:
        words = rng.integers(0, pool, size=(V, D)).astype(np.uint32) * np.uint32(0x01010101)
    idx = rng.integers(0, max(1, V - V // 10), size=(E, K)).astype(np.uint32)
    return words, idx


@pytest.mark.parametrize("seed,V,D,E,K,pool", [
    (1, 100_000, 3, 40_000, 3, None), (2, 250_000, 2, 90_000, 4, 7), (3, 300_000, 4, 70_000, 4, None),
    (4, 70_000, 1, 30_000, 2, None), (5, 1_000_000, 3, 400_000, 3, 50), (6, 50_000, 7, 20_000, 3, 3),
    (7, 123_457, 5, 33_333, 5, None), (8, 2_000_000, 3, 700_000, 3, None)])
def test_random_bits_vs_oracle(rmx, seed, V, D, E, K, pool):
    words, idx = random_bits_mesh(seed, V, D, E, K, pool)
    ref = O.reindex(words, idx)
    out, sc = rmx.reindex(rmx.Mesh(words.view(np.float32), idx))
    assert np.array_equal(out.vertices.view(np.uint32), ref["vertices"].view(np.uint32))
    assert np.array_equal(out.elements, ref["elements"])
    if V <= 300_000:
        for f in FIELDS:
            assert np.array_equal(np.asarray(getattr(sc, f)), ref[f]), f


def _gen_device(rmx, kind, cells, seed, take=None):
    import torch
    from paper_2109_09812_b200 import _native
    lib = _native.lib()
    k = 0 if kind == "tri" else 1
    nz = cells[2] if len(cells) == 3 else 0
    E, V = ctypes.c_uint64(), ctypes.c_uint64()
    t = (1 << 63) if take is None else take
    assert lib.rmx_lattice_sizes(k, cells[0], cells[1], nz, t, ctypes.byref(E), ctypes.byref(V)) == 0
    n_take = E.value if take is None else min(take, E.value)
    D = 3 if kind == "tri" else 4
    vtx = torch.empty((V.value, D), dtype=torch.int32, device="cuda")
    idx = torch.empty((n_take, D), dtype=torch.int32, device="cuda")
    assert lib.rmx_gen_lattice_soup(k, cells[0], cells[1], nz, seed, t, vtx.data_ptr(), idx.data_ptr(),
                                    torch.cuda.current_stream().cuda_stream) == 0
    return vtx, idx


@pytest.mark.parametrize("kind,cells,take", [("tri", (7, 5), None), ("tet", (3, 4, 2), None),
                                             ("tri", (300, 200), None), ("tet", (20, 21, 22), 5000)])
def test_device_generator_matches_numpy(rmx, kind, cells, take):
    v, e = lattice.lattice_soup(kind, cells, seed=11, n_elem_take=take)
    dv, de = _gen_device(rmx, kind, cells, 11, take)
    assert np.array_equal(dv.cpu().numpy().view(np.uint32), v.view(np.uint32))
    assert np.array_equal(de.cpu().numpy().view(np.uint32), e)


def test_config1_full_vs_oracle(rmx):
    kind, cells = lattice.CONFIGS["C1"]
    v, e = lattice.lattice_soup(kind, cells, seed=0)
    ref = O.reindex(v, e)
    out, sc = rmx.reindex(rmx.Mesh(v, e))
    assert out.n_vertices == 501_426 == ref["new_count"]
    assert np.array_equal(out.vertices.view(np.uint32), ref["vertices"].view(np.uint32))
    assert np.array_equal(out.elements, ref["elements"])
    for f in FIELDS:
        assert np.array_equal(np.asarray(getattr(sc, f)), ref[f]), f


def _u64(t):
    import torch
    return t.to(torch.int64) & 0xFFFFFFFF


def check_determining_properties(vtx, idx, out_v, out_e, expect_count):
    """Strictly increasing rows + every row used + soup preserved <=> the reference output."""
    import torch
    U, D = out_v.shape
    assert U == expect_count
    a, b = _u64(out_v[:-1]), _u64(out_v[1:])
    lt = torch.zeros(U - 1, dtype=torch.bool, device=out_v.device)
    eq = torch.ones_like(lt)
    for c in range(D):
        lt |= eq & (a[:, c] < b[:, c])
        eq &= a[:, c] == b[:, c]
    assert bool(lt.all())
    used = torch.zeros(U, dtype=torch.bool, device=out_v.device)
    used[out_e.reshape(-1).long()] = True
    assert bool(used.all())
    chunk = 1 << 24
    fi, fo = idx.reshape(-1), out_e.reshape(-1)
    for s in range(0, fi.numel(), chunk):
        assert torch.equal(vtx[fi[s:s + chunk].long()], out_v[fo[s:s + chunk].long()])


@pytest.mark.parametrize("cfg", ["C2", "C3"])
def test_full_size_configs(rmx, cfg):
    import torch
    kind, cells = lattice.CONFIGS[cfg]
    vtx, idx = _gen_device(rmx, kind, cells, 0)
    res = rmx.reindex_tensors(vtx, idx)
    check_determining_properties(vtx, idx, res.vertices, res.elements, lattice.shape_of(kind, cells)["n_points"])
    # exact global ranks of the first elements against the closed form
    E = lattice.shape_of(kind, cells)["n_elem"]
    t = lattice.permute(np.arange(2000, dtype=np.uint64), E, 0).astype(np.int64)
    want = lattice.point_rank(kind, cells, lattice.element_points(kind, cells, t)).astype(np.uint32)
    assert np.array_equal(res.elements[:2000].cpu().numpy().view(np.uint32), want)
    del res, vtx, idx
    torch.cuda.empty_cache()


def test_c5_shard_full_size(rmx):
    """One GPU's shard of C5 at 8 GPUs (first 1/8 of the 1B-triangle soup, 393.75M vertex slots):
    index arithmetic past 2^28 rows, 128K+ tiles per pass, output determined by properties."""
    import torch
    from paper_2109_09812_b200 import gen
    kind, cells = lattice.CONFIGS["C5"]
    E_all, _ = gen.lattice_sizes(kind, cells)
    vtx, idx = gen.lattice_soup_tensors(kind, cells, seed=0, n_elem_take=E_all // 8)
    assert vtx.shape[0] == 393_750_000
    res = rmx.reindex_tensors(vtx, idx)
    U = res.vertices.shape[0]
    assert 0 < U < vtx.shape[0]
    check_determining_properties(vtx, idx, res.vertices, res.elements, U)
    del res, vtx, idx
    torch.cuda.empty_cache()


def test_native_library_is_the_loaded_code(rmx):
    rmx.reindex(rmx.Mesh(np.zeros((2, 2), np.float32), np.array([(0, 1)], np.uint32)))
    import os
    from paper_2109_09812_b200 import _native
    maps = open("/proc/self/maps").read()
    assert os.path.basename(_native.LIB_PATH) in maps and "librmx_b200" in maps


def test_c4_merge_full_size(rmx):
    """BASELINE configs[3] at one GPU: 8 welded 5000 x 5000 tiles (500 shared rows) merged on the
    device -- 210,084,008 vertex slots in, 182,541,501 out; determining properties + closed-form
    ranks of sampled elements of every tile."""
    import torch
    C, S, T = lattice.COLS_C4, lattice.ROW_STEP_C4, lattice.TILES_C4
    pieces = [rmx.gen.welded_tile_tensors(C, S * k, k) for k in range(T)]
    vtx = torch.cat([p[0] for p in pieces])
    offs = np.cumsum([0] + [p[0].shape[0] for p in pieces])[:-1]
    res = rmx.merge_tensors(pieces)
    assert vtx.shape[0] == 210_084_008
    assert res.vertices.shape[0] == 182_541_501
    E = 2 * C * C
    for k in (0, 3, T - 1):
        t = np.arange(E - 500, E, dtype=np.int64)
        corners = lattice.element_points("tri", (C, C), t)
        want = ((corners[..., 0] + S * k) * (C + 1) + corners[..., 1]).astype(np.uint32)
        got = res.elements[k * E + E - 500:(k + 1) * E].cpu().numpy().view(np.uint32)
        assert np.array_equal(got, want)
    idx = torch.cat([(p[1].to(torch.int64) + int(o)).to(torch.int32) for p, o in zip(pieces, offs)])
    del pieces
    check_determining_properties(vtx, idx, res.vertices, res.elements, 182_541_501)
    del res, vtx, idx
    torch.cuda.empty_cache()


def test_more_than_2_31_vertices(rmx):
    """V = 2^31 + 4099 one-word vertices, every row used once (arity 1): indices and positions past
    the int32 range, 700K tiles per pass.  Output checked by the determining properties, chunked."""
    import torch
    V = (1 << 31) + 4099
    free, _ = torch.cuda.mem_get_info()
    if free < 120 * (1 << 30):
        pytest.skip(f"needs ~120 GB free device memory, have {free / 2**30:.0f} GB")
    dev = torch.device("cuda")
    ar = torch.arange(V, dtype=torch.int64, device=dev)
    # 2^30 distinct values (x * odd constant mod 2^30), bit 31 set on half of them
    vals = ((ar * 2654435761) & ((1 << 30) - 1)) | ((ar & 1) << 31)
    vtx = torch.where(vals >= 2**31, vals - 2**32, vals).to(torch.int32).view(V, 1)
    idx = torch.where(ar >= 2**31, ar - 2**32, ar).to(torch.int32).view(V, 1)
    del ar, vals
    res = rmx.reindex_tensors(vtx, idx)
    out_v, out_e = res.vertices, res.elements
    U = out_v.shape[0]
    assert 0 < U <= V
    chunk = 1 << 27
    for s in range(0, U - 1, chunk):
        a = out_v[s:s + chunk + 1].view(-1).to(torch.int64) & 0xFFFFFFFF
        assert bool((a[1:] > a[:-1]).all())
    for s in range(0, V, chunk):
        e = out_e[s:s + chunk].view(-1).to(torch.int64) & 0xFFFFFFFF
        assert torch.equal(out_v.view(-1)[e], vtx.view(-1)[s:s + chunk])
    del res, out_v, out_e, vtx, idx
    torch.cuda.empty_cache()


@pytest.mark.parametrize("V,D,E,K", [(1, 1, 1, 1), (3072, 8, 3000, 3), (8192, 3, 65_536, 4), (1000, 5, 1, 2),
                                     (8191, 1, 5000, 1), (4500, 2, 32_768, 4), (2049, 7, 999, 3),
                                     (8192, 3, 70_000, 4)])
def test_small_path_limits_vs_oracle(rmx, V, D, E, K, mesh_path):
    """Edges of the one-CTA path (V = 8192, V D = 24576, I = 2^18) and just past them, both paths."""
    rng = np.random.default_rng(V + D + E)
    words = rng.integers(0, 8, size=(V, D)).astype(np.uint32) * np.uint32(0x9E3779B1)
    idx = rng.integers(0, V, size=(E, K)).astype(np.uint32)
    ref = O.reindex(words, idx)
    out, sc = rmx.reindex(rmx.Mesh(words.view(np.float32), idx))
    assert np.array_equal(out.vertices.view(np.uint32), ref["vertices"].view(np.uint32))
    assert np.array_equal(out.elements, ref["elements"])
    for f in FIELDS:
        assert np.array_equal(np.asarray(getattr(sc, f)), ref[f]), f


@pytest.mark.parametrize("D,pool", [(9, None), (16, None), (32, None), (12, 3), (32, 2), (6, 5)])
def test_wide_dims_vs_oracle(rmx, D, pool, mesh_path):
    """D up to RMX_MAX_DIM = 32 words per vertex: the generic-width AoS rows (random bits) and the
    generic packed path (few varying bits), both mesh paths where they apply, scratch included."""
    words, idx = random_bits_mesh(D * 7 + (pool or 0), 20_000, D, 9_000, 3, pool)
    ref = O.reindex(words, idx)
    out, sc = rmx.reindex(rmx.Mesh(words.view(np.float32), idx))
    assert np.array_equal(out.vertices.view(np.uint32), ref["vertices"].view(np.uint32))
    assert np.array_equal(out.elements, ref["elements"])
    for f in FIELDS:
        assert np.array_equal(np.asarray(getattr(sc, f)), ref[f]), f


@pytest.mark.parametrize("env", [{"RMX_PDL": "0"}, {"RMX_VALUE_RANK": "0"}, {"RMX_PDL": "0", "RMX_VALUE_RANK": "0"},
                                 {"RMX_DS": "2"}, {"RMX_DS": "2", "RMX_DS2": "24x256x2"},
                                 {"RMX_DS": "2", "RMX_DS2": "12x256x4"}, {"RMX_HASH": "0"}],
                         ids=["no-pdl", "no-value-rank", "neither", "ds2", "ds2-24x256", "ds2-12x256", "no-hash"])
def test_switches_keep_results(rmx, monkeypatch, env):
    """The A/B switches change speed, never results: golden cases through the
    large-mesh pipeline and a lattice soup with value ranks, each switch off."""
    monkeypatch.setenv("RMX_SMALL", "0")
    for k, v in env.items():
        monkeypatch.setenv(k, v)
    for name, case in CASES[::7]:
        out, sc = rmx.reindex(as_mesh(rmx, case["in_vtx"], case["in_idx"]))
        assert np.array_equal(out.vertices.view(np.uint32), case["out_vtx"]), name
        assert np.array_equal(out.elements, case["out_idx"]), name
        assert np.array_equal(np.asarray(sc.org_id), case["org_id"]), name
    v, e = lattice.lattice_soup("tri", (60, 70), seed=3)
    ref = O.reindex(v.view(np.uint32), e)
    out, sc = rmx.reindex(rmx.Mesh(v, e))
    assert np.array_equal(out.vertices.view(np.uint32), ref["vertices"].view(np.uint32))
    assert np.array_equal(out.elements, ref["elements"])
    assert np.array_equal(np.asarray(sc.org_id), ref["org_id"])
    # u64 packed keys (> 32 varying bits, several partial tiles) through the same passes
    rng = np.random.default_rng(5)
    words = (rng.integers(0, 1 << 12, size=(50_000, 4)).astype(np.uint32) << np.uint32(9)) | np.uint32(0x3F800000)
    idx = rng.integers(0, 50_000, size=(30_000, 3)).astype(np.uint32)
    ref = O.reindex(words, idx)
    out, sc = rmx.reindex(rmx.Mesh(words.view(np.float32), idx))
    assert np.array_equal(out.vertices.view(np.uint32), ref["vertices"].view(np.uint32))
    assert np.array_equal(out.elements, ref["elements"])
    assert np.array_equal(np.asarray(sc.org_id), ref["org_id"])


def test_misaligned_workspace_is_einval(rmx):
    """The workspace is carved into 256-byte aligned arrays that bulk copies and 16-byte loads
    read: a misaligned workspace pointer is rejected before any launch."""
    import torch
    from paper_2109_09812_b200 import _native
    V, D, E, K = 4096, 3, 1024, 3
    g = torch.Generator().manual_seed(3)
    vtx = torch.randint(0, 1 << 20, (V, D), generator=g, dtype=torch.int32).cuda()
    idx = torch.randint(0, V, (E, K), generator=g, dtype=torch.int32).cuda()
    out_v = torch.empty((V, D), dtype=torch.int32, device="cuda")
    out_e = torch.empty((E, K), dtype=torch.int32, device="cuda")
    info = torch.zeros(2, dtype=torch.int64, device="cuda")
    lib = _native.lib()
    wsb = lib.rmx_workspace_bytes(V, D, E, K)
    ws = torch.empty(wsb + 256, dtype=torch.uint8, device="cuda")
    args = [vtx.data_ptr(), V, D, idx.data_ptr(), E, K, out_v.data_ptr(), out_e.data_ptr(),
            info.data_ptr(), info.data_ptr() + 8]
    stream = torch.cuda.current_stream().cuda_stream
    rc = lib.rmx_reindex(*args, ws.data_ptr() + 16, wsb, None, stream)
    assert rc == _native.RMX_EINVAL and b"aligned" in lib.rmx_strerror(rc)
    assert lib.rmx_reindex(*args, ws.data_ptr(), wsb, None, stream) == _native.RMX_OK
    torch.cuda.synchronize()
    count, status = (int(x) for x in info.cpu())
    assert status == 0 and 0 < count <= V
