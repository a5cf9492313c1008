"""GPU: the host-to-host entry points (Reindexer, ReindexStream) against the oracle.

Both wrap the same ``rmx_reindex`` call as :func:`reindex`; these tests pin the
buffer handling around it -- pinned copies, capacity slicing, double-buffered
slots, the count-dependent vertex read-back, errors in the middle of a stream.
"""
import numpy as np
import pytest
import torch

from oracle import remesh_oracle as O

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def rmx(cuda_ok):
    import paper_2109_09812_b200 as p
    return p


def random_mesh(seed, V, D, E, K, pool=64):
    rng = np.random.default_rng(seed)
    vals = rng.integers(0, 1 << 32, size=pool, dtype=np.uint64).astype(np.uint32)
    v = vals[rng.integers(0, pool, size=(V, D))]
    # leave the tail unused, repeat rows so duplicates exist
    v[V // 2:] = v[rng.integers(0, max(1, V // 2), size=V - V // 2)]
    e = rng.integers(0, max(1, (V * 9) // 10), size=(E, K)).astype(np.uint32)
    return v, e


def pinned(v, e):
    hv = torch.from_numpy(np.ascontiguousarray(v).view(np.int32)).pin_memory()
    he = torch.from_numpy(np.ascontiguousarray(e).view(np.int32)).pin_memory()
    return hv, he


def expect(v, e):
    r = O.reindex(v.view(np.float32), e)
    return np.asarray(r["vertices"]).view(np.uint32), np.asarray(r["elements"])


def test_reindexer_repeated_calls(rmx):
    v, e = random_mesh(1, 5000, 3, 3000, 3)
    rx = rmx.Reindexer(5000, 3, 3000, 3)
    hv, he = pinned(v, e)
    ev, ee = expect(v, e)
    for _ in range(3):
        gv, ge = rx.run(hv, he)
        assert np.array_equal(gv.view(np.uint32), ev)
        assert np.array_equal(ge, ee)


@pytest.mark.parametrize("depth", [2, 3])
def test_stream_matches_oracle_in_order(rmx, depth):
    shapes = [(5000, 3000), (1, 4), (777, 50), (5000, 3000), (4096, 2999), (300, 0), (2, 1), (4999, 1234)]
    meshes = [random_mesh(10 + i, V, 3, E, 4) for i, (V, E) in enumerate(shapes)]
    rs = rmx.ReindexStream(5000, 3, 3000, 4, depth=depth)
    got = [(gv.copy(), ge.copy()) for gv, ge in rs.run(pinned(v, e) for v, e in meshes)]
    assert len(got) == len(meshes)
    for (v, e), (gv, ge) in zip(meshes, got):
        if e.shape[0] == 0:
            assert gv.shape == (0, 3) and ge.shape == (0, 4)
            continue
        ev, ee = expect(v, e)
        assert np.array_equal(gv.view(np.uint32), ev)
        assert np.array_equal(ge, ee)
    assert rs.last_counts[0] == expect(*meshes[0])[0].shape[0]


def test_stream_views_valid_until_next(rmx):
    meshes = [random_mesh(40 + i, 2000, 2, 1500, 3, pool=16) for i in range(5)]
    rs = rmx.ReindexStream(2000, 2, 1500, 3)
    for (v, e), (gv, ge) in zip(meshes, rs.run(pinned(v, e) for v, e in meshes)):
        ev, ee = expect(v, e)
        assert np.array_equal(gv.view(np.uint32), ev)
        assert np.array_equal(ge, ee)


def test_stream_out_of_range_raises(rmx):
    good = random_mesh(3, 100, 3, 80, 3)
    bad_v, bad_e = random_mesh(4, 100, 3, 80, 3)
    bad_e = bad_e.copy()
    bad_e[7, 1] = 100
    rs = rmx.ReindexStream(100, 3, 80, 3)
    it = rs.run(pinned(v, e) for v, e in [good, (bad_v, bad_e), good])
    gv, ge = next(it)
    assert np.array_equal(ge, expect(*good)[1])
    with pytest.raises(rmx.InvalidMeshError) as ei:
        next(it)
    assert ei.value.issues[0] == rmx.Issue(7, 1, 100)


def test_stream_capacity_and_shape_errors(rmx):
    rs = rmx.ReindexStream(100, 3, 80, 3)
    v, e = random_mesh(5, 101, 3, 80, 3)
    with pytest.raises(rmx.MeshError):
        list(rs.run([pinned(v, e)]))
    v, e = random_mesh(5, 50, 2, 40, 3)
    with pytest.raises(rmx.MeshError):
        list(rs.run([pinned(v, e)]))


def _graph_run(rmx, g, bufs, v, e, expect_ok=True):
    vt, it, ov, oe, info = bufs
    vt.copy_(torch.from_numpy(np.ascontiguousarray(v).view(np.int32)))
    it.copy_(torch.from_numpy(np.ascontiguousarray(e).view(np.int32)))
    s = torch.cuda.current_stream()
    g.launch(s)
    s.synchronize()
    count, status = (int(x) for x in info.cpu())
    return count, status, ov[:count].cpu().numpy().view(np.uint32), oe.cpu().numpy().view(np.uint32)


@pytest.mark.parametrize("D,K", [(1, 2), (2, 4), (3, 3), (4, 4), (7, 3)])
def test_graph_switches_paths_per_launch(rmx, D, K):
    """One captured graph, relaunched on packed-key data, then wide-key data (> 64 varying bits:
    hash mode for D = 3..8), then packed again: the kernels follow each input's plan on the device;
    every result matches the oracle."""
    from paper_2109_09812_b200 import pipeline
    V, E = 20_000, 9_000
    dev = torch.device("cuda")
    vt = torch.empty((V, D), dtype=torch.int32, device=dev)
    it = torch.empty((E, K), dtype=torch.int32, device=dev)
    ov, oe = torch.empty_like(vt), torch.empty_like(it)
    info = torch.zeros(2, dtype=torch.int64, device=dev)
    ws = torch.empty(pipeline.workspace_bytes(V, D, E, K), dtype=torch.uint8, device=dev)
    g = pipeline.PipelineGraph(vt, V, D, it, E, K, ov, oe, info, ws)
    rng = np.random.default_rng(D)
    for mode in ("pool", "raw", "pool", "raw"):
        if mode == "pool":
            v = rng.integers(0, 40, size=(V, D)).astype(np.uint32) * np.uint32(0x00010001)
        else:
            v = rng.integers(0, 1 << 32, size=(V, D), dtype=np.uint64).astype(np.uint32)
        e = rng.integers(0, V - 100, size=(E, K)).astype(np.uint32)
        count, status, gv, ge = _graph_run(rmx, g, (vt, it, ov, oe, info), v, e)
        ev, ee = expect(v, e)
        assert status == 0 and count == ev.shape[0]
        assert np.array_equal(gv, ev)
        assert np.array_equal(ge, ee)


def test_graph_out_of_range_status(rmx):
    from paper_2109_09812_b200 import pipeline
    V, D, E, K = 1000, 3, 500, 3
    dev = torch.device("cuda")
    vt = torch.empty((V, D), dtype=torch.int32, device=dev)
    it = torch.empty((E, K), dtype=torch.int32, device=dev)
    ov, oe = torch.empty_like(vt), torch.empty_like(it)
    info = torch.zeros(2, dtype=torch.int64, device=dev)
    ws = torch.empty(pipeline.workspace_bytes(V, D, E, K), dtype=torch.uint8, device=dev)
    g = pipeline.PipelineGraph(vt, V, D, it, E, K, ov, oe, info, ws)
    v, e = random_mesh(9, V, D, E, K)
    bad = e.copy()
    bad[3, 2] = V + 5
    _, status, _, _ = _graph_run(rmx, g, (vt, it, ov, oe, info), v, bad)
    assert status & 1
    count, status, gv, ge = _graph_run(rmx, g, (vt, it, ov, oe, info), v, e)   # status resets per launch
    ev, ee = expect(v, e)
    assert status == 0 and np.array_equal(gv, ev) and np.array_equal(ge, ee)


def test_concurrent_calls_from_threads(rmx):
    """The C-ABI is reentrant: 8 host threads re-index meshes of different sizes and dims at once
    (small-mesh and large-mesh paths, different shared-memory needs) on one device."""
    import threading
    jobs = []
    for t in range(8):
        D = 1 + t % 4
        V = [300, 5000, 8000, 40_000][t % 4]
        jobs.append(random_mesh(100 + t, V, D, V // 2, 3, pool=50))
    results, errors = [None] * len(jobs), []

    def run(k):
        try:
            out = []
            for _ in range(4):
                v, e = jobs[k]
                res = rmx.reindex_tensors(torch.from_numpy(v.view(np.int32)).cuda(),
                                          torch.from_numpy(e.view(np.int32)).cuda())
                out.append((res.vertices.cpu().numpy().view(np.uint32), res.elements.cpu().numpy().view(np.uint32)))
            results[k] = out
        except BaseException as exc:  # noqa: BLE001
            errors.append(exc)

    threads = [threading.Thread(target=run, args=(k,)) for k in range(len(jobs))]
    for th in threads:
        th.start()
    for th in threads:
        th.join()
    assert not errors, errors[0]
    for (v, e), outs in zip(jobs, results):
        ev, ee = expect(v, e)
        for gv, ge in outs:
            assert np.array_equal(gv, ev) and np.array_equal(ge, ee)


@pytest.mark.parametrize("V,D,E,K", [(50_000, 3, 30_000, 3), (20_000, 4, 9_000, 4), (300, 3, 200, 3)])
def test_unaligned_device_buffers(rmx, V, D, E, K):
    """Vertex/index tensors that start off a 16-byte boundary (slices of bigger buffers): the
    vectorised and bulk-copy paths must fall back, results unchanged."""
    v, e = random_mesh(7 + D, V, D, E, K, pool=40)
    ev, ee = expect(v, e)
    big_v = torch.zeros((V + 1) * D + 1, dtype=torch.int32, device="cuda")
    big_e = torch.zeros(E * K + 3, dtype=torch.int32, device="cuda")
    tv = big_v[1:1 + V * D].view(V, D)          # 4-byte offset
    te = big_e[3:3 + E * K].view(E, K)          # 12-byte offset
    tv.copy_(torch.from_numpy(v.view(np.int32)))
    te.copy_(torch.from_numpy(e.view(np.int32)))
    assert tv.data_ptr() % 16 and te.data_ptr() % 16
    res = rmx.reindex_tensors(tv, te)
    assert np.array_equal(res.vertices.cpu().numpy().view(np.uint32), ev)
    assert np.array_equal(res.elements.cpu().numpy().view(np.uint32), ee)


@pytest.mark.parametrize("V,D,E,K", [(320, 3, 128, 3), (20_000, 3, 9_000, 4), (60_000, 5, 30_000, 3),
                                     (100_000, 2, 60_000, 3)])
def test_small_call_path_matches_staged_path(rmx, monkeypatch, V, D, E, K):
    """reindex() stages meshes <= SMALL_CALL_BYTES through one pinned round trip; with the limit at
    0 the same meshes take the general path (separate copies, pageable staging).  Both match the
    oracle incl. the lazy scratch, and errors are the same."""
    from paper_2109_09812_b200 import pipeline
    v, e = random_mesh(7 + V, V, D, E, K, pool=40)
    ev, ee = expect(v, e)
    ref = O.reindex(v.view(np.float32), e)
    for limit in (pipeline.SMALL_CALL_BYTES, 0):
        monkeypatch.setattr(pipeline, "SMALL_CALL_BYTES", limit)
        out, sc = rmx.reindex(rmx.Mesh(v.view(np.float32), e))
        assert np.array_equal(out.vertices.view(np.uint32), ev)
        assert np.array_equal(out.elements, ee)
        assert sc.new_count == len(ev)
        assert np.array_equal(np.asarray(sc.org_id), ref["org_id"])
        bad = e.copy()
        bad[E // 2, 0] = V + 3
        with pytest.raises(rmx.InvalidMeshError) as ei:
            rmx.reindex(rmx.Mesh(v.view(np.float32), bad))
        assert [(i.element, i.slot, i.index) for i in ei.value.issues] == [(E // 2, 0, V + 3)]


def test_small_call_path_threads(rmx):
    """Per-thread staging buffers: concurrent small reindex() calls do not interfere."""
    import threading
    jobs = [random_mesh(300 + t, [300, 4000, 9000, 30_000][t % 4], 1 + t % 4, 500 + 100 * t, 3, pool=30)
            for t in range(8)]
    want = [expect(v, e) for v, e in jobs]
    errors = []

    def run(k):
        try:
            v, e = jobs[k]
            for _ in range(10):
                out, _ = rmx.reindex(rmx.Mesh(v.view(np.float32), e))
                assert np.array_equal(out.vertices.view(np.uint32), want[k][0])
                assert np.array_equal(out.elements, want[k][1])
        except BaseException as exc:  # noqa: BLE001
            errors.append(exc)

    threads = [threading.Thread(target=run, args=(k,)) for k in range(len(jobs))]
    for th in threads:
        th.start()
    for th in threads:
        th.join()
    assert not errors, errors[0]
