"""Composition ops: host-side argument checks (CPU) and GPU parity with the
reference remeshx.merge / soup_to_mesh / subset golden vectors."""
import numpy as np
import pytest

from conftest import load_group


def test_merge_argument_errors_cpu():
    import paper_2109_09812_b200 as rmx
    with pytest.raises(rmx.MeshError):
        rmx.merge([])
    tri = rmx.Mesh(np.zeros((3, 2), np.float32), np.array([(0, 1, 2)], np.uint32))
    quad = rmx.Mesh(np.zeros((4, 2), np.float32), np.array([(0, 1, 2, 3)], np.uint32))
    with pytest.raises(rmx.MeshError):
        rmx.merge([tri, quad])
    bad = rmx.Mesh(np.zeros((1, 2), np.float32), np.array([(0, 0, 5)], np.uint32))
    with pytest.raises(rmx.InvalidMeshError):
        rmx.merge([bad])


def test_subset_selector_errors_cpu():
    import paper_2109_09812_b200 as rmx
    m = rmx.Mesh(np.zeros((3, 2), np.float32), np.array([(0, 1, 2)] * 4, np.uint32))
    for keep in ([0, 9], [2, 1], np.array([True, False]), [0.5]):
        with pytest.raises(rmx.MeshError):
            rmx.subset(m, keep)


def test_soup_errors_cpu():
    import paper_2109_09812_b200 as rmx
    with pytest.raises(rmx.MeshError):
        rmx.soup_to_mesh([[[0, 0], [1, 1], [2, 2]], [[0, 0], [1, 1]]])
    with pytest.raises(rmx.MeshError):
        rmx.soup_to_mesh(np.zeros((3, 3), np.float32))
    e = rmx.soup_to_mesh(np.empty((0, 3, 2), np.float32))
    assert e.n_vertices == 0 and e.arity == 3 and e.dim == 2


def _cases(prefix):
    g = load_group("ops")
    return sorted((k, v) for k, v in g.items() if k.startswith(prefix))


@pytest.mark.gpu
@pytest.mark.parametrize("name,case", _cases("merge"), ids=[c[0] for c in _cases("merge")])
def test_merge_matches_reference(cuda_ok, name, case):
    import paper_2109_09812_b200 as rmx
    parts = [rmx.Mesh(case[f"piece_vtx_{k}"].view(np.float32), case[f"piece_idx_{k}"])
             for k in range(int(case["n_pieces"]))]
    out = rmx.merge(parts)
    assert np.array_equal(out.vertices.view(np.uint32), case["out_vtx"])
    assert np.array_equal(out.elements, case["out_idx"])


@pytest.mark.gpu
@pytest.mark.parametrize("name,case", _cases("soup"), ids=[c[0] for c in _cases("soup")])
def test_soup_to_mesh_matches_reference(cuda_ok, name, case):
    import paper_2109_09812_b200 as rmx
    out = rmx.soup_to_mesh(case["soup"].view(np.float32))
    assert np.array_equal(out.vertices.view(np.uint32), case["out_vtx"])
    assert np.array_equal(out.elements, case["out_idx"])


@pytest.mark.gpu
@pytest.mark.parametrize("name,case", _cases("subset"), ids=[c[0] for c in _cases("subset")])
def test_subset_matches_reference(cuda_ok, name, case):
    import paper_2109_09812_b200 as rmx
    m = rmx.Mesh(case["in_vtx"].view(np.float32), case["in_idx"])
    keep = case["keep"]
    out = rmx.subset(m, keep)
    assert np.array_equal(out.vertices.view(np.uint32), case["out_vtx"])
    assert np.array_equal(out.elements, case["out_idx"])
    mask = np.zeros(m.n_elements, bool)
    mask[keep] = True
    assert rmx.bitwise_equal(rmx.subset(m, mask), out)


@pytest.mark.gpu
def test_merge_empties_and_single(cuda_ok):
    import paper_2109_09812_b200 as rmx
    e = rmx.merge([rmx.Mesh.empty(), rmx.Mesh.empty()])
    assert e.n_vertices == 0 and e.n_elements == 0
    c = load_group("worked")["worked"]
    w = rmx.Mesh(c["in_vtx"].view(np.float32), c["in_idx"])
    assert rmx.bitwise_equal(rmx.merge([w]), rmx.reindex(w)[0])


@pytest.mark.gpu
@pytest.mark.parametrize("name,case", _cases("merge"), ids=[c[0] for c in _cases("merge")])
def test_merge_tensors_matches_reference(cuda_ok, name, case):
    """The device-resident merge (offset kernel + re-index) against the reference merge."""
    import torch

    import paper_2109_09812_b200 as rmx
    pieces = []
    for k in range(int(case["n_pieces"])):
        v = torch.from_numpy(case[f"piece_vtx_{k}"].view(np.int32).copy()).cuda()
        e = torch.from_numpy(case[f"piece_idx_{k}"].view(np.int32).copy()).cuda()
        pieces.append((v, e))
    res = rmx.merge_tensors(pieces)
    assert np.array_equal(res.vertices.cpu().numpy().view(np.uint32), case["out_vtx"])
    assert np.array_equal(res.elements.cpu().numpy().view(np.uint32), case["out_idx"])


@pytest.mark.gpu
@pytest.mark.parametrize("n,row0,seed,shuffle", [(1, 0, 0, False), (6, 4, 1, True), (13, 100, 7, False),
                                                  (40, 36, 3, True), (17, 9, 2, True)])
def test_welded_tile_generator_matches_oracle(cuda_ok, n, row0, seed, shuffle):
    from oracle import lattice

    from paper_2109_09812_b200 import gen
    vtx, idx = gen.welded_tile_tensors(n, row0, seed, shuffle)
    v, e = lattice.welded_tile(n, row0, seed, shuffle)
    assert np.array_equal(vtx.cpu().numpy().view(np.uint32), v.view(np.uint32))
    assert np.array_equal(idx.cpu().numpy().view(np.uint32), e)


@pytest.mark.gpu
def test_merge_tensors_welded_tiles_closed_form(cuda_ok):
    from oracle import lattice

    import paper_2109_09812_b200 as rmx
    n, row0s = 30, [0, 25, 50, 75]
    for shuffle in (False, True):
        pieces = [rmx.gen.welded_tile_tensors(n, r0, k, shuffle) for k, r0 in enumerate(row0s)]
        res = rmx.merge_tensors(pieces)
        ev, ei = lattice.welded_merge_expected(n, row0s, shuffle=shuffle)
        assert np.array_equal(res.vertices.cpu().numpy().view(np.uint32), ev.view(np.uint32))
        assert np.array_equal(res.elements.cpu().numpy().view(np.uint32), ei)
    ev, ei = lattice.welded_merge_expected(n, row0s, shuffle=True)
    assert np.array_equal(res.vertices.cpu().numpy().view(np.uint32), ev.view(np.uint32))
    assert np.array_equal(res.elements.cpu().numpy().view(np.uint32), ei)


@pytest.mark.gpu
def test_merge_tensors_errors(cuda_ok):
    import torch

    import paper_2109_09812_b200 as rmx
    with pytest.raises(rmx.MeshError):
        rmx.merge_tensors([])
    a = (torch.zeros((3, 2), dtype=torch.int32, device="cuda"), torch.zeros((1, 3), dtype=torch.int32, device="cuda"))
    b = (torch.zeros((3, 3), dtype=torch.int32, device="cuda"), torch.zeros((1, 3), dtype=torch.int32, device="cuda"))
    with pytest.raises(rmx.MeshError):
        rmx.merge_tensors([a, b])


@pytest.mark.gpu
@pytest.mark.parametrize("name,case", _cases("subset"), ids=[c[0] for c in _cases("subset")])
def test_subset_tensors_matches_reference(cuda_ok, name, case):
    """The device-resident subset (compaction kernel + re-index) against the reference subset."""
    import torch

    import paper_2109_09812_b200 as rmx
    v = torch.from_numpy(case["in_vtx"].view(np.int32).copy()).cuda()
    e = torch.from_numpy(case["in_idx"].view(np.int32).copy()).cuda()
    keep = torch.from_numpy(case["keep"]).cuda()
    for sel in (keep, torch.zeros(e.shape[0], dtype=torch.bool, device="cuda").index_fill_(0, keep, True)):
        res = rmx.subset_tensors(v, e, sel)
        assert np.array_equal(res.vertices.cpu().numpy().view(np.uint32), case["out_vtx"])
        assert np.array_equal(res.elements.cpu().numpy().view(np.uint32), case["out_idx"])


@pytest.mark.gpu
def test_subset_tensors_large_and_errors(cuda_ok):
    import torch

    import paper_2109_09812_b200 as rmx
    from oracle import remesh_oracle as O
    rng = np.random.default_rng(3)
    V, E, K = 100_000, 150_000, 3
    words = (rng.integers(0, 50, size=(V, 3)).astype(np.uint32) * np.uint32(0x01000193))
    idx = rng.integers(0, V, size=(E, K)).astype(np.uint32)
    mask = rng.random(E) < 0.3
    ref = O.reindex(words, idx[mask])
    res = rmx.subset_tensors(torch.from_numpy(words.view(np.int32)).cuda(), torch.from_numpy(idx.view(np.int32)).cuda(),
                             torch.from_numpy(mask).cuda())
    assert np.array_equal(res.vertices.cpu().numpy().view(np.uint32), ref["vertices"].view(np.uint32))
    assert np.array_equal(res.elements.cpu().numpy().view(np.uint32), ref["elements"])
    with pytest.raises(rmx.MeshError):
        rmx.subset_tensors(torch.zeros((3, 2), dtype=torch.int32, device="cuda"),
                           torch.zeros((4, 3), dtype=torch.int32, device="cuda"),
                           torch.tensor([2, 1], device="cuda"))
