"""GPU: memory-lean mode (rmx_reindex_lean, pipeline.reindex_tensors_lean) --
the vertex buffer becomes the second sort buffer and the result is left in the final sort buffer.
Results must equal the ordinary pipeline bit for bit; keys that do not pack into 64 bits are refused."""
import numpy as np
import pytest

from oracle import lattice
from oracle import remesh_oracle as O

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def rmx(cuda_ok):
    import paper_2109_09812_b200 as p
    return p


@pytest.mark.parametrize("kind,cells", [("tri", (120, 90)), ("tet", (20, 18, 16)), ("tri", (700, 600))])
def test_lean_equals_the_pipeline(rmx, kind, cells):
    import torch
    v, e = lattice.lattice_soup(kind, cells, seed=5)
    if v.shape[0] % 2:
        v, e = v[:-1], e[e.max(axis=1) < v.shape[0] - 1]
    vt = torch.from_numpy(v.view(np.int32).copy()).cuda()
    et = torch.from_numpy(e.view(np.int32).copy()).cuda()
    ref = rmx.reindex_tensors(vt, et)
    res = rmx.reindex_tensors_lean(vt.clone(), et)
    assert res.new_count == ref.new_count
    assert torch.equal(res.vertices, ref.vertices) and torch.equal(res.elements, ref.elements)


def test_lean_u64_keys_and_random_indices(rmx):
    """> 32 packed key bits (u64 keys, 5+ passes: the result lands in either buffer), indexed mesh."""
    import torch
    rng = np.random.default_rng(2)
    V = 200_000
    words = (rng.integers(0, 1 << 13, size=(V, 3)).astype(np.uint32) << np.uint32(10)) | np.uint32(0x3F800000)
    idx = rng.integers(0, V, size=(V // 3, 4)).astype(np.uint32)
    ref = O.reindex(words, idx)
    res = rmx.reindex_tensors_lean(torch.from_numpy(words.view(np.int32).copy()).cuda(),
                                   torch.from_numpy(idx.view(np.int32)).cuda())
    assert np.array_equal(res.vertices.cpu().numpy().view(np.uint32), ref["vertices"].view(np.uint32))
    assert np.array_equal(res.elements.cpu().numpy().view(np.uint32), ref["elements"])


def test_lean_refuses_wide_keys(rmx):
    import torch
    rng = np.random.default_rng(3)
    V = 50_000
    words = rng.integers(0, 2**32, size=(V, 3), dtype=np.uint64).astype(np.uint32)
    idx = rng.integers(0, V, size=(V // 3, 3)).astype(np.uint32)
    with pytest.raises(rmx.MeshError):
        rmx.reindex_tensors_lean(torch.from_numpy(words.view(np.int32).copy()).cuda(),
                                 torch.from_numpy(idx.view(np.int32)).cuda())


def test_lean_out_of_range(rmx):
    import torch
    v, e = lattice.lattice_soup("tri", (100, 100), seed=1)
    e = e.copy()
    e[7, 1] = v.shape[0] + 3
    with pytest.raises(rmx.InvalidMeshError):
        rmx.reindex_tensors_lean(torch.from_numpy(v.view(np.int32).copy()).cuda(),
                                 torch.from_numpy(e.view(np.int32)).cuda())
