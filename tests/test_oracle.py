"""CPU: pin the oracle (numpy restatement + lattice closed form) to the reference's golden vectors."""
import numpy as np
import pytest

from conftest import FIELDS, all_golden, load_group
from oracle import lattice, remesh_oracle as O

CASES = all_golden()


@pytest.mark.parametrize("name,case", CASES, ids=[c[0] for c in CASES])
def test_oracle_matches_reference_golden(name, case):
    r = O.reindex(case["in_vtx"], case["in_idx"])
    assert np.array_equal(r["vertices"].view(np.uint32), case["out_vtx"])
    assert np.array_equal(r["elements"], case["out_idx"])
    assert r["new_count"] == int(case["new_count"])
    for f in FIELDS:
        assert np.array_equal(np.asarray(r[f]), case[f]), f


@pytest.mark.parametrize("name,case", CASES, ids=[c[0] for c in CASES])
def test_closed_form_matches_reference_golden(name, case):
    v, e = O.closed_form(case["in_vtx"], case["in_idx"])
    assert np.array_equal(v.view(np.uint32), case["out_vtx"])
    assert np.array_equal(e, case["out_idx"])


def test_worked_example_intermediates():
    # reference test_pipeline.py:18-155 / test_acceptance.py:28-39 printed values
    c = load_group("worked")["worked"]
    r = O.reindex(c["in_vtx"], c["in_idx"])
    assert r["is_used"].astype(int).tolist() == [1, 1, 1, 0, 1, 1, 1, 1, 0, 1]
    assert r["org_id"].tolist() == [0, 3, 8, 1, 2, 5, 4, 9, 6, 7]
    assert r["nodup"].astype(int).tolist() == [1, 0, 0, 1, 1, 0, 1, 0, 1, 1]
    assert r["new_idx"].tolist() == [0, 0, 0, 1, 2, 2, 3, 3, 4, 5]
    assert r["perm"].tolist() == [0, 3, 4, 1, 6, 5, 8, 9, 2, 7]
    assert r["elements"].tolist() == [[0, 1, 2], [0, 2, 3], [2, 4, 5], [2, 5, 3]]
    assert r["new_count"] == 6


def test_table1_counts():
    g = load_group("grid")
    assert int(g["grid_8"]["new_count"]) == 81
    assert int(g["grid_64"]["new_count"]) == 4225
    assert int(g["grid_2"]["new_count"]) == 9


def test_oracle_rejects_out_of_range():
    with pytest.raises(O.OracleIndexError) as err:
        O.reindex(np.zeros((1, 2), np.float32), np.array([[0, 5, 7], [9, 0, 0]], np.uint32))
    assert err.value.issues[0] == (0, 1, 5) and len(err.value.issues) == 3


def test_oracle_thread_count_invariant():
    c = load_group("random")["random_big"]
    a = O.reindex(c["in_vtx"], c["in_idx"], threads=1)
    b = O.reindex(c["in_vtx"], c["in_idx"], threads=8)
    for k in ("elements", "org_id", "perm"):
        assert np.array_equal(a[k], b[k])


@pytest.mark.parametrize("kind,cells,take", [("tri", (9, 4), None), ("tet", (2, 3, 4), None),
                                             ("tri", (30, 31), 100), ("tet", (4, 4, 4), 77)])
def test_lattice_closed_form_matches_oracle(kind, cells, take):
    v, e = lattice.lattice_soup(kind, cells, seed=5, n_elem_take=take)
    ev, ee = lattice.lattice_expected(kind, cells, seed=5, n_elem_take=take)
    r = O.reindex(v, e)
    assert np.array_equal(r["vertices"].view(np.uint32), ev.view(np.uint32))
    assert np.array_equal(r["elements"], ee)


def test_lattice_sizes_of_configs():
    for cfg, (V, U) in {"C1": (3_150_000, 501_426), "C2": (157_500_000, 25_010_001),
                        "C3": (83_916_000, 3_397_349)}.items():
        kind, cells = lattice.CONFIGS[cfg]
        s = lattice.soup_sizes(kind, cells)
        assert s["n_vertices"] == V and s["n_points"] == U


def test_permutation_is_bijection():
    for n in (1, 2, 3, 17, 1000, 4097):
        p = lattice.permute(np.arange(n, dtype=np.uint64), n, seed=9)
        assert sorted(p.tolist()) == list(range(n))


@pytest.mark.parametrize("n,row0s,shuffle", [(6, [0, 4, 8], False), (5, [0], True), (9, [0, 3, 6, 9, 12], True),
                                             (4, [0, 4], False), (7, [0, 5, 10], True)])
def test_welded_merge_closed_form_matches_oracle(n, row0s, shuffle):
    """C4 recipe: merging welded tiles (overlapping rows) re-indexes to the lattice closed form."""
    tiles = [lattice.welded_tile(n, r0, seed=k, shuffle=shuffle) for k, r0 in enumerate(row0s)]
    offs = np.cumsum([0] + [t[0].shape[0] for t in tiles])[:-1]
    v = np.concatenate([t[0] for t in tiles])
    e = np.concatenate([t[1] + np.uint32(o) for t, o in zip(tiles, offs)])
    ref = O.reindex(v, e)
    ev, ei = lattice.welded_merge_expected(n, row0s, shuffle=shuffle)
    assert np.array_equal(ref["vertices"].view(np.uint32), ev.view(np.uint32))
    assert np.array_equal(ref["elements"], ei)
    s = lattice.welded_sizes(n)
    assert tiles[0][0].shape[0] == s["n_vertices"] and tiles[0][1].shape[0] == s["n_elem"]


def test_c4_counts():
    s = lattice.welded_sizes(lattice.COLS_C4)
    assert lattice.TILES_C4 * s["n_vertices"] == 210_084_008
    rows = lattice.ROW_STEP_C4 * (lattice.TILES_C4 - 1) + lattice.COLS_C4 + 1
    assert rows * (lattice.COLS_C4 + 1) == 182_541_501
