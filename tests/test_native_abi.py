"""CPU: the C-ABI library loads (no GPU needed) and exports every symbol the header declares."""
import os
import re

import pytest

from conftest import ROOT


def header_functions():
    text = open(os.path.join(ROOT, "include", "remesh_b200.h")).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(rmx_\w+)\s*\(", text)))


def test_header_lists_the_binding_table():
    from paper_2109_09812_b200 import _native
    assert header_functions() == sorted(_native.EXPORTS)


def test_library_exports_every_header_symbol():
    from paper_2109_09812_b200 import _native
    lib = _native.lib()
    for name in header_functions():
        assert hasattr(lib, name), name
    assert b"sm_100a" in lib.rmx_version()


def test_workspace_and_stage_queries():
    from paper_2109_09812_b200 import _native
    lib = _native.lib()
    small = lib.rmx_workspace_bytes(10, 2, 4, 3)
    big = lib.rmx_workspace_bytes(157_500_000, 3, 50_000_000, 3)
    assert 0 < small < big
    assert big > 2 * 157_500_000 * 16          # two row buffers of 16-byte rows
    assert lib.rmx_workspace_bytes(10, 0, 4, 3) == 0
    assert lib.rmx_workspace_bytes(10, 33, 4, 3) == 0
    n = lib.rmx_stage_count(3)
    names = [lib.rmx_stage_name(3, k).decode() for k in range(n)]
    assert names[:6] == ["start", "mark", "vary", "plan", "pack", "build_rows"]
    assert names[6] == "pk_pass_0" and names[13] == "pk_pass_7"
    assert names[14:16] == ["hash_groups", "first_hist"]
    assert names[16] == "sort_pass_0" and names[27] == "sort_pass_11"
    assert names[-5:] == ["unique", "window", "unique_pk", "map_fill", "remap"] and n == 33


def test_lattice_sizes_match_oracle():
    import ctypes
    from paper_2109_09812_b200 import _native
    from oracle import lattice
    lib = _native.lib()
    for kind, cells, take in (("tri", (625, 800), None), ("tet", (150, 150, 148), None), ("tri", (7, 5), 9)):
        E = ctypes.c_uint64()
        V = ctypes.c_uint64()
        nz = cells[2] if len(cells) == 3 else 0
        t = (1 << 63) if take is None else take
        assert lib.rmx_lattice_sizes(0 if kind == "tri" else 1, cells[0], cells[1], nz, t,
                                     ctypes.byref(E), ctypes.byref(V)) == 0
        v, e = lattice.lattice_soup(kind, cells, 0, take) if take is not None or cells[0] < 700 else (None, None)
        s = lattice.soup_sizes(kind, cells)
        assert E.value == s["n_elem"]
        if take is None:
            assert V.value == s["n_vertices"]
        else:
            assert V.value == len(v)


def test_cpu_only_box_fails_loudly():
    import torch
    if torch.cuda.is_available():
        pytest.skip("has a GPU")
    import numpy as np
    import paper_2109_09812_b200 as p
    with pytest.raises(RuntimeError, match="CUDA"):
        p.reindex(p.Mesh(np.zeros((3, 2), np.float32), np.array([[0, 1, 2]], np.uint32)))
