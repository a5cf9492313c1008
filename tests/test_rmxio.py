"""RMX1 container on the host: reference-written files, round trips, errors.

Fixtures in tests/golden/rmx1/ were written by the reference ``write_bin``
(tools/make_golden.py); error cases follow the reference tests
(test_io.py:84-124).
"""
import os

import numpy as np
import pytest

from paper_2109_09812_b200 import Mesh, MeshError, bitwise_equal
from paper_2109_09812_b200 import rmxio

GOLD = os.path.join(os.path.dirname(__file__), "golden", "rmx1")
NAMES = ["worked", "empty", "nan_bits", "random_quads3d"]


@pytest.mark.parametrize("name", NAMES)
def test_reads_reference_files_and_writes_identical_bytes(tmp_path, name):
    src = os.path.join(GOLD, f"{name}.rmx")
    m = rmxio.read_bin(src)
    out = tmp_path / "x.rmx"
    rmxio.write_bin(m, out)
    assert out.read_bytes() == open(src, "rb").read()


def test_worked_contents():
    m = rmxio.read_bin(os.path.join(GOLD, "worked.rmx"))
    assert m.vertices.shape == (10, 2) and m.elements.shape == (4, 3)
    assert m.elements.tolist() == [[0, 1, 2], [0, 2, 4], [5, 6, 7], [5, 7, 9]]
    assert m.vertices[3].tolist() == [9.0, 9.0]


def test_empty_is_28_bytes_and_keeps_shape(tmp_path):
    p = tmp_path / "e.rmx"
    rmxio.write_bin(Mesh.empty(), p)
    assert p.stat().st_size == 28
    back = rmxio.read_bin(p)
    assert back.n_vertices == 0 and back.n_elements == 0 and back.dim == 2 and back.arity == 3


def test_nan_and_negative_zero_bits_survive(tmp_path):
    m = rmxio.read_bin(os.path.join(GOLD, "nan_bits.rmx"))
    assert m.vertices.view(np.uint32).tolist() == [[0x7FC00123, 0x80000000]]
    p = tmp_path / "n.rmx"
    rmxio.write_bin(m, p)
    assert bitwise_equal(rmxio.read_bin(p), m)


def test_bad_magic(tmp_path):
    p = tmp_path / "bad.rmx"
    p.write_bytes(b"XXXX" + b"\0" * 24)
    with pytest.raises(rmxio.FormatError):
        rmxio.read_bin(p)


def test_truncated_short_and_trailing(tmp_path):
    good = open(os.path.join(GOLD, "worked.rmx"), "rb").read()
    for name, data in [("cut", good[:-3]), ("short", good[:10]), ("trail", good + b"\0")]:
        p = tmp_path / f"{name}.rmx"
        p.write_bytes(data)
        with pytest.raises(rmxio.FormatError):
            rmxio.read_bin(p)


def test_zero_dim_rejected(tmp_path):
    p = tmp_path / "z.rmx"
    p.write_bytes(rmxio.HEADER.pack(b"RMX1", 0, 3, 0, 0))
    with pytest.raises(rmxio.FormatError):
        rmxio.read_bin(p)


def test_format_error_is_mesh_error():
    assert issubclass(rmxio.FormatError, MeshError)


def test_write_rejects_invalid_mesh(tmp_path):
    m = Mesh(np.zeros((2, 2), np.float32), np.array([[0, 1, 2]], np.uint32))
    with pytest.raises(MeshError):
        rmxio.write_bin(m, tmp_path / "x.rmx")
