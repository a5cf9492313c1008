"""Host-side mesh value type and error classes of the drop-in.

Mirrors the reference data model (``pkg/src/remeshx/mesh.py``) so code written
against ``remeshx`` keeps working: an immutable ``(n, dim)`` float32 vertex
array plus an ``(m, arity)`` uint32 element array, compared on raw bits.

* ``Mesh``              <- ``remeshx.Mesh``            (mesh.py:45-88)
* ``MeshError``         <- ``remeshx.MeshError``       (mesh.py:20-21)
* ``InvalidMeshError``  <- ``remeshx.InvalidMeshError`` (mesh.py:24-33)
* ``Issue``             <- ``remeshx.Issue``           (mesh.py:36-42)
* ``vertex_bits`` / ``validate`` / ``require_valid`` / ``dereference`` /
  ``soups_equal`` / ``bitwise_equal``                  (mesh.py:91-126)

The helpers here are host-side input checks and comparisons; the
re-indexing arithmetic itself runs only in the CUDA library.
"""
from __future__ import annotations

from typing import NamedTuple

import numpy as np

MAX_VERTICES = 1 << 32


class MeshError(Exception):
    """Base class of every error this package raises (reference mesh.py:20)."""


class Issue(NamedTuple):
    """One out-of-range index: element position, slot in the element, bad value."""

    element: int
    slot: int
    index: int


class InvalidMeshError(MeshError):
    """Some element index is >= the vertex count (reference mesh.py:24-33)."""

    def __init__(self, issues):
        self.issues = list(issues)
        head = self.issues[0]
        super().__init__(
            f"{len(self.issues)} out-of-range index(es); first: element "
            f"{head.element} slot {head.slot} references vertex {head.index}")


def _frozen_copy(data, dtype, what: str) -> np.ndarray:
    arr = np.array(data, dtype=dtype, order="C", copy=True)
    if arr.ndim != 2 or arr.shape[1] < 1:
        raise MeshError(f"{what} must be (n, {'dim' if what == 'vertices' else 'arity'}) "
                        f"with {'dim' if what == 'vertices' else 'arity'} >= 1, got {arr.shape}")
    arr.flags.writeable = False
    return arr


class Mesh:
    """Immutable indexed mesh; both arrays are copied and frozen on construction."""

    __slots__ = ("_vertices", "_elements")

    def __init__(self, vertices, elements):
        v = _frozen_copy(vertices, np.float32, "vertices")
        e = _frozen_copy(elements, np.uint32, "elements")
        if v.shape[0] >= MAX_VERTICES:
            raise MeshError(f"vertex count {v.shape[0]} exceeds 32-bit index range")
        object.__setattr__(self, "_vertices", v)
        object.__setattr__(self, "_elements", e)

    @classmethod
    def _adopt(cls, vertices: np.ndarray, elements: np.ndarray) -> "Mesh":
        """Wrap freshly produced arrays without another copy (internal)."""
        obj = cls.__new__(cls)
        vertices.flags.writeable = False
        elements.flags.writeable = False
        object.__setattr__(obj, "_vertices", vertices)
        object.__setattr__(obj, "_elements", elements)
        return obj

    def __setattr__(self, name, value):
        raise AttributeError("Mesh is immutable")

    @classmethod
    def empty(cls, dim: int = 2, arity: int = 3) -> "Mesh":
        """No vertices, no elements (the reference's default shape: dim 2, arity 3)."""
        return cls._adopt(np.zeros((0, dim), dtype=np.float32), np.zeros((0, arity), dtype=np.uint32))

    @property
    def vertices(self) -> np.ndarray:
        return self._vertices

    @property
    def elements(self) -> np.ndarray:
        return self._elements

    @property
    def dim(self) -> int:
        return self._vertices.shape[1]

    @property
    def arity(self) -> int:
        return self._elements.shape[1]

    @property
    def n_vertices(self) -> int:
        return self._vertices.shape[0]

    @property
    def n_elements(self) -> int:
        return self._elements.shape[0]

    def __repr__(self):
        return f"Mesh(V={self.n_vertices}, D={self.dim}; E={self.n_elements}, K={self.arity})"


def vertex_bits(vertices) -> np.ndarray:
    """uint32 view of float32 vertex words (reference mesh.py:91-94)."""
    return np.ascontiguousarray(vertices, dtype=np.float32).view(np.uint32)


def validate(mesh) -> list[Issue]:
    """One Issue per out-of-range element index, in row-major order (mesh.py:97-100)."""
    elements = np.asarray(mesh.elements)
    bad = np.argwhere(elements >= len(mesh.vertices))
    return [Issue(int(e), int(s), int(elements[e, s])) for e, s in bad]


def require_valid(mesh) -> None:
    """Raise InvalidMeshError when any index is out of range (mesh.py:103-105)."""
    elements = np.asarray(mesh.elements)
    if elements.size and int(elements.max()) >= len(mesh.vertices):
        raise InvalidMeshError(validate(mesh))


def dereference(mesh) -> np.ndarray:
    """Element soup ``out[e, k] = vertices[elements[e, k]]`` (mesh.py:108-111)."""
    require_valid(mesh)
    return np.asarray(mesh.vertices)[np.asarray(mesh.elements)]


def soups_equal(a, b) -> bool:
    """Bitwise equality of two soups (mesh.py:114-118)."""
    a = np.ascontiguousarray(a, dtype=np.float32)
    b = np.ascontiguousarray(b, dtype=np.float32)
    return a.shape == b.shape and bool(np.array_equal(a.view(np.uint32), b.view(np.uint32)))


def bitwise_equal(a, b) -> bool:
    """Bit-identical vertex and element arrays (mesh.py:121-126)."""
    va, vb = np.asarray(a.vertices), np.asarray(b.vertices)
    ea, eb = np.asarray(a.elements), np.asarray(b.elements)
    return (va.shape == vb.shape and ea.shape == eb.shape
            and bool(np.array_equal(vertex_bits(va), vertex_bits(vb)))
            and bool(np.array_equal(ea, eb)))
