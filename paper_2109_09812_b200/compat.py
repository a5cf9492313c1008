"""Route an existing ``remeshx`` installation to the B200 path (drop-in switch).

``remeshx`` binds ``reindex`` by name in several modules (ops.py:7, bench.py:19,
testing.py:18, cli.py:17, the package __init__ re-export, and pipeline.py
itself), so replacing one attribute is not enough.  :func:`install_into_remeshx`
rebinds all of them to a wrapper that calls :func:`paper_2109_09812_b200.reindex`
and converts results and errors to the reference's own types
(``remeshx.Mesh``, ``remeshx.ReindexScratch``, ``remeshx.MeshError``,
``remeshx.InvalidMeshError`` with ``remeshx.Issue`` items).
"""
from __future__ import annotations

import importlib

_BINDINGS = ("remeshx", "remeshx.pipeline", "remeshx.ops", "remeshx.bench", "remeshx.testing", "remeshx.cli")


def make_reindex(remeshx, on_call=None):
    """A ``remeshx.reindex``-compatible function backed by the CUDA library."""
    from . import mesh as _mesh
    from .pipeline import reindex as _b200_reindex

    def reindex(mesh):
        if on_call is not None:
            on_call()
        try:
            out, sc = _b200_reindex(mesh)
        except _mesh.InvalidMeshError as err:
            raise remeshx.InvalidMeshError([remeshx.Issue(i.element, i.slot, i.index) for i in err.issues]) from None
        except _mesh.MeshError as err:
            raise remeshx.MeshError(str(err)) from None
        scratch = remeshx.ReindexScratch(sc.is_used, sc.org_id, sc.nodup, sc.new_idx, sc.perm, sc.new_count)
        return remeshx.Mesh(out.vertices, out.elements), scratch

    reindex.__wrapped_b200__ = True
    reindex.__doc__ = "B200 drop-in for remeshx.reindex (pipeline.py:133-157)."
    return reindex


def install_into_remeshx(on_call=None) -> list[str]:
    """Rebind every ``reindex`` name in the imported remeshx modules; returns the patched modules.
    ``on_call`` (optional) is called once per reindex call (instrumentation)."""
    remeshx = importlib.import_module("remeshx")
    fn = make_reindex(remeshx, on_call)
    patched = []
    for name in _BINDINGS:
        try:
            mod = importlib.import_module(name)
        except ImportError:
            continue
        if hasattr(mod, "reindex"):
            setattr(mod, "reindex", fn)
            patched.append(name)
    return patched
