"""paper_2109_09812_b200: B200-native re-indexing of indexed meshes (arXiv 2109.09812).

Drop-in for the reference hot path ``remeshx.reindex`` (pkg/src/remeshx/pipeline.py:133-157):
duplicate and unused vertices are removed by hand-written sm_100a kernels
(mark, replace, onesweep LSD radix sort, look-back scan/compaction, remap)
behind the C-ABI in include/remesh_b200.h.
"""
from .mesh import (InvalidMeshError, Issue, Mesh, MeshError, bitwise_equal, dereference,
                   require_valid, soups_equal, validate, vertex_bits)
from . import gen, rmxio
from .ops import merge, merge_tensors, soup_to_mesh, subset, subset_tensors
from .rmxio import FormatError, read_bin, write_bin
from .pipeline import (DeviceResult, PipelineGraph, ReindexScratch, Reindexer, ReindexStream, reindex,
                       reindex_tensors, reindex_tensors_lean, workspace_bytes)

__version__ = "0.1.0"

__all__ = [
    "Mesh", "Issue", "MeshError", "InvalidMeshError", "ReindexScratch", "DeviceResult",
    "Reindexer", "ReindexStream", "PipelineGraph", "reindex", "reindex_tensors", "reindex_tensors_lean", "workspace_bytes", "merge", "merge_tensors", "soup_to_mesh", "subset_tensors", "subset",
    "read_bin", "write_bin", "FormatError", "gen", "rmxio",
    "validate", "require_valid", "dereference", "soups_equal", "bitwise_equal", "vertex_bits",
]
