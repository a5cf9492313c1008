"""SHA-256 digests of the REFERENCE result on the full-size single-GPU configs.

Run in the build container (where /root/reference exists; C2 takes ~3 min and
~15 GB of RAM per config):

    python tools/make_digests.py [C2 C3 C2s]

For each config it generates the seeded soup on the host (``oracle/lattice.py``,
bit-identical to the device generator ``rmx_gen_lattice_soup`` -- checked by
tests/test_gpu_gen_io.py; C2s adds ``lattice.scramble_words``), runs
``remeshx.reindex(remeshx.Mesh(v, e))`` imported read-only from
/root/reference/pkg/src (BASELINE configs[1]: "bit-exact vs CPU reference on the
same seed"), and records the digest of every output array and every
ReindexScratch field (pipeline.py:24-38) in tests/golden/digests.json.
tests/test_gpu_digests.py hashes the device results of the same inputs.

Byte forms hashed: vertices as uint32 words, elements / org_id / new_idx / perm
as little-endian uint32, is_used / nodup as one byte 0/1 per vertex.
"""
from __future__ import annotations

import hashlib
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF_SRC = "/root/reference/pkg/src"
OUT = os.path.join(ROOT, "tests", "golden", "digests.json")
sys.path.insert(0, ROOT)
sys.path.insert(0, REF_SRC)

import remeshx  # noqa: E402  (reference, read-only)
from oracle import lattice  # noqa: E402

CONFIGS = {"C2": ("tri", (5000, 5000), False), "C3": ("tet", (150, 150, 148), False),
           "C2s": ("tri", (5000, 5000), True)}


def sha(a: np.ndarray) -> str:
    a = np.ascontiguousarray(a)
    if a.dtype == np.bool_:
        a = a.view(np.uint8)
    elif a.dtype == np.float32:
        a = a.view(np.uint32)
    return hashlib.sha256(a.astype(a.dtype.newbyteorder("<"), copy=False).tobytes()).hexdigest()


def digest(name: str) -> dict:
    kind, cells, scrambled = CONFIGS[name]
    t = time.time()
    v, e = lattice.lattice_soup(kind, cells, seed=0)
    if scrambled:
        v = lattice.scramble_words(v).view(np.float32)
    in_digest = {"in_vtx": sha(v), "in_idx": sha(e)}
    mesh = remeshx.Mesh(v, e)
    del v, e
    t_gen = time.time() - t
    t = time.time()
    out, sc = remeshx.reindex(mesh)
    t_ref = time.time() - t
    d = {"n_vertices": int(mesh.n_vertices), "n_elements": int(mesh.n_elements), "dim": int(mesh.dim),
         "arity": int(mesh.arity), "new_count": int(sc.new_count), **in_digest,
         "out_vtx": sha(out.vertices), "out_idx": sha(out.elements),
         "is_used": sha(np.asarray(sc.is_used)), "org_id": sha(np.asarray(sc.org_id)),
         "nodup": sha(np.asarray(sc.nodup)), "new_idx": sha(np.asarray(sc.new_idx)),
         "perm": sha(np.asarray(sc.perm)),
         "reference_s": round(t_ref, 1), "generate_s": round(t_gen, 1)}
    print(name, json.dumps(d), flush=True)
    return d


def main():
    names = sys.argv[1:] or list(CONFIGS)
    res = {}
    if os.path.exists(OUT):
        with open(OUT) as f:
            res = json.load(f)
    for n in names:
        res[n] = digest(n)
        with open(OUT, "w") as f:
            json.dump({"_note": "tools/make_digests.py: remeshx.reindex (reference, read-only) on the full "
                                "seeded soups; sha256 of every output and scratch array",
                       **{k: v for k, v in res.items() if not k.startswith("_")}}, f, indent=1)


if __name__ == "__main__":
    main()
