"""Golden digests of the REAL reference at BASELINE.json's FULL sizes (run in the
build container, where /root/reference exists; the GPU box only reads the json).

    python tests/golden/make_golden_full.py [cfg3] [cfg4] [cfg5] [cfg3_inverse] [cfg4_inverse]

Writes tests/golden/full.json: per config the input digest and, per level, the
sha256 of replace / mapping / facets / positions / features (and, for cfg3, of
the C=64 float32 max-pool and unpool of every level).  Runtime here: cfg3 ~40 s,
cfg4 ~10 s, cfg5 ~10 min and ~13 GB RSS (one 10M-vertex mesh, 4 levels).
"""

import json
import os
import sys
import time

import numpy as np

REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REF)
sys.path.insert(0, HERE)

import meshforge as mf  # noqa: E402
from meshforge import pooling as mpool  # noqa: E402
from meshforge import synthetic as msyn  # noqa: E402

from make_golden import einsum_order, input_digest, sha  # noqa: E402

OUT = os.path.join(HERE, "full.json")


def level_digests(r):
    base = r.mesh.mesh if isinstance(r.mesh, mf.BatchedMesh) else r.mesh
    d = {"n_out": int(base.n_vertices), "m_out": int(base.n_facets), "replace": sha(r.replace),
         "mapping": sha(r.mapping), "facets": sha(base.facets), "positions": sha(base.positions),
         "features": sha(base.features)}
    if isinstance(r.mesh, mf.BatchedMesh):
        d["vertex_offsets"] = sha(r.mesh.vertex_offsets)
        d["facet_offsets"] = sha(r.mesh.facet_offsets)
    return d


def chain(mesh, targets, feats=None, placement="average"):
    levels, cur, f = [], mesh, feats
    for tgt in targets:
        t = time.time()
        r = mf.decimate_parallel(cur, mf.DecimationConfig(target_vertices=tgt, placement=placement))
        d = level_digests(r)
        d["target"] = tgt
        d["ref_seconds"] = round(time.time() - t, 2)
        if f is not None:
            nxt = mpool.pool(f, r, mode="max")
            d["pool_max"] = sha(nxt)
            d["unpool"] = sha(mpool.unpool(nxt, r))
            f = nxt
        print(f"  level -> {tgt}: {d['ref_seconds']} s", flush=True)
        levels.append(d)
        cur = r.mesh
    return levels


def halving(n, k=4):
    out = []
    for _ in range(k):
        n = -(-n // 2)
        out.append(n)
    return out


def main():
    which = sys.argv[1:] or ["cfg3", "cfg4", "cfg5", "cfg3_inverse", "cfg4_inverse"]
    data = json.load(open(OUT)) if os.path.exists(OUT) else {}
    data.update({"einsum_order": einsum_order(), "numpy": np.__version__, "reference": "meshforge 0.1.0"})
    if "cfg3" in which:
        print("cfg3", flush=True)
        mesh = msyn.delaunay_terrain(500_000, 0.02, 3)
        feats = np.random.default_rng(0).standard_normal((mesh.n_vertices, 64)).astype(np.float32)
        data["cfg3"] = {"input": input_digest(mesh), "features": sha(feats),
                        "levels": chain(mesh, [125_000, 62_500, 31_250, 15_625], feats)}
    if "cfg4" in which:
        print("cfg4", flush=True)
        batch = mf.concat_batch([msyn.delaunay_terrain(2500, 0.02, b) for b in range(256)])
        data["cfg4"] = {"input": input_digest(batch), "levels": chain(batch, [1250])}
    if "cfg5" in which:
        print("cfg5", flush=True)
        mesh = msyn.perturbed_grid(3163, None, 0.02, 0)
        data["cfg5"] = {"input": input_digest(mesh), "levels": chain(mesh, halving(mesh.n_vertices))}
    # placement='inverse' at full size (the solve is restated in numpy.linalg.solve's order)
    if "cfg3_inverse" in which:
        print("cfg3_inverse", flush=True)
        mesh = msyn.delaunay_terrain(500_000, 0.02, 3)
        data["cfg3_inverse"] = {"input": input_digest(mesh),
                                "levels": chain(mesh, [125_000, 62_500, 31_250, 15_625], placement="inverse")}
    if "cfg4_inverse" in which:
        print("cfg4_inverse", flush=True)
        batch = mf.concat_batch([msyn.delaunay_terrain(2500, 0.02, b) for b in range(256)])
        data["cfg4_inverse"] = {"input": input_digest(batch), "levels": chain(batch, [1250], placement="inverse")}
    with open(OUT, "w") as fh:
        json.dump(data, fh, indent=1)
    print("wrote", OUT)


if __name__ == "__main__":
    main()
