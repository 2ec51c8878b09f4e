"""Golden fixtures for quality_report (decimate.py:580-602) from the REAL reference
(run in the build container where /root/reference exists):

    python tests/golden/make_golden_quality.py

Writes tests/golden/quality.json: per case the input digest, the reference's
QualityReport fields (float64 mean / max as exact hex, cluster-size counts) and the
sha256 of the per-output-vertex error array, computed with the reference's own
functions in the same sequence as quality_report.
"""

import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)
from make_golden import REF, build_mesh, einsum_order, input_digest, sha  # noqa: E402

sys.path.insert(0, REF)
import meshforge as mf  # noqa: E402
from meshforge.mesh import compute_facet_geometry  # noqa: E402
from meshforge.quadrics import accumulate_quadrics, facet_quadrics, vertex_quadrics  # noqa: E402


def T(n, seed, noise=0.05):
    return {"gen": "delaunay_terrain", "args": [n, noise, seed]}


CASES = [
    ("terrain500", T(500, 3, 0.02), dict(target=200), [None, 4]),
    ("terrain1000_auto", T(1000, 6), dict(target=130), [None]),
    ("icosphere3", {"gen": "icosphere", "args": [3]}, dict(target=230), [None, 7]),
    ("flat16_halve", {"flat": 16}, dict(target=128), [None]),
    ("grid300", {"gen": "perturbed_grid", "args": [300, None, 0.02, 0]}, dict(target=11250), [None]),
    ("terrain20k", T(20000, 1, 0.02), dict(target=5000), [None]),
    ("batch5", {"batch": [T(120 + 31 * b, 20 + b) for b in range(4)] + [{"gen": "icosphere", "args": [1]}]},
     dict(target=42), [None]),
]


def errors_of(mesh, result):
    base = mesh if isinstance(mesh, mf.TriMesh) else mesh.mesh
    vq = vertex_quadrics(base.n_vertices, base.facets, facet_quadrics(compute_facet_geometry(base)))
    cq = accumulate_quadrics(vq, result.replace, result.n_vertices_out)
    return cq.evaluate(result.mesh.positions)


def main():
    out = {"einsum_order": einsum_order(), "numpy": np.__version__, "cases": []}
    for name, spec, conf, seeds in CASES:
        mesh = build_mesh(spec)
        for seed in seeds:
            r = mf.decimate_parallel(mesh, mf.DecimationConfig(target_vertices=conf["target"], shuffle_seed=seed))
            q = mf.quality_report(mesh, r)
            err = errors_of(mesh, r)
            assert float(err.mean()) == q.mean_quadric_error and float(err.max()) == q.max_quadric_error
            out["cases"].append({
                "key": f"{name}|seed={seed}", "spec": spec, "target": conf["target"], "seed": seed,
                "input": input_digest(mesh), "replace": sha(r.replace), "positions": sha(r.mesh.positions),
                "errors": sha(err), "n_vertices_in": q.n_vertices_in, "n_facets_in": q.n_facets_in,
                "n_vertices_out": q.n_vertices_out, "n_facets_out": q.n_facets_out,
                "mean_hex": float(q.mean_quadric_error).hex(), "max_hex": float(q.max_quadric_error).hex(),
                "cluster_size_counts": q.cluster_size_counts.tolist(),
            })
            print(f"{name}|seed={seed}: mean {q.mean_quadric_error:.6g} max {q.max_quadric_error:.6g}")
    with open(os.path.join(HERE, "quality.json"), "w") as fh:
        json.dump(out, fh, indent=1)


if __name__ == "__main__":
    main()
