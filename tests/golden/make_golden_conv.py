"""Golden fixtures for the strided facet2vertex (conv.py:222-250 at
representative_vertices, test_conv.py:366-383) and vertex_facet_adjacency
(mesh.py:114-122) from the REAL reference (run in the build container):

    python tests/golden/make_golden_conv.py

Writes tests/golden/conv.npz: per case the inputs (facets, facet features, kernel
weights, GMM fuzzy coefficients from the reference's gmm_coefficients, the
representatives of a reference decimation) and the reference outputs (adjacency,
strided and full facet2vertex).
"""

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")

import meshforge as mf  # noqa: E402
from meshforge import synthetic as msyn  # noqa: E402
from meshforge.conv import ConvKernel, facet2vertex_forward  # noqa: E402
from meshforge.decimate import representative_vertices  # noqa: E402
from meshforge.gmm import SphereGMM, fibonacci_sphere, gmm_coefficients  # noqa: E402
from meshforge.mesh import compute_facet_geometry, vertex_facet_adjacency  # noqa: E402


def case(out, name, mesh, target, c, t, L, dtype, seed):
    rng = np.random.default_rng(seed)
    res = mf.decimate_parallel(mesh, mf.DecimationConfig(target_vertices=target))
    reps = representative_vertices(res)
    adj = vertex_facet_adjacency(mesh)
    feats = rng.standard_normal((mesh.n_facets, c)).astype(dtype)
    kernel = ConvKernel.random(t, c, L, rng)
    gmm = SphereGMM(means=fibonacci_sphere(t), sigmas=0.2 + 0.5 * rng.random(t))
    coeff = gmm_coefficients(compute_facet_geometry(mesh).normal, gmm)
    out[f"{name}|facets"] = mesh.facets
    out[f"{name}|n"] = np.array([mesh.n_vertices])
    out[f"{name}|feats"] = feats
    out[f"{name}|weights"] = kernel.weights
    out[f"{name}|coeff"] = coeff
    out[f"{name}|reps"] = reps
    out[f"{name}|adj_offsets"] = adj.offsets
    out[f"{name}|adj_facets"] = adj.facet_ids
    out[f"{name}|strided"] = facet2vertex_forward(adj, feats, kernel, coeff, vertex_ids=reps)
    out[f"{name}|full"] = facet2vertex_forward(adj, feats, kernel, coeff)
    print(name, mesh.n_vertices, mesh.n_facets, len(reps), out[f"{name}|strided"].dtype)


def main():
    out = {}
    case(out, "terrain400_f64", msyn.delaunay_terrain(400, 0.05, 12), 150, 4, 5, 2, np.float64, 1)
    case(out, "terrain400_f32", msyn.delaunay_terrain(400, 0.05, 12), 150, 3, 6, 1, np.float32, 2)
    case(out, "icosphere3_f64", msyn.icosphere(3), 230, 8, 18, 1, np.float64, 3)
    # an isolated vertex: empty adjacency -> zero row (test_conv.py:168-178)
    iso = mf.TriMesh(np.array([[0, 0, 0], [1, 0, 0], [0, 1, 0], [1, 1, 0.2], [5, 5, 5]], float),
                     np.array([[0, 1, 2], [1, 3, 2]]))
    case(out, "isolated_f64", iso, 4, 2, 3, 2, np.float64, 4)
    np.savez(os.path.join(HERE, "conv.npz"), **out)


if __name__ == "__main__":
    main()
