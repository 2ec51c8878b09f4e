"""Strided facet2vertex at the cluster representatives (conv.py:222-250,
test_conv.py:366-383) and vertex_facet_adjacency (mesh.py:114-122): the numpy
oracle (oracle/conv_oracle.py) is pinned to the REAL reference's outputs
(tests/golden/conv.npz, tests/golden/make_golden_conv.py); the GPU path must give
the same bits."""

import os

import numpy as np
import pytest

import paper_2103_15076_b200 as mfg

HERE = os.path.dirname(os.path.abspath(__file__))
G = np.load(os.path.join(HERE, "golden", "conv.npz"))
NAMES = sorted({k.split("|")[0] for k in G.files})


def _bits(a):
    a = np.ascontiguousarray(a)
    return a.view(np.uint32 if a.dtype == np.float32 else np.uint64)


@pytest.mark.parametrize("name", NAMES)
def test_conv_oracle_golden(name):
    from oracle import conv_oracle as CO

    F, n = G[f"{name}|facets"], int(G[f"{name}|n"][0])
    off, fid = CO.vertex_facet_adjacency(F, n)
    assert np.array_equal(off, G[f"{name}|adj_offsets"]) and np.array_equal(fid, G[f"{name}|adj_facets"])
    for key, vid in (("strided", G[f"{name}|reps"]), ("full", None)):
        got = CO.facet2vertex(off, fid, G[f"{name}|feats"], G[f"{name}|weights"], G[f"{name}|coeff"], vid)
        exp = G[f"{name}|{key}"]
        assert got.dtype == exp.dtype and np.array_equal(_bits(got), _bits(exp)), key


def test_conv_kernel_validation():
    with pytest.raises(ValueError):
        mfg.ConvKernel(np.zeros((2, 3)))
    k = mfg.ConvKernel.random(4, 2, 3, rng=5)
    assert (k.n_filters, k.in_channels, k.multiplier) == (4, 2, 3)
    adj = mfg.VertexFacetAdjacency(np.array([0, 1, 2, 3]), np.array([0, 0, 0]))
    with pytest.raises(ValueError):  # kernel / coefficient shape mismatch (conv.py:93-97)
        mfg.facet2vertex_forward(adj, np.ones((1, 2)), k, np.ones((1, 3)))
    with pytest.raises(ValueError):  # one coefficient row per facet
        mfg.facet2vertex_forward(adj, np.ones((1, 2)), k, np.ones((2, 4)))


@pytest.mark.gpu
@pytest.mark.parametrize("name", NAMES)
def test_gpu_f2v_golden(name):
    F, n = G[f"{name}|facets"], int(G[f"{name}|n"][0])
    mesh = mfg.TriMesh(np.zeros((n, 3)), F)
    adj = mfg.vertex_facet_adjacency(mesh)
    assert np.array_equal(adj.offsets, G[f"{name}|adj_offsets"])
    assert np.array_equal(adj.facet_ids, G[f"{name}|adj_facets"])
    kernel = mfg.ConvKernel(G[f"{name}|weights"])
    for key, vid in (("strided", G[f"{name}|reps"]), ("full", None)):
        got = mfg.facet2vertex_forward(adj, G[f"{name}|feats"], kernel, G[f"{name}|coeff"], vertex_ids=vid)
        exp = G[f"{name}|{key}"]
        assert got.dtype == exp.dtype and np.array_equal(_bits(got), _bits(exp)), key


@pytest.mark.gpu
def test_gpu_f2v_strided_after_decimation_large():
    """End to end on a 60k-vertex terrain: decimate on the GPU, representatives, strided
    facet2vertex vs the oracle (wide channels: several lane passes per row)."""
    from oracle import conv_oracle as CO
    from paper_2103_15076_b200 import synthetic

    mesh = synthetic.delaunay_terrain(60_000, 0.02, 4)
    res = mfg.decimate_parallel(mesh, mfg.DecimationConfig(target_vertices=20_000), device=0)
    reps = mfg.representative_vertices(res)
    rng = np.random.default_rng(0)
    feats = rng.standard_normal((mesh.n_facets, 40))
    kernel = mfg.ConvKernel.random(4, 40, 1, rng)
    coeff = rng.random((mesh.n_facets, 4))
    coeff /= coeff.sum(axis=1, keepdims=True)
    adj = mfg.vertex_facet_adjacency(mesh)
    off, fid = CO.vertex_facet_adjacency(mesh.facets, mesh.n_vertices)
    assert np.array_equal(adj.offsets, off) and np.array_equal(adj.facet_ids, fid)
    got = mfg.facet2vertex_forward(adj, feats, kernel, coeff, vertex_ids=reps[:2000])
    exp = CO.facet2vertex(off, fid, feats, kernel.weights, coeff, reps[:2000])
    assert np.array_equal(_bits(got), _bits(exp))
