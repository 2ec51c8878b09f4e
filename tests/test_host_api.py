"""Host-side boundary logic that needs no device: config validation, mesh
containers and their error types (reference decimate.py:45-71,
mesh.py:13-205, validation.py:8-65, io.py:434-457)."""

import numpy as np
import pytest

import paper_2103_15076_b200 as mfg
from paper_2103_15076_b200.numerics import einsum_order


def test_config_validation():
    with pytest.raises(ValueError):
        mfg.DecimationConfig(target_vertices=10, rounds=-1)
    with pytest.raises(ValueError):
        mfg.DecimationConfig(target_vertices=10, rounds="three")
    with pytest.raises(ValueError):
        mfg.DecimationConfig(target_vertices=0)
    with pytest.raises(ValueError):
        mfg.DecimationConfig(target_vertices=3, placement="median")
    c = mfg.DecimationConfig(target_vertices=3)
    assert c.placement == "average" and c.rounds == "auto" and c.shuffle_seed is None


def test_trimesh_validation():
    with pytest.raises(mfg.StructuralError):
        mfg.TriMesh(np.zeros((3, 2)), [[0, 1, 2]])
    with pytest.raises(mfg.StructuralError):
        mfg.TriMesh(np.array([[0, 0, 0], [1, 0, np.nan], [0, 1, 0]]), [[0, 1, 2]])
    with pytest.raises(mfg.StructuralError, match="references vertex 3"):
        mfg.TriMesh(np.eye(3), [[0, 1, 3]])
    with pytest.raises(mfg.StructuralError, match="repeats"):
        mfg.TriMesh(np.eye(3), [[0, 1, 1]])
    m = mfg.TriMesh(np.eye(3), np.zeros((0, 3)))
    assert m.n_facets == 0 and m.features.shape == (3, 3)
    f32 = mfg.TriMesh(np.eye(3), [[0, 1, 2]], np.ones((3, 2), np.float32))
    assert f32.features.dtype == np.float32


def test_concat_and_split_roundtrip():
    a = mfg.TriMesh(np.eye(3), [[0, 1, 2]])
    b = mfg.TriMesh(np.eye(3) * 2, [[2, 1, 0]])
    batch = mfg.concat_batch([a, b])
    assert batch.vertex_offsets.tolist() == [0, 3, 6]
    assert batch.facet_offsets.tolist() == [0, 1, 2]
    assert batch.facets.tolist() == [[0, 1, 2], [5, 4, 3]]
    parts = batch.split()
    np.testing.assert_array_equal(parts[1].facets, b.facets)
    with pytest.raises(mfg.StructuralError):
        mfg.BatchedMesh(batch.mesh, [0, 2, 6], [0, 1, 2])
    with pytest.raises(ValueError):
        mfg.concat_batch([])


def test_einsum_order_probe_matches_numpy():
    ones = np.ones((1, 3))
    v = np.einsum("ij,ij->i", np.array([[1e16, 1.0, -1e16]]), ones)[0]
    assert einsum_order() == (0 if v == 1.0 else 1)


def test_clusters_and_representatives_on_hand_result():
    rep = np.array([0, 0, 1, 1, 1, 0])
    res = mfg.DecimationResult(mesh=mfg.TriMesh(np.zeros((2, 3)), np.zeros((0, 3))), replace=rep,
                               mapping=rep.copy())
    assert [c.members for c in mfg.clusters(res)] == [(0, 1, 5), (2, 3, 4)]
    np.testing.assert_array_equal(mfg.representative_vertices(res), [0, 2])
    np.testing.assert_array_equal(res.cluster_sizes(), [3, 3])
