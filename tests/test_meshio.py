"""Binary PLY load / save (io.py:226-431) and the clusters sidecar (cli.py:95-96):
the numpy oracle (oracle/ply_oracle.py) is pinned to the REAL reference's outputs
(tests/golden/ply.npz, tests/golden/make_golden_ply.py); the GPU decode / encode
(mf_ply_decode / mf_ply_encode) must reproduce them bit for bit."""

import os

import numpy as np
import pytest

import paper_2103_15076_b200 as mfg
from paper_2103_15076_b200.meshio import parse_ply_header

HERE = os.path.dirname(os.path.abspath(__file__))
PLY = os.path.join(HERE, "golden", "ply")
G = np.load(os.path.join(HERE, "golden", "ply.npz"))
LOADS = sorted({k.split("|")[1] for k in G.files if k.startswith("load|")})
SAVES = sorted({k.split("|")[1] for k in G.files if k.startswith("save|")})


def _same(a, b):
    a, b = np.ascontiguousarray(a), np.ascontiguousarray(b)
    return a.dtype == b.dtype and a.shape == b.shape and a.tobytes() == b.tobytes()


@pytest.mark.parametrize("name", LOADS)
def test_ply_oracle_decode_golden(name):
    from oracle import ply_oracle

    P, F, X = ply_oracle.decode(open(os.path.join(PLY, name + ".ply"), "rb").read())
    for k, v in (("positions", P), ("facets", F), ("features", X)):
        assert _same(v, G[f"load|{name}|{k}"]), k


@pytest.mark.parametrize("name", SAVES)
def test_ply_oracle_encode_golden(name):
    from oracle import ply_oracle

    ref = G[f"save|{name}|bytes"].tobytes()
    body = ply_oracle.encode_body(G[f"save|{name}|positions"], G[f"save|{name}|facets"], G[f"save|{name}|features"])
    assert ref.endswith(body) and ref[: len(ref) - len(body)].endswith(b"end_header\n")


def test_ply_header_errors(tmp_path):
    with pytest.raises(mfg.MeshFormatError, match="missing header"):
        parse_ply_header(b"nope")
    with pytest.raises(mfg.MeshFormatError, match="unsupported PLY format"):
        parse_ply_header(b"ply\nformat binary_big_endian 1.0\nend_header\n")
    with pytest.raises(mfg.MeshFormatError, match="property before element"):
        parse_ply_header(b"ply\nformat ascii 1.0\nproperty float x\nend_header\n")
    with pytest.raises(mfg.MeshFormatError, match="cannot infer format"):
        mfg.load_mesh(tmp_path / "mesh.stl")


def test_clusters_sidecar(tmp_path):
    res = mfg.DecimationResult(mfg.TriMesh(np.zeros((2, 3)), np.zeros((0, 3), np.int64)),
                               np.array([0, 1, 1]), np.array([0, -1, 1]))
    side = mfg.save_clusters(tmp_path / "out.ply", res)
    assert side.endswith("out.ply.clusters.npz")
    z = np.load(side)
    assert z["replace"].tolist() == [0, 1, 1] and z["mapping"].tolist() == [0, -1, 1]


@pytest.mark.gpu
@pytest.mark.parametrize("name", LOADS)
def test_gpu_ply_load_golden(name):
    m = mfg.load_mesh(os.path.join(PLY, name + ".ply"))
    for k in ("positions", "facets", "features"):
        assert _same(getattr(m, k), G[f"load|{name}|{k}"]), k


@pytest.mark.gpu
@pytest.mark.parametrize("name", SAVES)
def test_gpu_ply_save_golden(name, tmp_path):
    m = mfg.TriMesh(G[f"save|{name}|positions"], G[f"save|{name}|facets"], G[f"save|{name}|features"])
    out = tmp_path / (name + ".ply")
    mfg.save_mesh(m, out)
    assert out.read_bytes() == G[f"save|{name}|bytes"].tobytes()


@pytest.mark.gpu
def test_gpu_ply_round_trip_large(tmp_path):
    """save -> load of a 200k-vertex mesh: float32 positions, int32 indices survive exactly."""
    from paper_2103_15076_b200 import synthetic

    mesh = synthetic.delaunay_terrain(200_000, 0.02, 5)
    path = tmp_path / "big.ply"
    mfg.save_mesh(mesh, path)
    back = mfg.load_mesh(path)
    assert np.array_equal(back.facets, mesh.facets)
    assert np.array_equal(back.positions, mesh.positions.astype(np.float32).astype(np.float64))


@pytest.mark.gpu
def test_gpu_ply_mixed_arity_rejected(tmp_path):
    rec = np.zeros(4, dtype=[("x", "<f4"), ("y", "<f4"), ("z", "<f4")])
    faces = bytes([3]) + np.array([0, 1, 2], "<i4").tobytes() + bytes([4]) + np.array([0, 1, 2, 3], "<i4").tobytes()
    head = b"ply\nformat binary_little_endian 1.0\nelement vertex 4\nproperty float x\nproperty float y\n" \
           b"property float z\nelement face 2\nproperty list uchar int vertex_indices\nend_header\n"
    p = tmp_path / "mixed.ply"
    p.write_bytes(head + rec.tobytes() + faces + bytes(3))
    with pytest.raises(mfg.MeshFormatError):
        mfg.load_mesh(p)
