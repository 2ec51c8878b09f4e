"""quality_report (decimate.py:580-602) against golden fixtures produced by the REAL
reference (tests/golden/make_golden_quality.py): the CPU oracle pins the arithmetic
(per-output-vertex errors bit-exact, mean / max / cluster-size counts equal), and the
GPU path (mf_quality_errors through paper_2103_15076_b200.quality_report) must give the
same bits."""

import json
import os

import numpy as np
import pytest

import paper_2103_15076_b200 as mfg
from test_oracle_golden import build_mesh, input_digest, sha

HERE = os.path.dirname(os.path.abspath(__file__))
GOLD = json.load(open(os.path.join(HERE, "golden", "quality.json")))
ORDER = GOLD["einsum_order"]
CASES = GOLD["cases"]


def _oracle_result(oracle, mesh, case):
    base = mesh.mesh if isinstance(mesh, mfg.BatchedMesh) else mesh
    kw = dict(target=case["target"], seed=case["seed"], order=ORDER)
    if isinstance(mesh, mfg.BatchedMesh):
        kw.update(vertex_offsets=mesh.vertex_offsets, facet_offsets=mesh.facet_offsets)
    return base, oracle.decimate(base.positions, base.facets, None, **kw)


def _check_report(rep, case, errors):
    assert sha(errors) == case["errors"]
    assert rep.mean_quadric_error == float.fromhex(case["mean_hex"])
    assert rep.max_quadric_error == float.fromhex(case["max_hex"])
    assert rep.cluster_size_counts.tolist() == case["cluster_size_counts"]
    for k in ("n_vertices_in", "n_facets_in", "n_vertices_out", "n_facets_out"):
        assert getattr(rep, k) == case[k], k


@pytest.mark.parametrize("case", CASES, ids=[c["key"] for c in CASES])
def test_quality_oracle_golden(oracle, case):
    mesh = build_mesh(case["spec"])
    assert input_digest(mesh) == case["input"]
    base, out = _oracle_result(oracle, mesh, case)
    assert sha(out["replace"]) == case["replace"] and sha(out["positions"]) == case["positions"]
    err = oracle.quality_errors(base.positions, base.facets, out["replace"], out["positions"], ORDER)
    sizes = np.bincount(out["replace"], minlength=len(out["positions"]))
    rep = mfg.QualityReport(base.n_vertices, base.n_facets, len(out["positions"]), len(out["facets"]),
                            float(err.mean()), float(err.max()), np.bincount(sizes))
    _check_report(rep, case, err)


def test_quality_report_describe():
    rep = mfg.QualityReport(10, 16, 5, 6, 0.5, 1.25, np.array([0, 1, 2]))
    assert rep.describe().splitlines()[-1] == "cluster sizes {1: 1, 2: 2}"


@pytest.mark.gpu
@pytest.mark.parametrize("case", CASES, ids=[c["key"] for c in CASES])
def test_gpu_quality_golden(case):
    from paper_2103_15076_b200 import quality
    from paper_2103_15076_b200.numerics import forced_order

    mesh = build_mesh(case["spec"])
    with forced_order(ORDER):
        res = mfg.decimate_parallel(mesh, mfg.DecimationConfig(target_vertices=case["target"],
                                                               shuffle_seed=case["seed"]), device=0)
        assert sha(res.replace) == case["replace"]
        _check_report(mfg.quality_report(mesh, res), case, quality.quadric_errors(mesh, res))


@pytest.mark.gpu
def test_gpu_quality_vs_oracle_large(oracle):
    """A 200k-vertex terrain (heavy tier + many clusters), replace given as a plain array."""
    from paper_2103_15076_b200 import quality, synthetic

    mesh = synthetic.delaunay_terrain(200_000, 0.02, 9)
    res = mfg.decimate_parallel(mesh, mfg.DecimationConfig(target_vertices=60_000), device=0)
    plain = mfg.DecimationResult(res.mesh, np.array(res.replace), np.array(res.mapping))  # re-uploaded path
    got = quality.quadric_errors(mesh, plain, 0)
    exp = oracle.quality_errors(mesh.positions, mesh.facets, res.replace, res.mesh.positions, 0)
    assert np.array_equal(got.view(np.uint64), exp.view(np.uint64))
