"""the device re-validation of a mesh (mf_validate_mesh) raises the
reference's StructuralError messages in the reference's check order (validation.py:8-41,
restated host-side by paper_2103_15076_b200.validation), and MF_DEBUG=1 re-validates every
decimation output on the device without changing a bit of it."""

import os
import subprocess
import sys

import numpy as np
import pytest

import paper_2103_15076_b200 as mfg
from paper_2103_15076_b200 import synthetic as S
from paper_2103_15076_b200 import validation as V

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _raw(P, F):
    t = mfg.TriMesh.__new__(mfg.TriMesh)
    t.positions, t.facets, t.features = np.asarray(P, float), np.asarray(F, np.int64).reshape(-1, 3), None
    return t


def _host_message(P, F):
    try:
        V.as_facets(F, len(V.as_positions(P)))
    except mfg.StructuralError as e:
        return str(e)
    return None


def test_valid_outputs_pass():
    mesh = S.delaunay_terrain(20_000, noise=0.02, seed=4)
    res = mfg.decimate_parallel(mesh, mfg.DecimationConfig(target_vertices=5_000))
    mfg.validate_on_device(res.mesh, check_duplicates=True)
    batch = mfg.concat_batch([S.delaunay_terrain(300 + 40 * b, seed=b) for b in range(6)])
    res = mfg.decimate_parallel(batch, mfg.DecimationConfig(target_vertices=150, shuffle_seed=3))
    mfg.validate_on_device(res.mesh, check_duplicates=True)


@pytest.mark.parametrize("case", ["nan", "inf", "range_hi", "range_neg", "repeat", "range_before_repeat"])
def test_reference_messages(case):
    rng = np.random.default_rng(0)
    P = rng.random((50, 3))
    F = np.array([[0, 1, 2], [2, 3, 4], [4, 5, 6], [6, 7, 8], [8, 9, 10]], np.int64)
    if case == "nan":
        P[7, 1] = np.nan
    elif case == "inf":
        P[3, 2] = -np.inf
    elif case == "range_hi":
        F[3] = [6, 50, 8]
    elif case == "range_neg":
        F[2] = [4, -1, 6]
    elif case == "repeat":
        F[4] = [8, 9, 8]
    else:  # the range check runs over every facet before the repeat check
        F[1] = [2, 2, 4]
        F[3] = [6, 7, 99]
    if case in ("nan", "inf"):
        exp = "positions contain NaN or infinite values"
    else:
        exp = _host_message(P, F)
    with pytest.raises(mfg.StructuralError) as err:
        mfg.validate_on_device(_raw(P, F))
    assert str(err.value) == exp


def test_duplicates_and_batch_entries():
    P = np.random.default_rng(1).random((12, 3))
    F = np.array([[0, 1, 2], [1, 2, 3], [3, 4, 5], [2, 1, 0], [6, 7, 8]], np.int64)
    mfg.validate_on_device(_raw(P, F), check_duplicates=False)
    with pytest.raises(mfg.StructuralError, match="facet 3 repeats the vertex set of facet 0"):
        mfg.validate_on_device(_raw(P, F), check_duplicates=True)
    # in range of the whole mesh, but facet 2 crosses from entry 0 into entry 1
    F = np.array([[0, 1, 2], [1, 2, 3], [3, 4, 6], [6, 7, 8]], np.int64)
    bm = mfg.BatchedMesh.__new__(mfg.BatchedMesh)
    bm.mesh, bm.vertex_offsets, bm.facet_offsets = _raw(P, F), np.array([0, 6, 12]), np.array([0, 3, 4])
    with pytest.raises(mfg.StructuralError, match="facet 2 references vertex 6 outside its batch entry"):
        mfg.validate_on_device(bm)


DEBUG_SCRIPT = r"""
import sys
sys.path.insert(0, {root!r})
import numpy as np
import paper_2103_15076_b200 as mfg
from paper_2103_15076_b200 import synthetic as S
from paper_2103_15076_b200.numerics import einsum_order
from oracle import oracle as O
cases = [(S.delaunay_terrain(20_000, noise=0.02, seed=4), 6_000, None),
         (S.icosphere(5), 3585, 7),
         (mfg.concat_batch([S.delaunay_terrain(300 + 40 * b, seed=b) for b in range(6)]), 150, 3)]
for mesh, target, seed in cases:
    res = mfg.decimate_parallel(mesh, mfg.DecimationConfig(target_vertices=target, shuffle_seed=seed))
    kw = dict(target=target, seed=seed, order=einsum_order())
    if hasattr(mesh, "vertex_offsets"):
        kw.update(vertex_offsets=mesh.vertex_offsets, facet_offsets=mesh.facet_offsets)
    ref = O.decimate(mesh.positions, mesh.facets, mesh.features, **kw)
    for key, got in (("replace", res.replace), ("mapping", res.mapping), ("facets", res.mesh.facets),
                     ("positions", res.mesh.positions)):
        assert np.array_equal(np.asarray(got).view(np.uint8), ref[key].view(np.uint8)), key
print("DEBUG-OK")
"""


def test_mf_debug_revalidates_every_output():
    out = subprocess.run([sys.executable, "-c", DEBUG_SCRIPT.format(root=ROOT)], cwd=ROOT,
                         env={**os.environ, "MF_DEBUG": "1"}, capture_output=True, text=True, timeout=600)
    assert "DEBUG-OK" in out.stdout, out.stdout[-2000:] + out.stderr[-4000:]
