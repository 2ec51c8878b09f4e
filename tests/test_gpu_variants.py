"""Every A/B switch of the CUDA path (matching / selection variants chosen by round
size, or forced through environment flags) must give the oracle's bits.  The flags
are read once per process, so each variant runs in its own interpreter."""

import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

SCRIPT = r"""
import sys
sys.path.insert(0, {root!r})
import paper_2103_15076_b200 as mfg
from paper_2103_15076_b200 import synthetic as S
from paper_2103_15076_b200.numerics import einsum_order
from oracle import oracle as O
import numpy as np
DEG_P = [[0, 0, 0], [1, 0, 0], [0, 1, 0], [9, 9, 9], [2, 0, 0], [1, 1, 0], [3, 3, 0]]
DEG_F = [[0, 1, 2], [1, 4, 5], [0, 1, 4], [1, 2, 5], [2, 1, 5], [0, 4, 6], [0, 1, 2]]

cases = [(S.delaunay_terrain(20_000, noise=0.02, seed=4), 6_000, None),
         (S.delaunay_terrain(20_000, noise=0.02, seed=4), 6_000, 7),
         (S.icosphere(5), 3585, None),
         (S.flat_grid(60), 1_800, None),
         (mfg.concat_batch([S.delaunay_terrain(300 + 40 * b, seed=b) for b in range(6)]), 150, 3),
         # duplicate + degenerate input facets (the dedupe keeps the first occurrence and its winding)
         (mfg.TriMesh(np.array(DEG_P, float), np.array(DEG_F)), 4, None),
         (mfg.TriMesh(np.array(DEG_P, float), np.array(DEG_F)), 5, 3),
         (S.perturbed_grid(120, None, 0.02, 2), 2_000, None)]
for mesh, target, seed in cases:
    res = mfg.decimate_parallel(mesh, mfg.DecimationConfig(target_vertices=target, shuffle_seed=seed))
    kw = dict(target=target, seed=seed, order=einsum_order())
    if hasattr(mesh, "vertex_offsets"):
        kw.update(vertex_offsets=mesh.vertex_offsets, facet_offsets=mesh.facet_offsets)
    ref = O.decimate(mesh.positions, mesh.facets, mesh.features, **kw)
    for key, got in (("replace", res.replace), ("mapping", res.mapping), ("facets", res.mesh.facets),
                     ("positions", res.mesh.positions), ("features", res.mesh.features)):
        exp = ref[key]
        assert got.shape == exp.shape and np.array_equal(np.ascontiguousarray(got).view(np.uint8),
                                                         np.ascontiguousarray(exp).view(np.uint8)), key
print("VARIANT-OK")
"""

VARIANTS = [
    {"MF_SUITOR": "1"},
    {"MF_SUITOR": "8"},
    {"MF_SUITOR": "4"},
    {"MF_SUITOR": "2"},
    {"MF_LD1_MIN": "1"},
    {"MF_LD1_MIN": "1", "MF_LD_MID": "5"},
    {"MF_LD_MIN": "1", "MF_SUITOR": "1"},
    {"MF_LD_MIN": "1", "MF_LD_BIG": "12"},
    {"MF_SELECT_CL": "1"},
    {"MF_SEL_CAP": "12288"},
    {"MF_SEL_PASSES": "1", "MF_LD1_MIN": "1"},
    {"MF_GRAPHS": "0"},
    {"MF_PDL": "0"},
    {"MF_COND": "1", "MF_PDL": "0"},
    {"MF_LD_MIN": "1", "MF_COND": "1", "MF_PDL": "0"},
    # size-gated branches that the defaults take only at cfg5 scale, forced at small sizes
    {"MF_WIDE_MIN": "0"},
    {"MF_SCAN4_MIN": "0"},
    {"MF_BIG_SEL_MIN": "0"},
    {"MF_BIG_SEL_MIN": "0", "MF_SEL_PASSES": "1"},
    {"MF_WIDE_MIN": "0", "MF_SCAN4_MIN": "0", "MF_BIG_SEL_MIN": "0", "MF_LD_MIN": "1", "MF_SUITOR": "1"},
    {"MF_FUSE_PLANE": "0"},
    {"MF_TWO_PASS_MIN": "0"},
    {"MF_TWO_PASS_MIN": "0", "MF_LD_MIN": "1"},
    {"MF_VT16": "1"},
    {"MF_RECOMPUTE_MIN": "0"},
    {"MF_SCAN_TICKET": "1"},
    {"MF_SEL_BULK": "0"},
    {"MF_SEL_FIRST": "0"},
    {"MF_RECOMPUTE_MIN": "0", "MF_VT16": "1", "MF_TWO_PASS_MIN": "0"},
    {"MF_EDGES_RANK": "1"},
    {"MF_EDGES_RANK": "1", "MF_LD_MIN": "1"},
    {"MF_VERTEX_SCAN": "1"},
    {"MF_VERTEX_SCAN": "2"},
    {"MF_POOL_SCALAR": "1", "MF_CSR_COOP": "0"},
]


@pytest.mark.parametrize("env", VARIANTS, ids=[",".join(f"{k}={v}" for k, v in e.items()) for e in VARIANTS])
def test_variant_matches_oracle(env):
    out = subprocess.run([sys.executable, "-c", SCRIPT.format(root=ROOT)], cwd=ROOT, env={**os.environ, **env},
                         capture_output=True, text=True, timeout=600)
    assert "VARIANT-OK" in out.stdout, out.stdout[-2000:] + out.stderr[-4000:]
