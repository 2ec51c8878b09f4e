"""Small decimation / pooling workload for compute-sanitizer runs (scripts/gpu_sanitize.sh).

Runs the golden toy fixtures, a 20k terrain (seeded and unseeded), a mixed batch and
pool / unpool / pool_backward once each through the public API and checks them against
the C oracle (test infrastructure, used as the checker only)."""

import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import paper_2103_15076_b200 as mfg  # noqa: E402
from oracle import oracle as O  # noqa: E402
from paper_2103_15076_b200 import synthetic as S  # noqa: E402
from paper_2103_15076_b200.numerics import einsum_order  # noqa: E402

DEG_P = [[0, 0, 0], [1, 0, 0], [0, 1, 0], [9, 9, 9], [2, 0, 0], [1, 1, 0], [3, 3, 0]]
DEG_F = [[0, 1, 2], [1, 4, 5], [0, 1, 4], [1, 2, 5], [2, 1, 5], [0, 4, 6], [0, 1, 2]]
n = int(os.environ.get("MF_SAN_N", "20000"))
cases = [(mfg.TriMesh(np.array(DEG_P, float), np.array(DEG_F)), 4, None),
         (S.delaunay_terrain(n, noise=0.02, seed=4), n * 3 // 10, None),
         (S.delaunay_terrain(n, noise=0.02, seed=4), n * 3 // 10, 7),
         (S.flat_grid(40), 800, None),
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
X = np.random.default_rng(0).standard_normal((res.n_vertices_in, 16)).astype(np.float32)
w = np.random.default_rng(1).random(res.n_vertices_in).astype(np.float32) + 0.5
for mode in mfg.POOL_MODES:
    got = mfg.pool(X, res, mode=mode, weights=w)
    assert np.array_equal(got.view(np.uint8), O.pool(X, res.replace, res.n_vertices_out, mode, w).view(np.uint8))
    mfg.pool_backward(got, X, res, mode=mode, weights=w)
up = mfg.unpool(got, res)
assert np.array_equal(up, O.unpool(got, res.replace))
mfg.validate_on_device(res.mesh)
# a batch whose lowest failing entry fails in a later round than a higher one (the prefix rerun)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import test_gpu_fuzz as FZ  # noqa: E402

mesh, target, seed, rounds = FZ._case(1120)
try:
    mfg.decimate_parallel(mesh, mfg.DecimationConfig(target_vertices=target, shuffle_seed=seed, rounds=rounds))
    raise AssertionError("expected InfeasibleTargetError")
except mfg.InfeasibleTargetError as e:
    assert e.achievable_vertices == 63, e
print("SANITIZE-CASES-OK")
