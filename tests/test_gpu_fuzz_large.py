"""Randomised cases at sizes that cross the size gates naturally (LD rounds from 2^17 vertices,
thread-per-proposer Suitor from 2^18, multi-block selection from 2^18, 4-item look-back tiles
from 2^20 facets, the two-phase single-CTA select below 27k candidates): terrains, grids and
shuffled-id meshes of 100k-700k vertices, single and batched, seeded or not, auto or fixed
rounds, both placements, with features -- bit for bit against the C oracle.
MF_FUZZL_SEEDS=a:b widens it (4 cases in the round-end suite)."""

import os

import numpy as np
import pytest

import paper_2103_15076_b200 as mfg
from paper_2103_15076_b200 import synthetic as S
from paper_2103_15076_b200.numerics import einsum_order

pytestmark = pytest.mark.gpu

_LO, _HI = (int(x) for x in os.environ.get("MF_FUZZL_SEEDS", "0:4").split(":"))


def _mesh(rng):
    kind = int(rng.integers(0, 3))
    if kind == 0:
        return S.delaunay_terrain(int(rng.integers(100_000, 700_000)), noise=float(rng.uniform(0, 0.05)),
                                  seed=int(rng.integers(1 << 30)))
    if kind == 1:
        return S.perturbed_grid(int(rng.integers(300, 800)), int(rng.integers(300, 800)), noise=0.02,
                                seed=int(rng.integers(1 << 30)))
    a = S.delaunay_terrain(int(rng.integers(100_000, 400_000)), seed=int(rng.integers(1 << 30)))
    perm = rng.permutation(a.n_vertices)
    inv = np.empty_like(perm)
    inv[perm] = np.arange(a.n_vertices)
    return mfg.TriMesh(a.positions[perm], inv[a.facets])


def _same(a, b):
    a, b = np.ascontiguousarray(a), np.ascontiguousarray(b)
    return a.shape == b.shape and a.dtype == b.dtype and np.array_equal(a.view(np.uint8), b.view(np.uint8))


@pytest.mark.parametrize("seed", range(_LO, _HI))
def test_large_random_configuration_matches_oracle(oracle, seed):
    rng = np.random.default_rng(777 + seed)
    if rng.random() < 0.3:
        parts = [_mesh(rng) for _ in range(int(rng.integers(2, 4)))]
        target = int(min(m.n_vertices for m in parts) * rng.uniform(0.2, 0.9))
        mesh = mfg.concat_batch(parts)
        base = mesh.mesh
    else:
        mesh = base = _mesh(rng)
        target = int(base.n_vertices * rng.uniform(0.1, 0.9))
    if rng.random() < 0.5:
        base.features = rng.standard_normal((base.n_vertices, int(rng.integers(1, 5)))).astype(
            np.float32 if rng.random() < 0.5 else np.float64)
    shuffle = None if rng.random() < 0.5 else int(rng.integers(1 << 31))
    rounds = "auto" if rng.random() < 0.7 else int(rng.integers(1, 4))
    placement = "inverse" if rng.random() < 0.2 else "average"
    kw = dict(target=target, seed=shuffle, rounds=rounds, order=einsum_order(), placement=placement)
    if isinstance(mesh, mfg.BatchedMesh):
        kw.update(vertex_offsets=mesh.vertex_offsets, facet_offsets=mesh.facet_offsets)
    cfg = mfg.DecimationConfig(target_vertices=target, shuffle_seed=shuffle, rounds=rounds, placement=placement)
    try:
        exp = oracle.decimate(base.positions, base.facets, base.features, **kw)
    except oracle.OracleInfeasible as e:
        with pytest.raises(mfg.InfeasibleTargetError) as err:
            mfg.decimate_parallel(mesh, cfg, device=0)
        assert err.value.achievable_vertices == e.achievable_vertices
        return
    res = mfg.decimate_parallel(mesh, cfg, device=0)
    out = res.mesh.mesh if isinstance(res.mesh, mfg.BatchedMesh) else res.mesh
    for key, got in (("replace", res.replace), ("mapping", res.mapping), ("facets", out.facets),
                     ("positions", out.positions), ("features", out.features)):
        assert _same(got, exp[key]), key
