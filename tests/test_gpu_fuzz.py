"""Seeded random configurations through every public entry point, bit for bit against the C
oracle: single meshes and batches (with entries already at the target, i.e. bypassed),
unseeded / seeded ranks, `rounds` fixed or auto, omitted / float32 / float64 features of
1-7 channels, shuffled vertex ids, disconnected unions, duplicate input facets; the numpy
API (pinned and pageable inputs), the device-tensor API, and a chained second level."""

import os

import numpy as np
import pytest
import torch

import paper_2103_15076_b200 as mfg
from paper_2103_15076_b200 import synthetic as S
from paper_2103_15076_b200 import tensor as T
from paper_2103_15076_b200.numerics import einsum_order

pytestmark = pytest.mark.gpu


def _mesh(rng):
    kind = rng.integers(0, 5)
    if kind == 0:
        m = S.delaunay_terrain(int(rng.integers(40, 6000)), noise=float(rng.uniform(0, 0.1)),
                               seed=int(rng.integers(1 << 30)))
    elif kind == 1:
        m = S.perturbed_grid(int(rng.integers(5, 70)), int(rng.integers(5, 70)), noise=0.02,
                             seed=int(rng.integers(1 << 30)))
    elif kind == 2:
        m = S.icosphere(int(rng.integers(1, 5)))
    elif kind == 3:  # two disconnected pieces
        a = S.delaunay_terrain(int(rng.integers(40, 800)), seed=int(rng.integers(1 << 30)))
        b = S.delaunay_terrain(int(rng.integers(40, 800)), seed=int(rng.integers(1 << 30)))
        m = mfg.TriMesh(np.concatenate([a.positions, b.positions + 5.0]),
                        np.concatenate([a.facets, b.facets + a.n_vertices]))
    else:  # shuffled vertex ids + a few duplicated facets
        a = S.delaunay_terrain(int(rng.integers(60, 3000)), seed=int(rng.integers(1 << 30)))
        perm = rng.permutation(a.n_vertices)
        inv = np.empty_like(perm)
        inv[perm] = np.arange(a.n_vertices)
        F = inv[a.facets]
        dup = F[rng.integers(0, len(F), size=max(1, len(F) // 50))]
        m = mfg.TriMesh(a.positions[perm], np.concatenate([F, dup[:, ::-1]]))
    return m


def _features(rng, n):
    k = rng.integers(0, 3)
    if k == 0:
        return None
    c = int(rng.integers(1, 8))
    dt = np.float32 if k == 1 else np.float64
    return rng.standard_normal((n, c)).astype(dt)


def _case(seed):
    rng = np.random.default_rng(seed)
    if rng.random() < 0.35:
        metas = [_mesh(rng) for _ in range(int(rng.integers(2, 6)))]
        target = int(min(m.n_vertices for m in metas) * rng.uniform(0.3, 1.0))
        mesh = mfg.concat_batch(metas)
        base = mesh.mesh
    else:
        mesh = base = _mesh(rng)
        target = int(base.n_vertices * rng.uniform(0.2, 0.95))
    target = max(target, 1)
    feats = _features(rng, base.n_vertices)
    if feats is not None:
        base.features = feats
    seed_ = None if rng.random() < 0.5 else int(rng.integers(1 << 31))
    rounds = "auto" if rng.random() < 0.7 else int(rng.integers(1, 4))
    return mesh, target, seed_, rounds


def _placement(seed):
    # drawn from its own stream so the cases of _case(seed) stay what they were
    return "inverse" if np.random.default_rng([seed, 7]).random() < 0.25 else "average"


def _oracle(oracle, mesh, target, seed, rounds, placement="average"):
    base = mesh.mesh if isinstance(mesh, mfg.BatchedMesh) else mesh
    kw = dict(target=target, seed=seed, rounds=rounds, order=einsum_order(), placement=placement)
    if isinstance(mesh, mfg.BatchedMesh):
        kw.update(vertex_offsets=mesh.vertex_offsets, facet_offsets=mesh.facet_offsets)
    return oracle.decimate(base.positions, base.facets, base.features, **kw)


def _same(a, b):
    a, b = np.ascontiguousarray(a), np.ascontiguousarray(b)
    return a.shape == b.shape and a.dtype == b.dtype and np.array_equal(a.view(np.uint8), b.view(np.uint8))


# MF_FUZZ_SEEDS=a:b widens the sweep (the default 120 cases run in the round-end suite)
_LO, _HI = (int(x) for x in os.environ.get("MF_FUZZ_SEEDS", "0:120").split(":"))
# found by wider sweeps: batches whose lowest failing entry fails in a LATER round than a
# higher entry (decimate.py:354-361 raises the lowest entry's error)
_REGRESSIONS = [966, 1120, 3338, 8790]


@pytest.mark.parametrize("placement", ["average", "inverse"])
def test_identity_rounds_inside_a_chain(oracle, placement):
    """A fixed round count that interpolates to targets equal to the input size (16 -> 16 -> 16
    -> 15): those rounds are _identity_result (decimate.py:231-233), and 'inverse' singletons
    must not move; alone and as entries of a batch beside meshes with real rounds."""
    small = S.perturbed_grid(4, noise=0.01, seed=3)
    big = S.delaunay_terrain(40, seed=5)  # 40 -> 29 -> 21 -> 15: real rounds
    for mesh in (small, mfg.concat_batch([small, big, small])):
        base = mesh.mesh if isinstance(mesh, mfg.BatchedMesh) else mesh
        cfg = mfg.DecimationConfig(target_vertices=15, rounds=3, placement=placement)
        res = mfg.decimate_parallel(mesh, cfg, device=0)
        exp = _oracle(oracle, mesh, 15, None, 3, placement)
        got = res.mesh.mesh if isinstance(res.mesh, mfg.BatchedMesh) else res.mesh
        for key, g in (("replace", res.replace), ("mapping", res.mapping), ("facets", got.facets),
                       ("positions", got.positions)):
            assert _same(g, exp[key]), key


@pytest.mark.parametrize("seed", sorted(set(range(_LO, _HI)) | set(_REGRESSIONS)))
def test_random_configuration_matches_oracle(oracle, seed):
    mesh, target, shuffle, rounds = _case(seed)
    placement = _placement(seed)
    cfg = mfg.DecimationConfig(target_vertices=target, shuffle_seed=shuffle, rounds=rounds, placement=placement)
    try:
        exp = _oracle(oracle, mesh, target, shuffle, rounds, placement)
    except oracle.OracleInfeasible as e:
        with pytest.raises(mfg.InfeasibleTargetError) as err:
            mfg.decimate_parallel(mesh, cfg, device=0)
        assert err.value.achievable_vertices == e.achievable_vertices
        return
    res = mfg.decimate_parallel(mesh, cfg, device=0)
    base = res.mesh.mesh if isinstance(res.mesh, mfg.BatchedMesh) else res.mesh
    for key, got in (("replace", res.replace), ("mapping", res.mapping), ("facets", base.facets),
                     ("positions", base.positions), ("features", base.features)):
        assert _same(got, exp[key]), key
    if isinstance(mesh, mfg.BatchedMesh):
        assert np.array_equal(res.mesh.vertex_offsets, exp["vertex_offsets"])
        assert np.array_equal(res.mesh.facet_offsets, exp["facet_offsets"])
    # the device-tensor API gives the same bytes
    src = mesh.mesh if isinstance(mesh, mfg.BatchedMesh) else mesh
    nv = np.diff(mesh.vertex_offsets) if isinstance(mesh, mfg.BatchedMesh) else None
    nf = np.diff(mesh.facet_offsets) if isinstance(mesh, mfg.BatchedMesh) else None
    X = None if src.features is src.positions or src.features.shape[1] == 3 and np.array_equal(
        src.features, src.positions) else torch.from_numpy(np.ascontiguousarray(src.features)).cuda()
    dd = T.decimate(torch.from_numpy(src.positions).cuda(), torch.from_numpy(src.facets).cuda(), nv, nf,
                    target=target, seed=shuffle, rounds=rounds, features=X, placement=placement)
    assert np.array_equal(dd.replace.cpu().numpy(), exp["replace"])
    assert np.array_equal(dd.mapping.cpu().numpy(), exp["mapping"])
    assert np.array_equal(dd.faces.cpu().numpy(), exp["facets"])
    assert _same(dd.vertices.cpu().numpy(), exp["positions"])
    # a chained second level (the result's mesh fed back in) equals the oracle's second level
    t2 = max(1, target // 2)
    cfg2 = mfg.DecimationConfig(target_vertices=t2, shuffle_seed=shuffle, placement=placement)
    try:
        exp2 = _oracle(oracle, mfg.BatchedMesh(mfg.TriMesh(exp["positions"], exp["facets"], exp["features"]),
                                                exp["vertex_offsets"], exp["facet_offsets"])
                       if isinstance(mesh, mfg.BatchedMesh) else
                       mfg.TriMesh(exp["positions"], exp["facets"], exp["features"]), t2, shuffle, "auto", placement)
    except (oracle.OracleInfeasible, oracle.OracleStructural):
        return
    except ValueError:
        return
    res2 = mfg.decimate_parallel(res.mesh, cfg2, device=0)
    base2 = res2.mesh.mesh if isinstance(res2.mesh, mfg.BatchedMesh) else res2.mesh
    for key, got in (("replace", res2.replace), ("mapping", res2.mapping), ("facets", base2.facets),
                     ("positions", base2.positions), ("features", base2.features)):
        assert _same(got, exp2[key]), "level 2 " + key
