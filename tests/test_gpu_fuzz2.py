"""Structure fuzz, bit for bit against the C oracle: meshes the smooth generators of
test_gpu_fuzz.py never produce -- random facet soups (non-manifold edges, isolated vertices),
high-degree fans (the heavy / mid vertex tiers), flat grids (all-zero costs, ties broken by the
edge order), coincident vertices -- under both placements, followed by pool (4 modes, float32
and float64, weights), unpool and pool_backward of random features over the result, and
quality_report's per-output-vertex quadric errors."""

import os

import numpy as np
import pytest

import paper_2103_15076_b200 as mfg
from paper_2103_15076_b200 import synthetic as S
from paper_2103_15076_b200.numerics import einsum_order

pytestmark = pytest.mark.gpu

_LO, _HI = (int(x) for x in os.environ.get("MF_FUZZ2_SEEDS", "0:60").split(":"))
# found by wider sweeps: 'inverse' with a fixed round count whose first rounds are identities
_REGRESSIONS = [2709]


def _soup(rng):
    n = int(rng.integers(8, 3000))
    m = int(n * rng.uniform(0.5, 3.0))
    F = np.stack([rng.choice(n, 3, replace=False) for _ in range(m)])
    P = rng.standard_normal((n, 3))
    return mfg.TriMesh(P, F)


def _fan(rng):
    hubs = int(rng.integers(1, 4))
    P, F, base = [], [], 0
    for _ in range(hubs):
        d = int(rng.integers(3, 2500))
        t = np.sort(rng.uniform(0, 2 * np.pi, d))
        ring = np.stack([np.cos(t), np.sin(t), 0.05 * rng.standard_normal(d)], axis=1) * rng.uniform(0.5, 2)
        P.append(np.concatenate([[[0.0, 0.0, 0.0]], ring]) + base * 3.0)
        i = np.arange(d)
        F.append(np.stack([np.zeros(d, np.int64), 1 + i, 1 + (i + 1) % d], axis=1) + base)
        base += d + 1
    return mfg.TriMesh(np.concatenate(P), np.concatenate(F))


def _flat(rng):
    m = S.perturbed_grid(int(rng.integers(3, 60)), int(rng.integers(3, 60)), noise=0.0)
    P = m.positions.copy()
    P[:, 2] = 0.0  # exactly planar: every pair cost is 0, the rank order is the edge order
    return mfg.TriMesh(P, m.facets)


def _isolated(rng):
    a = S.delaunay_terrain(int(rng.integers(30, 2000)), seed=int(rng.integers(1 << 30)))
    k = int(rng.integers(1, 50))
    n = a.n_vertices + k
    perm = rng.permutation(n)  # the unreferenced vertices end up anywhere in the id range
    P = np.empty((n, 3))
    P[perm[: a.n_vertices]] = a.positions
    P[perm[a.n_vertices:]] = rng.standard_normal((k, 3))
    return mfg.TriMesh(P, perm[a.facets])


def _coincident(rng):
    a = S.perturbed_grid(int(rng.integers(4, 50)), noise=0.01, seed=int(rng.integers(1 << 30)))
    P = a.positions.copy()
    idx = rng.choice(len(P), size=max(1, len(P) // 10), replace=False)
    P[idx] = P[rng.choice(len(P), size=len(idx))]  # some vertices share coordinates
    return mfg.TriMesh(P, a.facets)


_KINDS = [_soup, _fan, _flat, _isolated, _coincident]


def _same(a, b):
    a, b = np.ascontiguousarray(a), np.ascontiguousarray(b)
    return a.shape == b.shape and a.dtype == b.dtype and np.array_equal(a.view(np.uint8), b.view(np.uint8))


@pytest.mark.parametrize("seed", sorted(set(range(_LO, _HI)) | set(_REGRESSIONS)))
def test_structure_fuzz_matches_oracle(oracle, seed):
    rng = np.random.default_rng(10_000 + seed)
    mesh = _KINDS[seed % len(_KINDS)](rng)
    n = mesh.n_vertices
    target = max(1, int(n * rng.uniform(0.2, 0.95)))
    placement = "inverse" if rng.random() < 0.3 else "average"
    shuffle = None if rng.random() < 0.6 else int(rng.integers(1 << 31))
    rounds = "auto" if rng.random() < 0.7 else int(rng.integers(1, 4))
    cfg = mfg.DecimationConfig(target_vertices=target, placement=placement, shuffle_seed=shuffle, rounds=rounds)
    try:
        exp = oracle.decimate(mesh.positions, mesh.facets, None, target=target, seed=shuffle, rounds=rounds,
                              order=einsum_order(), placement=placement)
    except oracle.OracleInfeasible as e:
        with pytest.raises(mfg.InfeasibleTargetError) as err:
            mfg.decimate_parallel(mesh, cfg, device=0)
        assert err.value.achievable_vertices == e.achievable_vertices
        return
    res = mfg.decimate_parallel(mesh, cfg, device=0)
    for key, got in (("replace", res.replace), ("mapping", res.mapping), ("facets", res.mesh.facets),
                     ("positions", res.mesh.positions), ("features", res.mesh.features)):
        assert _same(got, exp[key]), key
    # quality_report's per-output-vertex errors (decimate.py:580-602)
    from paper_2103_15076_b200.quality import quadric_errors

    qe = quadric_errors(mesh, res)
    assert _same(np.asarray(qe), oracle.quality_errors(mesh.positions, mesh.facets, exp["replace"], exp["positions"],
                                                       einsum_order()))
    # pooling over the result
    n_out = len(exp["positions"])
    dt = np.float32 if rng.random() < 0.5 else np.float64
    C = int(rng.integers(1, 40))
    X = rng.standard_normal((n, C)).astype(dt)
    if rng.random() < 0.2:
        X[rng.integers(0, n, size=max(1, n // 20)), rng.integers(0, C)] = X[0, 0]  # ties for max
    mode = ("average", "max", "weighted", "sum")[int(rng.integers(0, 4))]
    w = rng.uniform(0.1, 2.0, n).astype(dt) if mode == "weighted" else None
    got = mfg.pool(X, res, mode, weights=w)
    assert _same(got, oracle.pool(X, exp["replace"], n_out, mode, weights=w)), mode
    coarse = rng.standard_normal((n_out, C)).astype(dt)
    assert _same(mfg.unpool(coarse, res), oracle.unpool(coarse, exp["replace"]))
    if n <= 1500:
        G = rng.standard_normal((n_out, C)).astype(dt)
        gb = mfg.pool_backward(G, X, res, mode, weights=w)
        eb = oracle.pool_backward(G, X, exp["replace"], n_out, mode, weights=w)
        assert gb.dtype == eb.dtype and np.array_equal(gb, eb), mode
