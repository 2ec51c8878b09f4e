"""GPU decimation parity: CUDA path vs the CPU oracle, bitwise, on seeded
synthetic inputs (replace, mapping, facets, positions, features, offsets)."""

import numpy as np
import pytest

import paper_2103_15076_b200 as mfg
from paper_2103_15076_b200 import synthetic as S
from paper_2103_15076_b200.numerics import einsum_order

pytestmark = pytest.mark.gpu

TOY_P = np.array([[-0.8, 0.9, 0.0], [0.5, 1.8, 0.9], [0.0, 0.0, 0.0], [0.5, -0.9, 0.3], [1.0, 0.0, 0.0],
                  [1.8, 0.9, 0.0]])
TOY_F = np.array([[0, 2, 4], [5, 2, 4], [2, 3, 4], [0, 1, 5]])


def bits(a):
    a = np.ascontiguousarray(a)
    return a.view(np.uint8)


def assert_same(res, ref, batched=False):
    pairs = [("replace", res.replace), ("mapping", res.mapping), ("facets", res.mesh.facets),
             ("positions", res.mesh.positions), ("features", res.mesh.features)]
    if batched:
        pairs += [("vertex_offsets", res.mesh.vertex_offsets), ("facet_offsets", res.mesh.facet_offsets)]
    for key, got in pairs:
        exp = ref[key]
        assert got.shape == exp.shape, (key, got.shape, exp.shape)
        assert got.dtype == exp.dtype, (key, got.dtype, exp.dtype)
        if not np.array_equal(bits(got), bits(exp)):
            bad = np.flatnonzero((np.asarray(got) != exp).reshape(len(got), -1).any(axis=1)) if got.ndim else []
            raise AssertionError(f"{key} differs at {len(bad)} rows, first {bad[:5]}")


def run_both(oracle, mesh, target, seed=None, rounds="auto"):
    res = mfg.decimate_parallel(mesh, mfg.DecimationConfig(target_vertices=target, shuffle_seed=seed, rounds=rounds))
    if isinstance(mesh, mfg.BatchedMesh):
        ref = oracle.decimate(mesh.positions, mesh.facets, mesh.features, target=target, rounds=rounds, seed=seed,
                              order=einsum_order(), vertex_offsets=mesh.vertex_offsets,
                              facet_offsets=mesh.facet_offsets)
        assert_same(res, ref, batched=True)
    else:
        ref = oracle.decimate(mesh.positions, mesh.facets, mesh.features, target=target, rounds=rounds, seed=seed,
                              order=einsum_order())
        assert_same(res, ref)
    return res


def test_toy_fixture(oracle):
    res = run_both(oracle, mfg.TriMesh(TOY_P, TOY_F), 2, rounds=1)
    np.testing.assert_array_equal(res.replace, [0, 0, 1, 1, 1, 0])
    np.testing.assert_array_equal(res.mapping, [-1] * 6)
    assert [c.members for c in mfg.clusters(res)] == [(0, 1, 5), (2, 3, 4)]


@pytest.mark.parametrize("seed", [None, 0, 7])
def test_icosphere5(oracle, seed):
    run_both(oracle, S.icosphere(5), 3585, seed=seed)


@pytest.mark.parametrize("n,target,seed,rounds", [
    (1000, 130, None, "auto"), (400, 100, None, 2), (2000, 700, 3, "auto"), (300, 150, 7, "auto"),
    (200, 199, None, "auto"), (500, 250, None, 1),
])
def test_terrain_small(oracle, n, target, seed, rounds):
    run_both(oracle, S.delaunay_terrain(n, seed=n + 1), target, seed=seed, rounds=rounds)


@pytest.mark.parametrize("seed", [None, 1])
def test_flat_grid_ties(oracle, seed):
    run_both(oracle, S.flat_grid(40), 800, seed=seed)


def test_terrain_115k(oracle):
    run_both(oracle, S.delaunay_terrain(115_114, noise=0.02, seed=12), 41_449)


def test_terrain_115k_seeded(oracle):
    run_both(oracle, S.delaunay_terrain(115_114, noise=0.02, seed=12), 41_449, seed=3)


@pytest.mark.parametrize("seed", [None, 3])
def test_batch(oracle, seed):
    meshes = [S.delaunay_terrain(120 + 31 * b, seed=20 + b) for b in range(4)] + [S.icosphere(1)]
    run_both(oracle, mfg.concat_batch(meshes), 42, seed=seed)


def test_batch_mixed_chains(oracle):
    # 0/1/2-round chains and one entry already at target (bypassed)
    meshes = [S.delaunay_terrain(n, seed=n) for n in (60, 120, 250, 60, 90)]
    run_both(oracle, mfg.concat_batch(meshes), 60, seed=9)


def test_degenerate_and_duplicate_input(oracle):
    P = np.array([[0, 0, 0], [1, 0, 0], [0, 1, 0], [9, 9, 9], [2, 0, 0], [1, 1, 0], [3, 3, 0]], float)
    F = np.array([[0, 1, 2], [1, 4, 5], [0, 1, 4], [1, 2, 5], [2, 1, 5], [0, 4, 6], [0, 1, 2]])
    run_both(oracle, mfg.TriMesh(P, F), 4, rounds=1)
    run_both(oracle, mfg.TriMesh(P, F), 5, seed=3)


def test_infeasible(oracle):
    mesh = mfg.TriMesh(np.array([[0, 0, 0], [1, 0, 0], [0, 1, 0], [5, 5, 5], [6, 5, 5], [5, 6, 5]], float),
                       [[0, 1, 2], [3, 4, 5]])
    assert mfg.decimate_parallel(mesh, mfg.DecimationConfig(target_vertices=2, rounds=1)).mesh.n_vertices == 2
    with pytest.raises(mfg.InfeasibleTargetError) as err:
        mfg.decimate_parallel(mesh, mfg.DecimationConfig(target_vertices=1, rounds=1))
    assert err.value.achievable_vertices == 2


def test_features_float32_and_channels(oracle):
    mesh = S.delaunay_terrain(800, seed=5)
    feats = np.random.default_rng(0).standard_normal((800, 7)).astype(np.float32)
    m2 = mfg.TriMesh(mesh.positions, mesh.facets, feats)
    run_both(oracle, m2, 300, seed=2)


@pytest.mark.parametrize("n,where", [(800, "head"), (800, "tail"), (800_000, "tail")])
def test_features_like_positions_but_different(oracle, n, where):
    """float64 (n, 3) features are first assumed to be the positions (the default) and
    verified while the rounds run -- on the host for small meshes, on the device (side-stream
    upload) for large ones; one differing word must make the call carry them."""
    mesh = S.delaunay_terrain(n, seed=6)
    feats = mesh.positions.copy()
    feats[0 if where == "head" else -1, 2] += 0.5
    m2 = mfg.TriMesh(mesh.positions, mesh.facets, feats)
    run_both(oracle, m2, n // 3)
    # and the exact copy (aliased) still matches
    run_both(oracle, mfg.TriMesh(mesh.positions, mesh.facets, mesh.positions.copy()), n // 3)


def fan_mesh(k, seed=0, lift=0.0):
    """One hub vertex of degree k (heavy tier when k > 32) inside a ring."""
    rng = np.random.default_rng(seed)
    ang = np.sort(rng.random(k)) * 2 * np.pi
    ring = np.stack([np.cos(ang), np.sin(ang), lift * rng.standard_normal(k)], axis=1)
    P = np.concatenate([[[0.0, 0.0, 0.3]], ring])
    F = np.array([[0, 1 + i, 1 + (i + 1) % k] for i in range(k)])
    return mfg.TriMesh(P, F)


@pytest.mark.parametrize("k,target,seed", [(40, 20, None), (300, 100, None), (3000, 1000, 4), (5000, 2600, None)])
def test_heavy_hub(oracle, k, target, seed):
    run_both(oracle, fan_mesh(k, seed=k, lift=0.05), target, seed=seed)


def test_fan_absorb_to_achievable(oracle):
    # one round down to the achievable minimum: maximal matching + absorption
    run_both(oracle, fan_mesh(200, seed=1, lift=0.0), 88, rounds=1)
    with pytest.raises(mfg.InfeasibleTargetError) as err:
        mfg.decimate_parallel(fan_mesh(200, seed=1), mfg.DecimationConfig(87, rounds=1))
    assert err.value.achievable_vertices == 88


@pytest.mark.parametrize("seed", [None, 2])
def test_flat_grid_sweep(oracle, seed):
    run_both(oracle, S.flat_grid(150), 11250, seed=seed)


@pytest.mark.parametrize("i", range(12))
def test_random_small(oracle, i):
    rng = np.random.default_rng(100 + i)
    n = int(rng.integers(5, 400))
    mesh = S.delaunay_terrain(n, noise=float(rng.random()), seed=1000 + i)
    target = int(rng.integers(1, n))
    seed = None if i % 2 else int(rng.integers(0, 1000))
    rounds = ["auto", 1, 2, 3][i % 4]
    try:
        ref = oracle.decimate(mesh.positions, mesh.facets, None, target=target, rounds=rounds, seed=seed,
                              order=einsum_order())
    except oracle.OracleInfeasible as e:
        with pytest.raises(mfg.InfeasibleTargetError) as err:
            mfg.decimate_parallel(mesh, mfg.DecimationConfig(target, shuffle_seed=seed, rounds=rounds))
        assert err.value.achievable_vertices == e.achievable_vertices
        return
    res = mfg.decimate_parallel(mesh, mfg.DecimationConfig(target, shuffle_seed=seed, rounds=rounds))
    assert_same(res, ref)


def test_big_batch_random(oracle):
    rng = np.random.default_rng(5)
    meshes = [S.delaunay_terrain(int(rng.integers(40, 900)), seed=int(s)) for s in rng.integers(0, 10**6, 40)]
    run_both(oracle, mfg.concat_batch(meshes), 40, seed=13)
    run_both(oracle, mfg.concat_batch(meshes), 40)


@pytest.mark.parametrize("seed", [None, 5])
def test_large_grid_ld_path(oracle, seed):
    # >= 512k vertices: locally-dominant rounds + Suitor residual
    mesh = S.perturbed_grid(760, noise=0.02, seed=1)
    run_both(oracle, mesh, -(-mesh.n_vertices // 2), seed=seed)


def test_large_flat_grid_ld_then_suitor(oracle):
    # all costs tie: LD rounds sweep slowly, the residual frontier goes to Suitor
    mesh = S.flat_grid(730)
    run_both(oracle, mesh, -(-mesh.n_vertices // 2))


@pytest.mark.parametrize("seed", [None, 7])
def test_forced_ld_small(oracle, seed, monkeypatch):
    monkeypatch.setenv("MF_LD_MIN", "0")
    run_both(oracle, S.delaunay_terrain(20_000, noise=0.02, seed=4), 6_000, seed=seed)
    run_both(oracle, S.flat_grid(60), 1_800, seed=seed)
    meshes = [S.delaunay_terrain(300 + 40 * b, seed=b) for b in range(6)]
    run_both(oracle, mfg.concat_batch(meshes), 150, seed=seed)


@pytest.mark.parametrize("mesh_fn,target,seed", [
    (lambda: S.delaunay_terrain(20_000, noise=0.02, seed=1), 5_000, None),
    (lambda: S.icosphere(4), 900, None),
    (lambda: S.perturbed_grid(60, noise=0.02, seed=0), 900, 3),
    (lambda: S.flat_grid(40), 800, None),
])
def test_inverse_placement_matches_oracle(oracle, mesh_fn, target, seed):
    # same scalar algorithm on both sides (Jacobi |eig| range + partial-pivot LU, no FMA): bitwise
    mesh = mesh_fn()
    res = mfg.decimate_parallel(mesh, mfg.DecimationConfig(target, shuffle_seed=seed, placement="inverse"))
    ref = oracle.decimate(mesh.positions, mesh.facets, mesh.features, target=target, seed=seed,
                          order=einsum_order(), placement="inverse")
    assert_same(res, ref)
