"""The C oracle against the REAL reference, live (decimation and pooling), on the seeded fuzz
generators of the GPU suite
(test_gpu_fuzz.py: terrains / grids / icospheres / unions / shuffled ids with duplicate facets,
batches, float32 / float64 features, seeded ranks, fixed or auto rounds, both placements;
test_gpu_fuzz2.py: facet soups, hub fans, flat grids, isolated and coincident vertices).  The GPU
suite checks the CUDA path against the oracle on the same cases, so together they pin the CUDA
path to meshforge on inputs no committed fixture holds.  Runs only where the reference tree is
present (this container; it does not travel to the GPU box)."""

import os
import sys

import numpy as np
import pytest

REF = "/root/reference/pkg/src"
pytestmark = pytest.mark.skipif(not os.path.isdir(REF), reason="reference tree not present")

HERE = os.path.dirname(os.path.abspath(__file__))


@pytest.fixture(scope="module")
def ref():
    sys.path.insert(0, REF)
    try:
        import meshforge
    finally:
        sys.path.remove(REF)
    return meshforge


def _same(a, b):
    a, b = np.ascontiguousarray(a), np.ascontiguousarray(b)
    return a.shape == b.shape and a.dtype == b.dtype and np.array_equal(a.view(np.uint8), b.view(np.uint8))


def _compare(ref, oracle, mesh_parts, oracle_call, cfg):
    try:
        exp = oracle_call()
        oe = None
    except oracle.OracleInfeasible as e:
        exp, oe = None, e.achievable_vertices
    try:
        rm = mesh_parts[0] if len(mesh_parts) == 1 else ref.concat_batch(mesh_parts)
        r = ref.decimate_parallel(rm, ref.DecimationConfig(**cfg))
        re_ = None
    except ref.InfeasibleTargetError as e:
        r, re_ = None, e.achievable_vertices
    assert (r is None) == (exp is None) and oe == re_
    if r is None:
        return
    out = r.mesh if isinstance(r.mesh, ref.TriMesh) else r.mesh.mesh
    for key, got in (("replace", r.replace), ("mapping", r.mapping), ("facets", out.facets),
                     ("positions", out.positions), ("features", out.features)):
        assert _same(got, exp[key]), key


@pytest.mark.parametrize("seed", range(0, 400, 10))
def test_fuzz_cases_oracle_equals_reference(ref, oracle, seed):
    sys.path.insert(0, HERE)
    import test_gpu_fuzz as T

    import paper_2103_15076_b200 as mfg

    mesh, target, shuffle, rounds = T._case(seed)
    placement = T._placement(seed)
    base = mesh.mesh if isinstance(mesh, mfg.BatchedMesh) else mesh
    if isinstance(mesh, mfg.BatchedMesh):
        vo, fo = mesh.vertex_offsets, mesh.facet_offsets
        parts = [ref.TriMesh(base.positions[a:b], base.facets[c:d] - a,
                             None if base.features is None else base.features[a:b])
                 for a, b, c, d in zip(vo[:-1], vo[1:], fo[:-1], fo[1:])]
    else:
        parts = [ref.TriMesh(base.positions, base.facets, base.features)]
    _compare(ref, oracle, parts, lambda: T._oracle(oracle, mesh, target, shuffle, rounds, placement),
             dict(target_vertices=target, placement=placement, shuffle_seed=shuffle, rounds=rounds))


@pytest.mark.parametrize("seed", range(0, 400, 10))
def test_structure_cases_oracle_equals_reference(ref, oracle, seed):
    sys.path.insert(0, HERE)
    import test_gpu_fuzz2 as T2

    from paper_2103_15076_b200.numerics import einsum_order

    rng = np.random.default_rng(10_000 + seed)
    mesh = T2._KINDS[seed % len(T2._KINDS)](rng)
    n = mesh.n_vertices
    target = max(1, int(n * rng.uniform(0.2, 0.95)))
    placement = "inverse" if rng.random() < 0.3 else "average"
    shuffle = None if rng.random() < 0.6 else int(rng.integers(1 << 31))
    rounds = "auto" if rng.random() < 0.7 else int(rng.integers(1, 4))
    _compare(ref, oracle, [ref.TriMesh(mesh.positions, mesh.facets)],
             lambda: oracle.decimate(mesh.positions, mesh.facets, None, target=target, seed=shuffle, rounds=rounds,
                                     order=einsum_order(), placement=placement),
             dict(target_vertices=target, placement=placement, shuffle_seed=shuffle, rounds=rounds))


@pytest.mark.parametrize("seed", range(0, 200, 10))
def test_pooling_oracle_equals_reference(ref, oracle, seed):
    """pool (4 modes, f32 / f64, weights) and unpool over the reference's own decimation of a
    structure-fuzz mesh: the oracle's restatement against meshforge.pooling, bit for bit."""
    sys.path.insert(0, HERE)
    import test_gpu_fuzz2 as T2

    rng = np.random.default_rng(20_000 + seed)
    mesh = T2._KINDS[seed % len(T2._KINDS)](rng)
    n = mesh.n_vertices
    try:
        r = ref.decimate_parallel(ref.TriMesh(mesh.positions, mesh.facets),
                                  ref.DecimationConfig(target_vertices=max(1, n // 2)))
    except ref.InfeasibleTargetError:
        return
    n_out = r.n_vertices_out
    for dt in (np.float32, np.float64):
        X = rng.standard_normal((n, int(rng.integers(1, 9)))).astype(dt)
        X[rng.integers(0, n, 3), 0] = np.nan
        w = rng.uniform(0.1, 2.0, n).astype(dt)
        for mode in ("average", "max", "weighted", "sum"):
            got = ref.pool(X, r, mode=mode, weights=w if mode == "weighted" else None)
            exp = oracle.pool(X, r.replace, n_out, mode, weights=w if mode == "weighted" else None)
            assert _same(np.asarray(got), exp), (mode, dt)
        coarse = rng.standard_normal((n_out, X.shape[1])).astype(dt)
        assert _same(np.asarray(ref.unpool(coarse, r)), oracle.unpool(coarse, r.replace))
