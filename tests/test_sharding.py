"""Multi-GPU host logic: contiguous facet-balanced shards, the merge, and
world_size-2 gloo runs where each rank decimates its shard -- with the CPU
oracle standing in for the per-rank device (CPU tests) or with the real CUDA
path, both ranks on cuda:0 (GPU tests).  The merged result must equal the
whole batch decimated at once, bit for bit; a failing batch entry must raise
the lowest failing entry's exception on EVERY rank (decimate.py:354-361)."""

import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

import paper_2103_15076_b200 as mfg
from paper_2103_15076_b200 import sharding
from paper_2103_15076_b200 import synthetic as S


def small_batch():
    return mfg.concat_batch([S.delaunay_terrain(60 + 23 * b, seed=b) for b in range(7)])


def oracle_decimate(batch, config):
    from oracle import oracle as O

    out = O.decimate(batch.positions, batch.facets, batch.features, target=config.target_vertices,
                     rounds=config.rounds, seed=config.shuffle_seed, vertex_offsets=batch.vertex_offsets,
                     facet_offsets=batch.facet_offsets)
    tm = mfg.TriMesh(out["positions"], out["facets"], out["features"])
    return mfg.DecimationResult(mesh=mfg.BatchedMesh(tm, out["vertex_offsets"], out["facet_offsets"]),
                                replace=out["replace"], mapping=out["mapping"])


def iso_mesh(n=50):
    """One triangle plus n-3 isolated vertices: decimating it below n-2 is infeasible."""
    P = np.random.default_rng(n).random((n, 3))
    return mfg.TriMesh(P, np.array([[0, 1, 2]]))


def failing_batch():
    """Entries 3 and 5 fail at target 40 (InfeasibleTargetError, achievable 48); entry 6 is
    too small (ValueError).  The lowest failing entry is 3."""
    ms = [S.delaunay_terrain(60 + 23 * b, seed=b) for b in range(3)] + [iso_mesh(), S.delaunay_terrain(120, seed=4),
                                                                        iso_mesh(), S.delaunay_terrain(30, seed=6)]
    return mfg.concat_batch(ms)


def oracle_decimate_per_mesh(batch, config):
    """oracle_decimate, raising the package's exceptions with the failing entry's index."""
    from oracle import oracle as O

    for b in range(len(batch.vertex_offsets) - 1):
        v0, v1, f0, f1 = (batch.vertex_offsets[b], batch.vertex_offsets[b + 1], batch.facet_offsets[b],
                          batch.facet_offsets[b + 1])
        n = v1 - v0
        try:
            if config.target_vertices > n:
                raise ValueError(f"target_vertices={config.target_vertices} exceeds the input size {n}")
            O.decimate(batch.positions[v0:v1], batch.facets[f0:f1] - v0, None, target=config.target_vertices,
                       rounds=config.rounds, seed=config.shuffle_seed)
        except O.OracleInfeasible as e:
            err = mfg.InfeasibleTargetError(str(e), achievable_vertices=e.achievable_vertices)
            err.mesh_index = b
            raise err
        except ValueError as e:
            e.mesh_index = b
            raise
    return oracle_decimate(batch, config)


def test_shard_bounds_contiguous_and_balanced():
    fc = [100, 100, 100, 100, 400, 100, 100]
    b = sharding.shard_bounds(fc, 2)
    assert b[0][0] == 0 and b[-1][1] == len(fc) and b[0][1] == b[1][0]
    assert sharding.shard_bounds(fc, 1) == [(0, 7)]
    for w in (2, 3, 4, 8, 16):
        bb = sharding.shard_bounds(fc, w)
        assert len(bb) == w and all(lo <= hi for lo, hi in bb)
        assert [x for lo, hi in bb for x in range(lo, hi)] == list(range(7))


def test_merge_of_shards_equals_whole_batch():
    batch = small_batch()
    cfg = mfg.DecimationConfig(target_vertices=40, shuffle_seed=3)
    whole = oracle_decimate(batch, cfg)
    parts = []
    for r in range(3):
        sub, lo, hi = sharding.shard_batch(batch, 3, r)
        parts.append(oracle_decimate(sub, cfg) if sub is not None else None)
    merged = sharding.merge_results(parts)
    for a, b in ((merged.replace, whole.replace), (merged.mapping, whole.mapping),
                 (merged.mesh.facets, whole.mesh.facets), (merged.mesh.positions, whole.mesh.positions),
                 (merged.mesh.vertex_offsets, whole.mesh.vertex_offsets),
                 (merged.mesh.facet_offsets, whole.mesh.facet_offsets)):
        np.testing.assert_array_equal(a, b)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, queue, use_gpu):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        if use_gpu:  # the real CUDA path on every rank (one box has one GPU here: both on cuda:0)
            fn = whole_fn = fail_fn = lambda b, c: mfg.decimate_parallel(b, c, device=0)  # noqa: E731
        else:
            fn, whole_fn, fail_fn = oracle_decimate, oracle_decimate, oracle_decimate_per_mesh
        batch = small_batch()
        cfg = mfg.DecimationConfig(target_vertices=40, shuffle_seed=5)
        res = sharding.decimate_sharded(batch, cfg, decimate_fn=fn)
        whole = whole_fn(batch, cfg)
        ok = all(np.array_equal(np.asarray(a).view(np.uint8), np.asarray(b).view(np.uint8)) for a, b in (
            (res.replace, whole.replace), (res.mapping, whole.mapping), (res.mesh.facets, whole.mesh.facets),
            (res.mesh.positions, whole.mesh.positions), (res.mesh.features, whole.mesh.features),
            (res.mesh.vertex_offsets, whole.mesh.vertex_offsets), (res.mesh.facet_offsets, whole.mesh.facet_offsets)))
        # a failing entry: every rank raises the lowest failing entry's exception (global index)
        fb = failing_batch()
        errs = []
        try:
            sharding.decimate_sharded(fb, mfg.DecimationConfig(target_vertices=40), decimate_fn=fail_fn)
            errs.append(None)
        except Exception as e:  # noqa: BLE001
            errs.append((type(e).__name__, getattr(e, "mesh_index", None), getattr(e, "achievable_vertices", None)))
        if use_gpu:  # and the same exception as the whole batch on one device
            try:
                fail_fn(fb, mfg.DecimationConfig(target_vertices=40))
                errs.append(None)
            except Exception as e:  # noqa: BLE001
                errs.append((type(e).__name__, getattr(e, "mesh_index", None),
                             getattr(e, "achievable_vertices", None)))
        bounds = sharding.shard_bounds(np.diff(fb.facet_offsets), world)
        queue.put((rank, ok, errs, bounds))
    finally:
        dist.destroy_process_group()


def _run_world2(use_gpu):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q, use_gpu)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=300)
    assert all(p.exitcode == 0 for p in procs)
    out = sorted(q.get(timeout=5) for _ in procs)
    for rank, ok, errs, bounds in out:
        assert ok, f"rank {rank}: merged result differs from the whole batch"
        # entries 3 and 5 are infeasible (achievable 48 = 50 - 2), entry 6 too small: entry 3 wins
        for e in errs:
            assert e == ("InfeasibleTargetError", 3, 48), (rank, e)
    # the failing entries must span both ranks for the exchange to matter
    (lo0, hi0), (lo1, hi1) = out[0][3]
    assert lo0 <= 3 < hi0 or lo1 <= 3 < hi1
    assert lo1 <= 5 < hi1


def test_gloo_world2_sharded_decimation():
    _run_world2(use_gpu=False)


@pytest.mark.gpu
def test_gpu_gloo_world2_sharded_decimation():
    """decimate_sharded with the real CUDA decimation on 2 ranks (gloo, both on cuda:0)."""
    _run_world2(use_gpu=True)


@pytest.mark.gpu
def test_gpu_shard_equals_whole():
    batch = small_batch()
    cfg = mfg.DecimationConfig(target_vertices=40, shuffle_seed=5)
    whole = mfg.decimate_parallel(batch, cfg)
    parts = [mfg.decimate_parallel(sharding.shard_batch(batch, 2, r)[0], cfg) for r in range(2)]
    merged = sharding.merge_results(parts)
    np.testing.assert_array_equal(merged.replace, whole.replace)
    np.testing.assert_array_equal(merged.mesh.facets, whole.mesh.facets)
    np.testing.assert_array_equal(merged.mesh.positions, whole.mesh.positions)
