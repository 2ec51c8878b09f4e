"""Multi-GPU host logic on CPU: contiguous facet-balanced shards, the merge,
and a world_size-2 gloo run where each rank decimates its shard (with the CPU
oracle standing in for the per-rank device) -- the merged result must equal
the whole batch decimated at once, bit for bit."""

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


def _worker(rank, world, port, queue):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        batch = small_batch()
        cfg = mfg.DecimationConfig(target_vertices=40, shuffle_seed=5)
        res = sharding.decimate_sharded(batch, cfg, decimate_fn=oracle_decimate)
        if rank == 0:
            whole = oracle_decimate(batch, cfg)
            ok = all(np.array_equal(a, b) for a, b in (
                (res.replace, whole.replace), (res.mapping, whole.mapping), (res.mesh.facets, whole.mesh.facets),
                (res.mesh.positions, whole.mesh.positions), (res.mesh.vertex_offsets, whole.mesh.vertex_offsets)))
            queue.put(ok)
    finally:
        dist.destroy_process_group()


def test_gloo_world2_sharded_decimation():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=120)
    assert all(p.exitcode == 0 for p in procs)
    assert q.get(timeout=5) is True


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
