"""Batch sharding across GPUs (one process per GPU), SURVEY.md §8(e).

Meshes of a BatchedMesh are independent (decimate.py:347-361: a batch is
decimated entry by entry), so a batch splits into contiguous slices, one per
rank, balanced by facet count; each rank decimates its slice on its own
device with no inter-GPU traffic, and the per-rank results are merged with
the same offset bookkeeping as the reference's _merge_batch_results
(decimate.py:319-341).  A single mesh does not shard (the greedy matching is
global over its rank order): N GPUs then run independent replicas.
"""

from __future__ import annotations

import numpy as np

from .decimate import DecimationResult, decimate_parallel
from .mesh import BatchedMesh, TriMesh


def shard_bounds(facet_counts, world: int) -> list:
    """Contiguous [lo, hi) mesh ranges per rank, balanced by cumulative facet count."""
    fc = np.asarray(facet_counts, dtype=np.int64)
    n = len(fc)
    if world <= 1 or n == 0:
        return [(0, n)] + [(n, n)] * max(0, world - 1)
    cum = np.concatenate([[0], np.cumsum(fc)])
    total = cum[-1]
    cuts = [0]
    for r in range(1, world):
        target = total * r / world
        k = int(np.searchsorted(cum, target, side="left"))
        k = min(max(k, cuts[-1]), n)
        cuts.append(k)
    cuts.append(n)
    return [(cuts[r], cuts[r + 1]) for r in range(world)]


def shard_batch(batch: BatchedMesh, world: int, rank: int) -> tuple:
    """(sub-batch or None, lo, hi) of the meshes rank `rank` owns."""
    lo, hi = shard_bounds(np.diff(batch.facet_offsets), world)[rank]
    if hi <= lo:
        return None, lo, hi
    vo, fo = batch.vertex_offsets, batch.facet_offsets
    v0, v1, f0, f1 = vo[lo], vo[hi], fo[lo], fo[hi]
    sub = TriMesh.__new__(TriMesh)
    sub.positions = batch.positions[v0:v1]
    sub.facets = batch.facets[f0:f1] - v0
    sub.features = batch.features[v0:v1]
    out = BatchedMesh.__new__(BatchedMesh)
    out.mesh, out.vertex_offsets, out.facet_offsets = sub, vo[lo:hi + 1] - v0, fo[lo:hi + 1] - f0
    return out, lo, hi


def merge_results(parts: list) -> DecimationResult:
    """Concatenate per-rank batch results in rank order (decimate.py:319-341 offsets)."""
    parts = [p for p in parts if p is not None]
    meshes = [p.mesh for p in parts]
    nv = [m.n_vertices for m in meshes]
    vbase = np.concatenate([[0], np.cumsum(nv)]).astype(np.int64)
    fbase = np.concatenate([[0], np.cumsum([m.n_facets for m in meshes])]).astype(np.int64)
    positions = np.concatenate([m.positions for m in meshes])
    facets = np.concatenate([m.facets + vbase[i] for i, m in enumerate(meshes)]).reshape(-1, 3)
    features = np.concatenate([m.features for m in meshes])
    vo = np.concatenate([[0]] + [m.vertex_offsets[1:] + vbase[i] for i, m in enumerate(meshes)]).astype(np.int64)
    fo = np.concatenate([[0]] + [m.facet_offsets[1:] + fbase[i] for i, m in enumerate(meshes)]).astype(np.int64)
    replace = np.concatenate([p.replace + vbase[i] for i, p in enumerate(parts)])
    mapping = np.concatenate([np.where(p.mapping < 0, -1, p.mapping + vbase[i]) for i, p in enumerate(parts)])
    tm = TriMesh.__new__(TriMesh)
    tm.positions, tm.facets, tm.features = positions, facets, features
    bm = BatchedMesh.__new__(BatchedMesh)
    bm.mesh, bm.vertex_offsets, bm.facet_offsets = tm, vo, fo
    return DecimationResult(mesh=bm, replace=replace, mapping=mapping,
                            reached_target=all(p.reached_target for p in parts))


def _error_record(exc: BaseException, lo: int) -> tuple:
    """(global batch index, type, message, achievable_vertices) of a rank's failure: a plain
    tuple travels through all_gather_object where the exception itself would not round-trip
    (InfeasibleTargetError's pickle drops achievable_vertices)."""
    idx = getattr(exc, "mesh_index", None)
    return (lo + (idx or 0), type(exc).__name__, str(exc), getattr(exc, "achievable_vertices", None))


def _raise_record(rec: tuple):
    from . import errors

    _, name, msg, achievable = rec
    if name == "InfeasibleTargetError":
        err = errors.InfeasibleTargetError(msg, achievable_vertices=achievable)
    elif name in ("StructuralError", "MeshError", "NativeError"):
        err = getattr(errors, name)(msg)
    elif name in ("ValueError", "RuntimeError", "TypeError", "IndexError"):
        err = {"ValueError": ValueError, "RuntimeError": RuntimeError, "TypeError": TypeError,
               "IndexError": IndexError}[name](msg)
    else:
        err = RuntimeError(f"{name}: {msg}")
    err.mesh_index = rec[0]
    raise err


def decimate_sharded(batch: BatchedMesh, config, group=None, decimate_fn=None, device=None):
    """Decimate `batch` across the ranks of a torch.distributed group.

    Every rank decimates its contiguous slice (no collective on the data
    path).  The ranks then exchange one status record each: if any slice
    failed, every rank raises the exception of the LOWEST failing batch entry,
    with its global index in `mesh_index` -- what the reference's in-order
    `pool.map` re-raises (decimate.py:354-361) -- instead of leaving the
    healthy ranks blocked in the result exchange.  Otherwise the per-rank
    results are exchanged once with all_gather_object and every rank returns
    the merged result, identical to decimate_parallel(batch, config) on one
    device.
    """
    import torch.distributed as dist

    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    sub, lo, _ = shard_batch(batch, world, rank)
    fn = decimate_fn or (lambda b, c: decimate_parallel(b, c, device=device))
    mine, failure = None, None
    try:
        mine = fn(sub, config) if sub is not None else None
    except Exception as exc:  # noqa: BLE001 -- every failure is re-raised below, on every rank
        if world == 1:
            raise
        failure = _error_record(exc, lo)
    if mine is not None:
        mine = DecimationResult(mesh=mine.mesh, replace=np.asarray(mine.replace), mapping=mine.mapping,
                                reached_target=mine.reached_target)
    if world == 1:
        return merge_results([mine])
    statuses = [None] * world
    dist.all_gather_object(statuses, failure, group=group)
    failed = [s for s in statuses if s is not None]
    if failed:
        _raise_record(min(failed, key=lambda s: s[0]))
    parts = [None] * world
    dist.all_gather_object(parts, mine, group=group)
    return merge_results(parts)
