"""BASELINE.json configurations at their FULL sizes, compared BIT FOR BIT:

* against the real reference (tests/golden/full.json, digests produced by
  meshforge itself in the build container, tests/golden/make_golden_full.py) --
  run with the fixture host's numpy reduction order;
* against the C oracle run on this host with this host's order (every array, every
  level, cfg3's C=64 max / average pooling and unpooling included).

cfg5's levels 1-2 have >= 2^21 output vertices, so they exercise the wide-key facet
dedupe and the 4-item gather-chain scans that smaller inputs never reach
(tests/test_gpu_variants.py forces those branches at small sizes as well).  The
device-tensor API is exercised at full size too (cfg5 chain through
paper_2103_15076_b200.tensor, checked equal to the numpy API's bytes) plus the
size-independent properties a decimation must have (surjective ordered `replace`,
`mapping` = replace or -1, facets valid and unique).
"""

import functools
import hashlib
import json
import os

import numpy as np
import pytest
import torch

import paper_2103_15076_b200 as mfg
from paper_2103_15076_b200 import synthetic as S
from paper_2103_15076_b200 import tensor as T
from paper_2103_15076_b200.numerics import einsum_order, forced_order

pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))
_FULL_PATH = os.path.join(HERE, "golden", "full.json")
FULL = json.load(open(_FULL_PATH)) if os.path.exists(_FULL_PATH) else {}
ORDER = FULL.get("einsum_order", 0)


def sha(*arrays):
    h = hashlib.sha256()
    for a in arrays:
        a = np.ascontiguousarray(a)
        h.update(str(a.dtype).encode() + str(a.shape).encode())
        h.update(a.tobytes())
    return h.hexdigest()


def input_digest(mesh):
    base = mesh.mesh if isinstance(mesh, mfg.BatchedMesh) else mesh
    parts = [base.positions, base.facets, base.features]
    if isinstance(mesh, mfg.BatchedMesh):
        parts += [mesh.vertex_offsets, mesh.facet_offsets]
    return sha(*parts)


def halving(n, k=4):
    out = []
    for _ in range(k):
        n = -(-n // 2)
        out.append(n)
    return out


def placement_of(cfg):
    return "inverse" if cfg.endswith("_inverse") else "average"


@functools.lru_cache(maxsize=None)
def workload(cfg):
    if cfg.endswith("_inverse"):  # the same meshes and levels under placement='inverse', no pooling
        mesh, levels, _ = workload(cfg[: -len("_inverse")])
        return mesh, levels, None
    if cfg == "cfg3":
        mesh = S.delaunay_terrain(500_000, 0.02, 3)
        feats = np.random.default_rng(0).standard_normal((mesh.n_vertices, 64)).astype(np.float32)
        return mesh, [125_000, 62_500, 31_250, 15_625], feats
    if cfg == "cfg4":
        return mfg.concat_batch([S.delaunay_terrain(2500, 0.02, b) for b in range(256)]), [1250], None
    if cfg == "cfg5":
        mesh = S.perturbed_grid(3163, None, 0.02, 0)
        return mesh, halving(mesh.n_vertices), None
    raise ValueError(cfg)


def _arrays(res):
    base = res.mesh.mesh if isinstance(res.mesh, mfg.BatchedMesh) else res.mesh
    d = dict(replace=res.replace, mapping=res.mapping, facets=base.facets, positions=base.positions,
             features=base.features)
    if isinstance(res.mesh, mfg.BatchedMesh):
        d["vertex_offsets"] = res.mesh.vertex_offsets
        d["facet_offsets"] = res.mesh.facet_offsets
    return d


@functools.lru_cache(maxsize=None)
def gpu_chain(cfg, order):
    """The level chain through the drop-in numpy API (+ max / average pool and unpool)."""
    mesh, levels, feats = workload(cfg)
    out, cur, f = [], mesh, feats
    with forced_order(order):
        for tgt in levels:
            res = mfg.decimate_parallel(cur, mfg.DecimationConfig(target_vertices=tgt, placement=placement_of(cfg)),
                                        device=0)
            a = {k: np.array(v) for k, v in _arrays(res).items()}
            if f is not None:
                a["pool_max"] = mfg.pool(f, res, mode="max")
                a["pool_average"] = mfg.pool(f, res, mode="average")
                a["unpool"] = mfg.unpool(a["pool_max"], res)
                f = a["pool_max"]
            out.append(a)
            cur = res.mesh
    return out


def oracle_chain(oracle, cfg, order):
    mesh, levels, feats = workload(cfg)
    batched = isinstance(mesh, mfg.BatchedMesh)
    base = mesh.mesh if batched else mesh
    P, F, X = base.positions, base.facets, None
    kw = dict(vertex_offsets=mesh.vertex_offsets, facet_offsets=mesh.facet_offsets,
              threads=os.cpu_count() or 1) if batched else {}
    out, f = [], feats
    for tgt in levels:
        o = oracle.decimate(P, F, X, target=tgt, order=order, placement=placement_of(cfg), **kw)
        if f is not None:
            o["pool_max"] = oracle.pool(f, o["replace"], len(o["positions"]), "max")
            o["pool_average"] = oracle.pool(f, o["replace"], len(o["positions"]), "average")
            o["unpool"] = oracle.unpool(o["pool_max"], o["replace"])
            f = o["pool_max"]
        out.append(o)
        P, F, X = o["positions"], o["facets"], o["features"]
        if batched:
            kw.update(vertex_offsets=o["vertex_offsets"], facet_offsets=o["facet_offsets"])
    return out


def _check_reference(cfg):
    if cfg not in FULL:
        pytest.skip(f"tests/golden/full.json has no {cfg} entry (run tests/golden/make_golden_full.py {cfg})")
    g = FULL[cfg]
    mesh, levels, feats = workload(cfg)
    assert input_digest(mesh) == g["input"]
    if feats is not None:
        assert sha(feats) == g["features"]
    got = gpu_chain(cfg, ORDER)
    assert len(got) == len(g["levels"])
    for i, (a, exp) in enumerate(zip(got, g["levels"])):
        assert len(a["positions"]) == exp["n_out"] and len(a["facets"]) == exp["m_out"], f"level {i}"
        for k in ("replace", "mapping", "facets", "positions", "features", "vertex_offsets", "facet_offsets"):
            if k in exp:
                assert sha(a[k]) == exp[k], f"level {i}: {k} differs from the reference"
        if "pool_max" in exp:
            assert sha(a["pool_max"]) == exp["pool_max"], f"level {i}: max-pool differs from the reference"
            assert sha(a["unpool"]) == exp["unpool"], f"level {i}: unpool differs from the reference"


def _check_oracle(oracle, cfg):
    order = einsum_order()
    got = gpu_chain(cfg, order)
    exp = oracle_chain(oracle, cfg, order)
    for i, (a, o) in enumerate(zip(got, exp)):
        for k, v in a.items():
            e = o[k]
            assert v.shape == e.shape and v.dtype == e.dtype, f"level {i}: {k} shape/dtype"
            assert np.array_equal(np.ascontiguousarray(v).view(np.uint8), np.ascontiguousarray(e).view(np.uint8)), \
                f"level {i}: {k} differs from the oracle"


@pytest.mark.parametrize("cfg", ["cfg3", "cfg4", "cfg5", "cfg3_inverse", "cfg4_inverse"])
def test_full_size_matches_reference(cfg):
    """configs[2..4] at full size, digest-equal to meshforge's own outputs (cfg3 / cfg4 also
    under placement='inverse': its solve follows numpy.linalg.solve's operation order)."""
    _check_reference(cfg)


@pytest.mark.parametrize("cfg", ["cfg3", "cfg4", "cfg5", "cfg3_inverse"])
def test_full_size_matches_oracle(oracle, cfg):
    """configs[2..4] at full size, byte-equal to the C oracle on this host."""
    _check_oracle(oracle, cfg)


def _check_level(V, F, dd, target):
    n_in = V.shape[0]
    R, Mp, Vo, Fo = dd.replace, dd.mapping, dd.vertices, dd.faces
    assert dd.n_vertices_out == target and Vo.shape == (target, 3)
    assert R.shape == (n_in,) and int(R.min()) == 0 and int(R.max()) == target - 1
    counts = torch.bincount(R, minlength=target)
    assert int(counts.min()) >= 1  # surjective
    # output index order = order of each cluster's lowest member
    first = torch.full((target,), n_in, dtype=torch.int64, device=R.device)
    first.scatter_reduce_(0, R, torch.arange(n_in, device=R.device), reduce="amin")
    assert bool((first[1:] > first[:-1]).all())
    live = Mp >= 0
    assert bool((Mp[live] == R[live]).all())
    # facets: in range, non-degenerate, unique as sorted triples
    assert int(Fo.min()) >= 0 and int(Fo.max()) < target
    assert bool(((Fo[:, 0] != Fo[:, 1]) & (Fo[:, 1] != Fo[:, 2]) & (Fo[:, 0] != Fo[:, 2])).all())
    srt = torch.sort(Fo, dim=1).values
    key = (srt[:, 0] * target + srt[:, 1]) * target + srt[:, 2]
    assert torch.unique(key).numel() == key.numel()


def test_cfg5_tensor_api_equals_numpy_api():
    """The device-tensor API (north-star interface) at cfg5 size: same bytes as the numpy API,
    valid at every level, deterministic."""
    mesh, levels, _ = workload("cfg5")
    ref = gpu_chain("cfg5", einsum_order())
    V = torch.from_numpy(mesh.positions).cuda()
    F = torch.from_numpy(mesh.facets).cuda()
    for i, t in enumerate(levels):
        dd = T.decimate(V, F, target=t)
        _check_level(V, F, dd, t)
        for k, tv in (("replace", dd.replace), ("mapping", dd.mapping), ("facets", dd.faces),
                      ("positions", dd.vertices)):
            assert np.array_equal(tv.cpu().numpy(), ref[i][k]), f"level {i}: {k}"
        V, F = dd.vertices, dd.faces
