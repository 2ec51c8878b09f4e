"""BASELINE.json configurations at their FULL sizes, checked through size-independent
properties (the bitwise oracle comparisons run at sizes the CPU oracle finishes in
seconds -- tests/test_gpu_parity.py):

* every level: exact output vertex count, `replace` a surjection onto [0, n_out) whose
  output order is the order of each cluster's lowest member (decimate.py:130-137),
  `mapping` = replace or -1 (decimate.py:159-167), facets in range, non-degenerate and
  free of duplicate triples (decimate.py:147-157), positions = member means (one-round
  levels) or inside the members' bounding box (multi-round levels nest means);
* the whole chain is deterministic (two runs give identical bytes);
* a batch equals its entries decimated one by one (decimate.py:347-361, the reference's
  test_decimation.py:175-191) -- for the cfg4 batch of 256 meshes;
* max-pool / unpool of C=64 float32 features equal an independent scatter-max / gather.
"""

import hashlib

import numpy as np
import pytest
import torch

import paper_2103_15076_b200 as mfg
from paper_2103_15076_b200 import synthetic as S
from paper_2103_15076_b200 import tensor as T

pytestmark = pytest.mark.gpu


def _digest(*ts):
    h = hashlib.sha256()
    for t in ts:
        h.update(t.detach().cpu().numpy().tobytes())
    return h.hexdigest()


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
    if len(dd.round_stats()) == 1:
        # one round: positions are the member means (float64 sums in another order: tolerance)
        sums = torch.zeros((target, 3), dtype=torch.float64, device=V.device).index_add_(0, R, V)
        mean = sums / counts[:, None].to(torch.float64)
        assert torch.allclose(Vo, mean, rtol=1e-12, atol=1e-12)
    else:
        # a chain of rounds nests means: each output lies in its members' bounding box
        lo = torch.full((target, 3), float("inf"), dtype=torch.float64, device=V.device)
        hi = torch.full((target, 3), -float("inf"), dtype=torch.float64, device=V.device)
        idx = R[:, None].expand(-1, 3)
        lo.scatter_reduce_(0, idx, V, reduce="amin")
        hi.scatter_reduce_(0, idx, V, reduce="amax")
        assert bool((Vo >= lo - 1e-12).all()) and bool((Vo <= hi + 1e-12).all())


def _chain(mesh, levels):
    V = torch.from_numpy(mesh.positions).cuda()
    F = torch.from_numpy(mesh.facets).cuda()
    out = []
    for t in levels:
        dd = T.decimate(V, F, target=t)
        out.append((V, F, dd, t))
        V, F = dd.vertices, dd.faces
    return out


def test_cfg5_full_grid_hierarchy():
    """configs[4]: perturbed_grid(3163) -- 10,004,569 vertices / 19,996,488 facets, 4 levels."""
    mesh = S.perturbed_grid(3163, noise=0.02, seed=0)
    n, levels = mesh.n_vertices, []
    for _ in range(4):
        n = -(-n // 2)
        levels.append(n)
    a = _chain(mesh, levels)
    for V, F, dd, t in a:
        _check_level(V, F, dd, t)
    b = _chain(mesh, levels)
    for (_, _, d1, _), (_, _, d2, _) in zip(a, b):
        assert _digest(d1.replace, d1.mapping, d1.faces, d1.vertices) == \
            _digest(d2.replace, d2.mapping, d2.faces, d2.vertices)


def test_cfg3_full_terrain_hierarchy_with_pooling():
    """configs[2]: delaunay_terrain(500000) -- ~1M facets, 125k/62.5k/31.25k/15.625k, C=64 max-pool/unpool."""
    mesh = S.delaunay_terrain(500_000, noise=0.02, seed=3)
    levels = [125_000, 62_500, 31_250, 15_625]
    chain = _chain(mesh, levels)
    X = torch.from_numpy(np.random.default_rng(0).standard_normal((mesh.n_vertices, 64)).astype(np.float32)).cuda()
    ups = []
    for V, F, dd, t in chain:
        _check_level(V, F, dd, t)
        P = T.pool(X, dd, mode="max")
        ref = torch.full((t, 64), -float("inf"), dtype=torch.float32, device=X.device)
        ref.scatter_reduce_(0, dd.replace[:, None].expand(-1, 64), X, reduce="amax")
        assert torch.equal(P, ref)
        U = T.unpool(P, dd)
        assert torch.equal(U, P[dd.replace])
        ups.append(U)
        X = P


def test_cfg4_full_batch_equals_per_mesh():
    """configs[3]: 256 x delaunay_terrain(2500) -> 1250 each; sampled entries equal their solo runs."""
    meshes = [S.delaunay_terrain(2500, noise=0.02, seed=b) for b in range(256)]
    batch = mfg.concat_batch(meshes)
    res = mfg.decimate_parallel(batch, mfg.DecimationConfig(target_vertices=1250), device=0)
    vo, fo = res.mesh.vertex_offsets, res.mesh.facet_offsets
    assert np.array_equal(np.diff(vo), np.full(256, 1250))
    vin = batch.vertex_offsets
    for b in (0, 1, 17, 128, 200, 255):
        solo = mfg.decimate_parallel(meshes[b], mfg.DecimationConfig(target_vertices=1250), device=0)
        sl = slice(vin[b], vin[b + 1])
        assert np.array_equal(res.replace[sl] - vo[b], solo.replace)
        m = res.mapping[sl]
        assert np.array_equal(np.where(m >= 0, m - vo[b], -1), solo.mapping)
        assert np.array_equal(res.mesh.facets[fo[b]:fo[b + 1]] - vo[b], solo.mesh.facets)
        assert np.array_equal(res.mesh.positions[vo[b]:vo[b + 1]].view(np.uint64),
                              solo.mesh.positions.view(np.uint64))
