"""GPU pooling / unpooling vs the oracle, bitwise: all modes x float32/float64,
signed zeros, NaN payloads, exact ties, clusters from 1 to 100k members
(thread tier and heavy tier of the member sort), host and device buffers."""

import os

import numpy as np
import pytest

import paper_2103_15076_b200 as mfg
from paper_2103_15076_b200 import synthetic as S

pytestmark = pytest.mark.gpu


def hand_result(replace, n_out):
    replace = np.asarray(replace, dtype=np.int64)
    return mfg.DecimationResult(mesh=mfg.TriMesh(np.zeros((n_out, 3)), np.zeros((0, 3))), replace=replace,
                                mapping=replace.copy())


def bits_equal(a, b):
    return a.shape == b.shape and a.dtype == b.dtype and np.array_equal(a.view(np.uint8), b.view(np.uint8))


@pytest.mark.parametrize("dtype", [np.float32, np.float64])
@pytest.mark.parametrize("sizes", [(400, 60), (5000, 1), (100_000, 3), (70_000, 20_000)])
def test_pool_modes(oracle, dtype, sizes):
    n, n_out = sizes
    rng = np.random.default_rng(n + n_out)
    rep = rng.integers(0, n_out, n)
    rep[:n_out] = np.arange(n_out)
    c = 5 if n < 10_000 else 33
    X = rng.standard_normal((n, c)).astype(dtype)
    X[rng.integers(0, n, 7), 0] = np.nan
    X[rep == rep[7], 1] = 0.0
    X[7, 1] = -0.0
    X[9, 2] = X[10, 2]
    w = (0.5 + rng.random(n)).astype(dtype)
    res = hand_result(rep, n_out)
    for mode in mfg.POOL_MODES:
        got = mfg.pool(X, res, mode=mode, weights=w)
        exp = oracle.pool(X, rep, n_out, mode, w)
        assert bits_equal(got, exp), mode
    coarse = oracle.pool(X, rep, n_out, "max")
    assert bits_equal(mfg.unpool(coarse, res), oracle.unpool(coarse, rep))


@pytest.mark.parametrize("dtype", [np.float32, np.float64])
@pytest.mark.parametrize("c", [1, 2, 3, 7, 63, 65, 129, 257, 1000])
def test_pool_channel_widths(oracle, dtype, c):
    """Row widths around the 16-byte vector / lane-count boundaries of k_pool_vec / k_unpool_rows
    (odd widths take the scalar path), and rows wider than one warp's vectors."""
    n, n_out = 3000, 900
    rng = np.random.default_rng(c)
    rep = rng.integers(0, n_out, n)
    rep[:n_out] = np.arange(n_out)
    X = rng.standard_normal((n, c)).astype(dtype)
    X[rng.integers(0, n, 5), rng.integers(0, c, 5)] = np.nan
    w = (0.5 + rng.random(n)).astype(dtype)
    res = hand_result(rep, n_out)
    for mode in mfg.POOL_MODES:
        assert bits_equal(mfg.pool(X, res, mode=mode, weights=w), oracle.pool(X, rep, n_out, mode, w)), mode
    coarse = rng.standard_normal((n_out, c)).astype(dtype)
    assert bits_equal(mfg.unpool(coarse, res), oracle.unpool(coarse, rep))


def test_pool_on_decimation_handle(oracle):
    mesh = S.delaunay_terrain(30_000, noise=0.02, seed=3)
    res = mfg.decimate_parallel(mesh, mfg.DecimationConfig(target_vertices=7_500))
    feats = np.random.default_rng(0).standard_normal((mesh.n_vertices, 64)).astype(np.float32)
    for mode in ("max", "average", "sum"):
        assert bits_equal(mfg.pool(feats, res, mode=mode), oracle.pool(feats, res.replace, 7_500, mode))
    coarse = mfg.pool(feats, res, mode="max")
    assert bits_equal(mfg.unpool(coarse, res), coarse[res.replace])


def test_pool_errors():
    res = hand_result([0, 0, 2], 3)
    with pytest.raises(RuntimeError, match="cover"):
        mfg.pool(np.zeros((3, 1)), res, mode="sum")
    ok = hand_result([0, 1, 1], 2)
    with pytest.raises(ValueError, match="weights"):
        mfg.pool(np.zeros((3, 1)), ok, mode="weighted")
    with pytest.raises(ValueError, match="mode"):
        mfg.pool(np.zeros((3, 1)), ok, mode="median")
    with pytest.raises(ValueError, match="zero total weight"):
        mfg.pool(np.ones((3, 1)), ok, mode="weighted", weights=np.array([0.0, 1.0, -1.0]))
    with pytest.raises(mfg.StructuralError):
        mfg.unpool(np.zeros((5, 2)), ok)


def test_tensor_api_pool_unpool(oracle):
    import torch

    from paper_2103_15076_b200 import tensor as T

    mesh = S.delaunay_terrain(5000, noise=0.02, seed=1)
    V = torch.from_numpy(mesh.positions).cuda()
    F = torch.from_numpy(mesh.facets).cuda()
    dd = T.decimate(V, F, target=1200)
    ref = oracle.decimate(mesh.positions, mesh.facets, target=1200)
    np.testing.assert_array_equal(dd.replace.cpu().numpy(), ref["replace"])
    np.testing.assert_array_equal(dd.faces.cpu().numpy(), ref["facets"])
    assert bits_equal(dd.vertices.cpu().numpy(), ref["positions"])
    X = torch.randn(5000, 64, device="cuda", dtype=torch.float32)
    pooled = T.pool(X, dd, mode="max")
    assert bits_equal(pooled.cpu().numpy(), oracle.pool(X.cpu().numpy(), ref["replace"], 1200, "max"))
    up = T.unpool(pooled, dd)
    assert torch.equal(up, pooled[dd.replace])


GOLDEN = np.load(os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "small.npz"))


@pytest.mark.parametrize("dt", ["float64", "float32"])
def test_pool_backward_matches_reference(dt):
    key = f"pool_handmade|{dt}"
    rep, X, w = GOLDEN[f"{key}|replace"], GOLDEN[f"{key}|X"], GOLDEN[f"{key}|w"]
    res = hand_result(rep, 60)
    for gdt in (dt, "float64"):
        G = GOLDEN[f"{key}|G_{gdt}"]
        for mode in mfg.POOL_MODES:
            Xb = X.copy()
            if mode == "max":
                Xb[np.isnan(Xb)] = 0.25
            got = mfg.pool_backward(G, Xb, res, mode=mode, weights=w)
            assert bits_equal(got, GOLDEN[f"{key}|bwd_{mode}_{gdt}"]), (mode, gdt)
        up = mfg.unpool(GOLDEN[f"{key}|max"], res).astype(gdt)
        assert bits_equal(mfg.unpool_backward(up, res), GOLDEN[f"{key}|unpool_bwd_{gdt}"])


def test_pool_backward_large_vs_oracle(oracle):
    mesh = S.delaunay_terrain(3000, noise=0.02, seed=9)
    res = mfg.decimate_parallel(mesh, mfg.DecimationConfig(target_vertices=800))
    rng = np.random.default_rng(2)
    X = rng.standard_normal((3000, 6)).astype(np.float32)
    X[::7, 2] = 0.5  # exact ties inside clusters
    G = rng.standard_normal((800, 6)).astype(np.float32)
    w = (0.5 + rng.random(3000)).astype(np.float32)
    for mode in mfg.POOL_MODES:
        got = mfg.pool_backward(G, X, res, mode=mode, weights=w)
        exp = oracle.pool_backward(G, X, res.replace, 800, mode, w)
        assert bits_equal(got, exp), mode


def test_adjoint_identities_gpu():
    mesh = S.delaunay_terrain(30, seed=4)
    res = mfg.decimate_parallel(mesh, mfg.DecimationConfig(target_vertices=15))
    rng = np.random.default_rng(3)
    x, y = rng.standard_normal((30, 2)), rng.standard_normal((15, 2))
    assert (mfg.pool(x, res, "sum") * y).sum() == pytest.approx((x * mfg.unpool(y, res)).sum(), rel=1e-12)
    g = mfg.pool_backward(y, x, res, mode="average")
    assert (mfg.pool(x, res, "average") * y).sum() == pytest.approx((x * g).sum(), rel=1e-12)


POOL_VARIANT_SCRIPT = r"""
import sys
sys.path.insert(0, {root!r})
import numpy as np
import torch
import paper_2103_15076_b200 as mfg
from paper_2103_15076_b200 import synthetic as S
from paper_2103_15076_b200 import tensor as T
from oracle import oracle as O
mesh = S.delaunay_terrain(30_000, noise=0.02, seed=8)
res = mfg.decimate_parallel(mesh, mfg.DecimationConfig(target_vertices=9_001))
dd = T.decimate(torch.from_numpy(mesh.positions).cuda(), torch.from_numpy(mesh.facets).cuda(), target=9_001)
rng = np.random.default_rng(3)
for c, dt in ((64, np.float32), (16, np.float64), (4, np.float32), (3, np.float64), (100, np.float32)):
    X = rng.standard_normal((mesh.n_vertices, c)).astype(dt)
    for mode in mfg.POOL_MODES:
        w = rng.random(mesh.n_vertices).astype(dt) + 0.5
        got = mfg.pool(X, res, mode=mode, weights=w if mode == "weighted" else None)
        exp = O.pool(X, res.replace, res.n_vertices_out, mode, w)
        assert np.array_equal(got.view(np.uint8), exp.view(np.uint8)), (c, mode)
        gt = T.pool(torch.from_numpy(X).cuda(), dd, mode=mode,
                    weights=torch.from_numpy(w).cuda() if mode == "weighted" else None)
        assert np.array_equal(gt.cpu().numpy().view(np.uint8), exp.view(np.uint8)), (c, mode, "tensor")
    up = mfg.unpool(got, res)
    assert np.array_equal(up.view(np.uint8), O.unpool(got, res.replace).view(np.uint8)), c
    ut = T.unpool(torch.from_numpy(got).cuda(), dd).cpu().numpy()
    assert np.array_equal(ut.view(np.uint8), O.unpool(got, res.replace).view(np.uint8)), (c, "tensor")
print("POOL-VARIANT-OK")
"""

POOL_VARIANTS = [{}, {"MF_UNPOOL_TMA": "1"}, {"MF_POOL_SCALAR": "1"}, {"MF_CSR_COOP": "0"}, {"MF_CSR_PER_BLOCK": "1"},
                 {"MF_CSR_PER_BLOCK": "100000000"}]


@pytest.mark.parametrize("env", POOL_VARIANTS, ids=[",".join(f"{k}={v}" for k, v in e.items()) or "default"
                                                     for e in POOL_VARIANTS])
def test_pool_unpool_variants_match_oracle(env):
    """Every pooling kernel variant (vectorised / scalar pool, LSU / TMA bulk-copy unpool,
    cooperative / multi-launch cluster CSR) bit-exact against the oracle, host and device API."""
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    out = subprocess.run([sys.executable, "-c", POOL_VARIANT_SCRIPT.format(root=root)], cwd=root,
                         env={**os.environ, **env}, capture_output=True, text=True, timeout=600)
    assert "POOL-VARIANT-OK" in out.stdout, out.stdout[-2000:] + out.stderr[-4000:]
