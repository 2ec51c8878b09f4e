"""Non-finite FEATURES (positions must be finite, validation.py): quiet and signalling NaNs with
payloads and either sign, and infinities, through the decimation's feature means and every
pooling mode -- bit for bit against the oracle, i.e. with x86's NaN-payload propagation (the
operand's payload survives an add; the GPU's own arithmetic would return its canonical NaN)."""

import numpy as np
import pytest

import paper_2103_15076_b200 as mfg
from paper_2103_15076_b200 import synthetic as S
from paper_2103_15076_b200.numerics import einsum_order

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("dt", [np.float64, np.float32])
def test_nan_payload_features_match_oracle(oracle, dt):
    m = S.delaunay_terrain(3000, seed=1)
    rng = np.random.default_rng(0)
    ut = np.uint64 if dt == np.float64 else np.uint32
    X = rng.standard_normal((m.n_vertices, 4)).astype(dt)
    X[rng.integers(0, m.n_vertices, 40), 0] = np.nan
    X[rng.integers(0, m.n_vertices, 40), 1] = -np.nan
    bits = X.view(ut).copy()
    idx = rng.integers(0, m.n_vertices, 40)
    if dt == np.float64:
        bits[idx, 2] = 0x7FF0000000000123  # signalling NaN with a payload
        bits[idx[:10], 3] = 0xFFF8000000000ABC
    else:
        bits[idx, 2] = 0x7F800123
        bits[idx[:10], 3] = 0xFFC00ABC
    X = bits.view(dt)
    X[rng.integers(0, m.n_vertices, 20), 3] = np.inf
    res = mfg.decimate_parallel(mfg.TriMesh(m.positions, m.facets, X), mfg.DecimationConfig(target_vertices=1000),
                                device=0)
    with np.errstate(invalid="ignore"):
        exp = oracle.decimate(m.positions, m.facets, X, target=1000, order=einsum_order())
    got = np.ascontiguousarray(res.mesh.features)
    assert got.dtype == exp["features"].dtype and np.array_equal(got.view(np.uint8), exp["features"].view(np.uint8))
    w = rng.uniform(0.5, 1.5, m.n_vertices).astype(dt)
    for mode in ("average", "max", "sum", "weighted"):
        g = mfg.pool(X, res, mode, weights=w if mode == "weighted" else None)
        e = oracle.pool(X, res.replace, res.n_vertices_out, mode, weights=w if mode == "weighted" else None)
        assert np.array_equal(g.view(np.uint8), e.view(np.uint8)), mode
