"""The CPU oracle (oracle/mf_oracle.c) against golden fixtures produced by the
REAL reference (tests/golden/make_golden.py): every input rebuilt by the
package's synthetic generators must hash like the reference's inputs, and
every oracle output must hash like the reference output.  CPU only."""

import hashlib
import json
import os

import numpy as np
import pytest

import paper_2103_15076_b200 as mfg
from paper_2103_15076_b200 import synthetic as S

HERE = os.path.dirname(os.path.abspath(__file__))
MANIFEST = json.load(open(os.path.join(HERE, "golden", "manifest.json")))
SMALL = np.load(os.path.join(HERE, "golden", "small.npz"))
ORDER = MANIFEST["einsum_order"]

# the slow reference-scale cases run here too (the C oracle takes < 1 s each)
CASES = MANIFEST["decimate"]


def sha(*arrays):
    h = hashlib.sha256()
    for a in arrays:
        a = np.ascontiguousarray(a)
        h.update(str(a.dtype).encode() + str(a.shape).encode())
        h.update(a.tobytes())
    return h.hexdigest()


def build_mesh(spec):
    if "gen" in spec:
        return getattr(S, spec["gen"])(*spec["args"])
    if "inline" in spec:
        return mfg.TriMesh(np.array(spec["inline"][0], float), np.array(spec["inline"][1]))
    if "flat" in spec:
        return S.flat_grid(spec["flat"])
    if "batch" in spec:
        return mfg.concat_batch([build_mesh(s) for s in spec["batch"]])
    if "features_f32" in spec:
        m = build_mesh(spec["base"])
        f = np.random.default_rng(spec["features_f32"][0]).standard_normal((m.n_vertices, spec["features_f32"][1]))
        return mfg.TriMesh(m.positions, m.facets, f.astype(np.float32))
    raise ValueError(spec)


def input_digest(mesh):
    base = mesh.mesh if isinstance(mesh, mfg.BatchedMesh) else mesh
    parts = [base.positions, base.facets, base.features]
    if isinstance(mesh, mfg.BatchedMesh):
        parts += [mesh.vertex_offsets, mesh.facet_offsets]
    return sha(*parts)


def run_oracle(oracle, mesh, case):
    base = mesh.mesh if isinstance(mesh, mfg.BatchedMesh) else mesh
    kw = dict(target=case["target"], rounds=case["rounds"], seed=case["seed"], order=ORDER,
              placement=case.get("placement", "average"))
    if isinstance(mesh, mfg.BatchedMesh):
        kw.update(vertex_offsets=mesh.vertex_offsets, facet_offsets=mesh.facet_offsets)
    return oracle.decimate(base.positions, base.facets, base.features, **kw)


def check_inverse(out, case):
    """placement='inverse': the solve runs in numpy.linalg.solve's own operation order
    (mf_inverse.h), so topology AND positions are bit-exact against the reference; only the
    rcond test's eigenvalue range is approximated (it decides solve vs fallback, never the bits
    of a solution) -- the north-star bar would be 1e-5 relative."""
    key = case["key"]
    for k in ("replace", "mapping", "facets", "positions"):
        got, ref = np.ascontiguousarray(out[k]), np.ascontiguousarray(SMALL[f"{key}|{k}"])
        assert got.dtype == ref.dtype and np.array_equal(got.view(np.uint8), ref.view(np.uint8)), k
    np.testing.assert_array_equal(out["features"], SMALL[f"{key}|features"])


@pytest.mark.parametrize("case", CASES, ids=[c["key"] for c in CASES])
def test_decimate_golden(oracle, case):
    mesh = build_mesh(case["spec"])
    assert input_digest(mesh) == case["input"], "synthetic generator drifted from the reference"
    exp = case["expect"]
    if "error" in exp:
        with pytest.raises(oracle.OracleInfeasible) as err:
            run_oracle(oracle, mesh, case)
        assert err.value.achievable_vertices == exp["achievable_vertices"]
        return
    out = run_oracle(oracle, mesh, case)
    assert len(out["positions"]) == exp["n_out"] and len(out["facets"]) == exp["m_out"]
    if case.get("placement") == "inverse":
        check_inverse(out, case)
        return
    for k in ("replace", "mapping", "facets", "positions"):
        assert sha(out[k]) == exp[k], k
    feats = out["features"]
    if exp["features_dtype"] == "float32":
        feats = feats.astype(np.float32)
    assert sha(feats) == exp["features"]
    if "vertex_offsets" in exp:
        assert out["vertex_offsets"].tolist() == exp["vertex_offsets"]
        assert out["facet_offsets"].tolist() == exp["facet_offsets"]
    if case.get("arrays"):
        np.testing.assert_array_equal(out["replace"], SMALL[f"{case['key']}|replace"])


@pytest.mark.parametrize("entry", MANIFEST["pool"], ids=[e["key"] for e in MANIFEST["pool"]])
def test_pool_golden(oracle, entry):
    key = entry["key"]
    rep, X, w = SMALL[f"{key}|replace"], SMALL[f"{key}|X"], SMALL[f"{key}|w"]
    for mode, digest in entry["modes"].items():
        out = oracle.pool(X, rep, entry["n_out"], mode, w)
        assert sha(out) == digest, mode
        np.testing.assert_array_equal(out.view(np.uint8), SMALL[f"{key}|{mode}"].view(np.uint8))
    assert sha(oracle.unpool(SMALL[f"{key}|max"], rep)) == entry["unpool_max"]


def test_hierarchy_golden(oracle):
    h = MANIFEST["hierarchy20k"]
    mesh = S.delaunay_terrain(20_000, 0.02, 3)
    assert input_digest(mesh) == h["input"]
    feats = np.random.default_rng(0).standard_normal((mesh.n_vertices, 64)).astype(np.float32)
    assert sha(feats) == h["features"]
    P, F, X, f = mesh.positions, mesh.facets, mesh.features, feats
    for lvl in h["levels"]:
        out = oracle.decimate(P, F, X, target=lvl["target"], order=ORDER)
        assert sha(out["replace"]) == lvl["replace"]
        assert sha(out["facets"]) == lvl["facets"]
        assert sha(out["positions"]) == lvl["positions"]
        n_out = len(out["positions"])
        for mode, digest in lvl["pool"].items():
            assert sha(oracle.pool(f, out["replace"], n_out, mode)) == digest
        nxt = oracle.pool(f, out["replace"], n_out, "max")
        assert sha(oracle.unpool(nxt, out["replace"])) == lvl["unpool"]
        P, F, X, f = out["positions"], out["facets"], out["features"], nxt


def test_pcg64_matches_numpy(oracle):
    for seed in (0, 7, 12345):
        np.testing.assert_array_equal(oracle.pcg64_random(seed, 1000), np.random.default_rng(seed).random(1000))


def test_host_einsum_order_recorded():
    # the fixtures pin numpy's lane-split einsum order of the generating host
    assert ORDER in (0, 1)


@pytest.mark.parametrize("entry", MANIFEST["pool"], ids=[e["key"] for e in MANIFEST["pool"]])
def test_pool_backward_golden(oracle, entry):
    key = entry["key"]
    rep, X, w = SMALL[f"{key}|replace"], SMALL[f"{key}|X"], SMALL[f"{key}|w"]
    dt = key.split("|")[1]
    for gdt in (dt, "float64"):
        G = SMALL[f"{key}|G_{gdt}"]
        for mode in ("average", "max", "weighted", "sum"):
            Xb = X.copy()
            if mode == "max":
                Xb[np.isnan(Xb)] = 0.25
            out = oracle.pool_backward(G, Xb, rep, entry["n_out"], mode, w)
            exp = SMALL[f"{key}|bwd_{mode}_{gdt}"]
            assert out.dtype == exp.dtype and np.array_equal(out.view(np.uint8), exp.view(np.uint8)), (mode, gdt)


FULL_PATH = os.path.join(HERE, "golden", "full.json")
FULL = json.load(open(FULL_PATH)) if os.path.exists(FULL_PATH) else {}


@pytest.mark.parametrize("cfg", ["cfg3", "cfg4", "cfg5", "cfg3_inverse", "cfg4_inverse"])
def test_oracle_matches_reference_at_full_size(oracle, cfg):
    """The C oracle at BASELINE.json's full sizes (cfg5: 10M vertices, 4 levels) against the
    real reference's digests (tests/golden/make_golden_full.py) -- pins the checker the GPU
    full-size tests compare with, on every level, pooled features included."""
    import test_gpu_fullsize as G  # workload builders + digest helpers (no GPU needed for these)

    if cfg not in FULL:
        pytest.skip(f"no {cfg} in tests/golden/full.json")
    g = FULL[cfg]
    mesh, levels, feats = G.workload(cfg)
    assert G.input_digest(mesh) == g["input"]
    got = G.oracle_chain(oracle, cfg, FULL["einsum_order"])
    for i, (o, exp) in enumerate(zip(got, g["levels"])):
        assert len(o["positions"]) == exp["n_out"] and len(o["facets"]) == exp["m_out"]
        for k in ("replace", "mapping", "facets", "positions", "features", "vertex_offsets", "facet_offsets"):
            if k in exp:
                assert sha(o[k]) == exp[k], f"level {i}: {k}"
        if "pool_max" in exp:
            assert sha(o["pool_max"]) == exp["pool_max"] and sha(o["unpool"]) == exp["unpool"], f"level {i}"
