"""Generate golden fixtures from the REAL reference package (run in the build
container, where /root/reference exists; the GPU box only reads the output).

    python tests/golden/make_golden.py

Writes tests/golden/manifest.json (per case: input spec + sha256 of every
input and output array, exception + achievable_vertices for error cases)
and tests/golden/small.npz (full arrays of the small cases).  Inputs come
from deterministic generators; tests rebuild them with
paper_2103_15076_b200.synthetic and check the input digests first.
"""

import hashlib
import json
import os
import sys
import time

import numpy as np

REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REF)

import meshforge as mf  # noqa: E402
from meshforge import pooling as mpool  # noqa: E402
from meshforge import synthetic as msyn  # noqa: E402


def sha(*arrays):
    h = hashlib.sha256()
    for a in arrays:
        a = np.ascontiguousarray(a)
        h.update(str(a.dtype).encode() + str(a.shape).encode())
        h.update(a.tobytes())
    return h.hexdigest()


def einsum_order():
    a = float(np.einsum("ij,ij->i", np.array([[1e16, 1.0, -1e16]]), np.ones((1, 3)))[0])
    return 0 if a == 1.0 else 1


TOY_P = [[-0.8, 0.9, 0.0], [0.5, 1.8, 0.9], [0.0, 0.0, 0.0], [0.5, -0.9, 0.3], [1.0, 0.0, 0.0], [1.8, 0.9, 0.0]]
TOY_F = [[0, 2, 4], [5, 2, 4], [2, 3, 4], [0, 1, 5]]
TWO_TRI_P = [[0, 0, 0], [1, 0, 0], [0, 1, 0], [5, 5, 5], [6, 5, 5], [5, 6, 5]]
TWO_TRI_F = [[0, 1, 2], [3, 4, 5]]
ISO_P = [[0, 0, 0], [1, 0, 0], [0, 1, 0], [9, 9, 9]]
ISO_F = [[0, 1, 2]]
DEG_P = [[0, 0, 0], [1, 0, 0], [0, 1, 0], [9, 9, 9], [2, 0, 0], [1, 1, 0], [3, 3, 0]]
DEG_F = [[0, 1, 2], [1, 4, 5], [0, 1, 4], [1, 2, 5], [2, 1, 5], [0, 4, 6], [0, 1, 2]]


def build_mesh(spec):
    """spec: {"gen": name, "args": [...]} | {"inline": [P, F]} | {"batch": [spec...]} | {"flat": n}."""
    if "gen" in spec:
        return getattr(msyn, spec["gen"])(*spec["args"])
    if "inline" in spec:
        return mf.TriMesh(np.array(spec["inline"][0], float), np.array(spec["inline"][1]))
    if "flat" in spec:
        base = msyn.perturbed_grid(spec["flat"], noise=0.0, seed=0)
        p = base.positions.copy()
        p[:, 2] = 0.0
        return mf.TriMesh(p, base.facets)
    if "batch" in spec:
        return mf.concat_batch([build_mesh(s) for s in spec["batch"]])
    if "features_f32" in spec:
        m = build_mesh(spec["base"])
        f = np.random.default_rng(spec["features_f32"][0]).standard_normal((m.n_vertices, spec["features_f32"][1]))
        return mf.TriMesh(m.positions, m.facets, f.astype(np.float32))
    raise ValueError(spec)


def input_digest(mesh):
    base = mesh.mesh if isinstance(mesh, mf.BatchedMesh) else mesh
    parts = [base.positions, base.facets, base.features]
    if isinstance(mesh, mf.BatchedMesh):
        parts += [mesh.vertex_offsets, mesh.facet_offsets]
    return sha(*parts)


def T(n, seed, noise=0.05):
    return {"gen": "delaunay_terrain", "args": [n, noise, seed]}


DECIMATE_CASES = [
    ("toy", {"inline": [TOY_P, TOY_F]}, dict(target=2, rounds=1), [None, 0, 1, 12345], True),
    ("two_triangles_ok", {"inline": [TWO_TRI_P, TWO_TRI_F]}, dict(target=2, rounds=1), [None], True),
    ("two_triangles_infeasible", {"inline": [TWO_TRI_P, TWO_TRI_F]}, dict(target=1, rounds=1), [None], True),
    ("isolated_vertex", {"inline": [ISO_P, ISO_F]}, dict(target=3, rounds=1), [None], True),
    ("degenerate_dup", {"inline": [DEG_P, DEG_F]}, dict(target=4, rounds=1), [None, 3], True),
    ("degenerate_dup_auto", {"inline": [DEG_P, DEG_F]}, dict(target=5), [3], True),
    ("min_cost_edge", T(200, 4), dict(target=199), [None], True),
    ("terrain400_r2", T(400, 12), dict(target=100, rounds=2), [None], True),
    ("terrain1000_auto", T(1000, 6), dict(target=130), [None, 5], True),
    ("terrain300_seed7", T(300, 5), dict(target=150), [7], True),
    ("flat40", {"flat": 40}, dict(target=800), [None, 1], True),
    ("flat16_halve", {"flat": 16}, dict(target=128), [None], True),
    ("features_f32", {"features_f32": [0, 7], "base": T(800, 5)}, dict(target=300), [2], True),
    ("identity_rounds0", T(50, 7), dict(target=50, rounds=0), [None], True),
    ("cfg1_icosphere5", {"gen": "icosphere", "args": [5]}, dict(target=3585), [None, 7], False),
    ("grid300", {"gen": "perturbed_grid", "args": [300, None, 0.02, 0]}, dict(target=11250), [None], False),
    ("terrain20k", T(20000, 1, 0.02), dict(target=5000), [None, 11], False),
    ("cfg2_terrain115k", T(115_114, 12, 0.02), dict(target=41_449), [None, 3], False),
    ("batch5", {"batch": [T(120 + 31 * b, 20 + b) for b in range(4)] + [{"gen": "icosphere", "args": [1]}]},
     dict(target=42), [None, 3], True),
    ("batch_mixed", {"batch": [T(n, n) for n in (60, 120, 250, 60, 90)]}, dict(target=60), [9], True),
    ("batch16_cfg4lite", {"batch": [T(2500, b, 0.02) for b in range(16)]}, dict(target=1250), [None, 5], False),
    # placement='inverse' (quadrics.py:89-114): LAPACK eigvalsh/solve -> tolerance-only parity;
    # small meshes whose rank order is not decided by rounding noise
    ("inv_toy", {"inline": [TOY_P, TOY_F]}, dict(target=2, rounds=1, placement="inverse"), [None], True),
    ("inv_terrain300", T(300, 5), dict(target=150, placement="inverse"), [None], True),
    ("inv_terrain1000", T(1000, 6), dict(target=130, placement="inverse"), [None, 3], True),
    ("inv_batch", {"batch": [T(120 + 31 * b, 20 + b) for b in range(3)]}, dict(target=50, placement="inverse"),
     [None], True),
]


def run_decimate(mesh, target, rounds, seed, placement="average"):
    cfg = mf.DecimationConfig(target_vertices=target, shuffle_seed=seed, rounds=rounds, placement=placement)
    try:
        r = mf.decimate_parallel(mesh, cfg)
    except mf.InfeasibleTargetError as e:
        return {"error": "InfeasibleTargetError", "achievable_vertices": e.achievable_vertices, "message": str(e)}, None
    out = {
        "n_out": int(r.mesh.n_vertices), "m_out": int(r.mesh.n_facets),
        "replace": sha(r.replace), "mapping": sha(r.mapping), "facets": sha(r.mesh.facets),
        "positions": sha(r.mesh.positions), "features": sha(r.mesh.features),
        "features_dtype": str(r.mesh.features.dtype),
    }
    arrays = dict(replace=r.replace, mapping=r.mapping, facets=r.mesh.facets, positions=r.mesh.positions,
                  features=r.mesh.features)
    if isinstance(r.mesh, mf.BatchedMesh):
        out["vertex_offsets"] = r.mesh.vertex_offsets.tolist()
        out["facet_offsets"] = r.mesh.facet_offsets.tolist()
    return out, arrays


def main():
    manifest = {"einsum_order": einsum_order(), "numpy": np.__version__, "reference": "meshforge 0.1.0",
                "decimate": [], "pool": [], "cfg3": None}
    small = {}
    for name, spec, conf, seeds, keep_arrays in DECIMATE_CASES:
        mesh = build_mesh(spec)
        for seed in seeds:
            t = time.time()
            placement = conf.get("placement", "average")
            out, arrays = run_decimate(mesh, conf["target"], conf.get("rounds", "auto"), seed, placement)
            key = f"{name}|seed={seed}"
            case = {"key": key, "name": name, "spec": spec, "target": conf["target"],
                    "rounds": conf.get("rounds", "auto"), "seed": seed, "placement": placement,
                    "input": input_digest(mesh),
                    "expect": out, "ref_seconds": round(time.time() - t, 3)}
            if keep_arrays and arrays is not None:
                for k, v in arrays.items():
                    small[f"{key}|{k}"] = v
                case["arrays"] = True
            manifest["decimate"].append(case)
            print(f"{key:45s} {case['ref_seconds']:8.3f}s {out.get('n_out', out.get('error'))}")
    # pooling: hand-built clusterings with +-0, NaN and exact ties (pooling.py:36-71)
    rng = np.random.default_rng(0)
    for dt in ("float64", "float32"):
        n, n_out, c = 400, 60, 5
        rep = rng.integers(0, n_out, n)
        rep[:n_out] = np.arange(n_out)
        X = rng.standard_normal((n, c)).astype(dt)
        X[5, 0] = np.nan
        X[rep == rep[7], 1] = 0.0
        X[7, 1] = -0.0
        X[9, 2] = X[10, 2]
        w = (0.5 + rng.random(n)).astype(dt)
        res = mf.DecimationResult(mesh=mf.TriMesh(np.zeros((n_out, 3)), np.zeros((0, 3), np.int64)),
                                  replace=rep, mapping=rep.copy())
        key = f"pool_handmade|{dt}"
        small[f"{key}|replace"] = rep
        small[f"{key}|X"] = X
        small[f"{key}|w"] = w
        entry = {"key": key, "n_out": n_out, "modes": {}}
        for mode in mpool.POOL_MODES:
            out = mpool.pool(X, res, mode=mode, weights=w)
            small[f"{key}|{mode}"] = out
            entry["modes"][mode] = sha(out)
        up = mpool.unpool(small[f"{key}|max"], res)
        entry["unpool_max"] = sha(up)
        # adjoints (pooling.py:80-102), grad of the pooled shape, same dtype and float64
        for gdt in (dt, "float64"):
            G = rng.standard_normal((n_out, c)).astype(gdt)
            G[0, 0] = -0.0
            small[f"{key}|G_{gdt}"] = G
            for mode in mpool.POOL_MODES:
                Xb = X.copy()
                if mode == "max":
                    Xb[np.isnan(Xb)] = 0.25  # a NaN maximum has no winner row in the reference (IndexError)
                small[f"{key}|bwd_{mode}_{gdt}"] = mpool.pool_backward(G, Xb, res, mode=mode, weights=w)
            small[f"{key}|unpool_bwd_{gdt}"] = mpool.unpool_backward(np.asarray(up, dtype=gdt), res)
        manifest["pool"].append(entry)
    # cfg3-lite hierarchy: terrain 20k, C=64 float32 features, max-pool down / unpool up
    mesh = msyn.delaunay_terrain(20_000, 0.02, 3)
    feats = np.random.default_rng(0).standard_normal((mesh.n_vertices, 64)).astype(np.float32)
    levels = []
    cur, f = mesh, feats
    for tgt in (5000, 2500, 1250, 625):
        r = mf.decimate_parallel(cur, mf.DecimationConfig(target_vertices=tgt))
        pooled = {m: sha(mpool.pool(f, r, mode=m)) for m in ("max", "average")}
        nxt = mpool.pool(f, r, mode="max")
        levels.append({"target": tgt, "replace": sha(r.replace), "facets": sha(r.mesh.facets),
                       "positions": sha(r.mesh.positions), "pool": pooled, "unpool": sha(mpool.unpool(nxt, r))})
        cur, f = r.mesh, nxt
    manifest["hierarchy20k"] = {"input": input_digest(mesh), "features": sha(feats), "levels": levels}
    with open(os.path.join(HERE, "manifest.json"), "w") as fh:
        json.dump(manifest, fh, indent=1)
    np.savez_compressed(os.path.join(HERE, "small.npz"), **small)
    print("wrote", len(manifest["decimate"]), "decimate cases,", len(small), "arrays")


if __name__ == "__main__":
    main()
