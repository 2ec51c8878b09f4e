"""ctypes front-end of the CPU oracle (TEST INFRASTRUCTURE ONLY).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
--impl reference legs import this module, and only as the checker or the
CPU timing arm.  The product package never imports it.

The per-mesh work is done by mf_oracle.c; this file restates the
surrounding control flow of the reference:
  decimate_parallel  decimate.py:344-382  (validation order, identity path)
  batch split/merge  decimate.py:319-341, 354-361; mesh.py:192-205
  _round_targets     decimate.py:294-316  (delegated to C)
  pool / unpool      pooling.py:18-77
"""

from __future__ import annotations

import ctypes
import os
from concurrent.futures import ThreadPoolExecutor

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "_build", "libmforacle.so")
_lib = None

_i64p = ctypes.POINTER(ctypes.c_int64)
_f64p = ctypes.POINTER(ctypes.c_double)
_f32p = ctypes.POINTER(ctypes.c_float)
_u64p = ctypes.POINTER(ctypes.c_uint64)

POOL_MODES = ("average", "max", "weighted", "sum")


class OracleInfeasible(Exception):
    def __init__(self, msg, achievable_vertices):
        super().__init__(msg)
        self.achievable_vertices = achievable_vertices


class OracleStructural(Exception):
    pass


def build() -> str:
    """Compile the oracle with its Makefile (gcc, -ffp-contract=off)."""
    import subprocess

    subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return _LIB_PATH


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            build()
        L = ctypes.CDLL(_LIB_PATH)
        L.mfo_round_targets.restype = ctypes.c_int64
        L.mfo_round_targets.argtypes = [ctypes.c_int64, ctypes.c_int64, ctypes.c_int64, _i64p, ctypes.c_int64]
        L.mfo_decimate_mesh.restype = ctypes.c_int
        L.mfo_decimate_mesh.argtypes = [
            _f64p, ctypes.c_int64, _i64p, ctypes.c_int64, _f64p, ctypes.c_int64,
            _i64p, ctypes.c_int64, ctypes.c_int, _u64p, ctypes.c_int, ctypes.c_int,
            ctypes.POINTER(ctypes.c_void_p), _i64p,
        ]
        L.mfo_result_sizes.argtypes = [ctypes.c_void_p, _i64p, _i64p, _i64p, _i64p]
        L.mfo_result_copy.argtypes = [ctypes.c_void_p, _f64p, _i64p, _f64p, _i64p, _i64p]
        L.mfo_result_free.argtypes = [ctypes.c_void_p]
        L.mfo_vertex_quadrics.argtypes = [_f64p, ctypes.c_int64, _i64p, ctypes.c_int64, ctypes.c_int, _f64p]
        L.mfo_quality_errors.argtypes = [_f64p, ctypes.c_int64, _i64p, ctypes.c_int64, _i64p, ctypes.c_int64, _f64p,
                                         ctypes.c_int, _f64p]
        L.mfo_quality_errors.restype = ctypes.c_int
        L.mfo_edge_costs.restype = ctypes.c_int64
        L.mfo_edge_costs.argtypes = [_f64p, ctypes.c_int64, _i64p, ctypes.c_int64, ctypes.c_int, _i64p, _f64p]
        L.mfo_pcg64_random.argtypes = [_u64p, ctypes.c_int64, _f64p]
        L.mfo_pool_f64.restype = ctypes.c_int
        L.mfo_pool_f64.argtypes = [_f64p, ctypes.c_int64, ctypes.c_int64, _i64p, ctypes.c_int64, ctypes.c_int,
                                   _f64p, _f64p]
        L.mfo_pool_f32.restype = ctypes.c_int
        L.mfo_pool_f32.argtypes = [_f32p, ctypes.c_int64, ctypes.c_int64, _i64p, ctypes.c_int64, ctypes.c_int,
                                   _f32p, _f32p]
        _lib = L
    return _lib


def _p(a, t):
    return a.ctypes.data_as(t)


def pcg_words(seed) -> np.ndarray:
    """(state_hi, state_lo, inc_hi, inc_lo) of np.random.default_rng(seed)."""
    st = np.random.default_rng(seed).bit_generator.state["state"]
    s, inc = int(st["state"]), int(st["inc"])
    m = (1 << 64) - 1
    return np.array([s >> 64, s & m, inc >> 64, inc & m], dtype=np.uint64)


def round_targets(n_in: int, target: int, rounds) -> list[int]:
    r = -1 if rounds == "auto" else int(rounds)
    cap = 4096
    buf = np.zeros(cap, dtype=np.int64)
    k = lib().mfo_round_targets(n_in, target, r, _p(buf, _i64p), cap)
    return buf[:k].tolist()


def vertex_quadrics(positions, facets, order=0) -> np.ndarray:
    P = np.ascontiguousarray(positions, dtype=np.float64)
    F = np.ascontiguousarray(facets, dtype=np.int64).reshape(-1, 3)
    Q = np.zeros((len(P), 13))
    lib().mfo_vertex_quadrics(_p(P, _f64p), len(P), _p(F, _i64p), len(F), order, _p(Q, _f64p))
    return Q


def quality_errors(positions, facets, replace, positions_out, order=0) -> np.ndarray:
    """quality_report's per-output-vertex errors (decimate.py:580-602 before the numpy reductions)."""
    P = np.ascontiguousarray(positions, dtype=np.float64)
    F = np.ascontiguousarray(facets, dtype=np.int64).reshape(-1, 3)
    R = np.ascontiguousarray(replace, dtype=np.int64)
    Po = np.ascontiguousarray(positions_out, dtype=np.float64).reshape(-1, 3)
    err = np.zeros(len(Po))
    rc = lib().mfo_quality_errors(_p(P, _f64p), len(P), _p(F, _i64p), len(F), _p(R, _i64p), len(Po), _p(Po, _f64p),
                                  order, _p(err, _f64p))
    if rc:
        raise ValueError("replace holds indices outside [0, n_out)")
    return err


def edge_costs(positions, facets, order=0):
    P = np.ascontiguousarray(positions, dtype=np.float64)
    F = np.ascontiguousarray(facets, dtype=np.int64).reshape(-1, 3)
    E = np.zeros((3 * len(F), 2), dtype=np.int64)
    C = np.zeros(3 * len(F))
    ne = lib().mfo_edge_costs(_p(P, _f64p), len(P), _p(F, _i64p), len(F), order, _p(E, _i64p), _p(C, _f64p))
    return E[:ne].copy(), C[:ne].copy()


def pcg64_random(seed, n) -> np.ndarray:
    w = pcg_words(seed)
    out = np.zeros(n)
    lib().mfo_pcg64_random(_p(w, _u64p), n, _p(out, _f64p))
    return out


def _decimate_one(P, F, X, target, rounds, seed, order, placement="average"):
    """decimate_parallel on one TriMesh (decimate.py:363-382)."""
    n = len(P)
    if target > n:
        raise ValueError(f"target_vertices={target} exceeds the input size {n}")
    if rounds == 0 or target == n:
        if target != n:
            raise ValueError("rounds=0 requires target_vertices == input vertex count")
        idx = np.arange(n, dtype=np.int64)
        return dict(positions=P.copy(), facets=F.copy(), features=X.copy(), replace=idx, mapping=idx.copy())
    if n < 3 or len(F) < 1:
        raise OracleStructural("decimate_parallel requires a mesh with at least 3 vertices and 1 facet")
    chain = np.asarray(round_targets(n, target, rounds), dtype=np.int64)
    Xd = np.ascontiguousarray(X, dtype=np.float64)
    c = Xd.shape[1]
    words = pcg_words(seed) if seed is not None else np.zeros(4, dtype=np.uint64)
    res = ctypes.c_void_p()
    ach = ctypes.c_int64(0)
    st = lib().mfo_decimate_mesh(
        _p(P, _f64p), n, _p(F, _i64p), len(F), _p(Xd, _f64p), c,
        _p(chain, _i64p), len(chain), int(seed is not None), _p(words, _u64p), order,
        int(placement == "inverse"), ctypes.byref(res), ctypes.byref(ach),
    )
    if st == 4:
        raise OracleInfeasible(f"achievable minimum is {ach.value}", ach.value)
    if st != 0:
        raise RuntimeError(f"oracle status {st}")
    n_in, n_out, m_out, cc = (ctypes.c_int64() for _ in range(4))
    lib().mfo_result_sizes(res, ctypes.byref(n_in), ctypes.byref(n_out), ctypes.byref(m_out), ctypes.byref(cc))
    out = dict(
        positions=np.zeros((n_out.value, 3)),
        facets=np.zeros((m_out.value, 3), dtype=np.int64),
        features=np.zeros((n_out.value, cc.value)),
        replace=np.zeros(n_in.value, dtype=np.int64),
        mapping=np.zeros(n_in.value, dtype=np.int64),
    )
    lib().mfo_result_copy(
        res, _p(out["positions"], _f64p), _p(out["facets"], _i64p), _p(out["features"], _f64p),
        _p(out["replace"], _i64p), _p(out["mapping"], _i64p),
    )
    lib().mfo_result_free(res)
    return out


def decimate(positions, facets, features=None, target=None, rounds="auto", seed=None, order=0,
             vertex_offsets=None, facet_offsets=None, threads=1, placement="average"):
    """Oracle decimate_parallel; batch when offsets are given.

    Returns a dict with positions, facets, features, replace, mapping and,
    for batches, vertex_offsets / facet_offsets of the output.
    """
    P = np.ascontiguousarray(positions, dtype=np.float64)
    F = np.ascontiguousarray(facets, dtype=np.int64).reshape(-1, 3)
    X = P.copy() if features is None else np.asarray(features)
    if X.ndim == 1:
        X = X[:, None]
    if vertex_offsets is None:
        return _decimate_one(P, F, X, target, rounds, seed, order, placement)
    vo = np.asarray(vertex_offsets, dtype=np.int64)
    fo = np.asarray(facet_offsets, dtype=np.int64)
    parts = [(P[vo[b]:vo[b + 1]], F[fo[b]:fo[b + 1]] - vo[b], X[vo[b]:vo[b + 1]]) for b in range(len(vo) - 1)]
    run = lambda p: _decimate_one(p[0], p[1], p[2], target, rounds, seed, order, placement)  # noqa: E731
    if threads > 1 and len(parts) > 1:
        with ThreadPoolExecutor(max_workers=min(threads, len(parts))) as ex:
            results = list(ex.map(run, parts))
    else:
        results = [run(p) for p in parts]
    nv = np.array([len(r["positions"]) for r in results], dtype=np.int64)
    nf = np.array([len(r["facets"]) for r in results], dtype=np.int64)
    ov = np.zeros(len(results) + 1, dtype=np.int64)
    of = np.zeros(len(results) + 1, dtype=np.int64)
    np.cumsum(nv, out=ov[1:])
    np.cumsum(nf, out=of[1:])
    return dict(
        positions=np.concatenate([r["positions"] for r in results]),
        facets=np.concatenate([r["facets"] + ov[b] for b, r in enumerate(results)]).reshape(-1, 3),
        features=np.concatenate([r["features"] for r in results]),
        replace=np.concatenate([r["replace"] + ov[b] for b, r in enumerate(results)]),
        mapping=np.concatenate([np.where(r["mapping"] < 0, -1, r["mapping"] + ov[b]) for b, r in enumerate(results)]),
        vertex_offsets=ov,
        facet_offsets=of,
    )


def pool(features, replace, n_out, mode="average", weights=None):
    """pooling.pool (pooling.py:49-71) over a replace tensor."""
    if mode not in POOL_MODES:
        raise ValueError(f"mode must be one of {POOL_MODES}")
    X = np.asarray(features)
    if X.dtype not in (np.float32, np.float64):
        X = X.astype(np.float64)
    X = np.ascontiguousarray(X)
    if X.ndim == 1:
        X = X[:, None]
    r = np.ascontiguousarray(replace, dtype=np.int64)
    if np.bincount(r, minlength=n_out).min() == 0:
        raise RuntimeError("replace tensor does not cover every output vertex")
    m = POOL_MODES.index(mode)
    out = np.zeros((n_out, X.shape[1]), dtype=X.dtype)
    if X.dtype == np.float64:
        w = np.ascontiguousarray(weights, dtype=np.float64) if mode == "weighted" else np.zeros(1)
        st = lib().mfo_pool_f64(_p(X, _f64p), len(X), X.shape[1], _p(r, _i64p), n_out, m, _p(w, _f64p),
                                _p(out, _f64p))
    else:
        w = np.ascontiguousarray(weights, dtype=np.float32) if mode == "weighted" else np.zeros(1, np.float32)
        st = lib().mfo_pool_f32(_p(X, _f32p), len(X), X.shape[1], _p(r, _i64p), n_out, m, _p(w, _f32p),
                                _p(out, _f32p))
    if st:
        raise ValueError("weighted pooling: some cluster has zero total weight")
    return out


def unpool(coarse, replace):
    """pooling.unpool (pooling.py:74-77): row gather."""
    c = np.asarray(coarse)
    if c.ndim == 1:
        c = c[:, None]
    return c[np.asarray(replace, dtype=np.int64)]


def pool_backward(grad_output, features, replace, n_out, mode="average", weights=None):
    """pooling.pool_backward (pooling.py:80-97) restated with explicit loops (small inputs only)."""
    X = np.asarray(features)
    if X.dtype not in (np.float32, np.float64):
        X = X.astype(np.float64)
    X = X.reshape(len(X), -1)
    G = np.asarray(grad_output)
    if G.dtype not in (np.float32, np.float64):
        G = G.astype(np.float64)
    G = G.reshape(n_out, -1)
    r = np.asarray(replace, dtype=np.int64)
    n, c = X.shape
    members = [[] for _ in range(n_out)]
    for v in range(n):
        members[r[v]].append(v)
    if mode == "sum":
        return np.array([G[r[v]] for v in range(n)], dtype=G.dtype).reshape(n, c)
    if mode == "average":
        return np.array([[np.float64(G[r[v], k]) / np.float64(len(members[r[v]])) for k in range(c)]
                         for v in range(n)], dtype=np.float64).reshape(n, c)
    if mode == "weighted":
        w = np.asarray(weights, dtype=X.dtype)
        den = np.zeros(n_out, dtype=X.dtype)
        for v in range(n):
            den[r[v]] = den[r[v]] + w[v]
        odt = np.result_type(G.dtype, X.dtype)
        out = np.zeros((n, c), dtype=odt)
        for v in range(n):
            q = w[v] / den[r[v]]
            for k in range(c):
                out[v, k] = odt.type(G[r[v], k]) * odt.type(q)
        return out
    out = np.zeros((n, c), dtype=X.dtype)
    for cl in range(n_out):
        for k in range(c):
            acc = X.dtype.type(-np.inf)
            for v in members[cl]:
                acc = acc if (np.isnan(acc) or acc > X[v, k]) else X[v, k]
            for v in members[cl]:
                if X[v, k] == acc:
                    out[v, k] = X.dtype.type(0) + X.dtype.type(G[cl, k])
                    break
    return out
