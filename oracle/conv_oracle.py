"""CPU oracle (TEST INFRASTRUCTURE ONLY -- never imported by the product path):
restatement of the reference's vertex_facet_adjacency (mesh.py:114-122) and
facet2vertex_forward (conv.py:222-250) with explicit loops in the reference's
operation order, for the strided facet2vertex parity tests.  Pinned against the
reference's own outputs in tests/golden/conv.npz (tests/test_conv_f2v.py).
"""

import numpy as np


def vertex_facet_adjacency(facets, n):
    """offsets (n+1,), facet_ids (3m,): stable argsort of the flat corner list (mesh.py:116-122)."""
    flat_v = np.asarray(facets, dtype=np.int64).ravel()
    counts = np.zeros(n, dtype=np.int64)
    for v in flat_v:  # bincount
        counts[v] += 1
    offsets = np.zeros(n + 1, dtype=np.int64)
    offsets[1:] = np.cumsum(counts)
    cursor = offsets[:-1].copy()
    facet_ids = np.empty(len(flat_v), dtype=np.int64)
    for i, v in enumerate(flat_v):  # stable: flat index order = (facet, corner) order
        facet_ids[cursor[v]] = i // 3
        cursor[v] += 1
    return offsets, facet_ids


def facet2vertex(offsets, facet_ids, feats, weights, coeff, vertex_ids=None):
    """conv.py:238-250: eff = sum_t coeff[f,t] w[t,c,l] (sequential t), folded over the
    row's facets from +0 in adjacency order in the features' dtype, / count."""
    X = np.asarray(feats)
    dt = X.dtype
    w = np.asarray(weights).astype(dt).astype(np.float64)
    coeff = np.asarray(coeff, dtype=np.float64)
    T, C, L = w.shape
    n = len(offsets) - 1
    rows = np.arange(n) if vertex_ids is None else np.asarray(vertex_ids, dtype=np.int64)
    out = np.zeros((len(rows), C, L), dtype=dt)
    for r, v in enumerate(rows):
        a, b = offsets[v], offsets[v + 1]
        acc = np.zeros((C, L), dtype=dt)
        for f in facet_ids[a:b]:
            eff = np.zeros((C, L))
            for t in range(T):
                eff = eff + coeff[f, t] * w[t]
            contrib = eff * X[f].astype(np.float64)[:, None]
            acc = (acc.astype(np.float64) + contrib).astype(dt)
        if b > a:
            acc = (acc.astype(np.float64) / np.float64(b - a)).astype(dt)
        out[r] = acc
    return out.reshape(len(rows), C * L)
