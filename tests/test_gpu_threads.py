"""Concurrent calls from Python threads (the reference runs batch entries on a thread pool,
decimate.py:356-358, and its operations are pure): every thread gets its own library context
(workspace, streams, graph cache), the GIL is released inside the library, and the results
equal the sequential ones bit for bit."""

from concurrent.futures import ThreadPoolExecutor

import numpy as np
import pytest

import paper_2103_15076_b200 as mfg
from paper_2103_15076_b200 import synthetic as S

pytestmark = pytest.mark.gpu


def _work(i):
    mesh = S.delaunay_terrain(3000 + 1500 * (i % 4), noise=0.02, seed=100 + i)
    cfg = mfg.DecimationConfig(target_vertices=mesh.n_vertices // 3, shuffle_seed=None if i % 2 else i)
    res = mfg.decimate_parallel(mesh, cfg, device=0)
    X = np.random.default_rng(i).standard_normal((mesh.n_vertices, 8)).astype(np.float32)
    pooled = mfg.pool(X, res, "max")
    res2 = mfg.decimate_parallel(res.mesh, mfg.DecimationConfig(target_vertices=res.n_vertices_out // 2), device=0)
    return (res.replace.copy(), res.mapping.copy(), np.array(res.mesh.facets), np.array(res.mesh.positions),
            pooled.copy(), mfg.unpool(pooled, res).copy(), res2.replace.copy(), np.array(res2.mesh.positions))


def test_threaded_calls_match_sequential():
    jobs = list(range(12))
    seq = [_work(i) for i in jobs]
    with ThreadPoolExecutor(max_workers=4) as ex:
        par = list(ex.map(_work, jobs))
    for i, (a, b) in enumerate(zip(seq, par)):
        for x, y in zip(a, b):
            assert x.dtype == y.dtype and np.array_equal(x.view(np.uint8), y.view(np.uint8)), i
