"""The meshforge-side ctypes binding printed in INTEGRATION.md §2 is executed as written (only
its library path and its package-relative import are substituted) and must give the same bytes
as this package's own API -- the documentation a maintainer would copy stays correct."""

import os
import re

import numpy as np
import pytest

import paper_2103_15076_b200 as mfg
from paper_2103_15076_b200 import _native
from paper_2103_15076_b200 import synthetic as S

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def binding():
    text = open(os.path.join(ROOT, "INTEGRATION.md")).read()
    m = re.search(r"```python\n(# meshforge/_gpu\.py.*?)```", text, re.S)
    assert m, "INTEGRATION.md lost its binding block"
    code = m.group(1)
    code = code.replace("from .errors import InfeasibleTargetError, StructuralError",
                        "from paper_2103_15076_b200.errors import InfeasibleTargetError, StructuralError")
    code = code.replace('ctypes.CDLL("libmfgpu.so")', f'ctypes.CDLL({_native.LIB_PATH!r})')
    ns = {}
    exec(compile(code, "INTEGRATION.md#binding", "exec"), ns)
    return ns


@pytest.mark.parametrize("placement", ["average", "inverse"])
@pytest.mark.parametrize("seed", [None, 5])
def test_documented_binding_matches_package(binding, placement, seed):
    mesh = S.delaunay_terrain(3000, noise=0.02, seed=11)
    cfg = mfg.DecimationConfig(target_vertices=1100, placement=placement, shuffle_seed=seed)
    pos, fac, feats, rep, mp, vo, fo = binding["decimate_parallel_gpu"](mesh, cfg)
    res = mfg.decimate_parallel(mesh, cfg, device=0)
    assert np.array_equal(pos.view(np.uint8), np.ascontiguousarray(res.mesh.positions).view(np.uint8))
    assert np.array_equal(fac, res.mesh.facets)
    assert np.array_equal(rep, res.replace) and np.array_equal(mp, res.mapping)
    assert np.array_equal(feats.view(np.uint8), np.ascontiguousarray(res.mesh.features).view(np.uint8))
    X = np.random.default_rng(0).standard_normal((mesh.n_vertices, 6)).astype(np.float32)
    for mode in ("average", "max", "sum"):
        assert np.array_equal(binding["pool_gpu"](X, res, mode), mfg.pool(X, res, mode))
    coarse = mfg.pool(X, res, "max")
    assert np.array_equal(binding["unpool_gpu"](coarse, res), mfg.unpool(coarse, res))


def test_documented_binding_raises_reference_errors(binding):
    mesh = S.delaunay_terrain(200, seed=2)
    with pytest.raises(mfg.InfeasibleTargetError) as err:
        binding["decimate_parallel_gpu"](mesh, mfg.DecimationConfig(target_vertices=10, rounds=1))
    assert err.value.achievable_vertices > 10


def test_documented_binding_from_a_thread_pool(binding):
    """meshforge decimates batch entries on a thread pool (decimate.py:356-358): the binding's
    per-thread contexts give every concurrent call the same bytes as a sequential one."""
    from concurrent.futures import ThreadPoolExecutor

    meshes = [S.delaunay_terrain(2000 + 500 * i, noise=0.02, seed=40 + i) for i in range(8)]
    cfg = lambda m: mfg.DecimationConfig(target_vertices=m.n_vertices // 3)  # noqa: E731
    seq = [binding["decimate_parallel_gpu"](m, cfg(m)) for m in meshes]
    with ThreadPoolExecutor(max_workers=4) as ex:
        par = list(ex.map(lambda m: binding["decimate_parallel_gpu"](m, cfg(m)), meshes))
    for a, b in zip(seq, par):
        for x, y in zip(a, b):
            assert np.array_equal(np.ascontiguousarray(x).view(np.uint8), np.ascontiguousarray(y).view(np.uint8))
