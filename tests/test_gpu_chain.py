"""Device-resident hierarchies through the drop-in numpy API: feeding a result's mesh back in
(the next level) reads the library's device copy instead of re-uploading it.  The chained
levels must be bit-identical to levels computed from fresh host copies, for single meshes and
batches, seeded or not; the output arrays are read-only (so the device copy cannot go stale),
and a modified copy is uploaded as usual."""

import numpy as np
import pytest

import paper_2103_15076_b200 as mfg
from paper_2103_15076_b200 import decimate as D
from paper_2103_15076_b200 import synthetic as S

pytestmark = pytest.mark.gpu


def _arrays(res):
    base = res.mesh.mesh if isinstance(res.mesh, mfg.BatchedMesh) else res.mesh
    return [res.replace, res.mapping, base.positions, base.facets, base.features]


def _fresh(mesh):
    if isinstance(mesh, mfg.BatchedMesh):
        b = mesh.mesh
        return mfg.BatchedMesh(mfg.TriMesh(np.array(b.positions), np.array(b.facets)), np.array(mesh.vertex_offsets),
                               np.array(mesh.facet_offsets))
    return mfg.TriMesh(np.array(mesh.positions), np.array(mesh.facets))


@pytest.mark.parametrize("case", ["terrain", "grid_seeded", "batch"])
def test_chained_levels_equal_fresh_uploads(case):
    if case == "terrain":
        mesh, levels, seed = S.delaunay_terrain(60_000, noise=0.02, seed=3), [20_000, 9_000, 4_000, 1_500], None
    elif case == "grid_seeded":
        mesh, levels, seed = S.perturbed_grid(200, None, 0.02, 1), [20_000, 10_000, 5_000], 7
    else:
        mesh = mfg.concat_batch([S.delaunay_terrain(3000 + 500 * b, seed=b) for b in range(5)])
        levels, seed = [1500, 700, 300], 2
    cur_a, cur_b = mesh, mesh
    for t in levels:
        cfg = mfg.DecimationConfig(target_vertices=t, shuffle_seed=seed)
        src = D._device_source(cur_a.mesh if hasattr(cur_a, "vertex_offsets") else cur_a, 0)
        assert (src is not None) == (cur_a is not mesh)  # every level after the first is chained
        ra = mfg.decimate_parallel(cur_a, cfg, device=0)
        rb = mfg.decimate_parallel(_fresh(cur_b), cfg, device=0)
        for x, y in zip(_arrays(ra), _arrays(rb)):
            assert x.shape == y.shape and np.array_equal(x.view(np.uint8), y.view(np.uint8))
        cur_a, cur_b = ra.mesh, rb.mesh


def test_outputs_are_read_only_and_copies_upload():
    mesh = S.delaunay_terrain(20_000, noise=0.02, seed=5)
    r1 = mfg.decimate_parallel(mesh, mfg.DecimationConfig(target_vertices=8_000), device=0)
    for a in (r1.mesh.positions, r1.mesh.facets, r1.mesh.features, r1.replace):
        assert not a.flags.writeable
        with pytest.raises(ValueError):
            a[0] = a[0]
    moved = mfg.TriMesh(np.array(r1.mesh.positions) + 1.0, np.array(r1.mesh.facets))
    assert D._device_source(moved, 0) is None
    r2 = mfg.decimate_parallel(moved, mfg.DecimationConfig(target_vertices=3_000), device=0)
    r3 = mfg.decimate_parallel(_fresh(moved), mfg.DecimationConfig(target_vertices=3_000), device=0)
    assert np.array_equal(r2.mesh.positions, r3.mesh.positions) and np.array_equal(r2.replace, r3.replace)


def test_begin_end_split_and_abandoned_call():
    """mf_decimate_begin / _end (the APIs launch before allocating their outputs): equal to the
    one-shot call; a begun call that is never ended is finished by the next begin."""
    import ctypes

    import torch

    from paper_2103_15076_b200 import _native
    from paper_2103_15076_b200 import tensor as T

    mesh = S.delaunay_terrain(30_000, noise=0.02, seed=9)
    V = torch.from_numpy(mesh.positions).cuda()
    F = torch.from_numpy(mesh.facets).cuda()
    ref = mfg.decimate_parallel(mesh, mfg.DecimationConfig(target_vertices=9_000), device=0)
    dd = T.decimate(V, F, target=9_000)
    assert np.array_equal(dd.replace.cpu().numpy(), ref.replace)
    assert np.array_equal(dd.faces.cpu().numpy(), ref.mesh.facets)
    # abandon a begun call, then decimate again on the same context
    view = _native.MeshView()
    view.positions, view.facets, view.n, view.m, view.c = V.data_ptr(), F.data_ptr(), V.shape[0], F.shape[0], 3
    cfg = D._make_config(mfg.DecimationConfig(target_vertices=9_000))
    st = _native.Status()
    assert _native.lib().mf_decimate_begin(_native.context(0), ctypes.byref(view), ctypes.byref(cfg),
                                           ctypes.c_void_p(torch.cuda.current_stream().cuda_stream),
                                           ctypes.byref(st)) == 0
    dd2 = T.decimate(V, F, target=9_000)
    assert np.array_equal(dd2.replace.cpu().numpy(), ref.replace)
    assert torch.equal(dd2.nv, torch.tensor([9_000])) and int(dd2.mf[0]) == ref.mesh.n_facets


@pytest.mark.parametrize("zero_copy", ["1", "0"])
def test_pinned_host_inputs_read_in_place(zero_copy):
    """Pinned host inputs are read by the conversion kernel through their mapped addresses (no
    staging copy, MF_ZERO_COPY_IN=1) -- same bytes as staged and as pageable inputs."""
    import os
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    script = r'''
import sys
sys.path.insert(0, %r)
import numpy as np, torch
import paper_2103_15076_b200 as mfg
from paper_2103_15076_b200 import synthetic as S
mesh = S.delaunay_terrain(40_000, noise=0.02, seed=2)
P = torch.empty((mesh.n_vertices, 3), dtype=torch.float64, pin_memory=True).numpy(); P[:] = mesh.positions
F = torch.empty((mesh.n_facets, 3), dtype=torch.int64, pin_memory=True).numpy(); F[:] = mesh.facets
cfg = mfg.DecimationConfig(target_vertices=12_000, shuffle_seed=4)
a = mfg.decimate_parallel(mfg.TriMesh(P, F), cfg)
b = mfg.decimate_parallel(mesh, cfg)
for x, y in ((a.replace, b.replace), (a.mapping, b.mapping), (a.mesh.facets, b.mesh.facets),
             (a.mesh.positions, b.mesh.positions)):
    assert np.array_equal(x.view(np.uint8), y.view(np.uint8))
print("PINNED-OK")
''' % root
    out = subprocess.run([sys.executable, "-c", script], cwd=root, env={**os.environ, "MF_ZERO_COPY_IN": zero_copy},
                         capture_output=True, text=True, timeout=300)
    assert "PINNED-OK" in out.stdout, out.stdout[-2000:] + out.stderr[-3000:]
