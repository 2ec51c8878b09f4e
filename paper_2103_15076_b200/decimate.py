"""decimate_parallel on the GPU -- drop-in for the reference's decimate.py:45-382.

`DecimationConfig`, `DecimationResult`, `VertexCluster`, `clusters`,
`representative_vertices` and `decimate_parallel` keep the reference
signatures, validation order, exception types and output dtypes
(int64 replace/mapping/facets, float64 positions/features).  All compute runs
in libmfgpu.so: one call decimates a TriMesh or a whole BatchedMesh through
every round of its chain on one device.
"""

from __future__ import annotations

import ctypes
import weakref
from dataclasses import dataclass, field

import numpy as np

from . import _native, hostmem
from .mesh import BatchedMesh, TriMesh
from .numerics import einsum_order

SHUFFLE_BUCKET_FRACTION = 1e-12  # decimate.py:42 (the kernels use the same constant)


@dataclass(frozen=True)
class DecimationConfig:
    """Settings of decimate_parallel (decimate.py:45-71)."""

    target_vertices: int
    placement: str = "average"
    shuffle_seed: int | None = None
    rounds: int | str = "auto"

    def __post_init__(self):
        if self.target_vertices < 1:
            raise ValueError("target_vertices must be >= 1")
        if self.placement not in ("average", "inverse"):
            raise ValueError(f"unknown placement {self.placement!r}")
        if self.rounds != "auto" and (not isinstance(self.rounds, int) or self.rounds < 0):
            raise ValueError("rounds must be 'auto' or a non-negative integer")


@dataclass
class DecimationResult:
    """Decimated mesh and the cluster tensors over the input vertices (decimate.py:74-92)."""

    mesh: TriMesh | BatchedMesh
    replace: np.ndarray
    mapping: np.ndarray
    reached_target: bool = True
    _native: object = field(default=None, repr=False, compare=False)

    @property
    def n_vertices_in(self) -> int:
        return len(self.replace)

    @property
    def n_vertices_out(self) -> int:
        return self.mesh.n_vertices

    def cluster_sizes(self) -> np.ndarray:
        return np.bincount(self.replace, minlength=self.n_vertices_out)


@dataclass(frozen=True)
class VertexCluster:
    members: tuple
    representative: int


def clusters(result: DecimationResult) -> list:
    """Clusters ordered by output index, members ascending (decimate.py:103-115)."""
    order = np.argsort(result.replace, kind="stable")
    ids = result.replace[order]
    cuts = np.flatnonzero(np.diff(ids)) + 1
    groups = np.split(order, cuts) if len(order) else []
    return [VertexCluster(tuple(int(v) for v in np.sort(g)), int(result.replace[g[0]])) for g in groups]


def representative_vertices(result: DecimationResult) -> np.ndarray:
    """Lowest input index of every output vertex's cluster (decimate.py:118-123)."""
    n_in = len(result.replace)
    rep = np.full(result.n_vertices_out, n_in, dtype=np.int64)
    np.minimum.at(rep, result.replace, np.arange(n_in, dtype=np.int64))
    return rep


def round_targets(n_in: int, target: int, rounds) -> list:
    """_round_targets (decimate.py:294-316), computed by the library."""
    cap = 4096
    buf = (ctypes.c_int64 * cap)()
    k = _native.lib().mf_round_targets(n_in, target, -1 if rounds == "auto" else int(rounds), buf, cap)
    return [int(buf[i]) for i in range(min(k, cap))]


def pcg_state(seed) -> tuple:
    """(state_hi, state_lo, inc_hi, inc_lo) of np.random.default_rng(seed) -- host setup of the
    device PCG64 jump-ahead (decimate.py:190)."""
    st = np.random.default_rng(seed).bit_generator.state["state"]
    s, inc = int(st["state"]), int(st["inc"])
    m = (1 << 64) - 1
    return (s >> 64, s & m, inc >> 64, inc & m)


def _trusted_trimesh(positions, facets, features) -> TriMesh:
    # outputs are valid by construction (no degenerate / out-of-range facets)
    t = TriMesh.__new__(TriMesh)
    t.positions, t.facets, t.features = positions, facets, features
    return t


def _make_config(config: DecimationConfig) -> _native.Config:
    cfg = _native.Config()
    cfg.target_vertices = int(config.target_vertices)
    cfg.rounds = -1 if config.rounds == "auto" else int(config.rounds)
    cfg.placement = 0 if config.placement == "average" else 1
    cfg.seeded = 0 if config.shuffle_seed is None else 1
    cfg.einsum_order = einsum_order()
    if config.shuffle_seed is not None:
        for i, w in enumerate(pcg_state(config.shuffle_seed)):
            cfg.pcg_state[i] = w
    return cfg


# Output meshes of this package whose device copy is still alive: id(positions) -> weak refs of
# (positions, facets, features, handle).  A later call given exactly those (read-only) arrays --
# the next level of a hierarchy -- reads the handle's device arrays instead of uploading them.
_CHAIN: dict = {}


def _register_chain(pos, fac, feats, dec) -> None:
    key = id(pos)

    def _drop(_ref, key=key):
        _CHAIN.pop(key, None)

    _CHAIN[key] = (weakref.ref(pos, _drop), weakref.ref(fac), weakref.ref(feats), weakref.ref(dec))


def _device_source(base, device):
    """The live handle whose output arrays `base` still is (unmodified: they are read-only)."""
    ent = _CHAIN.get(id(base.positions))
    if ent is None:
        return None
    pos, fac, feats, dec = (r() for r in ent)
    if pos is not base.positions or fac is not base.facets or feats is not base.features or dec is None:
        return None
    if pos.flags.writeable or fac.flags.writeable or feats.flags.writeable or dec.device != device:
        return None
    p, f, alias = ctypes.c_void_p(), ctypes.c_void_p(), ctypes.c_int32()
    _native.lib().mf_decimation_device_arrays(dec.handle, ctypes.byref(p), ctypes.byref(f), ctypes.byref(alias))
    if not alias.value:  # only the default features (a copy of the positions) travel implicitly
        return None
    return dec, p.value, f.value


def decimate_parallel(mesh, config: DecimationConfig, device: int | None = None) -> DecimationResult:
    """Cluster decimation to an exact vertex count (decimate.py:344-382), on the GPU.

    Accepts a TriMesh or a BatchedMesh (every entry decimated to
    config.target_vertices); raises InfeasibleTargetError naming the
    achievable minimum, ValueError / StructuralError as the reference does.
    """
    batched = hasattr(mesh, "vertex_offsets")  # duck-typed: the reference's containers work too
    base = mesh.mesh if batched else mesh
    P = np.ascontiguousarray(base.positions, dtype=np.float64)
    F = np.ascontiguousarray(base.facets, dtype=np.int64)
    X = base.features
    # features that are a bitwise copy of the positions (mesh.py:28-29) are detected on the
    # device (mf_decimate), so they are always handed over
    Xc = None if X is P else np.ascontiguousarray(X)
    view = _native.MeshView()
    view.positions = P.ctypes.data
    view.facets = F.ctypes.data if F.size else None
    view.features = None if Xc is None else Xc.ctypes.data
    view.features_dtype = _native.DTYPE_F32 if (Xc is not None and Xc.dtype == np.float32) else _native.DTYPE_F64
    view.n, view.m = P.shape[0], F.shape[0]
    view.c = X.shape[1]
    if device is None:
        device = _native.default_device()
    src = None
    if config.rounds != 0 and not _all_identity(mesh, config):
        src = _device_source(base, device)
    if src is not None:  # the previous level's device arrays, no upload (features = positions)
        view.positions, view.facets, view.features, view.facets_i32 = src[1], src[2] if F.size else None, None, 1
    if batched:
        vo = np.ascontiguousarray(mesh.vertex_offsets, dtype=np.int64)
        fo = np.ascontiguousarray(mesh.facet_offsets, dtype=np.int64)
        view.vertex_offsets, view.facet_offsets, view.n_meshes = vo.ctypes.data, fo.ctypes.data, len(vo) - 1
    cfg = _make_config(config)
    ctx = _native.context(device)
    handle = ctypes.c_void_p()
    st = _native.Status()
    B = len(mesh.vertex_offsets) - 1 if batched else 1
    nv = np.diff(np.asarray(mesh.vertex_offsets)) if batched else np.array([view.n])
    c = view.c
    feats_dtype = np.float64
    # the identity result keeps the input feature dtype (decimate.py:172-174); any real round folds into float64
    if Xc is not None and Xc.dtype == np.float32 and _all_identity(mesh, config):
        feats_dtype = np.float32
    if B > 0 and int(config.target_vertices) <= int(nv.min()):
        # every entry ends at exactly target_vertices (or the call raises): pinned outputs allocated up
        # front, emitted by the launch that fills the handle (mf_decimate_into, one synchronisation);
        # the facet buffer holds the input facet count and is narrowed to the output count
        n_out = int(config.target_vertices) * B
        # the round chain is launched first; the pinned outputs are allocated while it runs
        if _native.lib().mf_decimate_begin(ctx, ctypes.byref(view), ctypes.byref(cfg), None, ctypes.byref(st)):
            _native.raise_for(st)
        pos = hostmem.empty((n_out, 3), np.float64)
        fac_cap = hostmem.empty((max(view.m, 1), 3), np.int64)
        feats = hostmem.empty((n_out, c), feats_dtype)
        rep = hostmem.empty((view.n,), np.int64)
        mp = hostmem.empty((view.n,), np.int64)
        vo_out = np.empty(B + 1, dtype=np.int64)
        fo_out = np.empty(B + 1, dtype=np.int64)
        outs = _native.Outputs()
        outs.positions = pos.ctypes.data if pos.size else None
        outs.facets, outs.facets_capacity = fac_cap.ctypes.data, fac_cap.shape[0]
        outs.features = feats.ctypes.data if feats.size else None
        outs.features_dtype = _native.DTYPE_F32 if feats_dtype == np.float32 else _native.DTYPE_F64
        # features that turn out to be the positions (the default) are not copied out: the result
        # shares the (read-only) positions array
        share = c == 3 and feats_dtype == np.float64
        outs.features_if_distinct = int(share)
        outs.replace = rep.ctypes.data if rep.size else None
        outs.mapping = mp.ctypes.data if mp.size else None
        outs.vertex_offsets, outs.facet_offsets = vo_out.ctypes.data, fo_out.ctypes.data
        if _native.lib().mf_decimate_end(ctx, ctypes.byref(outs), ctypes.byref(handle), ctypes.byref(st)):
            _native.raise_for(st)
        m_out = int(fo_out[-1])
        dec = _native.Decimation(handle, device, (view.n, n_out, m_out, c, B))
        fac = fac_cap[:m_out]
        if share and _native.features_alias(dec):
            feats = pos
    else:  # the library raises the reference's error for an oversized target
        _native.lib().mf_decimate(ctx, ctypes.byref(view), ctypes.byref(cfg), None, ctypes.byref(handle),
                                  ctypes.byref(st))
        _native.raise_for(st)
        dec = _native.Decimation(handle, device)
        n_out, m_out = dec.n_out, dec.m_out
        pos = hostmem.empty((n_out, 3), np.float64)
        fac = hostmem.empty((m_out, 3), np.int64)
        feats = hostmem.empty((n_out, c), feats_dtype)
        rep = hostmem.empty((dec.n_in,), np.int64)
        mp = hostmem.empty((dec.n_in,), np.int64)
        vo_out = np.empty(B + 1, dtype=np.int64)
        fo_out = np.empty(B + 1, dtype=np.int64)
        st = _native.Status()
        _native.lib().mf_decimation_copy(
            dec.handle, pos.ctypes.data, fac.ctypes.data if fac.size else None,
            feats.ctypes.data if feats.size else None,
            _native.DTYPE_F32 if feats_dtype == np.float32 else _native.DTYPE_F64,
            rep.ctypes.data if rep.size else None, mp.ctypes.data if mp.size else None,
            vo_out.ctypes.data, fo_out.ctypes.data, None, ctypes.byref(st),
        )
        _native.raise_for(st)
    rep.flags.writeable = False
    dec.replace_ref = rep  # pool/unpool reuse the device replace only for this very array
    # the output mesh arrays are read-only views of library-owned pinned memory (np.array(x) gives a
    # writable copy): a hierarchy's next level then reads their device copy instead of uploading
    for a in (pos, fac, feats):
        a.flags.writeable = False
    _register_chain(pos, fac, feats, dec)
    out_mesh = _trusted_trimesh(pos, fac, feats)
    if batched:
        bm = BatchedMesh.__new__(BatchedMesh)
        bm.mesh, bm.vertex_offsets, bm.facet_offsets = out_mesh, vo_out, fo_out
        out_mesh = bm
    return DecimationResult(mesh=out_mesh, replace=rep, mapping=mp, _native=dec)


def _all_identity(mesh, config) -> bool:
    if hasattr(mesh, "vertex_offsets"):
        nv = np.diff(mesh.vertex_offsets)
        return bool(np.all(nv == config.target_vertices))
    return mesh.n_vertices == config.target_vertices
