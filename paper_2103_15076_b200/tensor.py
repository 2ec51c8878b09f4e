"""Device-tensor API: decimation and pooling on CUDA tensors (no host copies).

`decimate(vertices, faces, nv, mf, target, ...)` takes batched float64
vertices [N,3] and int64 faces [M,3] resident on a CUDA device plus per-mesh
vertex / facet counts, and returns decimated vertices / faces / counts and
the cluster `replace` / `mapping` index tensors on the same device -- the
north-star interface ("batched vertices/faces/nv/mf go in, decimated
vertices/faces plus cluster representative and map indices come out").
torch is only the allocator / stream here; all compute runs in libmfgpu.so.
"""

from __future__ import annotations

import ctypes
import functools

import numpy as np
import torch

from . import _native
from .decimate import DecimationConfig, _make_config
from .numerics import einsum_order

_POOL_MODES = ("average", "max", "weighted", "sum")


class DeviceDecimation:
    """Outputs of one device decimation plus the library handle (reused by pool/unpool).
    `nv` / `mf` (per-mesh output vertex / facet counts) are built from the offsets on first use."""

    def __init__(self, dec, vertices, faces, features, vo, fo, replace, mapping):
        self._dec = dec
        self.vertices, self.faces, self.features = vertices, faces, features
        self._vo, self._fo = vo, fo
        self.replace, self.mapping = replace, mapping

    @property
    def nv(self):
        return None if self._vo is None else torch.from_numpy(np.diff(self._vo))

    @property
    def mf(self):
        return None if self._fo is None else torch.from_numpy(np.diff(self._fo))

    @property
    def n_vertices_out(self) -> int:
        return self._dec.n_out

    def round_stats(self) -> list:
        return _native.round_stats(self._dec)


def _offsets(counts, total) -> np.ndarray:
    if counts is None:
        return None
    c = np.asarray(counts.cpu() if torch.is_tensor(counts) else counts, dtype=np.int64)
    off = np.zeros(len(c) + 1, dtype=np.int64)
    np.cumsum(c, out=off[1:])
    if off[-1] != total:
        raise ValueError(f"counts sum to {off[-1]}, expected {total}")
    return off


@functools.lru_cache(maxsize=64)
def _config(target, placement, seed, rounds, order):
    """The validated mf_decimate_config of these settings (the C side copies it; order = the
    host's numpy reduction order, part of the key because tests may force it)."""
    return _make_config(DecimationConfig(target_vertices=target, placement=placement, shuffle_seed=seed,
                                         rounds=rounds))


def _current_stream(index: int) -> int:
    raw = getattr(torch._C, "_cuda_getCurrentRawStream", None)
    return raw(index) if raw is not None else torch.cuda.current_stream(index).cuda_stream


def _dtype_code(t: torch.Tensor, what: str) -> int:
    """Feature-like tensors are float32 or float64 (pooling.py:18-33 / mesh.py:25-31 accept no other)."""
    if t.dtype == torch.float32:
        return _native.DTYPE_F32
    if t.dtype == torch.float64:
        return _native.DTYPE_F64
    raise ValueError(f"{what} must be float32 or float64, got {t.dtype}")


def _same_device(t: torch.Tensor, dev: torch.device, what: str) -> None:
    if not t.is_cuda or t.device != dev:
        raise ValueError(f"{what} must be a CUDA tensor on {dev}, got {t.device}")


def decimate(vertices: torch.Tensor, faces: torch.Tensor, nv=None, mf=None, target: int = 1,
             placement: str = "average", seed=None, rounds="auto", features: torch.Tensor | None = None,
             copy_outputs: bool = True) -> DeviceDecimation:
    if not vertices.is_cuda or not faces.is_cuda:
        raise ValueError("vertices / faces must be CUDA tensors")
    dev = vertices.device
    _same_device(faces, dev, "faces")
    if vertices.dtype != torch.float64 or faces.dtype != torch.int64:
        raise ValueError("vertices must be float64 and faces int64")
    if vertices.dim() != 2 or vertices.shape[1] != 3:
        raise ValueError(f"vertices must have shape (N, 3), got {tuple(vertices.shape)}")
    if faces.dim() != 2 or faces.shape[1] != 3:
        raise ValueError(f"faces must have shape (M, 3), got {tuple(faces.shape)}")
    if features is not None:
        _same_device(features, dev, "features")
        _dtype_code(features, "features")
        if features.dim() != 2 or features.shape[0] != vertices.shape[0]:
            raise ValueError(f"features must have shape ({vertices.shape[0]}, C), got {tuple(features.shape)}")
    vertices = vertices.contiguous()
    faces = faces.contiguous()
    view = _native.MeshView()
    view.positions = vertices.data_ptr()
    view.facets = faces.data_ptr() if faces.numel() else None
    view.n, view.m = vertices.shape[0], faces.shape[0]
    if features is not None:
        features = features.contiguous()
        view.features = features.data_ptr()
        view.features_dtype = _dtype_code(features, "features")
        view.c = features.shape[1]
    else:
        view.c = 3
    vo = _offsets(nv, view.n)
    fo = _offsets(mf, view.m)
    if vo is not None:
        view.vertex_offsets, view.facet_offsets, view.n_meshes = vo.ctypes.data, fo.ctypes.data, len(vo) - 1
    cfg = _config(int(target), placement, seed, rounds, einsum_order())
    stream = _current_stream(dev.index)
    ctx = _native.context(dev.index)
    handle = ctypes.c_void_p()
    st = _native.Status()
    if not copy_outputs:
        _native.lib().mf_decimate(ctx, ctypes.byref(view), ctypes.byref(cfg), ctypes.c_void_p(stream),
                                  ctypes.byref(handle), ctypes.byref(st))
        _native.raise_for(st)
        return DeviceDecimation(_native.Decimation(handle, dev.index), None, None, None, None, None, None, None)
    # the round chain is launched first (mf_decimate_begin); the result tensors are allocated while
    # it runs -- every entry ends at exactly `target` vertices or the call raises, and the facet
    # buffer holds the input facet count -- and mf_decimate_end emits into them, synchronising once
    B = 1 if vo is None else len(vo) - 1
    n_out = int(target) * B
    c = view.c
    if _native.lib().mf_decimate_begin(ctx, ctypes.byref(view), ctypes.byref(cfg), ctypes.c_void_p(stream),
                                       ctypes.byref(st)):
        _native.raise_for(st)
    V = torch.empty((n_out, 3), dtype=torch.float64, device=dev)
    Fo = torch.empty((max(view.m, 1), 3), dtype=torch.int64, device=dev)
    X = torch.empty((n_out, c), dtype=torch.float64, device=dev)
    R = torch.empty(view.n, dtype=torch.int64, device=dev)
    Mp = torch.empty(view.n, dtype=torch.int64, device=dev)
    vo_out = np.empty(B + 1, dtype=np.int64)
    fo_out = np.empty(B + 1, dtype=np.int64)
    # features that turn out to be the positions (the default) share the positions' tensor
    share = c == 3
    outs = _native.Outputs(V.data_ptr() if n_out else None, Fo.data_ptr(), Fo.shape[0],
                           X.data_ptr() if n_out * c else None, _native.DTYPE_F64, int(share),
                           R.data_ptr() if view.n else None, Mp.data_ptr() if view.n else None,
                           vo_out.ctypes.data, fo_out.ctypes.data)
    if _native.lib().mf_decimate_end(ctx, ctypes.byref(outs), ctypes.byref(handle), ctypes.byref(st)):
        _native.raise_for(st)
    m_out = int(fo_out[-1])
    dec = _native.Decimation(handle, dev.index, (view.n, n_out, m_out, c, B))
    if share and _native.features_alias(dec):
        X = V
    return DeviceDecimation(dec, V, Fo[:m_out], X, vo_out, fo_out, R, Mp)


def pool(features: torch.Tensor, dd: DeviceDecimation, mode: str = "average", weights=None) -> torch.Tensor:
    if mode not in _POOL_MODES:
        raise ValueError(f"mode must be one of {_POOL_MODES}, got {mode!r}")
    dev = torch.device("cuda", dd._dec.device)
    _same_device(features, dev, "features")
    code = _dtype_code(features, "features")
    if features.dim() != 2 or features.shape[0] != dd._dec.n_in:
        raise ValueError(f"features must have shape ({dd._dec.n_in}, C), got {tuple(features.shape)}")
    features = features.contiguous()
    out = torch.empty((dd.n_vertices_out, features.shape[1]), dtype=features.dtype, device=dev)
    w = None
    if weights is not None:
        _same_device(weights, dev, "weights")
        _dtype_code(weights, "weights")
        if tuple(weights.shape) != (dd._dec.n_in,):
            raise ValueError(f"weights must have shape ({dd._dec.n_in},)")
        w = weights.to(dtype=features.dtype).contiguous()
    st = _native.Status()
    _native.lib().mf_pool(
        _native.context(dev.index), dd._dec.handle, None, dd._dec.n_in, dd._dec.n_out, features.data_ptr(),
        code, features.shape[1], _POOL_MODES.index(mode), None if w is None else w.data_ptr(), out.data_ptr(),
        ctypes.c_void_p(_current_stream(dev.index)), ctypes.byref(st))
    _native.raise_for(st)
    return out


def unpool(coarse: torch.Tensor, dd: DeviceDecimation) -> torch.Tensor:
    dev = torch.device("cuda", dd._dec.device)
    _same_device(coarse, dev, "coarse")
    code = _dtype_code(coarse, "coarse")
    if coarse.dim() != 2 or coarse.shape[0] != dd._dec.n_out:
        raise ValueError(f"coarse must have shape ({dd._dec.n_out}, C), got {tuple(coarse.shape)}")
    coarse = coarse.contiguous()
    out = torch.empty((dd._dec.n_in, coarse.shape[1]), dtype=coarse.dtype, device=dev)
    st = _native.Status()
    _native.lib().mf_unpool(
        _native.context(dev.index), dd._dec.handle, None, dd._dec.n_in, dd._dec.n_out, coarse.data_ptr(),
        code, coarse.shape[1], out.data_ptr(), ctypes.c_void_p(_current_stream(dev.index)),
        ctypes.byref(st))
    _native.raise_for(st)
    return out
