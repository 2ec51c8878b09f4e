"""Strided facet2vertex on the GPU -- the first network consumer of a decimation.

Drop-in for the reference's conv.py:23-53 (`ConvKernel`), mesh.py:91-122
(`VertexFacetAdjacency`, `vertex_facet_adjacency`) and conv.py:222-250
(`facet2vertex_forward`), evaluated at every vertex or -- the strided / down-sampling
use (test_conv.py:366-383) -- only at `vertex_ids = representative_vertices(result)`.
The adjacency is built by a GPU counting sort (mf_vertex_facet_adjacency) and the
convolution runs as one warp per output row (mf_facet2vertex); results equal the
reference's bit for bit for float64 features (float32 follows numpy's float32
accumulation).  Only this operator of the reference's conv subsystem is on the path.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np

from . import _native


@dataclass
class ConvKernel:
    """Depthwise filter bank: weights has shape (filters, in_channels, multiplier) (conv.py:23-53)."""

    weights: np.ndarray

    def __post_init__(self):
        self.weights = np.asarray(self.weights, dtype=np.float64)
        if self.weights.ndim != 3:
            raise ValueError(
                f"kernel weights must be (filters, in_channels, multiplier), got shape {self.weights.shape}"
            )

    @property
    def n_filters(self) -> int:
        return self.weights.shape[0]

    @property
    def in_channels(self) -> int:
        return self.weights.shape[1]

    @property
    def multiplier(self) -> int:
        return self.weights.shape[2]

    @classmethod
    def random(cls, n_filters, in_channels, multiplier=1, rng=None, scale=0.5) -> "ConvKernel":
        rng = np.random.default_rng(rng)
        return cls(scale * rng.standard_normal((n_filters, in_channels, multiplier)))


@dataclass
class VertexFacetAdjacency:
    """facet_ids[offsets[v]:offsets[v+1]] = facets adjacent to v, ascending (mesh.py:91-111)."""

    offsets: np.ndarray    # (n + 1,) int64
    facet_ids: np.ndarray  # (3 m,) int64

    @property
    def counts(self) -> np.ndarray:
        return np.diff(self.offsets)

    @property
    def n_vertices(self) -> int:
        return len(self.offsets) - 1

    def facets_of(self, vertex: int) -> np.ndarray:
        return self.facet_ids[self.offsets[vertex]:self.offsets[vertex + 1]]


def vertex_facet_adjacency(mesh) -> VertexFacetAdjacency:
    """Vertex -> adjacent-facet CSR of the whole mesh (mesh.py:114-122), built on the GPU."""
    F = np.ascontiguousarray(mesh.facets, dtype=np.int64)
    n, m = int(mesh.n_vertices), len(F)
    offsets = np.empty(n + 1, dtype=np.int64)
    facet_ids = np.empty(3 * m, dtype=np.int64)
    st = _native.Status()
    _native.lib().mf_vertex_facet_adjacency(
        _native.context(_native.default_device()), F.ctypes.data if m else None, m, n, offsets.ctypes.data,
        facet_ids.ctypes.data if m else None, None, ctypes.byref(st))
    _native.raise_for(st)
    return VertexFacetAdjacency(offsets=offsets, facet_ids=facet_ids)


def _check_kernel(kernel: ConvKernel, n_filters: int, channels: int, who: str):
    if kernel.n_filters != n_filters or kernel.in_channels != channels:
        raise ValueError(
            f"{who} expects kernel shape ({n_filters}, {channels}, multiplier), got {kernel.weights.shape}"
        )


def facet2vertex_forward(adjacency: VertexFacetAdjacency, facet_features, kernel: ConvKernel, coeff,
                         vertex_ids=None) -> np.ndarray:
    """Per-vertex features averaged over adjacent facets (conv.py:222-250); `vertex_ids`
    restricts (and orders) the output rows -- the strided layer after a decimation."""
    facet_features = np.asarray(facet_features)
    m, c = facet_features.shape
    coeff = np.asarray(coeff)
    _check_kernel(kernel, coeff.shape[1], c, "facet2vertex")
    if coeff.shape[0] != m:
        raise ValueError("fuzzy coefficients must have one row per facet")
    dtype = np.float32 if facet_features.dtype == np.float32 else np.float64
    X = np.ascontiguousarray(facet_features, dtype=dtype)
    # w = kernel.weights.astype(features dtype) (conv.py:241), then promoted by einsum
    W = np.ascontiguousarray(kernel.weights.astype(dtype, copy=False).astype(np.float64))
    Cf = np.ascontiguousarray(coeff, dtype=np.float64)
    offsets = np.ascontiguousarray(adjacency.offsets, dtype=np.int64)
    facet_ids = np.ascontiguousarray(adjacency.facet_ids, dtype=np.int64)
    n = len(offsets) - 1
    vid = None
    if vertex_ids is not None:
        vid = np.ascontiguousarray(vertex_ids, dtype=np.int64)
        if vid.size and (vid.min() < -n or vid.max() >= n):
            raise IndexError(f"vertex_ids out of bounds for {n} vertices")
        vid = np.where(vid < 0, vid + n, vid)  # numpy fancy-index semantics (conv.py:212-214)
    rows = n if vid is None else len(vid)
    L = kernel.multiplier
    out = np.empty((rows, c * L), dtype=dtype)
    st = _native.Status()
    _native.lib().mf_facet2vertex(
        _native.context(_native.default_device()), offsets.ctypes.data, n,
        facet_ids.ctypes.data if facet_ids.size else None, X.ctypes.data if X.size else None,
        _native.DTYPE_F32 if dtype == np.float32 else _native.DTYPE_F64, m, c, W.ctypes.data if W.size else None,
        kernel.n_filters, L, Cf.ctypes.data if Cf.size else None, None if vid is None else vid.ctypes.data, rows,
        out.ctypes.data if out.size else None, None, ctypes.byref(st))
    _native.raise_for(st)
    return out
