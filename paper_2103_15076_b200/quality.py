"""Decimation quality summary -- drop-in for decimate.py:551-602 (`QualityReport`,
`quality_report`).

The per-output-vertex errors (the original mesh's vertex quadrics summed over each
cluster, evaluated at the output position) come from the GPU (`mf_quality_errors`,
bit-exact with the reference's arithmetic); the three reductions are numpy's own
(`errors.mean()`, `errors.max()`, `np.bincount(sizes)`, decimate.py:594-602), so the
report equals the reference's on the same inputs.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass, field

import numpy as np

from . import _native
from .mesh import BatchedMesh, TriMesh
from .numerics import einsum_order


@dataclass
class QualityReport:
    """Decimation quality summary against the original facet planes (decimate.py:553-577)."""

    n_vertices_in: int
    n_facets_in: int
    n_vertices_out: int
    n_facets_out: int
    mean_quadric_error: float
    max_quadric_error: float
    cluster_size_counts: np.ndarray = field(repr=False)  # index = cluster size

    def describe(self) -> str:
        sizes = ", ".join(
            f"{size}: {count}" for size, count in enumerate(self.cluster_size_counts) if size > 0 and count > 0
        )
        return (
            f"vertices {self.n_vertices_in} -> {self.n_vertices_out}, "
            f"facets {self.n_facets_in} -> {self.n_facets_out}\n"
            f"quadric error vs original planes: mean {self.mean_quadric_error:.6g}, "
            f"max {self.max_quadric_error:.6g}\n"
            f"cluster sizes {{{sizes}}}"
        )


def quadric_errors(original, result, order: int | None = None) -> np.ndarray:
    """float64[n_out]: cluster quadric of the original vertex quadrics at each output position."""
    base = original.mesh if isinstance(original, BatchedMesh) else original
    if not isinstance(base, TriMesh):
        base = TriMesh(base.positions, base.facets)
    P = np.ascontiguousarray(base.positions, dtype=np.float64)
    F = np.ascontiguousarray(base.facets, dtype=np.int64)
    replace = np.ascontiguousarray(result.replace, dtype=np.int64)
    if len(replace) != len(P):
        raise ValueError(f"replace has {len(replace)} entries for a mesh of {len(P)} vertices")
    n_out = result.n_vertices_out
    Pout = np.ascontiguousarray(result.mesh.positions, dtype=np.float64)
    err = np.empty(n_out, dtype=np.float64)
    view = _native.MeshView()
    view.positions = P.ctypes.data if P.size else None
    view.facets = F.ctypes.data if F.size else None
    view.n, view.m, view.c = len(P), len(F), 3
    dec = getattr(result, "_native", None)
    if dec is not None and (dec.n_in != len(P) or dec.n_out != n_out or result.replace.flags.writeable):
        dec = None
    device = dec.device if dec is not None else _native.default_device()
    st = _native.Status()
    _native.lib().mf_quality_errors(
        _native.context(device), ctypes.byref(view), dec.handle if dec is not None else None,
        replace.ctypes.data if replace.size else None, n_out, Pout.ctypes.data if Pout.size else None,
        einsum_order() if order is None else order, err.ctypes.data if err.size else None, None, ctypes.byref(st),
    )
    _native.raise_for(st)
    return err


def quality_report(original, result) -> QualityReport:
    """Counts, per-output-vertex quadric error, and the cluster-size histogram (decimate.py:580-602)."""
    errors = quadric_errors(original, result)
    n_out = result.n_vertices_out
    sizes = result.cluster_sizes()
    return QualityReport(
        n_vertices_in=int(original.n_vertices),
        n_facets_in=int(original.n_facets),
        n_vertices_out=n_out,
        n_facets_out=int(result.mesh.n_facets),
        mean_quadric_error=float(errors.mean()) if n_out else 0.0,
        max_quadric_error=float(errors.max()) if n_out else 0.0,
        cluster_size_counts=np.bincount(sizes),
    )
