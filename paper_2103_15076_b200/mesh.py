"""Mesh containers of the decimation boundary.

`TriMesh` (reference mesh.py:13-52), `BatchedMesh` (mesh.py:137-205) and
`concat_batch` (io.py:434-457) with the same fields, validation and
defaults, so reference callers construct inputs unchanged.  Arrays stay
host numpy; the CUDA path uploads them once per `decimate_parallel`.
"""

from dataclasses import dataclass

import numpy as np

from .errors import StructuralError
from .validation import as_facets, as_feature_matrix, as_positions


class TriMesh:
    """positions (n,3) float64, facets (m,3) int64, features (n,c) float32/64 (copy of positions by default)."""

    __slots__ = ("positions", "features", "facets")

    def __init__(self, positions, facets, features=None):
        self.positions = as_positions(positions)
        self.facets = as_facets(facets, self.positions.shape[0])
        self.features = (
            self.positions.copy() if features is None else as_feature_matrix(features, self.positions.shape[0])
        )

    @property
    def n_vertices(self) -> int:
        return self.positions.shape[0]

    @property
    def n_facets(self) -> int:
        return self.facets.shape[0]

    @property
    def n_channels(self) -> int:
        return self.features.shape[1]

    def copy(self) -> "TriMesh":
        return TriMesh(self.positions.copy(), self.facets.copy(), self.features.copy())

    def __repr__(self):
        return f"TriMesh(n_vertices={self.n_vertices}, n_facets={self.n_facets}, n_channels={self.n_channels})"


@dataclass
class BatchedMesh:
    """Meshes concatenated with global vertex ids; entry b owns vertices
    [vertex_offsets[b], vertex_offsets[b+1]) and facets [facet_offsets[b], facet_offsets[b+1])."""

    mesh: TriMesh
    vertex_offsets: np.ndarray
    facet_offsets: np.ndarray

    def __post_init__(self):
        self.vertex_offsets = np.ascontiguousarray(self.vertex_offsets, dtype=np.int64)
        self.facet_offsets = np.ascontiguousarray(self.facet_offsets, dtype=np.int64)
        for name, offs, total in (
            ("vertex_offsets", self.vertex_offsets, self.mesh.n_vertices),
            ("facet_offsets", self.facet_offsets, self.mesh.n_facets),
        ):
            if offs.ndim != 1 or len(offs) < 1 or offs[0] != 0 or offs[-1] != total or (np.diff(offs) < 0).any():
                raise StructuralError(f"{name} must be monotone from 0 to {total}")
        if len(self.vertex_offsets) != len(self.facet_offsets):
            raise StructuralError("vertex_offsets and facet_offsets must have the same length")
        # every facet of entry b must stay inside entry b's vertex range
        f = self.mesh.facets
        if len(f):
            owner = np.repeat(np.arange(self.n_meshes), np.diff(self.facet_offsets))
            lo = self.vertex_offsets[owner][:, None]
            hi = self.vertex_offsets[owner + 1][:, None]
            bad = np.flatnonzero(((f < lo) | (f >= hi)).any(axis=1))
            if bad.size:
                b = int(owner[bad[0]])
                raise StructuralError(
                    f"facets of batch entry {b} reference vertices outside "
                    f"[{self.vertex_offsets[b]}, {self.vertex_offsets[b + 1]})"
                )

    @property
    def n_meshes(self) -> int:
        return len(self.vertex_offsets) - 1

    @property
    def n_vertices(self) -> int:
        return self.mesh.n_vertices

    @property
    def n_facets(self) -> int:
        return self.mesh.n_facets

    @property
    def positions(self) -> np.ndarray:
        return self.mesh.positions

    @property
    def features(self) -> np.ndarray:
        return self.mesh.features

    @property
    def facets(self) -> np.ndarray:
        return self.mesh.facets

    def split(self) -> list:
        """Entries as standalone TriMesh objects (inverse of concat_batch)."""
        vo, fo = self.vertex_offsets, self.facet_offsets
        return [
            TriMesh(
                self.mesh.positions[vo[b]:vo[b + 1]],
                self.mesh.facets[fo[b]:fo[b + 1]] - vo[b],
                self.mesh.features[vo[b]:vo[b + 1]],
            )
            for b in range(self.n_meshes)
        ]


def concat_batch(meshes) -> BatchedMesh:
    """Concatenate meshes into one batch with shifted facet indices (io.py:434-457)."""
    meshes = list(meshes)
    if not meshes:
        raise ValueError("concat_batch needs at least one mesh")
    channels = sorted({m.n_channels for m in meshes})
    if len(channels) != 1:
        raise StructuralError(f"meshes have mismatched channel counts: {channels}")
    nv = np.array([m.n_vertices for m in meshes], dtype=np.int64)
    nf = np.array([m.n_facets for m in meshes], dtype=np.int64)
    vo = np.concatenate([[0], np.cumsum(nv)]).astype(np.int64)
    fo = np.concatenate([[0], np.cumsum(nf)]).astype(np.int64)
    positions = np.concatenate([m.positions for m in meshes], axis=0)
    features = np.concatenate([m.features for m in meshes], axis=0)
    facets = np.concatenate([m.facets + vo[b] for b, m in enumerate(meshes)], axis=0).reshape(-1, 3)
    return BatchedMesh(mesh=TriMesh(positions, facets, features), vertex_offsets=vo, facet_offsets=fo)
