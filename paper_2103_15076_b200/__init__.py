"""B200-native cluster-parallel mesh decimation and cluster pooling.

Drop-in for the reference package's hot path (meshforge decimate.py /
pooling.py): decimate_parallel, pool and unpool run as hand-written sm_100a
CUDA kernels in libmfgpu.so behind a C ABI (include/mfgpu.h).
"""

from .decimate import (
    DecimationConfig,
    DecimationResult,
    VertexCluster,
    clusters,
    decimate_parallel,
    representative_vertices,
    round_targets,
)
from .conv import ConvKernel, VertexFacetAdjacency, facet2vertex_forward, vertex_facet_adjacency
from .errors import InfeasibleTargetError, MeshError, MeshFormatError, NativeError, StructuralError
from .mesh import BatchedMesh, TriMesh, concat_batch
from .meshio import load_mesh, save_clusters, save_mesh
from .pooling import POOL_MODES, pool, pool_backward, unpool, unpool_backward
from .quality import QualityReport, quality_report
from .validation import validate_on_device

__version__ = "0.1.0"

__all__ = [
    "BatchedMesh",
    "ConvKernel",
    "DecimationConfig",
    "DecimationResult",
    "InfeasibleTargetError",
    "MeshError",
    "MeshFormatError",
    "NativeError",
    "POOL_MODES",
    "QualityReport",
    "StructuralError",
    "TriMesh",
    "VertexFacetAdjacency",
    "VertexCluster",
    "clusters",
    "concat_batch",
    "decimate_parallel",
    "facet2vertex_forward",
    "load_mesh",
    "pool",
    "pool_backward",
    "quality_report",
    "representative_vertices",
    "round_targets",
    "save_clusters",
    "save_mesh",
    "unpool",
    "unpool_backward",
    "validate_on_device",
    "vertex_facet_adjacency",
]
