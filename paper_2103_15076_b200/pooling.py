"""Cluster pooling / unpooling on the GPU -- drop-in for pooling.py:15-77.

`pool(features, result, mode, weights)` and `unpool(coarse, result)` keep
the reference signatures, dtype preservation (float32 stays float32),
validation order and exception types.  When `result` came from this
package's decimate_parallel, its device-resident replace tensor and cluster
CSR are reused instead of being uploaded again.
"""

from __future__ import annotations

import ctypes

import numpy as np

from . import _native, hostmem
from .validation import as_feature_matrix

POOL_MODES = ("average", "max", "weighted", "sum")


def _handle_for(result):
    """The decimation's device handle, when result.replace is still the (read-only) array that
    handle emitted; any other replace -- reassigned, or made writable again -- is uploaded."""
    dec = getattr(result, "_native", None)
    if dec is None or result.replace is not dec.replace_ref or result.replace.flags.writeable:
        return None
    if dec.n_in != len(result.replace) or dec.n_out != result.n_vertices_out:
        return None
    return dec


def pool(features, result, mode: str = "average", weights=None) -> np.ndarray:
    """Reduce per-input-vertex features over the clusters of a decimation (pooling.py:49-71)."""
    if mode not in POOL_MODES:
        raise ValueError(f"mode must be one of {POOL_MODES}, got {mode!r}")
    replace = np.ascontiguousarray(result.replace, dtype=np.int64)
    X = as_feature_matrix(features, len(replace))
    n_out = result.n_vertices_out
    W = None
    if mode == "weighted" and weights is not None:
        W = np.ascontiguousarray(np.asarray(weights, dtype=X.dtype))
        if W.shape != (len(replace),):
            # coverage is checked first in the reference (pooling.py:26-28)
            if np.bincount(replace, minlength=n_out).min() == 0:
                raise RuntimeError("replace tensor does not cover every output vertex")
            raise ValueError(f"weights must have shape ({len(replace)},)")
    out = hostmem.empty((n_out, X.shape[1]), X.dtype)
    dec = _handle_for(result)
    device = dec.device if dec is not None else _native.default_device()
    st = _native.Status()
    _native.lib().mf_pool(
        _native.context(device), dec.handle if dec is not None else None,
        replace.ctypes.data if replace.size else None, len(replace), n_out,
        X.ctypes.data if X.size else None, _native.DTYPE_F32 if X.dtype == np.float32 else _native.DTYPE_F64,
        X.shape[1], POOL_MODES.index(mode), None if W is None else W.ctypes.data,
        out.ctypes.data if out.size else None, None, ctypes.byref(st),
    )
    _native.raise_for(st)
    return out


def unpool(coarse_features, result) -> np.ndarray:
    """Broadcast every output vertex's row to its whole cluster (pooling.py:74-77)."""
    coarse = as_feature_matrix(coarse_features, result.n_vertices_out, "coarse_features")
    replace = np.ascontiguousarray(result.replace, dtype=np.int64)
    out = hostmem.empty((len(replace), coarse.shape[1]), coarse.dtype)
    dec = _handle_for(result)
    device = dec.device if dec is not None else _native.default_device()
    st = _native.Status()
    _native.lib().mf_unpool(
        _native.context(device), dec.handle if dec is not None else None,
        replace.ctypes.data if replace.size else None, len(replace), result.n_vertices_out,
        coarse.ctypes.data if coarse.size else None,
        _native.DTYPE_F32 if coarse.dtype == np.float32 else _native.DTYPE_F64, coarse.shape[1],
        out.ctypes.data if out.size else None, None, ctypes.byref(st),
    )
    _native.raise_for(st)
    return out


def _dtype_code(dt) -> int:
    return _native.DTYPE_F32 if dt == np.float32 else _native.DTYPE_F64


def pool_backward(grad_output, features, result, mode: str = "average", weights=None) -> np.ndarray:
    """Gradient of pool() w.r.t. the input features (pooling.py:80-97).

    sum: grad_output[replace]; average: grad_output[replace] / count (float64, numpy's
    promotion); weighted: grad_output[replace] * w / sum(w); max: routed to the lowest
    input row achieving the maximum, zeros elsewhere (features dtype).
    """
    if mode not in POOL_MODES:
        raise ValueError(f"mode must be one of {POOL_MODES}, got {mode!r}")
    replace = np.ascontiguousarray(result.replace, dtype=np.int64)
    X = as_feature_matrix(features, len(replace))
    n_out = result.n_vertices_out
    if np.bincount(replace, minlength=n_out).min() == 0:
        raise RuntimeError("replace tensor does not cover every output vertex")
    W = None
    if mode == "weighted":
        if weights is None:
            raise ValueError("weighted pooling requires per-input-vertex weights")
        W = np.ascontiguousarray(np.asarray(weights, dtype=X.dtype))
        if W.shape != (len(replace),):
            raise ValueError(f"weights must have shape ({len(replace)},)")
    G = as_feature_matrix(grad_output, n_out, "grad_output")
    if mode == "average":
        odt = np.float64
    elif mode == "sum":
        odt = G.dtype
    elif mode == "weighted":
        odt = np.result_type(G.dtype, X.dtype)
    else:
        odt = X.dtype
    c = G.shape[1]
    out = hostmem.empty((len(replace), c), odt)
    dec = _handle_for(result)
    device = dec.device if dec is not None else _native.default_device()
    st = _native.Status()
    _native.lib().mf_pool_backward(
        _native.context(device), dec.handle if dec is not None else None,
        replace.ctypes.data if replace.size else None, len(replace), n_out,
        G.ctypes.data if G.size else None, _dtype_code(G.dtype), X.ctypes.data if X.size else None,
        _dtype_code(X.dtype), c, POOL_MODES.index(mode), None if W is None else W.ctypes.data,
        out.ctypes.data if out.size else None, _dtype_code(odt), None, ctypes.byref(st),
    )
    _native.raise_for(st)
    return out


def unpool_backward(grad_output, result) -> np.ndarray:
    """Gradient of unpool(): sum pooling of the fine-level gradient (pooling.py:100-102)."""
    return pool(grad_output, result, mode="sum")
