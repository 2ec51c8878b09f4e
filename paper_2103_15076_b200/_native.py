"""ctypes binding of libmfgpu.so (C ABI in include/mfgpu.h).

The CUDA library is the only compute path: if the shared object is missing
or no CUDA device is usable, every entry point raises `NativeError` --
there is no CPU fallback.
"""

from __future__ import annotations

import ctypes
import os
import threading

from .errors import InfeasibleTargetError, NativeError, StructuralError

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libmfgpu.so")

MF_OK, MF_ERR_VALUE, MF_ERR_STRUCTURAL, MF_ERR_INFEASIBLE, MF_ERR_CUDA, MF_ERR_RUNTIME, MF_ERR_LIMIT = range(7)
DTYPE_F64, DTYPE_F32 = 0, 1


class MeshView(ctypes.Structure):
    _fields_ = [
        ("positions", ctypes.c_void_p),
        ("facets", ctypes.c_void_p),
        ("features", ctypes.c_void_p),
        ("features_dtype", ctypes.c_int32),
        ("facets_i32", ctypes.c_int32),
        ("n", ctypes.c_int64),
        ("m", ctypes.c_int64),
        ("c", ctypes.c_int64),
        ("vertex_offsets", ctypes.c_void_p),
        ("facet_offsets", ctypes.c_void_p),
        ("n_meshes", ctypes.c_int64),
    ]


class Config(ctypes.Structure):
    _fields_ = [
        ("target_vertices", ctypes.c_int64),
        ("rounds", ctypes.c_int32),
        ("placement", ctypes.c_int32),
        ("seeded", ctypes.c_int32),
        ("einsum_order", ctypes.c_int32),
        ("pcg_state", ctypes.c_uint64 * 4),
    ]


class Outputs(ctypes.Structure):
    """mf_outputs (include/mfgpu.h): caller buffers of mf_decimate_into."""

    _fields_ = [
        ("positions", ctypes.c_void_p),
        ("facets", ctypes.c_void_p),
        ("facets_capacity", ctypes.c_int64),
        ("features", ctypes.c_void_p),
        ("features_dtype", ctypes.c_int32),
        ("features_if_distinct", ctypes.c_int32),
        ("replace", ctypes.c_void_p),
        ("mapping", ctypes.c_void_p),
        ("vertex_offsets", ctypes.c_void_p),
        ("facet_offsets", ctypes.c_void_p),
    ]


class Status(ctypes.Structure):
    _fields_ = [
        ("code", ctypes.c_int32),
        ("mesh_index", ctypes.c_int32),
        ("achievable_vertices", ctypes.c_int64),
        ("target_vertices", ctypes.c_int64),
        ("no_edges", ctypes.c_int32),
        ("reserved", ctypes.c_int32),
        ("message", ctypes.c_char * 256),
    ]


_lib = None
_lock = threading.Lock()
_tls = threading.local()

_vp = ctypes.c_void_p
_i64 = ctypes.c_int64
_i32 = ctypes.c_int32


def lib():
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(LIB_PATH):
            raise NativeError(
                f"{LIB_PATH} is not built; run `python -c 'import __graft_entry__ as g; g.build()'` "
                "(there is no CPU fallback)"
            )
        L = ctypes.CDLL(LIB_PATH)
        L.mf_context_create.argtypes = [ctypes.c_int, ctypes.POINTER(_vp)]
        L.mf_context_create.restype = ctypes.c_int
        L.mf_context_destroy.argtypes = [_vp]
        L.mf_decimate.argtypes = [_vp, ctypes.POINTER(MeshView), ctypes.POINTER(Config), _vp, ctypes.POINTER(_vp),
                                  ctypes.POINTER(Status)]
        L.mf_decimate.restype = ctypes.c_int
        L.mf_decimate_into.argtypes = [_vp, ctypes.POINTER(MeshView), ctypes.POINTER(Config), _vp,
                                       ctypes.POINTER(Outputs), ctypes.POINTER(_vp), ctypes.POINTER(Status)]
        L.mf_decimate_into.restype = ctypes.c_int
        L.mf_decimate_begin.argtypes = [_vp, ctypes.POINTER(MeshView), ctypes.POINTER(Config), _vp,
                                        ctypes.POINTER(Status)]
        L.mf_decimate_begin.restype = ctypes.c_int
        L.mf_decimate_end.argtypes = [_vp, ctypes.POINTER(Outputs), ctypes.POINTER(_vp), ctypes.POINTER(Status)]
        L.mf_decimate_end.restype = ctypes.c_int
        L.mf_decimation_sizes.argtypes = [_vp] + [ctypes.POINTER(_i64)] * 5
        L.mf_decimation_copy.argtypes = [_vp, _vp, _vp, _vp, _i32, _vp, _vp, _vp, _vp, _vp, ctypes.POINTER(Status)]
        L.mf_decimation_copy.restype = ctypes.c_int
        L.mf_decimation_free.argtypes = [_vp]
        L.mf_decimation_device_arrays.argtypes = [_vp, ctypes.POINTER(_vp), ctypes.POINTER(_vp),
                                                  ctypes.POINTER(_i32)]
        L.mf_decimation_device_arrays.restype = ctypes.c_int
        L.mf_pool.argtypes = [_vp, _vp, _vp, _i64, _i64, _vp, _i32, _i64, _i32, _vp, _vp, _vp, ctypes.POINTER(Status)]
        L.mf_pool.restype = ctypes.c_int
        L.mf_pool_backward.argtypes = [_vp, _vp, _vp, _i64, _i64, _vp, _i32, _vp, _i32, _i64, _i32, _vp, _vp, _i32,
                                       _vp, ctypes.POINTER(Status)]
        L.mf_pool_backward.restype = ctypes.c_int
        L.mf_unpool.argtypes = [_vp, _vp, _vp, _i64, _i64, _vp, _i32, _i64, _vp, _vp, ctypes.POINTER(Status)]
        L.mf_unpool.restype = ctypes.c_int
        L.mf_round_targets.argtypes = [_i64, _i64, _i32, ctypes.POINTER(_i64), _i64]
        L.mf_quality_errors.argtypes = [_vp, ctypes.POINTER(MeshView), _vp, _vp, _i64, _vp, _i32, _vp, _vp,
                                        ctypes.POINTER(Status)]
        L.mf_quality_errors.restype = ctypes.c_int
        L.mf_ply_decode.argtypes = [_vp, _vp, _i64, _i64, _vp, _i64, _i64, _i32, _i32, _vp, _vp, _i32, _vp, _vp,
                                    ctypes.POINTER(Status)]
        L.mf_ply_decode.restype = ctypes.c_int
        L.mf_ply_encode.argtypes = [_vp, _vp, _i64, _vp, _i64, _vp, _i64, _vp, _vp, ctypes.POINTER(Status)]
        L.mf_ply_encode.restype = ctypes.c_int
        L.mf_vertex_facet_adjacency.argtypes = [_vp, _vp, _i64, _i64, _vp, _vp, _vp, ctypes.POINTER(Status)]
        L.mf_vertex_facet_adjacency.restype = ctypes.c_int
        L.mf_facet2vertex.argtypes = [_vp, _vp, _i64, _vp, _vp, _i32, _i64, _i64, _vp, _i64, _i64, _vp, _vp, _i64,
                                      _vp, _vp, ctypes.POINTER(Status)]
        L.mf_facet2vertex.restype = ctypes.c_int
        L.mf_round_targets.restype = _i64
        L.mf_validate_mesh.argtypes = [_vp, _vp, _i64, _vp, _i64, _vp, _vp, _i64, _i32, _vp, ctypes.POINTER(Status)]
        L.mf_validate_mesh.restype = ctypes.c_int
        L.mf_kernel_launch_count.argtypes = [_i32]
        L.mf_kernel_launch_count.restype = _i64
        L.mf_version.restype = ctypes.c_char_p
        L.mf_profile.argtypes = [_i32, ctypes.c_char_p]
        L.mf_profile_read.argtypes = [ctypes.c_char_p, _i32, ctypes.POINTER(ctypes.c_double), ctypes.POINTER(_i64),
                                      _i32]
        L.mf_profile_read.restype = _i32
        L.mf_decimation_round_stats.argtypes = [_vp, ctypes.POINTER(_i64), _i32]
        L.mf_decimation_round_stats.restype = _i32
        _lib = L
    return _lib


def default_device() -> int:
    dev = os.environ.get("MF_DEVICE")
    if dev is not None:
        return int(dev)
    try:
        import torch

        if torch.cuda.is_available():
            return torch.cuda.current_device()
    except Exception:  # pragma: no cover - torch is plumbing only
        pass
    return 0


def context(device: int | None = None):
    """Per-thread, per-device library context (workspace arena + pinned staging)."""
    if device is None:
        device = default_device()
    ctxs = getattr(_tls, "ctxs", None)
    if ctxs is None:
        ctxs = _tls.ctxs = {}
    h = ctxs.get(device)
    if h is None:
        h = _vp()
        rc = lib().mf_context_create(device, ctypes.byref(h))
        if rc != MF_OK:
            raise NativeError(f"mf_context_create(device={device}) failed with code {rc}: no usable CUDA device")
        ctxs[device] = h
    return h


def raise_for(st: Status):
    code = st.code
    if code == MF_OK:
        return
    msg = st.message.decode(errors="replace")
    if code == MF_ERR_VALUE:
        err = ValueError(msg)
    elif code == MF_ERR_STRUCTURAL:
        err = StructuralError(msg)
    elif code == MF_ERR_INFEASIBLE:
        err = InfeasibleTargetError(msg, achievable_vertices=int(st.achievable_vertices))
    elif code == MF_ERR_RUNTIME:
        err = RuntimeError(msg)
    else:
        err = NativeError(f"libmfgpu error {code}: {msg}")
    # batch entry the error belongs to (the lowest failing one, decimate.py:354-361); sharding
    # turns it into a global index
    err.mesh_index = int(st.mesh_index) if st.mesh_index >= 0 else None
    raise err


class Decimation:
    """Owner of a device-resident mf_decimation handle."""

    __slots__ = ("handle", "device", "n_in", "n_out", "m_out", "c", "n_meshes", "replace_ref", "__weakref__")

    def __init__(self, handle, device, sizes=None):
        self.handle = handle
        self.device = device
        self.replace_ref = None  # the host replace array emitted from this handle (pooling identity check)
        if sizes is None:  # (n_in, n_out, m_out, c, n_meshes) when the caller already knows them
            vals = [_i64() for _ in range(5)]
            lib().mf_decimation_sizes(handle, *[ctypes.byref(v) for v in vals])
            sizes = (int(v.value) for v in vals)
        self.n_in, self.n_out, self.m_out, self.c, self.n_meshes = sizes

    def __del__(self):
        h = getattr(self, "handle", None)
        if h and _lib is not None:
            try:
                _lib.mf_decimation_free(h)
            except Exception:
                pass
            self.handle = None


def features_alias(dec) -> bool:
    """Whether a result's features are its positions bitwise (then not emitted separately)."""
    alias = _i32()
    lib().mf_decimation_device_arrays(dec.handle, None, None, ctypes.byref(alias))
    return bool(alias.value)


def round_stats(dec) -> list:
    """Per-round dicts {N, M, E, N_out, M_out, ld_iters} of a decimation handle."""
    cap = 256
    buf = (_i64 * (6 * cap))()
    k = lib().mf_decimation_round_stats(dec.handle, buf, cap)
    keys = ("N", "M", "E", "N_out", "M_out", "ld_iters")
    return [dict(zip(keys, (int(buf[6 * r + j]) for j in range(6)))) for r in range(k)]


def profile(mode: int, only: str | None = None) -> None:
    """Per-kernel CUDA-event timing: 0 off, 1 every kernel, 2 only the kernel named `only`."""
    lib().mf_profile(mode, only.encode() if only else None)


def profile_read() -> dict:
    """{kernel: (total_ms, launches)} of the launches recorded since profile() was enabled."""
    cap, width = 128, 64
    names = ctypes.create_string_buffer(cap * width)
    ms = (ctypes.c_double * cap)()
    cnt = (_i64 * cap)()
    k = lib().mf_profile_read(names, width, ms, cnt, cap)
    out = {}
    for i in range(min(k, cap)):
        nm = names.raw[i * width:(i + 1) * width].split(b"\0", 1)[0].decode()
        out[nm] = (float(ms[i]), int(cnt[i]))
    return out


def launch_count(reset: bool = False) -> int:
    return int(lib().mf_kernel_launch_count(1 if reset else 0))
