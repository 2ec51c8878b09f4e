"""Binary PLY load / save on the GPU and the clusters sidecar -- the on-disk formats
either side of the decimation step (reference io.py:50-91, 182-431; cli.py:95-96).

The header is text and is parsed on the host (same rules and MeshFormatError
messages as io.py:182-223); the body -- fixed-size vertex records and uniform-arity
face records, the reference's vectorised fast path -- is decoded / encoded by
kernels (mf_ply_decode / mf_ply_encode).  ASCII PLY, OBJ and mixed-arity face
lists are not on this path and raise MeshFormatError.
"""

from __future__ import annotations

import ctypes
from pathlib import Path

import numpy as np

from . import _native
from .errors import MeshFormatError, StructuralError
from .mesh import TriMesh

_PLY_DTYPES = {  # io.py:12-20
    "char": "i1", "int8": "i1", "uchar": "u1", "uint8": "u1",
    "short": "i2", "int16": "i2", "ushort": "u2", "uint16": "u2",
    "int": "i4", "int32": "i4", "uint": "u4", "uint32": "u4",
    "float": "f4", "float32": "f4", "double": "f8", "float64": "f8",
}
_CODES = {"i1": 0, "u1": 1, "i2": 2, "u2": 3, "i4": 4, "u4": 5, "f4": 6, "f8": 7}
_SIZES = {"i1": 1, "u1": 1, "i2": 2, "u2": 2, "i4": 4, "u4": 4, "f4": 4, "f8": 8}


class PlyVertexSpec(ctypes.Structure):  # mf_ply_vertex_spec (include/mfgpu.h)
    _fields_ = [("record_size", ctypes.c_int32), ("offset", ctypes.c_int32 * 6), ("type", ctypes.c_int32 * 6)]


def _detect_format(path: Path) -> str:
    suffix = path.suffix.lower()
    if suffix == ".obj":
        return "obj"
    if suffix == ".ply":
        return "ply"
    raise MeshFormatError(f"cannot infer format from suffix {suffix!r}; pass format='obj' or 'ply'", path=path)


def parse_ply_header(data: bytes, path=None):
    """(format, [(name, count, [(prop, dtype | ('list', count_dt, item_dt))])], body offset) -- io.py:182-223."""
    end = data.find(b"end_header")
    if not data.startswith(b"ply") or end < 0:
        raise MeshFormatError("not a PLY file (missing header)", path=path)
    end = data.index(b"\n", end) + 1
    fmt, elements = None, []
    for lineno, line in enumerate(data[:end].decode("ascii", errors="replace").splitlines(), start=1):
        parts = line.split()
        if not parts or parts[0] in ("ply", "comment", "obj_info", "end_header"):
            continue
        if parts[0] == "format":
            fmt = parts[1]
            if fmt not in ("ascii", "binary_little_endian"):
                raise MeshFormatError(f"unsupported PLY format {fmt!r} (ascii and binary_little_endian are supported)",
                                      path=path, line=lineno)
        elif parts[0] == "element":
            elements.append((parts[1], int(parts[2]), []))
        elif parts[0] == "property":
            if not elements:
                raise MeshFormatError("property before element", path=path, line=lineno)
            if parts[1] == "list":
                if parts[2] not in _PLY_DTYPES or parts[3] not in _PLY_DTYPES:
                    raise MeshFormatError(f"unsupported list types {parts[2]}/{parts[3]}", path=path, line=lineno)
                elements[-1][2].append((parts[4], ("list", _PLY_DTYPES[parts[2]], _PLY_DTYPES[parts[3]])))
            else:
                if parts[1] not in _PLY_DTYPES:
                    raise MeshFormatError(f"unsupported property type {parts[1]!r}", path=path, line=lineno)
                elements[-1][2].append((parts[2], _PLY_DTYPES[parts[1]]))
    if fmt is None:
        raise MeshFormatError("PLY header has no format line", path=path)
    return fmt, elements, end


def _load_ply(path: Path) -> TriMesh:
    try:
        data = path.read_bytes()
    except OSError as exc:
        raise MeshFormatError(str(exc), path=path) from exc
    fmt, elements, body_at = parse_ply_header(data, path)
    if fmt != "binary_little_endian":
        raise MeshFormatError("only binary_little_endian PLY bodies are decoded on the GPU", path=path)
    body = np.frombuffer(data, dtype=np.uint8, offset=body_at)
    if not any(name == "vertex" for name, _, _ in elements):
        raise MeshFormatError("PLY file has no vertex element", path=path)
    cursor, nv, nf, face_off, arity, itype = 0, 0, 0, 0, 3, "i4"
    spec, colors = PlyVertexSpec(), False
    for name, count, props in elements:
        if name == "vertex":
            if any(isinstance(t, tuple) for _, t in props):
                raise MeshFormatError("list properties on vertices are not supported", path=path)
            offs, o = {}, 0
            for pname, t in props:
                offs[pname] = (o, t)
                o += _SIZES[t]
            missing = [ax for ax in ("x", "y", "z") if ax not in offs]
            if missing:
                raise MeshFormatError(f"vertex element lacks {missing} properties", path=path)
            colors = all(c in offs for c in ("red", "green", "blue"))
            if colors:
                for c in ("red", "green", "blue"):
                    if offs[c][1] != "u1":
                        raise MeshFormatError(f"color property {c!r} must be uchar", path=path)
            spec.record_size = o
            for k, pname in enumerate(("x", "y", "z", "red", "green", "blue")):
                spec.offset[k], spec.type[k] = (offs[pname][0], _CODES[offs[pname][1]]) if pname in offs else (-1, 0)
            nv, size = count, o * count
        elif name == "face":
            if len(props) != 1 or not isinstance(props[0][1], tuple) or props[0][0] not in ("vertex_indices",
                                                                                            "vertex_index"):
                raise MeshFormatError("face element must be a single vertex_indices list for the GPU loader",
                                      path=path)
            _, count_t, itype = props[0][1]
            if _SIZES[count_t] != 1:
                raise MeshFormatError("face list counts must be uchar for the GPU loader", path=path)
            nf, face_off = count, cursor
            arity = int(body[cursor]) if count and cursor < len(body) else 3
            if count and arity < 3:
                raise MeshFormatError(f"face 0 has {arity} vertices", path=path)
            size = (1 + arity * _SIZES[itype]) * count
        else:  # unknown element: skipped when its records have a fixed size
            if any(isinstance(t, tuple) for _, t in props):
                raise MeshFormatError(f"element {name!r} has list properties (not supported by the GPU loader)",
                                      path=path)
            size = sum(_SIZES[t] for _, t in props) * count
        if cursor + size > len(body):
            raise MeshFormatError("unexpected end of binary data", path=path, offset=body_at + cursor)
        cursor += size
    C = 6 if colors else 3
    P = np.empty((nv, 3), dtype=np.float64)
    X = np.empty((nv, C), dtype=np.float64)
    F = np.empty((nf * (arity - 2), 3), dtype=np.int64)
    st = _native.Status()
    _native.lib().mf_ply_decode(
        _native.context(_native.default_device()), body.ctypes.data if len(body) else None, len(body), nv,
        ctypes.byref(spec), face_off, nf, arity, _CODES[itype], P.ctypes.data if P.size else None,
        X.ctypes.data if X.size else None, C, F.ctypes.data if F.size else None, None, ctypes.byref(st))
    if st.code == 2:  # MF_ERR_STRUCTURAL: mixed face arity
        raise MeshFormatError(st.message.decode() + " (mixed-arity faces are not supported by the GPU loader)",
                              path=path)
    _native.raise_for(st)
    try:
        return TriMesh(P, F, X)
    except StructuralError as exc:
        raise MeshFormatError(str(exc), path=path) from exc


def _save_ply(mesh: TriMesh, path: Path) -> None:
    n, m = mesh.n_vertices, mesh.n_facets
    color = mesh.n_channels >= 6
    header = ["ply", "format binary_little_endian 1.0", f"element vertex {n}",
              "property float x", "property float y", "property float z"]
    if color:
        header += ["property uchar red", "property uchar green", "property uchar blue"]
    header += [f"element face {m}", "property list uchar int vertex_indices", "end_header"]
    head = ("\n".join(header) + "\n").encode("ascii")
    P = np.ascontiguousarray(mesh.positions, dtype=np.float64)
    F = np.ascontiguousarray(mesh.facets, dtype=np.int64)
    X = np.ascontiguousarray(mesh.features, dtype=np.float64) if color else None
    body = np.empty(n * (15 if color else 12) + m * 13, dtype=np.uint8)
    st = _native.Status()
    _native.lib().mf_ply_encode(
        _native.context(_native.default_device()), P.ctypes.data if P.size else None, n,
        None if X is None else X.ctypes.data, 0 if X is None else X.shape[1], F.ctypes.data if F.size else None, m,
        body.ctypes.data if body.size else None, None, ctypes.byref(st))
    _native.raise_for(st)
    path.write_bytes(head + body.tobytes())


def load_mesh(path, format: str = "auto") -> TriMesh:
    """Load a triangle mesh from a binary PLY file (io.py:62-76)."""
    path = Path(path)
    if format == "auto":
        format = _detect_format(path)
    if format == "ply":
        return _load_ply(path)
    if format == "obj":
        raise MeshFormatError("OBJ (text) is not on the GPU I/O path; use binary PLY", path=path)
    raise ValueError(f"unknown mesh format {format!r}")


def save_mesh(mesh: TriMesh, path, format: str = "auto") -> None:
    """Save a mesh as binary little-endian PLY (io.py:79-89)."""
    path = Path(path)
    if format == "auto":
        format = _detect_format(path)
    if format == "ply":
        _save_ply(mesh, path)
    elif format == "obj":
        raise MeshFormatError("OBJ (text) is not on the GPU I/O path; use binary PLY", path=path)
    else:
        raise ValueError(f"unknown mesh format {format!r}")


def save_clusters(path, result) -> str:
    """The `<output>.clusters.npz` sidecar of the CLI (cli.py:95-96): replace + mapping."""
    sidecar = str(path) + ".clusters.npz"
    np.savez(sidecar, replace=result.replace, mapping=result.mapping)
    return sidecar
