"""CPU oracle (TEST INFRASTRUCTURE ONLY -- never imported by the product path):
numpy restatement of the reference's binary PLY fast paths -- vertex records
(io.py:329-344, colours io.py:390-392), uniform-arity faces (io.py:277-306,
fan triangulation io.py:92-93) and the writer (io.py:404-431) -- over the host
header parse of paper_2103_15076_b200.meshio.  Pinned to the reference's own
outputs in tests/golden/ply.npz (tests/test_meshio.py).
"""

import numpy as np


def decode(data: bytes):
    from paper_2103_15076_b200.meshio import parse_ply_header

    fmt, elements, at = parse_ply_header(data)
    body = data[at:]
    cur, P, X, F = 0, None, None, np.zeros((0, 3), np.int64)
    for name, count, props in elements:
        if name == "vertex":
            rec = np.dtype([(p, "<" + t) for p, t in props])
            tab = np.frombuffer(body, dtype=rec, count=count, offset=cur)
            cur += rec.itemsize * count
            rows = {p: tab[p].astype(np.float64) for p, _ in props}
            P = np.stack([rows["x"], rows["y"], rows["z"]], axis=1)
            X = P.copy()
            if all(c in rows for c in ("red", "green", "blue")):
                X = np.concatenate([X, np.stack([rows[c] for c in ("red", "green", "blue")], 1) / 255.0 * 2.0 - 1.0], 1)
        elif name == "face":
            _, ct, it = props[0][1]
            arity = body[cur]
            rec = np.dtype([("n", "<" + ct), ("idx", "<" + it, arity)])
            tab = np.frombuffer(body, dtype=rec, count=count, offset=cur)
            cur += rec.itemsize * count
            idx = tab["idx"].astype(np.int64)
            tris = [(r[0], r[k], r[k + 1]) for r in idx.tolist() for k in range(1, arity - 1)]
            F = np.asarray(tris, dtype=np.int64).reshape(-1, 3)
        else:
            cur += sum(np.dtype("<" + t).itemsize for _, t in props) * count
    return P, F, X


def encode_body(P, F, X=None) -> bytes:
    color = X is not None and X.shape[1] >= 6
    if color:
        rec = np.empty(len(P), dtype=[("xyz", "<f4", 3), ("rgb", "u1", 3)])
        rec["xyz"] = P.astype("<f4")
        rec["rgb"] = np.clip(np.round((X[:, 3:6] + 1.0) * 127.5), 0, 255).astype("u1")
        vb = rec.tobytes()
    else:
        vb = P.astype("<f4").tobytes()
    face = np.empty(len(F), dtype=[("n", "u1"), ("idx", "<i4", 3)])
    face["n"], face["idx"] = 3, F.astype("<i4")
    return vb + face.tobytes()
