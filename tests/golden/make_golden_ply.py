"""Golden fixtures for binary PLY load / save (io.py:226-431) from the REAL reference
(run in the build container):

    python tests/golden/make_golden_ply.py

Writes tests/golden/ply/*.ply (inputs: files saved by the reference plus hand-built
variants -- float64 coords, extra vertex / element properties, uint indices, quads)
and tests/golden/ply.npz (the reference's load_mesh arrays for each file, and the
reference's saved bytes for two meshes).
"""

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")

import meshforge as mf  # noqa: E402
from meshforge import synthetic as msyn  # noqa: E402

OUT = os.path.join(HERE, "ply")


def write(name, header, body):
    with open(os.path.join(OUT, name), "wb") as fh:
        fh.write(("\n".join(header) + "\n").encode("ascii") + body)


def main():
    os.makedirs(OUT, exist_ok=True)
    arrays = {}
    # saved by the reference: plain and coloured (features -> uchar rgb)
    m1 = msyn.delaunay_terrain(300, 0.05, 2)
    mf.save_mesh(m1, os.path.join(OUT, "ref_plain.ply"))
    rng = np.random.default_rng(0)
    feats = np.concatenate([m1.positions, rng.uniform(-1.2, 1.2, (m1.n_vertices, 3))], axis=1)
    feats[:4, 3] = [-1.0, 1.0, 0.0, 2.0 / 255.0 - 1.0]  # exact / tie / clipped values
    m2 = mf.TriMesh(m1.positions, m1.facets, feats)
    mf.save_mesh(m2, os.path.join(OUT, "ref_color.ply"))
    for name, m in (("ref_plain", m1), ("ref_color", m2)):
        arrays[f"save|{name}|positions"] = m.positions
        arrays[f"save|{name}|facets"] = m.facets
        arrays[f"save|{name}|features"] = m.features
        arrays[f"save|{name}|bytes"] = np.frombuffer(open(os.path.join(OUT, name + ".ply"), "rb").read(), np.uint8)
    # hand-built: float64 coords + an extra float property + colours, uint indices
    n = 6
    P = rng.standard_normal((n, 3))
    rec = np.empty(n, dtype=[("x", "<f8"), ("y", "<f8"), ("z", "<f8"), ("confidence", "<f4"),
                             ("red", "u1"), ("green", "u1"), ("blue", "u1")])
    rec["x"], rec["y"], rec["z"] = P.T
    rec["confidence"] = 0.5
    rec["red"], rec["green"], rec["blue"] = [0, 128, 255, 7, 9, 200], 17, [255, 0, 1, 2, 3, 4]
    F = np.array([[0, 1, 2], [2, 1, 3], [3, 4, 5], [0, 2, 5]])
    face = np.empty(len(F), dtype=[("n", "u1"), ("idx", "<u4", 3)])
    face["n"], face["idx"] = 3, F
    write("hand_f64_uint.ply", ["ply", "format binary_little_endian 1.0", "comment made by make_golden_ply",
                                f"element vertex {n}", "property double x", "property double y", "property double z",
                                "property float confidence", "property uchar red", "property uchar green",
                                "property uchar blue", f"element face {len(F)}",
                                "property list uchar uint vertex_indices", "end_header"],
          rec.tobytes() + face.tobytes())
    # quads (fan-triangulated) with short coordinates and a trailing fixed-size element
    Q = np.array([[0, 1, 2, 3], [1, 4, 5, 2], [3, 2, 5, 6]])
    vs = np.array([[0, 0, 0], [1, 0, 0], [1, 1, 0], [0, 1, 0], [2, 0, 1], [2, 1, 1], [0, 2, 1]], dtype="<i2")
    qf = np.empty(len(Q), dtype=[("n", "u1"), ("idx", "<i4", 4)])
    qf["n"], qf["idx"] = 4, Q
    extra = np.arange(5, dtype="<f4")
    write("hand_quads_short.ply", ["ply", "format binary_little_endian 1.0", "element vertex 7",
                                   "property short x", "property short y", "property short z",
                                   "element face 3", "property list uchar int vertex_index",
                                   "element marker 5", "property float weight", "end_header"],
          vs.tobytes() + qf.tobytes() + extra.tobytes())
    for name in ("ref_plain", "ref_color", "hand_f64_uint", "hand_quads_short"):
        m = mf.load_mesh(os.path.join(OUT, name + ".ply"))
        arrays[f"load|{name}|positions"] = m.positions
        arrays[f"load|{name}|facets"] = m.facets
        arrays[f"load|{name}|features"] = m.features
        print(name, m.n_vertices, m.n_facets, m.n_channels)
    np.savez(os.path.join(HERE, "ply.npz"), **arrays)


if __name__ == "__main__":
    main()
