"""Debug: a multi-round call whose first rounds are identities vs the single real round."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np  # noqa: E402

import paper_2103_15076_b200 as mfg  # noqa: E402
import test_gpu_fuzz2 as T  # noqa: E402

seed = 2709
rng = np.random.default_rng(10_000 + seed)
mesh = T._KINDS[seed % len(T._KINDS)](rng)
for placement in ("inverse", "average"):
    one = mfg.decimate_parallel(mesh, mfg.DecimationConfig(target_vertices=15, placement=placement, rounds=1), device=0)
    for rounds in (2, 3):
        many = mfg.decimate_parallel(mesh, mfg.DecimationConfig(target_vertices=15, placement=placement, rounds=rounds),
                                     device=0)
        d = np.flatnonzero((one.mesh.positions != many.mesh.positions).any(axis=1))
        print(placement, "rounds", rounds, "replace equal", np.array_equal(one.replace, many.replace),
              "differing rows", d.tolist())
        for i in d[:3]:
            print("   ", one.mesh.positions[i].tolist(), many.mesh.positions[i].tolist(),
                  "members", np.flatnonzero(one.replace == i).tolist())
print("input has -0.0:", bool(np.any(np.signbit(mesh.positions) & (mesh.positions == 0))))
