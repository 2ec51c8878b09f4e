"""Debug: structure-fuzz seed 2709 ('inverse' placement) round by round against the oracle."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np  # noqa: E402

import paper_2103_15076_b200 as mfg  # noqa: E402
import test_gpu_fuzz2 as T  # noqa: E402
from oracle import oracle as O  # noqa: E402
from paper_2103_15076_b200.numerics import einsum_order  # noqa: E402

seed = int(sys.argv[1]) if len(sys.argv) > 1 else 2709
rng = np.random.default_rng(10_000 + seed)
mesh = T._KINDS[seed % len(T._KINDS)](rng)
n = mesh.n_vertices
target = max(1, int(n * rng.uniform(0.2, 0.95)))
placement = "inverse" if rng.random() < 0.3 else "average"
shuffle = None if rng.random() < 0.6 else int(rng.integers(1 << 31))
rounds = "auto" if rng.random() < 0.7 else int(rng.integers(1, 4))
chain = O.round_targets(n, target, rounds)
print("n", n, "target", target, placement, shuffle, rounds, "chain", chain)
P, F = mesh.positions, mesh.facets
for r, t in enumerate(chain):
    exp = O.decimate(P, F, None, target=t, seed=shuffle, rounds=1, order=einsum_order(), placement=placement)
    res = mfg.decimate_parallel(mfg.TriMesh(P, F), mfg.DecimationConfig(target_vertices=t, placement=placement,
                                                                        shuffle_seed=shuffle, rounds=1), device=0)
    same = {k: np.array_equal(np.asarray(g).view(np.uint8), exp[k].view(np.uint8))
            for k, g in (("replace", res.replace), ("facets", res.mesh.facets), ("positions", res.mesh.positions))}
    print("round", r, "target", t, same)
    if not same["positions"]:
        d = np.flatnonzero((res.mesh.positions != exp["positions"]).any(axis=1))
        for i in d[:4]:
            mem = np.flatnonzero(exp["replace"] == i)
            print("  out", i, "members", mem, "gpu", res.mesh.positions[i].tolist(), "oracle", exp["positions"][i].tolist())
            print("    member positions", P[mem].tolist())
        break
    P, F = exp["positions"], exp["facets"]
