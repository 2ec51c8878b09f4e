"""Phase timing of the public numpy API (host overheads vs device time)."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import cProfile  # noqa: E402
import pstats  # noqa: E402

import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2103_15076_b200 as mfg  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
wl = bench.with_features(bench.workload(cfg, 0))
mesh = wl["mesh"]
Pp = torch.empty((mesh.n_vertices, 3), dtype=torch.float64, pin_memory=True).numpy()
Fp = torch.empty((mesh.n_facets, 3), dtype=torch.int64, pin_memory=True).numpy()
Pp[:] = mesh.positions
Fp[:] = mesh.facets
pm = mfg.TriMesh(Pp, Fp)
X = wl.get("_features")


def step():
    cur, f, outs = pm, X, []
    for t in wl["levels"]:
        r = mfg.decimate_parallel(cur, mfg.DecimationConfig(target_vertices=t))
        outs.append(r)
        if f is not None:
            f = mfg.pool(f, r, mode="max")
        cur = r.mesh
    if f is not None:
        for r in reversed(outs):
            f = mfg.unpool(f, r)


for _ in range(3):
    step()
torch.cuda.synchronize()
t = time.perf_counter()
for _ in range(5):
    step()
print(cfg, "e2e ms", (time.perf_counter() - t) / 5 * 1e3)
pr = cProfile.Profile()
pr.enable()
for _ in range(5):
    step()
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(14)
