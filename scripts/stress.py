"""Repeat the bench step many times (tensor API + numpy API) to surface rare hangs / races.

    python scripts/stress.py [--config cfg2] [--iters 500]

Prints progress; run under `timeout -s INT` so a hang shows the Python frame it is stuck in."""
import argparse
import faulthandler
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
faulthandler.register(__import__("signal").SIGUSR1)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2103_15076_b200 as mfg  # noqa: E402
from paper_2103_15076_b200 import tensor as T  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="cfg2")
ap.add_argument("--iters", type=int, default=500)
args = ap.parse_args()
wl = bench.workload(args.config, 0)
mesh, levels = wl["mesh"], wl["levels"]
batched = hasattr(mesh, "vertex_offsets")
base = mesh.mesh if batched else mesh
nv0 = np.diff(mesh.vertex_offsets) if batched else None
nf0 = np.diff(mesh.facet_offsets) if batched else None
V0 = torch.from_numpy(base.positions).cuda()
F0 = torch.from_numpy(base.facets).cuda()
ref = None
t0 = time.time()
for it in range(args.iters):
    faulthandler.dump_traceback_later(30, exit=True)  # a stuck call prints its Python frame and exits
    V, F, nv, nf = V0, F0, nv0, nf0
    for t in levels:
        dd = T.decimate(V, F, nv, nf, target=t)
        V, F = dd.vertices, dd.faces
        if batched:
            nv, nf = dd.nv.numpy(), dd.mf.numpy()
    digest = (int(dd.replace.sum()), int(dd.faces.sum()), float(dd.vertices.sum()))
    if ref is None:
        ref = digest
    elif digest != ref:
        print(f"iter {it}: tensor-API result changed {digest} != {ref}", flush=True)
        sys.exit(3)
    if it % 4 == 0:
        cur = mesh
        for t in levels:
            res = mfg.decimate_parallel(cur, mfg.DecimationConfig(target_vertices=t))
            cur = res.mesh
        out = res.mesh.mesh if batched else res.mesh
        if (int(res.replace.sum()), int(out.facets.sum())) != ref[:2]:
            print(f"iter {it}: numpy-API result differs", flush=True)
            sys.exit(3)
    if it % 50 == 0:
        print(f"iter {it} ok ({time.time() - t0:.1f} s)", flush=True)
torch.cuda.synchronize()
faulthandler.cancel_dump_traceback_later()
print("STRESS-OK", flush=True)
