"""One bench step of a hierarchy config (cfg3 / cfg5) through the device-tensor API, after W
warm-up steps -- for ncu launch lists (sum of kernel durations vs the step's wall time).

    python scripts/hier_step.py [--config cfg3] [--warmup 2]
"""
import argparse
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2103_15076_b200 import _native  # noqa: E402
from paper_2103_15076_b200 import tensor as T  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="cfg3")
ap.add_argument("--warmup", type=int, default=2)
args = ap.parse_args()
wl = bench.with_features(bench.workload(args.config, 0))
mesh = wl["mesh"]
V0 = torch.from_numpy(mesh.positions).cuda()
F0 = torch.from_numpy(mesh.facets).cuda()
X0 = torch.from_numpy(wl["_features"]).cuda() if wl.get("_features") is not None else None


def step():
    dds, V, F, X = [], V0, F0, X0
    for tgt in wl["levels"]:
        dd = T.decimate(V, F, None, None, target=tgt)
        dds.append(dd)
        if X is not None:
            X = T.pool(X, dd, mode="max")
        V, F = dd.vertices, dd.faces
    if X is not None:
        for dd in reversed(dds):
            X = T.unpool(X, dd)
    return dds


for w in range(args.warmup):
    t = time.perf_counter()
    step()
    torch.cuda.synchronize()
    print(f"warm-up step {w}: wall_ms {1e3 * (time.perf_counter() - t):.3f}", file=sys.stderr)
_native.launch_count(reset=True)
t = time.perf_counter()
step()
torch.cuda.synchronize()
print(f"launches_per_step {_native.launch_count()} wall_ms {1e3 * (time.perf_counter() - t):.3f}", file=sys.stderr)
