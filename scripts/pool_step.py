"""cfg3's pooling half on its own (ncu windows): decimate the 4-level hierarchy once, then
run W warm-up + 1 measured pass of max-pool down / unpool up of C=64 float32 features.

    python scripts/pool_step.py [--warmup 2] [--mode max] [--fresh]

--fresh re-decimates before the measured pass so the cluster-CSR build is in the window."""

import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2103_15076_b200 import tensor as T  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--warmup", type=int, default=2)
ap.add_argument("--mode", default="max")
ap.add_argument("--fresh", action="store_true")
args = ap.parse_args()
wl = bench.workload("cfg3", 0)
mesh = wl["mesh"]
V0 = torch.from_numpy(mesh.positions).cuda()
F0 = torch.from_numpy(mesh.facets).cuda()
X0 = torch.from_numpy(np.random.default_rng(0).standard_normal((mesh.n_vertices, 64)).astype(np.float32)).cuda()


def chain():
    dds, V, F = [], V0, F0
    for t in wl["levels"]:
        dd = T.decimate(V, F, target=t)
        dds.append(dd)
        V, F = dd.vertices, dd.faces
    return dds


def passes(dds):
    X = X0
    for dd in dds:
        X = T.pool(X, dd, mode=args.mode)
    for dd in reversed(dds):
        X = T.unpool(X, dd)
    return X


dds = chain()
for _ in range(args.warmup):
    passes(dds)
torch.cuda.synchronize()
if args.fresh:
    dds = chain()
    torch.cuda.synchronize()
passes(dds)
torch.cuda.synchronize()
print("pool_step done", file=sys.stderr)
