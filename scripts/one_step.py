"""Run W warm-up decimation calls (first level of the config) then exactly one more (ncu windows).

    python scripts/one_step.py [--config cfg2] [--warmup 3]

Prints the number of library kernel launches per step on stderr so the
ncu skip count can be set to warmup * launches.
"""

import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import bench  # noqa: E402
from paper_2103_15076_b200 import _native  # noqa: E402
from paper_2103_15076_b200 import tensor as T  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="cfg2")
ap.add_argument("--warmup", type=int, default=3)
args = ap.parse_args()
wl = bench.workload(args.config, 0)
mesh = wl["mesh"]
base = mesh.mesh if hasattr(mesh, "vertex_offsets") else mesh
nv = [int(x) for x in (mesh.vertex_offsets[1:] - mesh.vertex_offsets[:-1])] if hasattr(mesh, "vertex_offsets") else None
nf = [int(x) for x in (mesh.facet_offsets[1:] - mesh.facet_offsets[:-1])] if hasattr(mesh, "facet_offsets") else None
V = torch.from_numpy(base.positions).cuda()
F = torch.from_numpy(base.facets).cuda()
torch.cuda.synchronize()
for _ in range(args.warmup):
    _native.launch_count(reset=True)
    T.decimate(V, F, nv, nf, target=wl["levels"][0])
print(f"launches_per_step {_native.launch_count()}", file=sys.stderr)
T.decimate(V, F, nv, nf, target=wl["levels"][0])
torch.cuda.synchronize()
