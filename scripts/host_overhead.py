"""Host-side cost of one tensor-API decimation (cfg2): wall time per call vs the GPU time of the
same calls (CUDA events), and a cProfile of the Python layer."""
import cProfile
import os
import pstats
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2103_15076_b200 import tensor as T  # noqa: E402

wl = bench.workload("cfg2", 0)
V = torch.from_numpy(wl["mesh"].positions).cuda()
F = torch.from_numpy(wl["mesh"].facets).cuda()
t = wl["levels"][0]
for _ in range(20):
    T.decimate(V, F, target=t)
torch.cuda.synchronize()
N = 200
ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(N)]
t0 = time.perf_counter()
for a, b in ev:
    a.record()
    T.decimate(V, F, target=t)
    b.record()
torch.cuda.synchronize()
wall = (time.perf_counter() - t0) / N * 1e3
gpu = sum(a.elapsed_time(b) for a, b in ev) / N
print(f"per call: wall {wall:.4f} ms, events {gpu:.4f} ms")
pr = cProfile.Profile()
pr.enable()
for _ in range(100):
    T.decimate(V, F, target=t)
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(14)
# per-call Python-side split: before the library call / inside it (the library prints its phases
# with MF_HOST_TIMING=1)
import ctypes  # noqa: E402

from paper_2103_15076_b200 import _native  # noqa: E402

orig = _native.lib().mf_decimate_into
stamps = []


class _Wrap:
    def __call__(self, *a):
        t = time.perf_counter()
        stamps.append(("enter", t))
        r = orig(*a)
        stamps.append(("leave", time.perf_counter()))
        return r


lib = _native.lib()
lib.mf_decimate_into = _Wrap()
for _ in range(5):
    torch.cuda.synchronize()
    stamps.clear()
    t_start = time.perf_counter()
    T.decimate(V, F, target=t)
    t_end = time.perf_counter()
    e, l = stamps[0][1], stamps[1][1]
    print(f"python before call {1e6 * (e - t_start):.1f} us, library {1e6 * (l - e):.1f} us, "
          f"python after {1e6 * (t_end - l):.1f} us", flush=True)
