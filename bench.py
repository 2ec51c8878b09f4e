"""Benchmark of the decimation hot path (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config cfg2]

One "step" = one decimate_parallel call from input to target, including every
internal round; facets/s = input facets / step time.  The
default workload is BASELINE.json configs[1]: delaunay_terrain(115_114,
noise=0.02, seed=12) decimated to 41,449 vertices (paper Fig. 1 size).  With
N > 1 GPUs (one process per GPU, torchrun) every rank decimates its own copy
of the workload with no inter-GPU traffic ("scaling": "weak") -- except cfg4, whose
fixed 256-mesh batch is sharded across the ranks ("scaling": "strong"); `value` is the
whole-job facets/s over the max-over-ranks device time.

Reported: `value` (device-resident inputs, CUDA events on the launching stream,
L2 flushed between steps), `e2e` (public numpy API with pinned host inputs,
H2D + D2H inside the timed region), `roofline` of the dominant kernel (timed
live with CUDA events inside the timed region; algorithmic bytes from the
per-round counts), `cpu_baseline` (the C oracle port of the reference on this
host, plus the UNMODIFIED reference from baseline/_ref as `stock_reference`),
`clocks` sampled during the timed region, `gpu_launches`.
`--impl reference` times the reference's CPU algorithm (oracle port, all
usable host threads) on the same workload, with the stock reference beside
it; rank 0 only.
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "ms per decimation step and facets/sec (1/2/4/8 B200) vs ref CPU; % HBM peak"
# Picasso GPU decimation of the Fig. 1 mesh (115,114 v / 231,293 f -> 41,449 v) in 65 ms.
PUBLISHED_FIG1_MS = 65.0
PUBLISHED_FIG1_FACETS = 231_293
L2_FLUSH_BYTES = 512 << 20  # > 126 MB L2


# ---------------------------------------------------------------- workloads
def workload(name: str, rank: int, world: int | None = None):
    """Synthetic input of a BASELINE.json config.  `levels` = successive
    decimate_parallel targets of one step (a hierarchy for cfg3 / cfg5);
    `pool_channels` > 0 adds max-pool down / unpool up of float32 features.
    cfg4 is the one sharded workload: rank `rank` of `world` (default WORLD_SIZE) gets its
    facet-balanced slice of the fixed 256-mesh batch (strong scaling)."""
    from paper_2103_15076_b200 import synthetic as S
    from paper_2103_15076_b200.mesh import concat_batch

    if name == "cfg2":
        return dict(mesh=S.delaunay_terrain(115_114, noise=0.02, seed=12), levels=[41_449], pool_channels=0,
                    desc="delaunay_terrain(115114, noise=0.02, seed=12) -> 41449 vertices (BASELINE configs[1])")
    if name == "cfg1":
        return dict(mesh=S.icosphere(5), levels=[3585], pool_channels=0,
                    desc="icosphere(5) -> 3585 vertices (configs[0])")
    if name == "cfg3":
        return dict(mesh=S.delaunay_terrain(500_000, noise=0.02, seed=3), levels=[125_000, 62_500, 31_250, 15_625],
                    pool_channels=64,
                    desc="delaunay_terrain(500000, 0.02, seed=3): 4 decimations 125000/62500/31250/15625 + "
                         "max-pool down / unpool up of C=64 float32 features (configs[2])")
    if name == "cfg4":
        from paper_2103_15076_b200 import sharding

        world = int(os.environ.get("WORLD_SIZE", "1")) if world is None else world
        batch = concat_batch([S.delaunay_terrain(2500, noise=0.02, seed=b) for b in range(256)])
        sub, lo, hi = sharding.shard_batch(batch, world, rank)  # facet-balanced contiguous slice (§8(e))
        return dict(mesh=sub, levels=[1250], pool_channels=0,
                    desc=f"batch of 256 delaunay_terrain(2500, 0.02, seed=b) -> 1250 each (configs[3]); "
                         f"{world} GPU(s), this rank's facet-balanced slice = meshes [{lo}, {hi})")
    if name == "cfg5":
        mesh = S.perturbed_grid(3163, noise=0.02, seed=rank)
        n, lv = mesh.n_vertices, []
        for _ in range(4):
            n = -(-n // 2)
            lv.append(n)
        return dict(mesh=mesh, levels=lv, pool_channels=0,
                    desc="perturbed_grid(3163, 0.02, seed=rank): 4 levels by ceil-halving "
                         + "/".join(str(x) for x in lv) + " (configs[4], one mesh per GPU)")
    raise SystemExit(f"unknown --config {name}")


# ---------------------------------------------------------------- helpers
def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as fh:
            d = json.load(fh)
        return float(d["hbm_gbs"]), "measured"
    return 6650.0, "fallback"


REASON_FIELDS = ["clocks_event_reasons.sw_power_cap", "clocks_event_reasons.hw_slowdown",
                 "clocks_event_reasons.hw_thermal_slowdown", "clocks_event_reasons.sw_thermal_slowdown"]


class ClockSampler:
    """nvidia-smi sampled every 50 ms while the timed region runs."""

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines = []

    def __enter__(self):
        q = "index,clocks.sm,clocks.max.sm,utilization.gpu," + ",".join(REASON_FIELDS)
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={q}", "--format=csv,noheader,nounits", "-lms",
                 "50"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
            time.sleep(0.15)
        except FileNotFoundError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *exc):
        if self.proc is not None:
            time.sleep(0.1)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except Exception:
                self.proc.kill()

    def summary(self):
        rows = []
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 4 + len(REASON_FIELDS):
                continue
            try:
                rows.append((float(parts[1]), float(parts[2]), float(parts[3]), parts[4:]))
            except ValueError:
                continue
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        loaded = [r for r in rows if r[2] > 0] or rows
        reasons = set()
        for r in rows:
            for name, val in zip(REASON_FIELDS, r[3]):
                if val.lower().startswith("active"):
                    reasons.add(name.split(".")[-1])
        return {"sm_mhz": float(np.median([r[0] for r in loaded])), "sm_max_mhz": rows[0][1],
                "reasons": sorted(reasons), "samples": len(rows), "samples_under_load": len(loaded)}


# Algorithmic bytes per launch of the main kernels, from one round's counts
# (N, M, E vertices/facets/edges in, Nn/Mn out; int32 indices, float64 values).
# Each byte a kernel must move at least once -- see DESIGN.md "Kernels".
def kernel_bytes(name: str, r: dict, C: int = 3) -> float | None:
    name = name.split("<")[0]  # template instances (k_edges<0>) share the model
    N, M, E, Nn, Mn = r["N"], r["M"], r["E"], r["N_out"], r["M_out"]
    table = {
        "k_facet_plane": 12 * M + 24 * N + 32 * M + 4 * N,
        "k_inc_scatter": 12 * M + 4 * N + 12 * M,
        "k_vertex": 4 * N + 12 * M + 32 * M + 12 * M + 80 * N + 8 * E + 8 * N,
        # per-vertex counts/offsets + quadric + position in, upper neighbours in, edge (e0, e1, key)
        # out, both adjacency slots (neighbour, edge id, key) out, per-vertex matching state init
        "k_edges": 16 * N + 80 * N + 24 * N + 4 * E + 16 * E + 32 * E + 24 * N,
        # slots (neighbour, edge id, key) in, rank-ordered (neighbour, edge id, key prefix) out, cursor
        "k_adj_rank": 12 * N + 32 * E + 24 * E,
        # adjacency (nbr + edge id) + rank key per slot, suitor word per vertex
        "k_suitor": 8 * E + 8 * E + 16 * E + 8 * N,
        "k_select": 16 * Nn,
        # one pass over the adjacency (nbr + edge id + key prefix) + pick / mate words: the matching
        # must read every incidence at least once; all LD-round launches of the round share it
        "k_ld_pick": 24 * E + 12 * N,
        "k_vertex_t": 4 * N + 12 * M + 32 * M + 12 * M + 80 * N + 8 * E + 8 * N,
        "k_contract": 4 * N + 4 * Nn + 24 * N + 24 * Nn,
        "k_facet_remap": 12 * M + 4 * N + 12 * M + 16 * M + 4 * M + N,
        "k_inc_scatter": 12 * M + 4 * N + 12 * M,
        "k_compose": 8 * r.get("N0", N) + 4 * N,
        # round 1 only: facets int64 in -> int32 out, positions in (+ copied into the workspace)
        "k_init_inputs": (24 * M + 12 * M + 24 * N + 24 * N) if r.get("first") else 0,
        # round epilogue + the NEXT round's facet planes (its facets are this round's outputs)
        "k_compose_plane": 8 * r.get("N0", N) + 4 * N + 12 * Mn + 24 * Nn + 32 * Mn + 4 * Nn,
        # one per call (after its last round): replace / mapping int32 -> int64, positions and
        # facets out (features alias the positions in the bench workloads)
        # after the call's last round: the result copy-out (int32 / float64 words as they are) and
        # the caller's emission (int32 -> int64, float64) -- two launches per call
        "k_emit": ((4 + 4 + 8 + 8) * r.get("N0", N) + 2 * (24 * Nn + 12 * Mn) + 24 * Nn + 24 * Mn + 24 * Nn)
        if r.get("last") else 0,
    }
    v = table.get(name)
    return None if v is None else float(v)


def call_bytes(name: str, call: dict) -> float | None:
    """Algorithmic bytes of the pooling-side kernels per decimate call (n_in -> n_out, C channels,
    float32): SURVEY.md §8(d) pool 4CN + 8N + 4CN', unpool 8N + 4CN' + 4CN; the cluster CSR build
    reads replace and writes offsets + members once (counts and the in-place sort included)."""
    name = name.split("<")[0].strip("(")
    n, no, C = call["n_in"], call["n_out"], call.get("C", 0)
    if not C:
        return None
    table = {"k_pool_vec": 4 * C * n + 8 * n + 4 * C * no, "k_pool": 4 * C * n + 8 * n + 4 * C * no,
             "k_unpool_rows": 8 * n + 4 * C * no + 4 * C * n, "k_unpool_vec": 8 * n + 4 * C * no + 4 * C * n,
             "k_csr_coop": 4 * n + 4 * no + 4 * n + 4 * no + 4 * n + 4 * n}
    return table.get(name)


def step_bytes(rounds: list, n0: int, C: int = 3) -> float:
    """SURVEY.md §8(d) whole-step model: Σ_r 24N+24M+8CN+160N+48E+24N'+24M'+8CN' + 16·N0."""
    b = 16.0 * n0
    for r in rounds:
        N, M, E, Nn, Mn = r["N"], r["M"], r["E"], r["N_out"], r["M_out"]
        b += 24 * N + 24 * M + 8 * C * N + 160 * N + 48 * E + 24 * Nn + 24 * Mn + 8 * C * Nn
    return b


def cpu_info() -> dict:
    model = None
    try:
        with open("/proc/cpuinfo") as fh:
            for ln in fh:
                if ln.startswith("model name"):
                    model = ln.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    try:
        usable = len(os.sched_getaffinity(0))
    except AttributeError:
        usable = os.cpu_count()
    return {"cpu_model": model, "cpu_count": os.cpu_count(), "usable_cores": usable}


def stock_reference(name: str, wl: dict, budget_s: float = 25.0) -> dict:
    """The UNMODIFIED reference (meshforge, pip-installed into baseline/_ref) through its own
    public API -- decimate_parallel (+ pool/unpool for cfg3) -- on a bounded sample of the
    workload: median of up to 3 steps within ~budget_s."""
    ref_dir = os.path.join(ROOT, "baseline", "_ref")
    if not os.path.isdir(os.path.join(ref_dir, "meshforge")):
        return {"unavailable": "baseline/_ref/meshforge not installed (see DESIGN.md §6)"}
    if ref_dir not in sys.path:
        sys.path.append(ref_dir)
    try:
        import meshforge as rmf
        from meshforge import pooling as rpool
    except Exception as e:  # noqa: BLE001
        return {"unavailable": f"importing the reference failed: {e!r}"}
    sw = with_features(dict(cpu_sample(name, wl)))
    mesh = sw["mesh"]
    batched = hasattr(mesh, "vertex_offsets")
    base = mesh.mesh if batched else mesh
    rm = rmf.TriMesh(base.positions, base.facets)
    if batched:
        rm = rmf.BatchedMesh(rm, mesh.vertex_offsets, mesh.facet_offsets)

    def one():
        cur, f, outs = rm, sw.get("_features"), []
        for tgt in sw["levels"]:
            r = rmf.decimate_parallel(cur, rmf.DecimationConfig(target_vertices=tgt))
            if f is not None:
                f = rpool.pool(f, r, mode="max")
                outs.append(r)
            cur = r.mesh
        for r in reversed(outs):
            f = rpool.unpool(f, r)

    times = []
    t0 = time.perf_counter()
    while len(times) < 3 and (not times or time.perf_counter() - t0 + times[-1] < budget_s):
        t = time.perf_counter()
        one()
        times.append(time.perf_counter() - t)
    ms = 1e3 * float(np.median(times))
    cores = (os.cpu_count() or 1) if batched else 1  # batches: the reference's own thread pool
    return {"value": facets_in(sw) / (ms / 1e3), "unit": "facets/s", "ms_per_step": ms, "cores": cores,
            "kind": "reference-stock",
            "sample": f"median of {len(times)} step(s) of {sw['desc']}; meshforge 0.1.0 from baseline/_ref, "
                      f"numpy {np.__version__}", **cpu_info()}


def scaling_of(name: str) -> str:
    """cfg4 shards one fixed batch across the ranks (total work fixed: strong); every other
    config gives each rank its own copy of the workload (per-GPU work fixed: weak)."""
    return "strong" if name == "cfg4" else "weak"


def dist_setup():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


# ---------------------------------------------------------------- CPU arm (oracle port of the reference)
def cpu_sample(name: str, wl: dict) -> dict:
    """Bounded CPU sample of a workload: the same workload when one oracle step
    takes a few seconds, else the same generator at reduced size."""
    if name == "cfg5":
        from paper_2103_15076_b200 import synthetic as S

        mesh = S.perturbed_grid(700, noise=0.02, seed=0)
        n, lv = mesh.n_vertices, []
        for _ in range(4):
            n = -(-n // 2)
            lv.append(n)
        return dict(mesh=mesh, levels=lv, pool_channels=0,
                    desc="perturbed_grid(700, 0.02, seed=0), same 4-level ceil-halving hierarchy (reduced size)")
    return wl


def oracle_step(wl: dict, threads: int = 1) -> None:
    """One step on the C oracle: the level chain, plus max-pool down / unpool up when configured."""
    from oracle import oracle as O

    mesh = wl["mesh"]
    batched = hasattr(mesh, "vertex_offsets")
    base = mesh.mesh if batched else mesh
    P, F, X = base.positions, base.facets, None
    kw = dict(vertex_offsets=mesh.vertex_offsets, facet_offsets=mesh.facet_offsets, threads=threads) if batched \
        else {}
    feats = wl.get("_features")
    reps = []
    for tgt in wl["levels"]:
        out = O.decimate(P, F, X, target=tgt, **kw)
        if feats is not None:
            reps.append((out["replace"], len(out["positions"])))
            feats = O.pool(feats, out["replace"], len(out["positions"]), "max")
        P, F, X = out["positions"], out["facets"], out["features"]
        if batched:
            kw.update(vertex_offsets=out["vertex_offsets"], facet_offsets=out["facet_offsets"])
    for rep, _ in reversed(reps):
        feats = O.unpool(feats, rep)


def with_features(wl: dict) -> dict:
    if wl.get("pool_channels"):
        n = (wl["mesh"].mesh if hasattr(wl["mesh"], "vertex_offsets") else wl["mesh"]).n_vertices
        wl["_features"] = np.random.default_rng(0).standard_normal((n, wl["pool_channels"])).astype(np.float32)
    return wl


def facets_in(wl: dict) -> int:
    m = wl["mesh"]
    return (m.mesh if hasattr(m, "vertex_offsets") else m).n_facets


def run_reference(args):
    world, rank, _ = dist_setup()
    if rank != 0:
        return 0
    wl = with_features(cpu_sample(args.config, workload(args.config, 0, world=1)))  # the whole job
    threads = os.cpu_count() or 1
    for _ in range(args.warmup):
        oracle_step(wl, threads)
    times = []
    for _ in range(args.steps):
        t = time.perf_counter()
        oracle_step(wl, threads)
        times.append(time.perf_counter() - t)
    ms = 1e3 * float(np.mean(times))
    value = facets_in(wl) / (ms / 1e3)
    batched = hasattr(wl["mesh"], "vertex_offsets")
    cores = threads if batched else 1
    sample = f"{wl['desc']}; oracle port of the reference, {'%d threads over meshes' % threads if batched else '1 thread'}"
    line = {"metric": METRIC, "value": value, "unit": "facets/s", "impl": "reference", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
            "scaling": scaling_of(args.config), "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": wl["desc"], "facets_in": facets_in(wl)},
            "cpu_baseline": {"value": value, "unit": "facets/s", "cores": cores, "kind": "port", "sample": sample,
                             **cpu_info()},
            "stock_reference": stock_reference(args.config, workload(args.config, 0, world=1)),
            "e2e": {"value": value, "unit": "facets/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


def cpu_baseline(name: str, wl: dict, budget_s: float = 12.0) -> dict:
    """The C oracle (port of the reference path) on this host, single thread, bounded sample."""
    sw = with_features(dict(cpu_sample(name, wl)))
    times = []
    t0 = time.perf_counter()
    while time.perf_counter() - t0 < budget_s and len(times) < 50:
        t = time.perf_counter()
        oracle_step(sw, 1)
        times.append(time.perf_counter() - t)
    ms = 1e3 * float(np.median(times))
    return {"value": facets_in(sw) / (ms / 1e3), "unit": "facets/s", "cores": 1, "kind": "port",
            "sample": f"{len(times)} step(s) of {sw['desc']} (median {ms:.1f} ms)", **cpu_info()}


# ---------------------------------------------------------------- our arm
def run_ours(args):
    import torch

    world, rank, local = dist_setup()
    ngpu = torch.cuda.device_count()
    if world > 1:
        import torch.distributed as dist

        torch.cuda.set_device(local % ngpu)
        backend = os.environ.get("MF_DIST_BACKEND", "nccl")
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local % ngpu))
        else:
            dist.init_process_group(backend)
    else:
        dist = None
        torch.cuda.set_device(0)
    dev = torch.device("cuda", torch.cuda.current_device())
    coll_dev = dev if (dist and dist.get_backend() == "nccl") else torch.device("cpu")

    def sum_over_ranks(x: float) -> float:
        if not dist:
            return x
        t = torch.tensor([x], dtype=torch.float64, device=coll_dev)
        dist.all_reduce(t, op=dist.ReduceOp.SUM)
        return float(t.item())

    def max_over_ranks(x: float) -> float:
        """The timing reduction (the only collective: the data path has none, §8(e))."""
        if not dist:
            return x
        t = torch.tensor([x], dtype=torch.float64, device=coll_dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    import paper_2103_15076_b200 as mfg
    from paper_2103_15076_b200 import _native
    from paper_2103_15076_b200 import tensor as T

    wl = with_features(workload(args.config, rank))
    mesh, levels = wl["mesh"], wl["levels"]
    batched = hasattr(mesh, "vertex_offsets")
    base = mesh.mesh if batched else mesh
    n_in, m_in = base.n_vertices, base.n_facets
    V0 = torch.from_numpy(base.positions).to(dev)
    F0 = torch.from_numpy(base.facets).to(dev)
    X0 = torch.from_numpy(wl["_features"]).to(dev) if wl.get("_features") is not None else None
    nv = np.diff(mesh.vertex_offsets) if batched else None
    nf = np.diff(mesh.facet_offsets) if batched else None
    flush = torch.empty(L2_FLUSH_BYTES, dtype=torch.uint8, device=dev)

    def step():
        dds = []
        V, F, X, cnv, cnf = V0, F0, X0, nv, nf
        for tgt in levels:
            dd = T.decimate(V, F, cnv, cnf, target=tgt)
            dds.append(dd)
            if X is not None:
                X = T.pool(X, dd, mode="max")
            V, F = dd.vertices, dd.faces
            if batched:
                cnv, cnf = dd.nv.numpy(), dd.mf.numpy()
        if X is not None:
            for dd in reversed(dds):
                X = T.unpool(X, dd)
        return dds

    # warm-up; the last warm-up step times every kernel to name the dominant one
    for _ in range(max(0, args.warmup - 1)):
        step()
    torch.cuda.synchronize()
    flush.zero_()
    _native.profile(1)
    dds = step()
    torch.cuda.synchronize()
    breakdown = _native.profile_read()
    _native.profile(0)
    rounds, calls = [], []
    for dd in dds:
        rs = dd.round_stats()
        for i, r in enumerate(rs):
            r["N0"] = dd._dec.n_in
            r["first"] = i == 0
            r["last"] = i == len(rs) - 1  # the call's outputs are emitted after its last round
            rounds.append(r)
        calls.append({"n_in": dd._dec.n_in, "n_out": dd._dec.n_out, "C": wl.get("pool_channels", 0)})
    total_ms = sum(v[0] for v in breakdown.values())
    dominant = max(breakdown.items(), key=lambda kv: kv[1][0])[0]
    # the timed region times the dominant kernel live: warm that graph variant first
    _native.profile(2, dominant)
    step()
    torch.cuda.synchronize()
    _native.profile(2, dominant)  # clears the warm-up record

    # ---------------- timed region: device-resident inputs
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    _native.launch_count(reset=True)
    starts = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    cvd = os.environ.get("CUDA_VISIBLE_DEVICES")
    phys = int(cvd.split(",")[local % ngpu]) if cvd else local % ngpu
    with ClockSampler(phys) as clk:
        for k in range(args.steps):
            flush.zero_()  # L2 flush between timed steps (outside the events)
            starts[k].record()
            step()
            ends[k].record()
        torch.cuda.synchronize()
    launches = _native.launch_count() // args.steps
    dom = _native.profile_read().get(dominant, (0.0, 0))
    _native.profile(0)
    if dist:
        dist.barrier()
    step_ms = float(np.sum([s.elapsed_time(e) for s, e in zip(starts, ends)])) / args.steps
    step_ms_max = max_over_ranks(step_ms)
    total_facets = sum_over_ranks(m_in)  # every rank's own work (replicas, or a batch slice)
    value = total_facets / (step_ms_max / 1e3)

    # ---------------- e2e: public numpy API, pinned host inputs, H2D + D2H inside
    Pp = torch.empty((n_in, 3), dtype=torch.float64, pin_memory=True).numpy()
    Fp = torch.empty((m_in, 3), dtype=torch.int64, pin_memory=True).numpy()
    Pp[:] = base.positions
    Fp[:] = base.facets
    Xp = None
    if wl.get("_features") is not None:
        Xp = torch.empty(wl["_features"].shape, dtype=torch.float32, pin_memory=True).numpy()
        Xp[:] = wl["_features"]
    pm = mfg.TriMesh(Pp, Fp)
    host_mesh = mfg.BatchedMesh(pm, mesh.vertex_offsets, mesh.facet_offsets) if batched else pm

    def e2e_step():
        cur, X, outs, d2h = host_mesh, Xp, [], 0
        for tgt in levels:
            res = mfg.decimate_parallel(cur, mfg.DecimationConfig(target_vertices=tgt))
            outs.append(res)
            o = res.mesh.mesh if batched else res.mesh
            d2h += o.positions.nbytes + o.facets.nbytes + res.replace.nbytes + res.mapping.nbytes
            if not np.shares_memory(o.features, o.positions):  # features that ARE the positions share it
                d2h += o.features.nbytes
            if X is not None:
                X = mfg.pool(X, res, mode="max")
                d2h += X.nbytes
            cur = res.mesh
        if X is not None:
            for res in reversed(outs):
                X = mfg.unpool(X, res)
                d2h += X.nbytes
        return d2h

    d2h = e2e_step()
    for _ in range(max(2, args.warmup)):  # warm the pinned host allocator and the graph cache on this path
        e2e_step()
    e2e_t = []
    for _ in range(max(3, min(args.steps, 20))):
        flush.zero_()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        e2e_step()
        e2e_t.append(time.perf_counter() - t0)
    e2e_ms = max_over_ranks(1e3 * float(np.mean(e2e_t)))
    h2d = Pp.nbytes + Fp.nbytes + (Xp.nbytes if Xp is not None else 0)

    if rank != 0:
        if dist:
            dist.destroy_process_group()
        return 0

    # ---------------- roofline of the dominant kernel
    peak, peak_kind = load_peaks()
    per_round = [kernel_bytes(dominant, r) for r in rounds]
    if any(b is None for b in per_round):  # a pooling-side kernel: its bytes follow the calls
        per_round = [call_bytes(dominant, c) for c in calls]
    dom_ms_per_step = dom[0] / args.steps if dom[1] else None
    roof = {"kernel": dominant, "bound": "hbm", "peak": peak, "unit": "GB/s", "peak_source": peak_kind}
    if dom_ms_per_step and all(b is not None for b in per_round):
        alg = float(sum(per_round))
        achieved = alg / (dom_ms_per_step / 1e3) / 1e9
        roof.update({"achieved": achieved, "frac": achieved / peak, "alg_bytes_per_step": alg,
                     "launches_per_step": dom[1] / args.steps, "ms_per_step": dom_ms_per_step,
                     "share_of_step": dom_ms_per_step / step_ms})
    else:
        roof.update({"achieved": None, "frac": None, "ms_per_step": dom_ms_per_step})
    traffic = None
    tp = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(tp):
        with open(tp) as fh:
            traffic = json.load(fh).get(args.config, {}).get(dominant)
    roof["traffic"] = traffic
    whole = sum(step_bytes([r], r["N0"]) - 16.0 * r["N0"] for r in rounds) + 16.0 * n_in
    roof["step_alg_bytes"] = whole
    if wl.get("pool_channels"):  # pool / unpool against the same peak (profiled warm-up step)
        pr = {}
        for fam in ("k_pool_vec", "k_unpool_rows", "k_csr_coop"):
            ms = sum(v[0] for k, v in breakdown.items() if fam in k)
            b = sum(call_bytes(fam, c) or 0 for c in calls)
            if ms > 0 and b > 0:
                pr[fam] = {"ms_per_step": ms, "alg_bytes_per_step": b, "achieved": b / (ms / 1e3) / 1e9,
                           "frac": b / (ms / 1e3) / 1e9 / peak, "source": "CUDA events, profiled warm-up step"}
        roof["pooling"] = pr
    roof["step_frac"] = whole / (step_ms / 1e3) / 1e9 / peak

    cpu = None
    if world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline(args.config, wl)
        cpu["stock_reference"] = stock_reference(args.config, wl)

    vs = None
    if args.config == "cfg2":
        vs = value / (PUBLISHED_FIG1_FACETS / (PUBLISHED_FIG1_MS / 1e3))
    line = {
        "metric": METRIC, "value": value, "unit": "facets/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": step_ms_max, "higher_is_better": True, "scaling": scaling_of(args.config),
        "vs_baseline": vs, "dtype": "f64", "data": "synthetic",
        "config": {"workload": wl["desc"], "facets_in": m_in, "facets_total": int(total_facets), "vertices_in": n_in, "levels": levels,
                   "rounds": len(rounds), "l2": "flushed between timed steps (512 MiB memset, outside events)",
                   "parallelism": (f"{world} GPUs, " + ("facet-balanced shards of one batch" if args.config == "cfg4"
                                                       else "independent work per GPU") + ", no collective")
                   if world > 1 else "1 GPU"},
        "clocks": clk.summary(),
        "e2e": {"value": total_facets / (e2e_ms / 1e3), "unit": "facets/s", "ms_per_step": e2e_ms,
                "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h),
                "path": "paper_2103_15076_b200.decimate_parallel / pool / unpool (numpy in, numpy out; pinned inputs)"},
        "gpu_launches": int(launches),
        "roofline": roof,
        "cpu_baseline": cpu,
        "kernels": {k: {"ms": round(v[0], 4), "share": round(v[0] / total_ms, 4), "launches": v[1]}
                    for k, v in sorted(breakdown.items(), key=lambda kv: -kv[1][0])[:40]},
        "round_stats": rounds,
    }
    if vs is not None:
        line["vs_baseline_note"] = "value / (231,293 facets / 65 ms): Picasso Fig. 1 GPU decimation (RTX 2080 Ti)"
    print(json.dumps(line), flush=True)
    if dist:
        dist.destroy_process_group()
    return 0


def main():
    import faulthandler

    # a stuck call prints every thread's Python stack and ends the run instead of hanging it
    faulthandler.dump_traceback_later(int(os.environ.get("MF_BENCH_WATCHDOG_S", "900")), exit=True)
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="cfg2")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if args.gpus > 1 and world == 1 and args.impl == "ours":
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
               "--master-addr=127.0.0.1", "--master-port=29533", os.path.abspath(__file__)] + sys.argv[1:]
        return subprocess.call(cmd)
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
