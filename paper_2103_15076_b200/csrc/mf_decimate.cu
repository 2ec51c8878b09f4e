// mf_decimate.cu -- host orchestration of decimate_parallel on one device.
//
// One call = the whole round chain of every batch entry as ONE stream-ordered
// launch sequence with no host synchronisation until the end: vertex counts
// per round are known on the host (they are the round targets), facet and
// edge counts stay on the device and every kernel reads them from there
// (grids are sized from host upper bounds).  The sequence is captured once
// per call shape into a CUDA graph and replayed: inputs are staged into fixed
// workspace buffers, outputs copied into the result allocation, and one small
// readback at the end carries status words, output facet offsets and the
// per-round counts.
//
// Batches (BatchedMesh, decimate.py:354-361) are processed as one segmented
// pipeline over the concatenated arrays: per-mesh budgets, per-mesh rank
// selection and per-mesh key-stream restart; a mesh whose chain is shorter
// (or that is already at its target) is bypassed in the remaining rounds,
// because a zero-budget round is not an identity (it drops duplicate facets
// and normalises -0.0), see SURVEY.md App. C.
#include <algorithm>
#include <climits>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <ctime>
#include <map>
#include <string>
#include <thread>
#include <vector>

#include "mf_internal.h"
#include "mf_kernels.cuh"

namespace mf {

thread_local int64_t g_launches = 0;

// ---- optional per-kernel timing (CUDA events on the launching stream) ----
struct ProfRec {
    const char* name;
    cudaEvent_t a, b;
};
thread_local int g_prof_mode = 0;  // 0 off, 1 every launch, 2 only kernels named g_prof_only
thread_local std::string g_prof_only;
thread_local std::vector<ProfRec> g_prof_recs;                         // recorded, not yet read
thread_local std::vector<std::pair<std::string, float>> g_prof_done;  // (kernel, ms)
thread_local std::vector<cudaEvent_t> g_prof_pool;
thread_local size_t g_prof_pool_used = 0;

static cudaEvent_t prof_event() {
    if (g_prof_pool_used == g_prof_pool.size()) {
        cudaEvent_t e;
        cudaEventCreate(&e);
        g_prof_pool.push_back(e);
    }
    return g_prof_pool[g_prof_pool_used++];
}
static bool prof_on(const char* name) {
    if (g_prof_mode == 1) return true;
    return g_prof_mode == 2 && g_prof_only == name;
}
// inside stream capture a plain cudaEventRecord only adds a dependency; the
// External flag turns it into an event-record node that fires on every replay
static void prof_record(cudaEvent_t e, cudaStream_t s) {
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    cudaStreamIsCapturing(s, &cs);
    if (cs == cudaStreamCaptureStatusActive) cudaEventRecordWithFlags(e, s, cudaEventRecordExternal);
    else cudaEventRecord(e, s);
}
void prof_pre(const char* name, cudaStream_t s) {
    if (!prof_on(name)) return;
    ProfRec r{name, prof_event(), prof_event()};
    prof_record(r.a, s);
    g_prof_recs.push_back(r);
}
void prof_post(const char* name, cudaStream_t s) {
    if (!prof_on(name)) return;
    prof_record(g_prof_recs.back().b, s);
}
// after the stream synchronised: fold event pairs into the tallies
static void prof_collect(const std::vector<ProfRec>& recs) {
    for (const ProfRec& r : recs) {
        float t = 0.f;
        cudaEventElapsedTime(&t, r.a, r.b);
        g_prof_done.emplace_back(r.name, t);
    }
}
void prof_collect_pending() {
    prof_collect(g_prof_recs);
    g_prof_recs.clear();
}

// first failing runtime call of the current recording (error attribution)
thread_local cudaError_t g_rec_err = cudaSuccess;
thread_local int g_rec_line = 0;
static void rec_check(cudaError_t e, int line) {
    if (e != cudaSuccess && g_rec_err == cudaSuccess) {
        g_rec_err = e;
        g_rec_line = line;
    }
}
#define RC(expr) rec_check((expr), __LINE__)
#define RCK() rec_check(cudaGetLastError(), __LINE__)

// Launch through cudaLaunchKernelEx; while the round chain is being recorded
// every launch carries the programmatic-stream-serialization attribute, so the
// captured graph's kernel->kernel edges are programmatic (PDL) edges.
thread_local bool g_pdl = false;
// Programmatic dependent launch on the graph's kernel->kernel edges: each node's launch overlaps
// its predecessor's tail.  Default on since round 2 (r2z: cfg2 0.4433 / 0.4432 vs 0.4458 / 0.4472
// ms, cfg5 11.48 vs 11.52 ms; measured a few % slower in round 1, before the graph lost its
// memset / memcpy nodes); MF_PDL=0 turns it off.
static bool pdl_enabled() {
    static int v = -1;
    if (v < 0) {
        const char* e = getenv("MF_PDL");
        v = (e && e[0] == '0') ? 0 : 1;
    }
    return v == 1;
}
template <typename... KArgs, typename... Args>
static cudaError_t launch_ex(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                             Args&&... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = (g_pdl && pdl_enabled()) ? 1 : 0;
    return cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}

#ifndef LAUNCH
// LAUNCH_AS: a kernel picked at run time (a function pointer) under a fixed profiling name
#define LAUNCH_AS(name, kernel, grid, block, smem, stream, ...)                                   \
    do {                                                                                          \
        prof_pre(name, stream);                                                                   \
        rec_check(launch_ex(kernel, dim3(grid), dim3(block), (smem), (stream), __VA_ARGS__),      \
                  __LINE__);                                                                      \
        prof_post(name, stream);                                                                  \
        g_launches++;                                                                             \
    } while (0)
#define LAUNCH(kernel, grid, block, smem, stream, ...) \
    LAUNCH_AS(#kernel, kernel, grid, block, smem, stream, __VA_ARGS__)
#endif

// Suitor variant per round size: 8 lanes per proposer below 2^18 vertices (more warps to hide
// the slot scans: cfg2 78 vs 119 us), one thread per proposer above (one wave of proposers:
// cfg4 136 vs 218 us, cfg3 326 vs 369 us).  MF_SUITOR=1 / 8 forces one (A/B runs).
// lanes per proposer: the rank-ordered adjacency makes the first winnable slot usually one of
// the first few, so lanes only pay while they fill the machine; measured (r1h): 8 lanes at cfg1
// (N*8 within one wave), 4 at both cfg2 rounds (0.569 -> 0.559 ms; 2 lanes 0.596; 8 lanes in
// round 2 only: 0.578), a thread each at cfg4 (640k)
static int suitor_lanes(int N, int sm_count) {
    static int v = -1;
    if (v < 0) {
        const char* e = getenv("MF_SUITOR");
        v = e ? atoi(e) : 0;
        if (v != 1 && v != 2 && v != 4 && v != 8) v = 0;
    }
    if (v) return v;
    if (N >= (1 << 18)) return 1;
    return (int64_t)N * 8 <= (int64_t)sm_count * 2048 ? 8 : 4;  // 8 lanes only within one wave
}

// MF_SEL_PASSES: multi-block selection passes in the graph before k_select resumes (default 5)
static int sel_passes() {
    static int v = -1;
    if (v < 0) {
        const char* e = getenv("MF_SEL_PASSES");
        v = e ? std::max(1, std::min(kSelPassesMax, atoi(e))) : kSelPasses;
    }
    return v;
}

// MF_SELECT_CL=1: 8-CTA cluster selection (DSMEM histogram merge) for mid-size meshes.  Measured
// no faster than the single CTA at cfg2 (75 vs 75 us) and slower at cfg1 (95 vs 53 us): the pass
// count, not the per-pass bandwidth, bounds these sizes -- so it is opt-in.
static bool select_cluster() {
    static int v = -1;
    if (v < 0) {
        const char* e = getenv("MF_SELECT_CL");
        v = (e && e[0] == '1') ? 1 : 0;
    }
    return v == 1;
}

static int select_cap() {  // MF_SEL_CAP: keys in k_select's shared-memory stage (A/B runs)
    static int v = -1;
    if (v < 0) {
        const char* e = getenv("MF_SEL_CAP");
        v = e ? std::max(kSelCap, std::min(kSelCapMax, atoi(e))) : kSelCap;
    }
    return v;
}

// MF_COND=1: conditional graph nodes (device-driven loop / skip).  Opt-in: measured neutral on
// B200, and Nsight Compute cannot profile the kernel nodes of a graph that holds conditional
// nodes -- the default graph stays fully profileable.
static bool use_cond() {
    static int v = -1;
    if (v < 0) {
        const char* e = getenv("MF_COND");
        v = (e && e[0] == '1') ? 1 : 0;
    }
    return v == 1;
}

// MF_VERTEX_SCAN=0: k_vertex_t + k_vertex_tiers + the offset scans instead of k_vertex_scan (A/B)
static int vertex_scan() {
    static int v = -1;
    if (v < 0) {
        // 0 off (default), 1 = 128 threads per 128-vertex tile, 2 = 256.  Measured (B200, r2i): cfg2
        // 0.501 / 0.518 / 0.504 ms, cfg5 11.98 / 13.07 / 13.35 ms -- the tile's mid-degree vertices
        // serialise on the block's few warps, which costs more than the two launches it saves
        const char* e = getenv("MF_VERTEX_SCAN");
        v = e ? atoi(e) : 0;
        if (v < 0 || v > 2) v = 0;
    }
    return v;
}

// MF_TWO_PASS_MIN=k: unseeded rounds from k vertices take the two-pass adjacency (k_edges lite +
// k_adj_build) instead of the lower-slot atomics + k_adj_rank_tiled.  Opt-in (default never):
// measured (r3c) cfg5 11.90 vs 11.74 ms -- k_edges 2.22 -> 1.78 ms, but k_adj_build's per-slot
// binary searches cost 1.67 vs 1.06 ms for k_adj_rank_tiled; cfg2 0.493 vs 0.449 ms (k = 0)
static int two_pass_min() {
    static int v = -2;
    if (v == -2) {
        const char* e = getenv("MF_TWO_PASS_MIN");
        v = e ? std::max(0, atoi(e)) : INT_MAX;
    }
    return v;
}

// rounds from this many vertices recompute facet planes in the vertex fold instead of reading the
// materialised k_facet_plane output (MF_RECOMPUTE_MIN; 0 = always). Off by default: on cfg5 the
// recomputing k_vertex_t<8> costs 2.33 ms against 1.31 + 0.63 ms for fold + plane pass
static int recompute_min() {
    static int v = -2;
    if (v == -2) {
        const char* e = getenv("MF_RECOMPUTE_MIN");
        v = e ? std::max(0, atoi(e)) : INT_MAX;
    }
    return v;
}

// MF_ZERO_COPY_IN=0: pinned host inputs are staged by a copy instead of read in place
static bool zero_copy_inputs() {
    static int v = -1;
    if (v < 0) {
        const char* e = getenv("MF_ZERO_COPY_IN");
        v = (e && e[0] == '0') ? 0 : 1;
    }
    return v == 1;
}

// MF_EDGES_RANK=1: unseeded rounds through the fused k_edges_rank instead of k_edges +
// k_adj_rank_tiled.  Opt-in: measured slower on B200 (r2n, 92 registers / 8 lanes per vertex:
// cfg2 0.557 vs 0.501 ms, cfg5 18.4 vs 12.0 ms) -- every pair cost evaluated twice plus a
// binary search of the lower end's list cost more latency than the atomics and the re-sort save.
static bool edges_rank() {
    static int v = -1;
    if (v < 0) {
        const char* e = getenv("MF_EDGES_RANK");
        v = (e && e[0] == '1') ? 1 : 0;
    }
    return v == 1;
}

// MF_VT16=1: thread tier up to degree 16 (90 registers) instead of 8 + the warp tier.  Opt-in:
// measured (r2o) cfg2 0.506 / 0.501 vs 0.496 / 0.494 ms -- the occupancy it costs outweighs the
// warp-tier launch it empties
static bool vt16(int N) {
    static int v = -1;
    if (v < 0) {
        const char* e = getenv("MF_VT16");
        v = (e && e[0] == '1') ? 1 : 0;
    }
    (void)N;
    return v == 1;
}

// MF_FUSE_PLANE=0: separate k_compose / k_facet_plane launches between rounds (A/B runs)
static bool fuse_plane() {
    static int v = -1;
    if (v < 0) {
        const char* e = getenv("MF_FUSE_PLANE");
        v = (e && e[0] == '0') ? 0 : 1;
    }
    return v == 1;
}

// grid-stride kernels launch at most MF_GRID_CAP blocks per SM
static int grid_cap_mult() {
    static int v = -1;
    if (v < 0) {
        const char* e = getenv("MF_GRID_CAP");
        v = e ? std::max(1, atoi(e)) : 64;  // blocks per SM at most (cfg5 12.56 -> 12.44 ms vs 16; 128: 12.53)
    }
    return v;
}
static int grid_for(const Context* ctx, int64_t n, int block = 256) {
    int64_t g = (n + block - 1) / block;
    int64_t cap = (int64_t)ctx->sm_count * grid_cap_mult();
    if (g > cap) g = cap;
    if (g < 1) g = 1;
    return (int)g;
}

// MF_HOST_TIMING=1: host-side phase timestamps of every mf_decimate call on stderr (profiling aid)
struct HostClock {
    bool on;
    double t0, last;
    std::string line;
    static double now() {
        timespec ts;
        clock_gettime(CLOCK_MONOTONIC, &ts);
        return ts.tv_sec * 1e6 + ts.tv_nsec * 1e-3;
    }
    HostClock() {
        static int v = -1;
        if (v < 0) {
            const char* e = getenv("MF_HOST_TIMING");
            v = (e && e[0] == '1') ? 1 : 0;
        }
        on = v == 1;
        t0 = last = on ? now() : 0.0;
    }
    void mark(const char* what) {
        if (!on) return;
        const double t = now();
        char b[64];
        snprintf(b, sizeof(b), " %s=%.1f", what, t - last);
        line += b;
        last = t;
    }
    ~HostClock() {
        if (on) fprintf(stderr, "mf_decimate host us:%s total=%.1f\n", line.c_str(), now() - t0);
    }
};

// _round_targets (decimate.py:294-316)
int64_t round_targets(int64_t n_in, int64_t target, int rounds, std::vector<int64_t>& chain) {
    chain.clear();
    if (rounds < 0) {
        int64_t cur = n_in;
        while ((cur + 1) / 2 > target) {
            cur = (cur + 1) / 2;
            chain.push_back(cur);
        }
        chain.push_back(target);
        return (int64_t)chain.size();
    }
    if (rounds == 1) {
        chain.push_back(target);
        return 1;
    }
    double ratio = std::pow((double)target / (double)n_in, 1.0 / (double)rounds);
    int64_t cur = n_in;
    for (int r = 1; r < rounds; r++) {
        int64_t step = (int64_t)std::ceil((double)n_in * std::pow(ratio, (double)r));
        step = std::min(std::max(step, target), cur);
        chain.push_back(step);
        cur = step;
    }
    chain.push_back(target);
    return (int64_t)chain.size();
}

// two look-back state buffers: each scan uses one and clears the other for the next
struct ScanBuf {
    unsigned long long* buf[2] = {nullptr, nullptr};
    int words = 0;
    int cur = 0;
    int resident = 0;  // tiles a ticketless launch may have (sm_count * 4)
};

// k_select's two-phase key stage by the bulk-copy engine (MF_SEL_BULK=0: per-thread loads, A/B)
static int sel_bulk() {
    static int v = -1;
    if (v < 0) {
        const char* e = getenv("MF_SEL_BULK");
        v = (e && e[0] == '0') ? 0 : 1;
    }
    return v;
}

// k_suitor<L> blocks per SM cap (MF_SUITOR_BPSM, 0 = one thread group per proposer; A/B)
static int suitor_bpsm() {
    static int v = -1;
    if (v < 0) {
        const char* e = getenv("MF_SUITOR_BPSM");
        v = e ? std::max(0, atoi(e)) : 0;
    }
    return v;
}

// k_select's first radix pass without the prefix test (MF_SEL_FIRST=0: with it, A/B)
static int sel_first() {
    static int v = -1;
    if (v < 0) {
        const char* e = getenv("MF_SEL_FIRST");
        v = (e && e[0] == '0') ? 0 : 1;
    }
    return v;
}

// k_vertex_tiers blocks per SM (MF_TIERS_PER_SM, A/B)
static int tiers_per_sm() {
    static int v = -1;
    if (v < 0) {
        const char* e = getenv("MF_TIERS_PER_SM");
        v = e ? std::max(1, atoi(e)) : 8;
    }
    return v;
}

// MF_SCAN_TICKET=1: every scan takes its tiles by ticket (A/B)
static bool scan_ticketless() {
    static int v = -1;
    if (v < 0) {
        const char* e = getenv("MF_SCAN_TICKET");
        v = (e && atoi(e) == 1) ? 0 : 1;
    }
    return v == 1;
}

template <typename LoadOp, typename Epi = EpiNone>
static void run_scan(ScanBuf& sb, LoadOp op, int* out, int n, cudaStream_t s, const char* name,
                     const int* abort_flag, Epi epi = Epi()) {
    const int tile = kScanBlock * ScanItems<LoadOp>::value;
    int tiles = std::max(1, (n + tile - 1) / tile);
    unsigned long long* st = sb.buf[sb.cur];
    unsigned long long* other = sb.buf[sb.cur ^ 1];
    // grids of at most 4 scan blocks per SM (of 8 resident) run all tiles at once: no ticket
    int* ticket = (scan_ticketless() && tiles <= sb.resident) ? nullptr : reinterpret_cast<int*>(st + tiles);
    prof_pre(name, s);
    rec_check(launch_ex(k_scan_excl<LoadOp, Epi>, dim3(tiles), dim3(kScanBlock), 0, s, op, n, out, st, ticket,
                        abort_flag, epi, other, sb.words),
              __LINE__);
    prof_post(name, s);
    g_launches++;
    sb.cur ^= 1;
}

// ------------------------------------------------------------------------
// plan: everything the host knows before touching the device
struct Plan {
    int64_t n = 0, m = 0, C = 3;
    bool alias = true;
    int fdtype = MF_DTYPE_F64;
    int B = 1, R = 0, first_err = 1, err_code = MF_OK;
    char err_msg[256] = {0};
    std::vector<int64_t> voff, foff;
    std::vector<std::vector<int64_t>> chains;
    std::vector<int> h_nin, h_act, h_budget, h_voff, h_N;
    int N0 = 0, M0 = 0, Nfin = 0, Mcap = 1, Ecap = 3, N1 = 0, nParamR = 1;
    bool seeded = false;
    int order = 0;
    uint64_t pcg[4] = {0, 0, 0, 0};
    size_t params_words = 0;
    int ld_min = kLDMinVertices;  // rounds with at least this many vertices start with LD rounds
    int ld1_min = 1 << 17;        // ... from this many, one LD round (measured: cfg4 1.07 -> 1.04 ms, cfg3
                                  // 2.97 -> 2.92; at cfg2 (115k) the two extra launches outweigh it)
    int ld_big = 4;               // LD rounds from ld_min (MF_LD_BIG; cfg5 13.06 -> 12.85 ms vs 12: the
                                  // frontier is small after 3-4 rounds and Suitor finishes it faster)
    int ld_mid = 2;               // LD rounds between ld1_min and ld_min (MF_LD_MID; cfg4 0.880 -> 0.865
                                  // ms with 2, 3 and 5 no better)
    int placement = 0;            // 0 = average, 1 = inverse (quadrics.py:89-114)
    // size gates of the kernel variants (env overrides force a branch at small sizes so the
    // parity tests reach it: MF_BIG_SEL_MIN / MF_SCAN4_MIN / MF_WIDE_MIN = 0 take it always)
    int big_sel_min = 1 << 18;    // one big mesh: multi-block selection passes before k_select
    int scan4_min = 1 << 20;      // 4-item tiles in the gather-chain scans (rep, keep)
    int wide_min = 1 << 21;       // output ids from here need the wide-key facet dedupe
};

static int make_plan(const mf_mesh_view* mv, const mf_decimate_config* cfg, Plan& p, mf_status* st) {
    p.n = mv->n;
    p.m = mv->m;
    if (cfg->placement != 0 && cfg->placement != 1) {
        st->code = MF_ERR_VALUE;
        snprintf(st->message, sizeof(st->message), "unknown placement %d", cfg->placement);
        return st->code;
    }
    p.placement = cfg->placement;
    if (p.n < 0 || p.m < 0 || p.n >= (int64_t)INT32_MAX - 1 || 6 * p.m >= (int64_t)INT32_MAX - 1) {  // edge ids: adjacency slots < 6m
        st->code = MF_ERR_LIMIT;
        snprintf(st->message, sizeof(st->message), "mesh too large for 32-bit device indices (n=%lld, m=%lld)",
                 (long long)p.n, (long long)p.m);
        return st->code;
    }
    // features omitted = a copy of the positions (mesh.py:28-29); their fold equals the position fold
    // only for 'average' placement, so 'inverse' carries them as a separate array
    p.alias = (mv->features == nullptr) && p.placement == 0;
    p.C = mv->features ? mv->c : 3;
    p.fdtype = mv->features ? mv->features_dtype : MF_DTYPE_F64;
    p.B = mv->vertex_offsets ? (int)mv->n_meshes : 1;
    const int B = p.B;
    p.voff.assign(B + 1, 0);
    p.foff.assign(B + 1, 0);
    if (mv->vertex_offsets) {
        for (int b = 0; b <= B; b++) {
            p.voff[b] = mv->vertex_offsets[b];
            p.foff[b] = mv->facet_offsets[b];
        }
        bool ok = p.voff[0] == 0 && p.foff[0] == 0 && p.voff[B] == p.n && p.foff[B] == p.m;
        for (int b = 0; b < B && ok; b++) ok = p.voff[b + 1] >= p.voff[b] && p.foff[b + 1] >= p.foff[b];
        if (!ok) {
            st->code = MF_ERR_STRUCTURAL;
            snprintf(st->message, sizeof(st->message), "vertex/facet offsets must be monotone from 0 to n/m");
            return st->code;
        }
    } else {
        p.voff[1] = p.n;
        p.foff[1] = p.m;
    }
    // per-mesh chains and host-side errors, in batch order (decimate.py:363-371)
    const int64_t target = cfg->target_vertices;
    p.first_err = B;
    p.chains.assign(B, {});
    for (int b = 0; b < B; b++) {
        int64_t nb = p.voff[b + 1] - p.voff[b], mb = p.foff[b + 1] - p.foff[b];
        if (target > nb) {
            p.err_code = MF_ERR_VALUE;
            snprintf(p.err_msg, sizeof(p.err_msg), "target_vertices=%lld exceeds the input size %lld",
                     (long long)target, (long long)nb);
        } else if (cfg->rounds == 0 || target == nb) {
            if (target != nb) {
                p.err_code = MF_ERR_VALUE;
                snprintf(p.err_msg, sizeof(p.err_msg), "rounds=0 requires target_vertices == input vertex count");
            }
        } else if (nb < 3 || mb < 1) {
            p.err_code = MF_ERR_STRUCTURAL;
            snprintf(p.err_msg, sizeof(p.err_msg),
                     "decimate_parallel requires a mesh with at least 3 vertices and 1 facet, got %lld vertices / "
                     "%lld facets",
                     (long long)nb, (long long)mb);
        } else {
            round_targets(nb, target, cfg->rounds, p.chains[b]);
        }
        if (p.err_code != MF_OK) {
            p.first_err = b;
            break;
        }
    }
    p.R = 0;
    for (int b = 0; b < p.first_err; b++) p.R = std::max(p.R, (int)p.chains[b].size());
    const int R = p.R;
    p.nParamR = std::max(R, 1);
    p.h_nin.assign((size_t)(R + 1) * B, 0);
    p.h_act.assign((size_t)p.nParamR * B, 0);
    p.h_budget.assign((size_t)p.nParamR * B, 0);
    p.h_voff.assign((size_t)(R + 1) * (B + 1), 0);
    for (int b = 0; b < B; b++) p.h_nin[b] = (int)(p.voff[b + 1] - p.voff[b]);
    for (int r = 0; r < R; r++)
        for (int b = 0; b < B; b++) {
            int nin = p.h_nin[(size_t)r * B + b];
            // a round whose target is its input size is _identity_result (decimate.py:231-233):
            // bypassed like a finished chain (positions and facets verbatim) -- run as a
            // zero-budget round it would move 'inverse' singletons to their optimal positions
            bool a = b < p.first_err && r < (int)p.chains[b].size() && p.chains[b][r] != nin;
            p.h_act[(size_t)r * B + b] = a;
            int tgt = a ? (int)p.chains[b][r] : nin;
            p.h_budget[(size_t)r * B + b] = nin - tgt;
            p.h_nin[(size_t)(r + 1) * B + b] = tgt;
        }
    for (int r = 0; r <= R; r++) {
        int acc = 0;
        for (int b = 0; b < B; b++) {
            acc += p.h_nin[(size_t)r * B + b];
            p.h_voff[(size_t)r * (B + 1) + b + 1] = acc;
        }
    }
    p.h_N.assign(R + 1, 0);
    for (int r = 0; r <= R; r++) p.h_N[r] = p.h_voff[(size_t)r * (B + 1) + B];
    p.N0 = (int)p.n;
    p.M0 = (int)p.m;
    p.Nfin = p.h_N[R];
    p.Mcap = std::max(p.M0, 1);
    p.Ecap = 3 * p.Mcap;
    p.N1 = R > 0 ? p.h_N[1] : p.N0;
    p.seeded = cfg->seeded != 0;
    p.order = cfg->einsum_order;
    if (const char* e = getenv("MF_LD_MIN")) p.ld_min = atoi(e);
    if (const char* e = getenv("MF_LD1_MIN")) p.ld1_min = atoi(e);
    if (const char* e = getenv("MF_LD_MID")) p.ld_mid = std::max(1, std::min(kLDRounds, atoi(e)));
    if (const char* e = getenv("MF_LD_BIG")) p.ld_big = std::max(1, std::min(kLDRounds, atoi(e)));
    if (const char* e = getenv("MF_BIG_SEL_MIN")) p.big_sel_min = std::max(0, atoi(e));
    if (const char* e = getenv("MF_SCAN4_MIN")) p.scan4_min = std::max(0, atoi(e));
    if (const char* e = getenv("MF_WIDE_MIN")) p.wide_min = std::max(0, atoi(e));
    for (int i = 0; i < 4; i++) p.pcg[i] = cfg->pcg_state[i];
    // device params: act | budget | nin | voff | foff0 (int32)
    p.params_words = (size_t)p.nParamR * B * 2 + (size_t)(R + 1) * B + (size_t)(R + 1) * (B + 1) + (B + 1);
    return MF_OK;
}

// ------------------------------------------------------------------------
// workspace
struct WS {
    int* params;
    int64_t *vo64, *fo64, *F64;
    float* Xf32;
    int* F0;
    double *P0, *X0, *Pa, *Pb, *Xa, *Xb, *Pfin, *Xfin;
    int *Fa, *Fb, *Ffin, *rt, *mt;
    int *foff_a, *foff_b;
    int* vmesh;
    Plane* plane;
    int *deg, *inc_off, *cursor, *inc, *inc_tmp;
    double* vq;
    unsigned* adj_k32;
    int* acur;
    int* snbr;    // adjacency slots in rank order (k_adj_rank output; nbr keeps neighbour order)
    int* seid_u;  // unseeded: edge ids of the unsorted slots (their neighbours / keys are e1 / key_hi)
    int* lowfill;
    unsigned long long* suitor;
    int *bestu, *front0, *front1, *ldc, *loose;
    unsigned* bar;
    int* selstate;
    int* ghist;
    int *nbr, *nbr_tmp, *adj_eid, *ucnt, *upcnt, *eoff, *aoff, *heavy, *mid, *counters, *e0, *e1;
    double* cost;
    uint64_t *key_hi, *key_lo;
    unsigned long long *mlo, *mhi;
    int *mate, *best, *pairlo;
    uint64_t *chi, *clo;
    int *cpay, *caux, *ksel, *mode;
    uint64_t *p_hi, *p_lo;
    int *segA, *segB, *removed, *absorbed, *minrep, *anchor, *outidx, *rstep, *ccount, *coff, *cmem, *repv, *abshead, *absnext;
    unsigned char* has_live;
    int* mapped;
    int4* canon;
    int *slot, *kout;
    unsigned tsize;
    int* table;
    unsigned long long* tkey;
    ScanBuf scan;
    unsigned long long* vs;  // k_vertex_scan look-back buffers (two, alternating by round)
    int vs_words;
    int* status;  // [8] flags | foff_final[B+1] | fail[3B] | stats[4R]
    size_t status_words, params_pad, status_pad, upload_bytes;
};

// memcmp(a, b, bytes) != 0, split over host threads above 8 MB
static bool host_differ(const void* a, const void* b, size_t bytes) {
    const size_t chunk = (size_t)8 << 20;
    unsigned hw = std::thread::hardware_concurrency();
    size_t T = std::min<size_t>(std::min<unsigned>(hw ? hw : 1, 16), (bytes + chunk - 1) / chunk);
    if (T <= 1) return memcmp(a, b, bytes) != 0;
    std::vector<std::thread> th;
    std::vector<char> diff(T, 0);
    const size_t per = (bytes + T - 1) / T;
    for (size_t t = 0; t < T; t++)
        th.emplace_back([&, t]() {
            const size_t o = t * per, e = std::min(bytes, o + per);
            if (o < e) diff[t] = memcmp((const char*)a + o, (const char*)b + o, e - o) != 0;
        });
    bool d = false;
    for (size_t t = 0; t < T; t++) {
        th[t].join();
        d = d || diff[t];
    }
    return d;
}

static void layout(Arena& A, WS& W, const Plan& p) {
    const int B = p.B, R = p.R, N0 = p.N0, N1 = p.N1, Mcap = p.Mcap, Ecap = p.Ecap, Nfin = p.Nfin;
    const int64_t C = p.C;
    const bool alias = p.alias;
    // one upload block: params | initial status words | vertex / facet offsets (int64)
    W.status_words = 8 + (size_t)(B + 1) + 3 * (size_t)B + 4 * (size_t)std::max(R, 1);
    W.params_pad = (p.params_words + 63) & ~size_t(63);
    W.status_pad = (W.status_words + 63) & ~size_t(63);
    W.upload_bytes = (W.params_pad + W.status_pad) * 4 + (size_t)2 * (B + 1) * 8;
    W.params = A.take<int>(W.upload_bytes / 4);
    W.status = W.params ? W.params + W.params_pad : nullptr;
    W.vo64 = W.params ? reinterpret_cast<int64_t*>(W.status + W.status_pad) : nullptr;
    W.fo64 = W.vo64 ? W.vo64 + (B + 1) : nullptr;
    W.F64 = A.take<int64_t>((size_t)Mcap * 3);
    W.Xf32 = (!alias && p.fdtype == MF_DTYPE_F32) ? A.take<float>((size_t)N0 * C) : nullptr;
    W.F0 = A.take<int>((size_t)Mcap * 3);
    W.P0 = A.take<double>((size_t)N0 * 3);
    W.X0 = alias ? nullptr : A.take<double>((size_t)N0 * C);
    W.Pa = A.take<double>((size_t)N1 * 3);
    W.Pb = A.take<double>((size_t)N1 * 3);
    W.Xa = alias ? nullptr : A.take<double>((size_t)N1 * C);
    W.Xb = alias ? nullptr : A.take<double>((size_t)N1 * C);
    W.Pfin = A.take<double>((size_t)Nfin * 3);
    W.Xfin = alias ? nullptr : A.take<double>((size_t)Nfin * C);
    W.Fa = A.take<int>((size_t)Mcap * 3);
    W.Fb = A.take<int>((size_t)Mcap * 3);
    W.Ffin = A.take<int>((size_t)Mcap * 3);
    W.rt = A.take<int>((size_t)N0);
    W.mt = A.take<int>((size_t)N0);
    W.foff_a = A.take<int>((size_t)B + 1);
    W.foff_b = A.take<int>((size_t)B + 1);
    W.vmesh = (B > 1) ? A.take<int>((size_t)N0) : nullptr;
    W.plane = A.take<Plane>((size_t)Mcap);
    W.deg = A.take<int>((size_t)N0 + 1);
    W.inc_off = A.take<int>((size_t)N0 + 1);
    W.cursor = A.take<int>((size_t)N0 + 1);
    W.inc = A.take<int>((size_t)Ecap);
    W.inc_tmp = A.take<int>((size_t)Ecap);
    W.vq = A.take<double>((size_t)N0 * 10);
    W.nbr = A.take<int>((size_t)2 * Ecap);
    W.nbr_tmp = A.take<int>((size_t)2 * Ecap);
    W.adj_eid = A.take<int>((size_t)2 * Ecap);
    W.adj_k32 = A.take<unsigned>((size_t)2 * Ecap);
    W.acur = A.take<int>((size_t)N0);
    W.snbr = A.take<int>((size_t)2 * Ecap);
    W.seid_u = p.seeded ? nullptr : A.take<int>((size_t)2 * Ecap);
    W.lowfill = A.take<int>((size_t)N0 + 1);
    W.suitor = A.take<unsigned long long>((size_t)N0);
    W.bestu = A.take<int>((size_t)N0);
    W.front0 = A.take<int>((size_t)N0);
    W.front1 = A.take<int>((size_t)N0);
    W.loose = A.take<int>((size_t)N0);
    W.ldc = A.take<int>(8);  // [0..5] LD rounds, [6] unmatched vertices listed by k_mates
    W.bar = A.take<unsigned>(8);
    W.selstate = A.take<int>((size_t)2 * B);
    W.ghist = A.take<int>(kSelScratch);
    W.ucnt = A.take<int>((size_t)N0);
    W.upcnt = A.take<int>((size_t)N0);
    W.eoff = A.take<int>((size_t)N0 + 1);
    W.aoff = A.take<int>((size_t)N0 + 1);
    W.heavy = A.take<int>((size_t)N0);
    W.mid = A.take<int>((size_t)N0);
    W.counters = A.take<int>(64);
    // unseeded edge ids are adjacency slot indices (sparse in [0, 2E)) and e1 / key_hi are the
    // unsorted slot arrays (neighbour, rank key) of k_edges, e0 the slot owner; seeded ids dense
    W.e0 = A.take<int>((size_t)2 * Ecap);
    W.e1 = A.take<int>((size_t)2 * Ecap);
    W.cost = A.take<double>((size_t)Ecap);
    W.key_hi = A.take<uint64_t>((size_t)2 * Ecap);
    W.key_lo = p.seeded ? A.take<uint64_t>((size_t)Ecap) : nullptr;
    W.mlo = A.take<unsigned long long>((size_t)B);
    W.mhi = A.take<unsigned long long>((size_t)B);
    W.mate = A.take<int>((size_t)N0);
    W.pairlo = A.take<int>((size_t)N0);
    W.best = A.take<int>((size_t)N0);
    W.chi = A.take<uint64_t>((size_t)N0);
    W.clo = A.take<uint64_t>((size_t)N0);
    W.cpay = A.take<int>((size_t)N0);
    W.caux = A.take<int>((size_t)N0);
    W.ksel = A.take<int>((size_t)B);
    W.mode = A.take<int>((size_t)B);
    W.p_hi = A.take<uint64_t>((size_t)B);
    W.p_lo = A.take<uint64_t>((size_t)B);
    W.segA = A.take<int>((size_t)B);
    W.segB = A.take<int>((size_t)B);
    W.removed = A.take<int>((size_t)B);
    W.absorbed = A.take<int>((size_t)N0);
    W.minrep = A.take<int>((size_t)N0);
    W.anchor = A.take<int>((size_t)N0);
    W.outidx = A.take<int>((size_t)N0 + 1);
    W.rstep = A.take<int>((size_t)N0);
    W.ccount = A.take<int>((size_t)N0 + 1);
    W.coff = A.take<int>((size_t)N0 + 1);
    W.cmem = A.take<int>((size_t)N0);
    W.repv = A.take<int>((size_t)N0);
    W.abshead = A.take<int>((size_t)N0);
    W.absnext = A.take<int>((size_t)N0);
    W.has_live = A.take<unsigned char>((size_t)N0);
    W.mapped = A.take<int>((size_t)Mcap * 3);
    W.canon = A.take<int4>((size_t)Mcap);
    W.slot = A.take<int>((size_t)Mcap);
    W.kout = A.take<int>((size_t)Mcap + 1);
    W.tsize = 1u;
    while (W.tsize < (unsigned)(2 * Mcap)) W.tsize <<= 1;
    W.table = A.take<int>((size_t)W.tsize);
    W.tkey = A.take<unsigned long long>((size_t)W.tsize);
    size_t maxn = (size_t)std::max(N0, Mcap) + 1;
    W.scan.words = (int)(maxn / kScanTileMin + 4);
    W.scan.buf[0] = A.take<unsigned long long>((size_t)W.scan.words);
    W.scan.buf[1] = A.take<unsigned long long>((size_t)W.scan.words);
    W.scan.cur = 0;
    W.vs_words = (N0 + kVsTile - 1) / kVsTile + 8;  // per buffer: tile words + ticket
    W.vs = A.take<unsigned long long>((size_t)2 * W.vs_words);
}

// ------------------------------------------------------------------------
// the device sequence (captured into a graph); inputs already staged in W
// Device-driven control flow while capturing: stages whose work is decided on the
// device become conditional graph nodes (WHILE for the locally-dominant rounds and the
// multi-block selection passes, IF for the absorb stage), their bodies captured on
// dedicated streams (nesting depth 2).  A kernel of the chain sets each condition
// (cudaGraphSetConditional), so converged rounds, finished passes and unneeded stages
// cost no launches.  Off (nullptr streams) when not capturing or when profiling.
struct CondCapture {
    cudaStream_t body[2] = {nullptr, nullptr};
    cudaStream_t outer[2] = {nullptr, nullptr};
    cudaGraphNode_t node[2] = {nullptr, nullptr};
    int depth = 0;
    bool on() const { return body[0] != nullptr; }
    cudaGraphConditionalHandle handle(cudaStream_t s, unsigned dflt) {
        cudaStreamCaptureStatus st;
        cudaGraph_t g = nullptr;
        const cudaGraphNode_t* d = nullptr;
        size_t nd = 0;
        RC(cudaStreamGetCaptureInfo(s, &st, nullptr, &g, &d, &nd));
        cudaGraphConditionalHandle h = 0;
        RC(cudaGraphConditionalHandleCreate(&h, g, dflt, cudaGraphCondAssignDefault));
        return h;
    }
    // adds the conditional node after the capture frontier of `s`; returns the body stream
    cudaStream_t begin(cudaStream_t s, cudaGraphConditionalHandle h, cudaGraphConditionalNodeType type) {
        cudaStreamCaptureStatus st;
        cudaGraph_t g = nullptr;
        const cudaGraphNode_t* d = nullptr;
        size_t nd = 0;
        RC(cudaStreamGetCaptureInfo(s, &st, nullptr, &g, &d, &nd));
        cudaGraphNodeParams cp = {};
        cp.type = cudaGraphNodeTypeConditional;
        cp.conditional.handle = h;
        cp.conditional.type = type;
        cp.conditional.size = 1;
        RC(cudaGraphAddNode(&node[depth], g, d, nd, &cp));
        outer[depth] = s;
        cudaStream_t b = body[depth];
        RC(cudaStreamBeginCaptureToGraph(b, cp.conditional.phGraph_out[0], nullptr, nullptr, 0,
                                         cudaStreamCaptureModeThreadLocal));
        depth++;
        return b;
    }
    cudaStream_t end() {  // closes the innermost body; returns the stream that continues
        depth--;
        cudaGraph_t bg = nullptr;
        RC(cudaStreamEndCapture(body[depth], &bg));
        RC(cudaStreamUpdateCaptureDependencies(outer[depth], &node[depth], 1, cudaStreamSetCaptureDependencies));
        return outer[depth];
    }
};

// k_init_inputs of the recording: its arguments and (when captured) its graph node, so a replay
// can point it at the call's own input buffers; g_in_* = this call's inputs when they are device
// buffers the kernel may read in place (else the staging buffers W.F64 / W.P0)
thread_local InitArgs g_init_args;
thread_local int g_init_grid = 1;
thread_local cudaGraphNode_t g_init_node = nullptr;
thread_local const void* g_in_F64 = nullptr;
thread_local int g_in_f32 = 0;
thread_local const double* g_in_P = nullptr;

static void record(const Context* ctx, const Plan& p, WS& W, cudaStream_t stream, cudaStream_t body0 = nullptr,
                   cudaStream_t body1 = nullptr) {
    CondCapture cc;
    cc.body[0] = body0;
    cc.body[1] = body1;
    W.scan.resident = ctx->sm_count * 4;
    const int B = p.B, R = p.R, N0 = p.N0, Mcap = p.Mcap, Ecap = p.Ecap;
    const int64_t n = p.n, m = p.m, C = p.C;
    const bool seeded = p.seeded;
    int* d_abort = W.status;  // [0] abort, [1] bad facet, [2] bad position
    int* d_badf = W.status + 1;
    int* d_badp = W.status + 2;
    int* d_foff_fin = W.status + 8;
    int* d_fail = W.status + 8 + (B + 1);
    int* d_stats = d_fail + 3 * B;
    int* d_act = W.params;
    int* d_budget = W.params + (size_t)p.nParamR * B;
    int* d_nin = W.params + (size_t)p.nParamR * B * 2;
    int* d_voff = d_nin + (size_t)(R + 1) * B;
    int* d_foff0 = d_voff + (size_t)(R + 1) * (B + 1);

    g_pdl = true;
    {
        // status words arrive initialised with the params upload; the input pointers (caller
        // device buffers or the host staging) are patched into this node on every replay
        InitArgs ia{W.foff_a, d_foff0, B, W.deg, W.cursor, W.lowfill, N0 + 1, W.counters, W.scan.buf[0],
                    W.scan.buf[1], W.scan.words, W.ghist, kSelScratch, m,
                    g_in_F64 ? g_in_F64 : (const void*)W.F64, g_in_F64 ? g_in_f32 : 0, W.F0, W.vo64,
                    W.fo64, d_badf, 3 * n, g_in_P ? g_in_P : W.P0, W.P0, d_badp, W.vs, 2 * W.vs_words};
        const int grid = grid_for(ctx, std::max<int64_t>({(int64_t)N0 + 1, (int64_t)W.scan.words, m, 3 * n}));
        // launched by hand (not LAUNCH): its graph node is read back right after the launch,
        // before a profiling event node can follow it
        prof_pre("k_init_inputs", stream);
        rec_check(launch_ex(k_init_inputs, dim3(grid), dim3(256), 0, stream, ia), __LINE__);
        g_launches++;
        g_init_args = ia;
        g_init_grid = grid;
        g_init_node = nullptr;
        cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
        const cudaGraphNode_t* deps = nullptr;
        size_t nd = 0;
        if (cudaStreamGetCaptureInfo(stream, &cs, nullptr, nullptr, &deps, &nd) == cudaSuccess &&
            cs == cudaStreamCaptureStatusActive && nd == 1) {
            cudaGraphNodeType t;
            if (cudaGraphNodeGetType(deps[0], &t) == cudaSuccess && t == cudaGraphNodeTypeKernel) g_init_node = deps[0];
        }
        cudaGetLastError();
        prof_post("k_init_inputs", stream);
    }
    if (W.Xf32 && n * C > 0) LAUNCH(k_f32_to_f64, grid_for(ctx, n * C), 256, 0, stream, n * C, W.Xf32, W.X0);

    const double* Pc = W.P0;
    const double* Xc = p.alias ? nullptr : W.X0;
    const int* Fc = W.F0;
    int* foff_c = W.foff_a;
    int* foff_n = W.foff_b;
    const int order = p.order;
    int* d_heavy_n = W.counters + 4;
    int* d_heavy_c = W.counters + 12;
    int* d_mid_n = W.counters + 20;
    int* d_scratch_used = W.counters + 24;
    bool plane_done = false;  // this round's facet planes were computed by the previous round's epilogue
    for (int r = 0; r < R; r++) {
        const int N = p.h_N[r];
        const int Nn = p.h_N[r + 1];
        const int* act = d_act + (size_t)r * B;
        const int* budget = d_budget + (size_t)r * B;
        const int* nin = d_nin + (size_t)r * B;
        const int* voff_r = d_voff + (size_t)r * (B + 1);
        const int* dM = foff_c + B;
        const bool last = (r == R - 1);
        double* Pn = last ? W.Pfin : ((r & 1) ? W.Pb : W.Pa);
        double* Xn = p.alias ? nullptr : (last ? W.Xfin : ((r & 1) ? W.Xb : W.Xa));
        int* Fn = last ? W.Ffin : ((r & 1) ? W.Fb : W.Fa);
        int* vmesh = nullptr;
        if (B > 1) {
            vmesh = W.vmesh;
            LAUNCH(k_vmesh, grid_for(ctx, N), 256, 0, stream, d_abort, N, voff_r, B, vmesh);
        }
        // facet planes + incidence CSR (corner-major order)
        // large rounds recompute each facet's plane in the vertex fold instead of materialising
        // 32 bytes per facet (write + gather); the plane kernel then only counts degrees
        const bool recompute = N >= recompute_min() && vertex_scan() == 0;  // k_vertex_scan reads planes
        const PlaneSrc ps{recompute ? nullptr : W.plane, Fc, Pc, order};
        if (!plane_done)
            LAUNCH(k_facet_plane, grid_for(ctx, Mcap), 256, 0, stream, d_abort, Fc, Pc, dM, vmesh, act,
                   recompute ? nullptr : W.plane, W.deg, order);
        plane_done = false;
        run_scan(W.scan, LoadArr{W.deg}, W.inc_off, N, stream, "k_scan<deg>", d_abort);
        LAUNCH(k_inc_scatter, grid_for(ctx, Mcap), 256, 0, stream, d_abort, Fc, dM, Mcap, vmesh, act, W.inc_off, W.cursor,
               W.inc);
        // vertex quadrics + unique neighbour lists (+ the adjacency / edge offset scans)
        if (vertex_scan()) {
            unsigned long long* vs_cur = W.vs + (size_t)(r & 1) * W.vs_words;
            unsigned long long* vs_nxt = W.vs + (size_t)((r + 1) & 1) * W.vs_words;
            const int tiles = (N + kVsTile - 1) / kVsTile;
            VertexScanArgs va{d_abort, N, W.inc_off, W.inc, W.inc_tmp, Fc, ps, Mcap, W.vq, W.nbr, W.nbr_tmp,
                              W.ucnt, W.upcnt, W.aoff, seeded ? W.eoff : nullptr, vs_cur,
                              reinterpret_cast<int*>(vs_cur + W.vs_words - 4), last ? nullptr : vs_nxt,
                              last ? 0 : W.vs_words};
            const int vg = std::max(1, std::min(tiles, ctx->sm_count * 16));
            if (vertex_scan() == 2) LAUNCH(k_vertex_scan<256>, vg, 256, 0, stream, va);
            else LAUNCH(k_vertex_scan<128>, vg, 128, 0, stream, va);
        } else {
            const bool t16 = vt16(N);
            auto* vt = t16 ? (recompute ? k_vertex_t<16, true> : k_vertex_t<16, false>)
                           : (recompute ? k_vertex_t<8, true> : k_vertex_t<8, false>);
            LAUNCH_AS(t16 ? "k_vertex_t<16>" : "k_vertex_t<8>", vt, grid_for(ctx, N, 128), 128, 0, stream, d_abort,
                      N, W.inc_off, W.inc, Fc, ps, Mcap, W.vq, W.nbr, W.ucnt, W.upcnt, W.mid, d_mid_n, W.heavy,
                      d_heavy_n);
            LAUNCH_AS("k_vertex_tiers", recompute ? k_vertex_tiers<true> : k_vertex_tiers<false>,
                      ctx->sm_count * tiers_per_sm(),
                      256, 0, stream, d_abort, W.mid, d_mid_n, W.heavy, d_heavy_n, W.inc_off, W.inc, W.inc_tmp, Fc,
                      ps, Mcap, W.vq, W.nbr, W.nbr_tmp, W.ucnt, W.upcnt);
            // compact adjacency offsets (2 slots per edge); seeded rounds also need the dense
            // lexicographic edge index (the PCG64 key-stream position, decimate.py:190)
            run_scan(W.scan, LoadArr{W.ucnt}, W.aoff, N, stream, "k_scan<adj>", d_abort);
            if (seeded) run_scan(W.scan, LoadArr{W.upcnt}, W.eoff, N, stream, "k_scan<edges>", d_abort);
        }
        const int ld_rounds = N >= p.ld_min ? p.ld_big : (N >= p.ld1_min ? p.ld_mid : 0);
        const bool use_ld = ld_rounds > 0;
        const bool fused_rank = !seeded && edges_rank();
        // unseeded large rounds: edge arrays only, then k_adj_build (no lower-slot atomics / re-sort)
        const bool two_pass = !seeded && !fused_rank && N >= two_pass_min();
        if (fused_rank) {  // edges + costs + rank-ordered adjacency in one pass (k_edges_rank)
            EdgeRankOut ro{W.e0,   W.e1,       W.key_hi, W.snbr,    W.adj_eid, W.adj_k32, W.acur,
                           use_ld ? W.best : nullptr, W.bestu, W.mate, W.minrep, W.absorbed, W.abshead,
                           W.suitor, W.mlo, W.mhi, W.segA, W.ldc, W.segB};
            const int eg = grid_for(ctx, (int64_t)N * 8);
            if (p.placement)
                LAUNCH(k_edges_rank<1>, eg, 256, 0, stream, d_abort, N, W.inc_off, W.nbr, W.ucnt, W.aoff, W.vq, Pc, ro,
                       order, B);
            else
                LAUNCH(k_edges_rank<0>, eg, 256, 0, stream, d_abort, N, W.inc_off, W.nbr, W.ucnt, W.aoff, W.vq, Pc, ro,
                       order, B);
        } else {
            // unseeded: the unsorted slots are written straight into e1 / key_hi (+ seid_u), and
            // k_adj_rank_tiled sorts them out of place into snbr / adj_eid / adj_k32
            EdgeOut eo{W.e0,      W.e1,   seeded ? W.cost : nullptr, nullptr, seeded ? W.snbr : W.e1,
                       seeded ? W.adj_eid : W.seid_u, seeded ? nullptr : W.key_hi,
                       W.lowfill, W.mate, W.minrep, W.absorbed, W.abshead, W.suitor, W.mlo, W.mhi,
                       W.segA,    W.ldc,  W.segB, two_pass ? 1 : 0};
            const int eg = grid_for(ctx, (int64_t)N * kEdgeLanes);
            if (p.placement)
                LAUNCH(k_edges<1>, eg, 256, 0, stream, d_abort, N, W.inc_off, W.nbr, W.ucnt, W.upcnt, W.aoff, W.eoff, W.vq,
                       Pc, eo, order, B);
            else
                LAUNCH(k_edges<0>, eg, 256, 0, stream, d_abort, N, W.inc_off, W.nbr, W.ucnt, W.upcnt, W.aoff, W.eoff, W.vq,
                       Pc, eo, order, B);
        }
        const int* dE = W.eoff + N;
        if (seeded) {
            LAUNCH(k_cost_minmax, grid_for(ctx, Ecap), 256, 0, stream, d_abort, dE, W.cost, W.e0, vmesh, W.mlo, W.mhi);
            LAUNCH(k_seed_keys, grid_for(ctx, (Ecap + kSeedRun - 1) / kSeedRun), 256, 0, stream, d_abort, dE, W.cost, W.e0,
                   vmesh, W.eoff, voff_r, W.mlo, W.mhi, p.pcg[0], p.pcg[1], p.pcg[2], p.pcg[3], W.key_hi, W.key_lo);
        }
        // large meshes: locally-dominant rounds first (round 0's picks written by k_adj_rank /
        // k_edges_rank), then Suitor proposals on the residual frontier; smaller meshes: Suitor only
        if (fused_rank) {
        } else if (two_pass)
            LAUNCH(k_adj_build, grid_for(ctx, N), 256, 0, stream, d_abort, N, W.inc_off, W.nbr, W.ucnt, W.upcnt, W.aoff,
                   W.key_hi, W.snbr, W.adj_eid, W.adj_k32, W.acur, use_ld ? W.best : nullptr, W.bestu);
        else if (seeded)
            LAUNCH(k_adj_rank<true>, grid_for(ctx, N), 256, 0, stream, d_abort, N, W.aoff, W.ucnt, W.snbr, W.adj_eid,
                   nullptr, W.key_hi, W.key_lo, W.adj_k32, W.acur, use_ld ? W.best : nullptr, W.bestu);
        else
            LAUNCH(k_adj_rank_tiled, std::min(grid_for(ctx, N), ctx->sm_count * 3), 256, kRankSmem, stream, d_abort, N, W.aoff, W.ucnt, W.e1, W.seid_u,
                   W.key_hi, W.snbr, W.adj_eid, W.adj_k32, W.acur, use_ld ? W.best : nullptr, W.bestu);
        if (use_ld) {
            LDArgs la{N, W.aoff, W.ucnt, W.snbr, W.adj_eid, W.adj_k32, W.key_hi, seeded ? W.key_lo : nullptr,
                      W.mate, W.best, W.bestu, W.front0, W.front1, W.ldc, W.bar, ld_rounds, d_abort, W.acur, 0};
            LAUNCH(k_ld_init, grid_for(ctx, N), 256, 0, stream, la);
            if (cc.on() && ld_rounds > 1) {  // as many rounds as the frontier needs (WHILE node)
                la.cond = cc.handle(stream, 1u);
                stream = cc.begin(stream, la.cond, cudaGraphCondTypeWhile);
                LAUNCH(k_ld_pick, grid_for(ctx, N), 256, 0, stream, la, -1);
                LAUNCH(k_ld_match, grid_for(ctx, N), 256, 0, stream, la, -1);
                stream = cc.end();
            } else {
                for (int round = 0; round < ld_rounds; round++) {
                    if (round > 0) LAUNCH(k_ld_pick, grid_for(ctx, N), 256, 0, stream, la, round);
                    LAUNCH(k_ld_match, grid_for(ctx, N), 256, 0, stream, la, round);
                }
            }
        }
        {
            MatchArgs ma{N, W.aoff, W.ucnt, W.snbr, W.adj_eid, W.adj_k32, W.e0, W.e1, W.key_hi,
                         seeded ? W.key_lo : nullptr, W.suitor, d_abort, use_ld ? W.mate : nullptr,
                         use_ld ? W.front0 : nullptr, W.front1, W.ldc, W.acur};
            const int sl = suitor_lanes(N, ctx->sm_count);
            auto sg = [&](int lanes) {  // MF_SUITOR_BPSM=k: at most k blocks per SM (grid-stride), A/B
                const int g = grid_for(ctx, (int64_t)N * lanes);
                return suitor_bpsm() > 0 ? std::min(g, ctx->sm_count * suitor_bpsm()) : g;
            };
            if (sl == 8) LAUNCH(k_suitor<8>, sg(8), 256, 0, stream, ma);
            else if (sl == 4) LAUNCH(k_suitor<4>, sg(4), 256, 0, stream, ma);
            else if (sl == 2) LAUNCH(k_suitor<2>, sg(2), 256, 0, stream, ma);
            else LAUNCH(k_suitor1, grid_for(ctx, N), 256, 0, stream, ma);
        }
        LAUNCH(k_mates, grid_for(ctx, N), 256, 0, stream, d_abort, N, W.suitor, W.e0, W.e1, W.mate, W.key_hi,
               seeded ? W.key_lo : nullptr, vmesh, voff_r, W.segA, W.chi, W.clo, W.cpay, W.pairlo, W.loose, W.ldc + 6);
        // per-mesh selection; one big mesh first narrows its rank prefix with multi-block passes
        const bool big = (B == 1 && N >= p.big_sel_min);  // below: one CTA (latency-bound sizes)
        auto select = [&](const int* seg_cnt, const int* removed_in) {
            SelectArgs sa{W.chi, W.clo, seg_cnt, voff_r, B, act, budget, removed_in, W.ksel, W.mode, W.p_hi, W.p_lo,
                          d_abort, W.selstate, W.selstate + B, 0, W.ghist, select_cap(), 0,
                          B == 1 ? kSelChiCap : 0, sel_bulk(), sel_first()};
            if (big) {
                const int hist_grid = std::min(grid_for(ctx, N / 2, 512), ctx->sm_count * 2);
                if (cc.on() && cc.depth < 2) {  // passes until decided / handed over (WHILE node)
                    sa.cond = cc.handle(stream, 1u);
                    stream = cc.begin(stream, sa.cond, cudaGraphCondTypeWhile);
                    LAUNCH(k_sel_hist, hist_grid, 512, 0, stream, sa, W.ghist, -1);
                    LAUNCH(k_sel_decide, 1, kSelThreads, 0, stream, sa, W.ghist, -1);
                    stream = cc.end();
                    sa.cond = 0;
                } else {
                    for (int pass = 0; pass < sel_passes(); pass++) {
                        LAUNCH(k_sel_hist, hist_grid, 512, 0, stream, sa, W.ghist, pass);
                        LAUNCH(k_sel_decide, 1, kSelThreads, 0, stream, sa, W.ghist, pass);
                    }
                }
                sa.resume = 1;
            }
            if (B == 1 && !big && select_cluster()) LAUNCH(k_select_cl, kClCTAs, kClThreads, kClSmem, stream, sa);
            else if (B == 1)
                LAUNCH(k_select<1024>, 1, 1024, kSelBins * 4 + 8 * std::max(2 * sa.cap, sa.chicap), stream, sa);
            else
                LAUNCH(k_select<512>, std::min(B, ctx->sm_count * 2), 512,
                       kSelBins * 4 + 8 * std::max(2 * sa.cap, sa.chicap), stream, sa);
        };
        // budget truncation: keep the `budget` lowest-ranked matched pairs per mesh
        select(W.segA, nullptr);
        // the absorb stage runs only when some mesh misses its budget after truncation (IF node,
        // condition set by k_trunc_apply); skipping it leaves removed / absorbed as they are
        const cudaGraphConditionalHandle absorb_cond = cc.on() ? cc.handle(stream, 1u) : 0;
        // truncation + absorb candidates (one pass is exact: the matching is maximal when the
        // budget is unmet), one launch: they act on disjoint meshes
        {
            TruncArgs ta{N,    vmesh,  voff_r, W.segA,    W.chi,     W.clo,    W.cpay,   W.mode, W.p_hi, W.p_lo,
                         W.e0, W.e1,   W.mate, B,         W.ksel,    W.removed, W.segB,  W.pairlo, act,  budget,
                         absorb_cond};
            AbsorbArgs aa{W.loose, W.ldc + 6, W.aoff, W.ucnt, W.snbr, W.adj_eid, seeded ? W.cost : nullptr, W.key_hi,
                          W.pairlo, vmesh, voff_r, act, budget, W.ksel, W.segB, W.chi, W.clo, W.caux};
            LAUNCH(k_trunc_absorb, grid_for(ctx, N), 256, 0, stream, d_abort, ta, aa);
        }
        if (absorb_cond) stream = cc.begin(stream, absorb_cond, cudaGraphCondTypeIf);
        select(W.segB, W.removed);
        RoundFail rf{d_abort, d_fail, d_fail + B, d_fail + 2 * B};
        LAUNCH(k_absorb_apply, grid_for(ctx, N), 256, 0, stream, N, vmesh, voff_r, W.segB, W.chi, W.clo, W.caux,
               W.mode, W.p_hi, W.p_lo, W.absorbed, W.minrep, B, act, budget, nin, W.ksel, W.removed, W.aoff, rf, r);
        if (absorb_cond) stream = cc.end();
        // relabel: output index = rank of the cluster's lowest member
        if (N >= p.scan4_min)  // 4-item tiles for large rounds (cfg5 0.27 -> 0.20 ms)
            run_scan(W.scan, LoadIsRepT<4>{W.pairlo, W.absorbed, W.minrep}, W.outidx, N, stream, "k_scan<rep>",
                     d_abort);
        else
            run_scan(W.scan, LoadIsRep{W.pairlo, W.absorbed, W.minrep}, W.outidx, N, stream, "k_scan<rep>", d_abort);
        const bool packed = Nn < p.wide_min;
        LAUNCH(k_relabel3, grid_for(ctx, std::max<int64_t>(N, W.tsize)), 256, 0, stream, N, d_abort, W.pairlo,
               W.absorbed, W.minrep, W.outidx, W.rstep, W.repv, W.abshead, W.absnext, W.table,
               packed ? W.tkey : nullptr, (int)W.tsize, packed ? 0x7f7f7f7f : -1, W.has_live, W.deg, W.cursor,
               W.lowfill, last ? 0 : Nn + 1);
        // contraction over member lists (no cluster CSR needed)
        // the heavy-cluster tier runs in k_contract's last block (counters[30] = finished blocks)
        if (p.placement)
            LAUNCH(k_contract<1>, grid_for(ctx, Nn), 256, 0, stream, Nn, d_abort, W.repv, W.mate, W.pairlo, W.e1,
                   W.absorbed, W.abshead, W.absnext, vmesh, act, Pc, Xc, (int)C, Pn, Xn, W.vq, W.heavy, d_heavy_c,
                   W.cmem, W.best, d_scratch_used, W.counters + 30);
        else
            LAUNCH(k_contract<0>, grid_for(ctx, Nn), 256, 0, stream, Nn, d_abort, W.repv, W.mate, W.pairlo, W.e1,
                   W.absorbed, W.abshead, W.absnext, vmesh, act, Pc, Xc, (int)C, Pn, Xn, W.vq, W.heavy, d_heavy_c,
                   W.cmem, W.best, d_scratch_used, W.counters + 30);
        // output facets: remap, drop degenerate, drop later duplicates (hash, min facet id wins)
        {
            const unsigned per_vertex = std::max(1u, W.tsize / (unsigned)std::max(Nn, 1));
            if (packed)
                LAUNCH(k_facet_remap<true>, grid_for(ctx, Mcap), 256, 0, stream, dM, d_abort, Fc, W.rstep, vmesh, act,
                       W.mapped, W.canon, W.slot, W.has_live, W.table, W.tkey, W.tsize - 1, per_vertex);
            else
                LAUNCH(k_facet_remap<false>, grid_for(ctx, Mcap), 256, 0, stream, dM, d_abort, Fc, W.rstep, vmesh,
                       act, W.mapped, W.canon, W.slot, W.has_live, W.table, W.tkey, W.tsize - 1, per_vertex);
        }
        // keep scan: 2-item tiles for latency-bound sizes, longer ones for large meshes (cfg5 0.64 -> 0.61 ms)
        if (Mcap >= p.scan4_min)  // (8-item tiles: 0.78 ms)
            run_scan(W.scan, LoadKeepT<4>{dM, W.slot, W.table}, W.kout, Mcap, stream, "k_scan<keep>", d_abort,
                     EpiFacetWrite{W.mapped, Fn});
        else
            run_scan(W.scan, LoadKeep{dM, W.slot, W.table}, W.kout, Mcap, stream, "k_scan<keep>", d_abort,
                     EpiFacetWrite{W.mapped, Fn});
        if (B == 1 && !last && fuse_plane()) {  // + the next round's facet planes, one launch
            LAUNCH(k_compose_plane, grid_for(ctx, std::max<int64_t>(N0, Mcap)), 256, 0, stream, N0, d_abort, W.rstep,
                   W.inc_off, W.has_live, act, W.rt, W.mt, r == 0, W.kout, foff_c, foff_n, d_stats + 4 * r,
                   W.aoff + N, W.ldc + 2, W.counters, Fn, Pn, d_act + (size_t)(r + 1) * B,
                   (Nn >= recompute_min() && vertex_scan() == 0) ? nullptr : W.plane, W.deg, order);
            plane_done = true;
        } else {
            LAUNCH(k_compose, grid_for(ctx, N0), 256, 0, stream, N0, d_abort, W.rstep, W.inc_off, W.has_live, vmesh,
                   act, W.rt, W.mt, r == 0, B, W.kout, foff_c, foff_n, last ? d_foff_fin : nullptr, d_stats + 4 * r,
                   W.aoff + N, W.ldc + 2, W.counters);
        }
        Pc = Pn;
        Xc = Xn;
        Fc = Fn;
        std::swap(foff_c, foff_n);
    }
    g_pdl = false;
}

// ------------------------------------------------------------------------
// graph cache (per context): key = every host value baked into the sequence
struct GraphEntry {
    cudaGraphExec_t exec = nullptr;
    cudaGraph_t graph = nullptr;  // kept alive: node updates address its nodes
    std::vector<ProfRec> prof;
    int64_t kernels = 0;  // kernel nodes (launch accounting on replay)
    cudaGraphNode_t init_node = nullptr;  // k_init_inputs (its input pointers change per call)
    InitArgs init_args;
    int init_grid = 1;
};
struct GraphCache {
    std::map<std::vector<int64_t>, GraphEntry> entries;
    void* arena = nullptr;
    cudaStream_t capture = nullptr;
    cudaStream_t body[2] = {nullptr, nullptr};  // conditional-node body captures
    ~GraphCache() { clear(); }
    void clear() {
        for (auto& kv : entries) {
            if (kv.second.exec) cudaGraphExecDestroy(kv.second.exec);
            if (kv.second.graph) cudaGraphDestroy(kv.second.graph);
        }
        entries.clear();
    }
};
static std::map<const Context*, GraphCache>& caches() {
    static thread_local std::map<const Context*, GraphCache> c;
    return c;
}
void drop_graphs(const Context* ctx) {
    auto& c = caches();
    auto it = c.find(ctx);
    if (it != c.end()) {
        if (it->second.capture) cudaStreamDestroy(it->second.capture);
        for (cudaStream_t b : it->second.body)
            if (b) cudaStreamDestroy(b);
        c.erase(it);
    }
}

static std::vector<int64_t> graph_key(const Plan& p) {
    std::vector<int64_t> k = {p.n, p.m, p.C, p.alias, p.fdtype, p.B, p.R, p.seeded, p.order, p.first_err,
                              (int64_t)p.pcg[0], (int64_t)p.pcg[1], (int64_t)p.pcg[2], (int64_t)p.pcg[3],
                              g_prof_mode, p.ld_min, p.ld1_min, p.ld_mid, p.ld_big, p.placement, fuse_plane(), vertex_scan(), edges_rank(),
                              vt16(1), vt16(1 << 21), two_pass_min(), recompute_min(), scan_ticketless(), tiers_per_sm(), sel_bulk(), sel_first(), suitor_bpsm(),
                              p.big_sel_min, p.scan4_min, p.wide_min};
    k.insert(k.end(), p.h_N.begin(), p.h_N.end());
    for (char ch : g_prof_only) k.push_back(ch);
    return k;
}

static bool use_graphs() {
    static int v = -1;
    if (v < 0) {
        const char* e = getenv("MF_GRAPHS");
        v = (e && e[0] == '0') ? 0 : 1;
    }
    return v == 1;
}

// ------------------------------------------------------------------------
// quality_report errors (decimate.py:580-602): the ORIGINAL mesh's vertex
// quadrics through the round kernels (facet planes, corner-major incidence
// CSR, ordered fold), then the cluster fold + evaluation (k_quality).
// d_off / d_mem: cluster CSR of replace over the original vertices.
int quality_run(Context* ctx, const mf_mesh_view* mv, const int* d_off, const int* d_mem, int64_t n_out,
                const double* positions_out, int order, double* errors, cudaStream_t stream, mf_status* st) {
    const int64_t n = mv->n, m = mv->m;
    if (n >= (int64_t)INT32_MAX - 1 || 6 * m >= (int64_t)INT32_MAX - 1) {
        st->code = MF_ERR_LIMIT;
        snprintf(st->message, sizeof(st->message), "mesh too large for 32-bit device indices");
        return st->code;
    }
    const int N = (int)n, Mc = (int)std::max<int64_t>(m, 1);
    const int scan_words = (int)((std::max<int64_t>(n, 1) + 1) / kScanTileMin + 4);
    Arena me;
    me.measuring = true;
    auto lay = [&](Arena& A, WS& W, int64_t*& vo, double*& Pin, double*& Pout, double*& err, int*& misc) {
        misc = A.take<int>(64);  // [0] abort [1] bad facet [2] m [3] act [8..] counters
        vo = A.take<int64_t>(4);
        W.F64 = A.take<int64_t>((size_t)Mc * 3);
        W.F0 = A.take<int>((size_t)Mc * 3);
        Pin = A.take<double>((size_t)std::max<int64_t>(n, 1) * 3);
        Pout = A.take<double>((size_t)std::max<int64_t>(n_out, 1) * 3);
        err = A.take<double>((size_t)std::max<int64_t>(n_out, 1));
        W.plane = A.take<Plane>((size_t)Mc);
        W.deg = A.take<int>((size_t)N + 1);
        W.inc_off = A.take<int>((size_t)N + 1);
        W.cursor = A.take<int>((size_t)N + 1);
        W.inc = A.take<int>((size_t)Mc * 3);
        W.inc_tmp = A.take<int>((size_t)Mc * 3);
        W.vq = A.take<double>((size_t)std::max(N, 1) * 10);
        W.nbr = A.take<int>((size_t)Mc * 6);
        W.nbr_tmp = A.take<int>((size_t)Mc * 6);
        W.ucnt = A.take<int>((size_t)N + 1);
        W.upcnt = A.take<int>((size_t)N + 1);
        W.heavy = A.take<int>((size_t)N + 1);
        W.mid = A.take<int>((size_t)N + 1);
        W.scan.words = scan_words;
        W.scan.buf[0] = A.take<unsigned long long>((size_t)scan_words);
        W.scan.buf[1] = A.take<unsigned long long>((size_t)scan_words);
    };
    WS W;
    int64_t* d_vo;
    double *d_P, *d_Pout, *d_err;
    int* misc;
    lay(me, W, d_vo, d_P, d_Pout, d_err, misc);
    void* block = nullptr;
    MF_CUDA_TRY(cudaMallocAsync(&block, me.off, stream));
    Arena A;
    A.base = (char*)block;
    A.cap = me.off;
    lay(A, W, d_vo, d_P, d_Pout, d_err, misc);
    int rc = MF_OK;
    int h_misc[4] = {0, 0x7f7f7f7f, (int)m, 1};
    int64_t h_vo[4] = {0, n, 0, m};
    auto fail = [&](cudaError_t e) {
        st->code = rc = MF_ERR_CUDA;
        snprintf(st->message, sizeof(st->message), "%s", cudaGetErrorString(e));
    };
    cudaError_t e = cudaSuccess;
#define QTRY(x)                               \
    do {                                      \
        if ((e = (x)) != cudaSuccess) {       \
            fail(e);                          \
            goto done;                        \
        }                                     \
    } while (0)
    QTRY(cudaMemsetAsync(misc, 0, 64 * sizeof(int), stream));
    QTRY(cudaMemcpyAsync(misc, h_misc, sizeof(h_misc), cudaMemcpyHostToDevice, stream));
    QTRY(cudaMemcpyAsync(d_vo, h_vo, sizeof(h_vo), cudaMemcpyHostToDevice, stream));
    QTRY(cudaMemsetAsync(W.deg, 0, ((size_t)N + 1) * 4, stream));
    QTRY(cudaMemsetAsync(W.cursor, 0, ((size_t)N + 1) * 4, stream));
    QTRY(cudaMemsetAsync(W.scan.buf[0], 0, (size_t)scan_words * 8, stream));
    QTRY(cudaMemsetAsync(W.scan.buf[1], 0, (size_t)scan_words * 8, stream));
    if (n) QTRY(cudaMemcpyAsync(d_P, mv->positions, (size_t)n * 24, cudaMemcpyDefault, stream));
    if (n_out) QTRY(cudaMemcpyAsync(d_Pout, positions_out, (size_t)n_out * 24, cudaMemcpyDefault, stream));
    if (m) {
        QTRY(cudaMemcpyAsync(W.F64, mv->facets, (size_t)m * 24, cudaMemcpyDefault, stream));
        LAUNCH(k_facets_in, grid_for(ctx, m), 256, 0, stream, m, W.F64, W.F0, 1, d_vo, d_vo + 2, misc + 1);
        LAUNCH(k_facet_plane, grid_for(ctx, m), 256, 0, stream, misc, W.F0, d_P, misc + 2, (const int*)nullptr,
               misc + 3, W.plane, W.deg, order);
    }
    if (n) {
        run_scan(W.scan, LoadArr{W.deg}, W.inc_off, N, stream, "k_scan<deg>", misc);
        if (m) LAUNCH(k_inc_scatter, grid_for(ctx, m), 256, 0, stream, misc, W.F0, misc + 2, Mc, (const int*)nullptr,
                      misc + 3, W.inc_off, W.cursor, W.inc);
        LAUNCH_AS("k_vertex_t<8>", (k_vertex_t<8, false>), grid_for(ctx, N, 128), 128, 0, stream, misc, N,
                  W.inc_off, W.inc, W.F0, PlaneSrc{W.plane, W.F0, d_P, order}, Mc, W.vq, W.nbr, W.ucnt, W.upcnt,
                  W.mid, misc + 12, W.heavy, misc + 8);
        LAUNCH(k_vertex_tiers<false>, ctx->sm_count * 8, 256, 0, stream, misc, W.mid, misc + 12, W.heavy, misc + 8,
               W.inc_off, W.inc, W.inc_tmp, W.F0, PlaneSrc{W.plane, W.F0, d_P, order}, Mc, W.vq, W.nbr, W.nbr_tmp,
               W.ucnt, W.upcnt);
    }
    if (n_out) LAUNCH(k_quality, grid_for(ctx, n_out), 256, 0, stream, (int)n_out, d_off, d_mem, W.vq, d_Pout, order,
                      d_err);
    QTRY(cudaGetLastError());
    if (n_out) QTRY(cudaMemcpyAsync(errors, d_err, (size_t)n_out * 8, cudaMemcpyDefault, stream));
    QTRY(cudaMemcpyAsync(h_misc, misc, 2 * sizeof(int), cudaMemcpyDeviceToHost, stream));
    QTRY(cudaStreamSynchronize(stream));
    if (m && h_misc[1] != 0x7f7f7f7f) {
        st->code = rc = MF_ERR_STRUCTURAL;
        snprintf(st->message, sizeof(st->message), "facet %d references an out-of-range vertex or repeats a vertex",
                 h_misc[1]);
    }
done:
#undef QTRY
    cudaFreeAsync(block, stream);
    return rc;
}

// One decimation between its two halves (decimate_begin launches the round chain, decimate_end
// emits the results and synchronises): the host may prepare the result buffers in between.
struct DecCall {
    Plan p;
    WS W;
    mf_mesh_view mv;
    mf_decimate_config cfg;
    cudaStream_t stream = nullptr;
    bool force_carry = false;
    bool active = false;
    const void* X_src = nullptr;
    void* alias_tmp = nullptr;
    int* d_diff = nullptr;
    bool host_check = false;
    size_t pbytes = 0;
    int* h_status = nullptr;
    std::vector<ProfRec>* graph_prof = nullptr;
};

// The caller's result buffers (mf_decimate_into) as k_emit jobs next to the copy-out; false when
// one of them cannot be written by the device (pageable host memory) or is too small.
static bool add_caller_jobs(EmitJobs& jobs, const mf_outputs* o, const double* P, const double* X, int64_t xc,
                            const int* F, int64_t fcap_rows, const int* frows, const int* rt, const int* mt,
                            int64_t n_out, int64_t n_in) {
    if (!o) return true;
    auto dev = [](void* p) { return p ? device_writable(p) : nullptr; };
    if (o->positions && n_out) {
        void* d = dev(o->positions);
        if (!d) return false;
        jobs.add(kEmitF64, P, d, n_out * 3);
    }
    if (o->features && n_out * xc > 0) {
        void* d = dev(o->features);
        if (!d) return false;
        jobs.add(o->features_dtype == MF_DTYPE_F32 ? kEmitF32 : kEmitF64, X, d, n_out * xc);
    }
    if (o->facets && fcap_rows) {
        void* d = dev(o->facets);
        if (!d || o->facets_capacity < fcap_rows) return false;
        jobs.add(kEmitI32, F, d, fcap_rows * 3, frows);
    }
    if (o->replace && n_in) {
        void* d = dev(o->replace);
        if (!d) return false;
        jobs.add(kEmitI32, rt, d, n_in);
    }
    if (o->mapping && n_in) {
        void* d = dev(o->mapping);
        if (!d) return false;
        jobs.add(kEmitI32, mt, d, n_in);
    }
    return true;
}

// First half of a call: plan, stage, launch the round chain (nothing waits for the device).
int decimate_begin(Context* ctx, const mf_mesh_view* mv, const mf_decimate_config* cfg, cudaStream_t stream,
                   mf_status* st, bool force_carry, DecCall& call) {
    call.mv = *mv;
    call.cfg = *cfg;
    call.stream = stream;
    call.force_carry = force_carry;
    st->code = MF_OK;
    st->mesh_index = -1;
    st->achievable_vertices = 0;
    st->message[0] = 0;
    HostClock hc;
    Plan& p = call.p;
    if (make_plan(mv, cfg, p, st) != MF_OK) return st->code;
    hc.mark("plan");
    const int B = p.B, R = p.R;
    const int64_t n = p.n, m = p.m, C = p.C;
    MF_CUDA_TRY(cudaSetDevice(ctx->device));
    // Features that are a bitwise copy of the positions (the default, mesh.py:28-29) fold like
    // the positions and need not be carried.  Optimistic: run as aliased and verify while the
    // round chain runs -- a host memcmp for small host arrays, else an upload on a side stream
    // plus a compare kernel after the chain; a mismatch (features of the right shape that are
    // NOT the positions) reruns the call carrying them.
    const bool verify = !force_carry && !p.alias && mv->features && p.fdtype == MF_DTYPE_F64 && C == 3 &&
                        p.placement == 0 && n > 0;
    if (verify) p.alias = true;
    const void* P_src = mv->positions;
    const void* X_src = mv->features;
    void* alias_tmp = nullptr;
    struct TmpFree {  // freed here only if the call fails before the device work is launched
        void*& p;
        cudaStream_t s;
        bool keep = false;
        ~TmpFree() {
            if (p && !keep) cudaFreeAsync(p, s);
        }
    } tmp_free{alias_tmp, stream};
    const size_t pbytes = (size_t)n * 24;
    // host arrays are compared in host memory (threads, while the GPU works): the PCIe link is
    // what bounds a call with host arrays, so the features are never uploaded just to be compared
    const bool host_check = verify && !is_device_ptr(mv->positions) && !is_device_ptr(mv->features);
    int* d_diff = nullptr;
    if (verify && !host_check) {
        const bool xd = is_device_ptr(mv->features);
        MF_CUDA_TRY(cudaMallocAsync(&alias_tmp, 256 + (xd ? 0 : ((pbytes + 255) & ~size_t(255))), stream));
        d_diff = (int*)alias_tmp;
        MF_CUDA_TRY(cudaMemsetAsync(d_diff, 0, 4, stream));
        if (!xd) {  // upload on the side stream: overlaps the round chain, joined before the compare
            if (!ctx->aux) {
                MF_CUDA_TRY(cudaStreamCreateWithFlags(&ctx->aux, cudaStreamNonBlocking));
                for (cudaEvent_t& e : ctx->aux_ev) MF_CUDA_TRY(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
            }
            MF_CUDA_TRY(cudaEventRecord(ctx->aux_ev[0], stream));  // alias_tmp allocated
            MF_CUDA_TRY(cudaStreamWaitEvent(ctx->aux, ctx->aux_ev[0], 0));
            X_src = (char*)alias_tmp + 256;
            MF_CUDA_TRY(cudaMemcpyAsync((void*)X_src, mv->features, pbytes, cudaMemcpyHostToDevice, ctx->aux));
            MF_CUDA_TRY(cudaEventRecord(ctx->aux_ev[1], ctx->aux));
        }
    }

    // ---- workspace (grown on demand; cached graphs are tied to the arena address)
    WS& W = call.W;
    {
        Arena meas;
        meas.measuring = true;
        layout(meas, W, p);
        if (ctx->arena_bytes < meas.off) {
            MF_CUDA_TRY(cudaStreamSynchronize(stream));
            drop_graphs(ctx);
            if (ctx->arena) cudaFree(ctx->arena);
            ctx->arena = nullptr;
            ctx->arena_bytes = 0;
            size_t want = meas.off + meas.off / 4;
            MF_CUDA_TRY(cudaMalloc(&ctx->arena, want));
            ctx->arena_bytes = want;
        }
        Arena A;
        A.base = (char*)ctx->arena;
        A.cap = ctx->arena_bytes;
        layout(A, W, p);
    }
    // ---- pinned staging: [params | initial status words | offsets] (one upload) + readback
    size_t pin_need = W.upload_bytes + W.status_words * 4 + 1024;
    if (ctx->pinned_bytes < pin_need) {
        MF_CUDA_TRY(cudaStreamSynchronize(stream));
        if (ctx->pinned) cudaFreeHost(ctx->pinned);
        ctx->pinned = nullptr;
        MF_CUDA_TRY(cudaMallocHost(&ctx->pinned, pin_need * 2));
        ctx->pinned_bytes = pin_need * 2;
    }
    int* hp = (int*)ctx->pinned;
    {
        int* q = hp;
        q = std::copy(p.h_act.begin(), p.h_act.end(), q);
        q = std::copy(p.h_budget.begin(), p.h_budget.end(), q);
        q = std::copy(p.h_nin.begin(), p.h_nin.end(), q);
        q = std::copy(p.h_voff.begin(), p.h_voff.end(), q);
        for (int b = 0; b <= B; b++) *q++ = (int)p.foff[b];
        // status words: [1] = no bad facet yet (atomicMin), fail words = -1, the rest 0
        int* hs = hp + W.params_pad;
        const size_t fail_lo = 8 + (size_t)(B + 1), fail_hi = fail_lo + 3 * (size_t)B;
        for (size_t i = 0; i < W.status_words; i++) hs[i] = (i == 1) ? 0x7f7f7f7f : ((i >= fail_lo && i < fail_hi) ? -1 : 0);
    }
    int64_t* h_o64 = (int64_t*)(hp + W.params_pad + W.status_pad);
    for (int b = 0; b <= B; b++) {
        h_o64[b] = p.voff[b];
        h_o64[B + 1 + b] = p.foff[b];
    }
    int* h_status = (int*)((char*)ctx->pinned + ((W.upload_bytes + 255) & ~size_t(255)));
    // ---- stage params + inputs (outside the graph: host pointers / caller buffers change per call).
    // Device-resident inputs of a real chain are read in place by k_init_inputs (its graph node is
    // re-pointed per call); host inputs are uploaded into the staging buffers it reads instead.
    MF_CUDA_TRY(cudaMemcpyAsync(W.params, hp, W.upload_bytes, cudaMemcpyHostToDevice, stream));
    // pinned host inputs may be read in place too, through their mapped addresses (the conversion
    // kernel then streams them over the link itself: no staging copy; MF_ZERO_COPY_IN=0 stages)
    auto readable = [&](const void* q) -> const void* {
        if (is_device_ptr(q)) return q;
        return zero_copy_inputs() ? device_writable(const_cast<void*>(q)) : nullptr;
    };
    const void* P_dev = (R > 0 && n) ? readable(P_src) : nullptr;
    const void* F_dev = (R > 0 && m) ? readable(mv->facets) : nullptr;
    const bool in_place = R > 0 && (n == 0 || P_dev) && (m == 0 || F_dev);
    if (mv->facets_i32 && (!in_place || R == 0)) {
        st->code = MF_ERR_VALUE;
        snprintf(st->message, sizeof(st->message),
                 "int32 facets (facets_i32) must be device arrays of a call with at least one round");
        return st->code;
    }
    g_in_P = in_place && n ? (const double*)P_dev : nullptr;
    g_in_F64 = in_place && m ? F_dev : nullptr;
    g_in_f32 = mv->facets_i32 ? 1 : 0;
    if (!in_place) {
        if (n) MF_CUDA_TRY(cudaMemcpyAsync(W.P0, P_src, (size_t)n * 24, cudaMemcpyDefault, stream));
        if (m) MF_CUDA_TRY(cudaMemcpyAsync(W.F64, mv->facets, (size_t)m * 24, cudaMemcpyDefault, stream));
    }
    if (!p.alias && n * C > 0) {
        if (!mv->features)
            MF_CUDA_TRY(cudaMemcpyAsync(W.X0, P_src, (size_t)n * 24, cudaMemcpyDefault, stream));
        else if (p.fdtype == MF_DTYPE_F64)
            MF_CUDA_TRY(cudaMemcpyAsync(W.X0, X_src, (size_t)(n * C) * 8, cudaMemcpyDefault, stream));
        else
            MF_CUDA_TRY(cudaMemcpyAsync(W.Xf32, mv->features, (size_t)(n * C) * 4, cudaMemcpyDefault, stream));
    }
    // ---- the round chain: replay (or capture once) the graph of this call shape
    g_rec_err = cudaSuccess;
    auto rec_fail = [&]() {
        st->code = MF_ERR_CUDA;
        snprintf(st->message, sizeof(st->message), "recording the round chain failed at mf_decimate.cu:%d: %s",
                 g_rec_line, cudaGetErrorString(g_rec_err));
        cudaGetLastError();
        return st->code;
    };
    std::vector<ProfRec>* graph_prof = nullptr;
    if (use_graphs()) {
        GraphCache& gc = caches()[ctx];
        if (gc.arena != ctx->arena) {
            gc.clear();
            gc.arena = ctx->arena;
        }
        if (!gc.capture) {
            MF_CUDA_TRY(cudaStreamCreateWithFlags(&gc.capture, cudaStreamNonBlocking));
            for (cudaStream_t& b : gc.body) MF_CUDA_TRY(cudaStreamCreateWithFlags(&b, cudaStreamNonBlocking));
        }
        std::vector<int64_t> key = graph_key(p);
        auto it = gc.entries.find(key);
        if (it == gc.entries.end()) {
            if (gc.entries.size() >= 16) gc.clear();
            size_t rec0 = g_prof_recs.size();
            int64_t l0 = g_launches;
            MF_CUDA_TRY(cudaStreamBeginCapture(gc.capture, cudaStreamCaptureModeThreadLocal));
            // conditional nodes unless profiling (event nodes cannot live in bodies) or PDL edges
            const bool cond = use_cond() && g_prof_mode == 0 && !pdl_enabled();
            record(ctx, p, W, gc.capture, cond ? gc.body[0] : nullptr, cond ? gc.body[1] : nullptr);
            int64_t nk = g_launches - l0;
            g_launches = l0;
            cudaGraph_t g = nullptr;
            cudaError_t ce = cudaStreamEndCapture(gc.capture, &g);
            if (g_rec_err != cudaSuccess) {
                if (g) cudaGraphDestroy(g);
                return rec_fail();
            }
            MF_CUDA_TRY(ce);
            GraphEntry e;
            cudaError_t ie = cudaGraphInstantiate(&e.exec, g, 0);
            if (ie != cudaSuccess) cudaGraphDestroy(g);
            MF_CUDA_TRY(ie);
            e.graph = g;
            e.prof.assign(g_prof_recs.begin() + rec0, g_prof_recs.end());
            e.kernels = nk;
            e.init_node = g_init_node;
            e.init_args = g_init_args;
            e.init_grid = g_init_grid;
            g_prof_recs.resize(rec0);
            it = gc.entries.emplace(key, std::move(e)).first;
        }
        {  // point k_init_inputs at this call's inputs (device buffers in place, else the staging)
            GraphEntry& ge = it->second;
            const void* f_src = g_in_F64 ? g_in_F64 : (const void*)W.F64;
            const int f32 = g_in_F64 ? g_in_f32 : 0;
            const double* p_src = g_in_P ? g_in_P : W.P0;
            if (ge.init_args.F64 != f_src || ge.init_args.Psrc != p_src || ge.init_args.f_is32 != f32) {
                if (!ge.init_node) return rec_fail();
                ge.init_args.F64 = f_src;
                ge.init_args.f_is32 = f32;
                ge.init_args.Psrc = p_src;
                cudaKernelNodeParams kp = {};
                void* kargs[] = {&ge.init_args};
                kp.func = (void*)k_init_inputs;
                kp.gridDim = dim3(ge.init_grid);
                kp.blockDim = dim3(256);
                kp.sharedMemBytes = 0;
                kp.kernelParams = kargs;
                MF_CUDA_TRY(cudaGraphExecKernelNodeSetParams(ge.exec, ge.init_node, &kp));
            }
        }
        hc.mark("pre-launch");
        MF_CUDA_TRY(cudaGraphLaunch(it->second.exec, stream));
        hc.mark("graph-launch");
        g_launches += it->second.kernels;
        graph_prof = &it->second.prof;
    } else {
        record(ctx, p, W, stream);
        if (g_rec_err != cudaSuccess) return rec_fail();
    }
    tmp_free.keep = true;
    call.X_src = X_src;
    call.alias_tmp = alias_tmp;
    call.d_diff = d_diff;
    call.host_check = host_check;
    call.pbytes = pbytes;
    call.h_status = h_status;
    call.graph_prof = graph_prof;
    call.active = true;
    return MF_OK;
}

// Second half: result arrays (+ the caller's buffers), the readback and the one synchronisation.
int decimate_end(Context* ctx, DecCall& call, const mf_outputs* outs, Result** out, mf_status* st) {
    HostClock hc;
    call.active = false;
    const Plan& p = call.p;
    WS& W = call.W;
    const mf_mesh_view* mv = &call.mv;
    const mf_decimate_config* cfg = &call.cfg;
    cudaStream_t stream = call.stream;
    const int B = p.B, R = p.R;
    const int64_t n = p.n, m = p.m, C = p.C;
    const void* X_src = call.X_src;
    int* d_diff = call.d_diff;
    const bool host_check = call.host_check;
    const size_t pbytes = call.pbytes;
    int* h_status = call.h_status;
    std::vector<ProfRec>* graph_prof = call.graph_prof;
    struct TmpFree {
        void* p;
        cudaStream_t s;
        ~TmpFree() {
            if (p) cudaFreeAsync(p, s);
        }
    } tmp_free{call.alias_tmp, stream};
    MF_CUDA_TRY(cudaSetDevice(ctx->device));
    // host features checked against the positions while the round chain still runs; features
    // known to BE the positions need not be emitted when the caller shares the positions' array
    const int host_diff = host_check ? (int)host_differ(mv->positions, mv->features, pbytes) : 0;
    const bool alias_known = p.alias && (!mv->features || (host_check && !host_diff));
    mf_outputs outs_local;
    if (outs && outs->features_if_distinct == 1 && alias_known) {
        outs_local = *outs;
        outs_local.features = nullptr;
        outs = &outs_local;
    }
    // ---- result: copy outputs out of the workspace
    Result* res = new Result();
    res->device = ctx->device;
    res->n_in = n;
    res->n_out = p.Nfin;
    res->c = C;
    res->n_meshes = B;
    res->features_alias = p.alias;
    {
        Arena ra;
        ra.measuring = true;
        ra.take<double>((size_t)p.Nfin * 3);
        if (!p.alias) ra.take<double>((size_t)p.Nfin * C);
        ra.take<int>((size_t)p.Mcap * 3);
        ra.take<int>((size_t)p.N0);
        ra.take<int>((size_t)p.N0);
        cudaError_t e = cudaMallocAsync(&res->block, ra.off, stream);
        if (e != cudaSuccess) {
            delete res;
            MF_CUDA_TRY(e);
        }
        Arena rb;
        rb.base = (char*)res->block;
        rb.cap = ra.off;
        res->positions = rb.take<double>((size_t)p.Nfin * 3);
        res->features = p.alias ? nullptr : rb.take<double>((size_t)p.Nfin * C);
        res->facets = rb.take<int>((size_t)p.Mcap * 3);
        res->replace = rb.take<int>((size_t)p.N0);
        res->mapping = rb.take<int>((size_t)p.N0);
    }
    if (R > 0) {  // the result arrays out of the workspace: one launch instead of five copies
        EmitJobs jobs;
        if (p.Nfin) jobs.add(kEmitF64, W.Pfin, res->positions, (int64_t)p.Nfin * 3);
        if (!p.alias && p.Nfin * C > 0) jobs.add(kEmitF64, W.Xfin, res->features, (int64_t)p.Nfin * C);
        jobs.add(kEmitW32, W.Ffin, res->facets, (int64_t)p.Mcap * 3, W.status + 8 + B);  // m_out rows
        if (n) {
            jobs.add(kEmitW32, W.rt, res->replace, n);
            jobs.add(kEmitW32, W.mt, res->mapping, n);
        }
        // mf_decimate_into: the caller's buffers in the same launch (int32 -> int64 widened there)
        if (!add_caller_jobs(jobs, outs, W.Pfin, p.alias ? W.Pfin : W.Xfin, C, W.Ffin, p.Mcap, W.status + 8 + B, W.rt,
                             W.mt, p.Nfin, n)) {
            cudaFreeAsync(res->block, stream);
            delete res;
            st->code = MF_ERR_VALUE;
            snprintf(st->message, sizeof(st->message),
                     "mf_decimate_into: outputs must be device or pinned host memory, facets >= the input facet count");
            return st->code;
        }
        LAUNCH(k_emit, grid_for(ctx, std::max<int64_t>(1, jobs.total() / 4)), 256, 0, stream, jobs);
    } else {
        // identity (decimate.py:172-174, 367-370): inputs verbatim, replace = mapping = arange
        if (m > 0) LAUNCH(k_facets_in, grid_for(ctx, m), 256, 0, stream, m, W.F64, res->facets, B, W.vo64, W.fo64,
                          W.counters);
        if (n) cudaMemcpyAsync(res->positions, W.P0, (size_t)n * 24, cudaMemcpyDeviceToDevice, stream);
        if (!p.alias && n * C > 0) {
            if (W.Xf32) LAUNCH(k_f32_to_f64, grid_for(ctx, n * C), 256, 0, stream, n * C, W.Xf32, res->features);
            else cudaMemcpyAsync(res->features, W.X0, (size_t)(n * C) * 8, cudaMemcpyDeviceToDevice, stream);
        }
        if (n) LAUNCH(k_identity_index, grid_for(ctx, n), 256, 0, stream, (int)n, res->replace, res->mapping);
        if (outs) {  // the caller's buffers from the handle's arrays (the identity has no graph)
            EmitJobs jobs;
            if (!add_caller_jobs(jobs, outs, res->positions, p.alias ? res->positions : res->features, C, res->facets,
                                 m, nullptr, res->replace, res->mapping, n, n)) {
                cudaFreeAsync(res->block, stream);
                delete res;
                st->code = MF_ERR_VALUE;
                snprintf(st->message, sizeof(st->message),
                         "mf_decimate_into: outputs must be device or pinned host memory, facets >= the input facet count");
                return st->code;
            }
            if (jobs.count) LAUNCH(k_emit, grid_for(ctx, std::max<int64_t>(1, jobs.total() / 4)), 256, 0, stream, jobs);
        }
    }
    // ---- verify the optimistic features alias (overlapped with the chain)
    int h_diff = 0;
    if (d_diff) {
        if (X_src != mv->features) MF_CUDA_TRY(cudaStreamWaitEvent(stream, ctx->aux_ev[1], 0));
        LAUNCH(k_words_differ, grid_for(ctx, 3 * n), 256, 0, stream, 3 * n, (const unsigned long long*)W.P0,
               (const unsigned long long*)X_src, d_diff);
        MF_CUDA_TRY(cudaMemcpyAsync(&h_diff, d_diff, 4, cudaMemcpyDeviceToHost, stream));
    }
    if (host_check) h_diff = host_diff;
    hc.mark("result-enqueued");
    // ---- single readback
    MF_CUDA_TRY(cudaMemcpyAsync(h_status, W.status, W.status_words * 4, cudaMemcpyDeviceToHost, stream));
    MF_CUDA_TRY(cudaStreamSynchronize(stream));
    MF_CUDA_TRY(cudaGetLastError());
    hc.mark("synced");
    if (h_diff) {  // features of the positions' shape that differ from them: carry them
        cudaFreeAsync(res->block, stream);
        delete res;
        const mf_mesh_view mv2 = *mv;
        const mf_decimate_config cfg2 = *cfg;
        return decimate_run(ctx, &mv2, &cfg2, stream, out, st, true, outs);
    }
    if (graph_prof) prof_collect(*graph_prof);
    prof_collect_pending();
    const int* h_fo = h_status + 8;
    const int* h_fail = h_status + 8 + (B + 1);
    const int* h_stats = h_fail + 3 * B;
    auto fail_out = [&](int code) {
        st->code = code;
        cudaFree(res->block);
        delete res;
        return code;
    };
    if (R > 0 && (h_status[1] != 0x7f7f7f7f || h_status[2] != 0)) {
        if (h_status[2]) snprintf(st->message, sizeof(st->message), "positions contain NaN or infinite values");
        else
            snprintf(st->message, sizeof(st->message),
                     "facet %d references an out-of-range vertex (or one outside its batch entry) or repeats a vertex",
                     h_status[1]);
        return fail_out(MF_ERR_STRUCTURAL);
    }
    if (R > 0 && h_status[0]) {
        int bf = -1;
        for (int b = 0; b < B; b++)
            if (h_fail[b] >= 0) {
                bf = b;
                break;
            }
        // read before a rerun below reuses the context's status buffer
        const int ach = bf >= 0 ? h_fail[bf] : 0, rr = bf >= 0 ? h_fail[B + bf] : 0;
        const int no_edges = bf >= 0 ? h_fail[2 * B + bf] : 0;
        if (bf > 0 && mv->vertex_offsets && mv->facet_offsets) {
            // the batch stopped at the round entry bf failed in; an earlier entry with a longer round
            // chain may fail in a later round, and the reference raises the LOWEST failing entry's
            // error (decimate.py:354-361, entries decimated independently) -- so decimate the
            // entries before bf on their own (a prefix of the same arrays) and report theirs if any
            bool later = false;
            for (int b = 0; b < bf && !later; b++) later = (int)p.chains[b].size() > rr + 1;
            if (later) {
                mf_mesh_view pre = *mv;
                pre.n_meshes = bf;
                pre.n = mv->vertex_offsets[bf];
                pre.m = mv->facet_offsets[bf];
                const mf_decimate_config cfg2 = *cfg;
                Result* r2 = nullptr;
                mf_status st2;
                const int rc2 = decimate_run(ctx, &pre, &cfg2, stream, &r2, &st2, call.force_carry, nullptr);
                if (rc2 != MF_OK) {
                    *st = st2;
                    return fail_out(rc2);
                }
                if (r2) {
                    cudaFree(r2->block);
                    delete r2;
                }
            }
        }
        st->mesh_index = bf;
        if (bf >= 0) {
            st->achievable_vertices = ach;
            st->target_vertices = p.chains[bf][rr];
            st->no_edges = no_edges;
            if (st->no_edges)
                snprintf(st->message, sizeof(st->message),
                         "mesh has no edges; cannot reach %lld vertices (achievable minimum is %d)",
                         (long long)st->target_vertices, ach);
            else
                snprintf(st->message, sizeof(st->message),
                         "cannot reach %lld vertices in one pass; achievable minimum is %d",
                         (long long)st->target_vertices, ach);
        }
        return fail_out(MF_ERR_INFEASIBLE);
    }
    if (p.first_err < B) {
        st->mesh_index = p.first_err;
        snprintf(st->message, sizeof(st->message), "%s", p.err_msg);
        return fail_out(p.err_code);
    }
    res->m_out = (R == 0) ? m : h_fo[B];
    res->vertex_offsets.resize(B + 1);
    res->facet_offsets.resize(B + 1);
    for (int b = 0; b <= B; b++) {
        res->vertex_offsets[b] = p.h_voff[(size_t)R * (B + 1) + b];
        res->facet_offsets[b] = (R == 0) ? p.foff[b] : h_fo[b];
    }
    for (int r = 0; r < R; r++) {
        int64_t row[6] = {p.h_N[r], h_stats[4 * r], h_stats[4 * r + 1], p.h_N[r + 1], h_stats[4 * r + 2],
                          h_stats[4 * r + 3]};
        res->round_stats.insert(res->round_stats.end(), row, row + 6);
    }
    if (outs) {  // host offsets of the caller's result
        if (outs->vertex_offsets) std::copy(res->vertex_offsets.begin(), res->vertex_offsets.end(), outs->vertex_offsets);
        if (outs->facet_offsets) std::copy(res->facet_offsets.begin(), res->facet_offsets.end(), outs->facet_offsets);
    }
    if (debug_validate() && R > 0) {  // row 16: the reference re-validates every output TriMesh
        int vr = validate_result(ctx, res, stream, st);
        if (vr != MF_OK) return fail_out(vr);
    }
    *out = res;
    return MF_OK;
}

int decimate_run(Context* ctx, const mf_mesh_view* mv, const mf_decimate_config* cfg, cudaStream_t stream,
                 Result** out, mf_status* st, bool force_carry, const mf_outputs* outs) {
    st->code = MF_OK;
    st->mesh_index = -1;
    st->achievable_vertices = 0;
    st->message[0] = 0;
    DecCall call;
    const int rc = decimate_begin(ctx, mv, cfg, stream, st, force_carry, call);
    if (rc != MF_OK) return rc;
    return decimate_end(ctx, call, outs, out, st);
}

}  // namespace mf
