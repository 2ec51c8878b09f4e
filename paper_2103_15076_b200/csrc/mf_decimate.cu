// mf_decimate.cu -- host orchestration of decimate_parallel on one device.
//
// One call = the whole round chain of every batch entry as ONE stream-ordered
// launch sequence with no host synchronisation until the end: vertex counts
// per round are known on the host (they are the round targets), facet and
// edge counts stay on the device and every kernel reads them from there
// (grids are sized from host upper bounds).  The single readback at the end
// carries the status words and the output facet offsets.
//
// Batches (BatchedMesh, decimate.py:354-361) are processed as one segmented
// pipeline over the concatenated arrays: per-mesh budgets, per-mesh rank
// selection and per-mesh key-stream restart; a mesh whose chain is shorter
// (or that is already at its target) is bypassed in the remaining rounds,
// because a zero-budget round is not an identity (it drops duplicate facets
// and normalises -0.0), see SURVEY.md App. C.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
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
thread_local std::vector<ProfRec> g_prof_recs;
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
void prof_pre(const char* name, cudaStream_t s) {
    if (!prof_on(name)) return;
    ProfRec r{name, prof_event(), prof_event()};
    cudaEventRecord(r.a, s);
    g_prof_recs.push_back(r);
}
void prof_post(const char* name, cudaStream_t s) {
    if (!prof_on(name)) return;
    cudaEventRecord(g_prof_recs.back().b, s);
}

#ifndef LAUNCH
#define LAUNCH(kernel, grid, block, smem, stream, ...)                 \
    do {                                                               \
        prof_pre(#kernel, stream);                                     \
        kernel<<<(grid), (block), (smem), (stream)>>>(__VA_ARGS__);    \
        prof_post(#kernel, stream);                                    \
        g_launches++;                                                  \
    } while (0)
#endif

static int grid_for(const Context* ctx, int64_t n, int block = 256) {
    int64_t g = (n + block - 1) / block;
    int64_t cap = (int64_t)ctx->sm_count * 16;
    if (g > cap) g = cap;
    if (g < 1) g = 1;
    return (int)g;
}

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

struct ScanBuf {
    unsigned long long* status = nullptr;
    int* ticket = nullptr;
    size_t words = 0;
};

static void run_scan(const Context* ctx, ScanBuf& sb, const int* in, int* out, int n, cudaStream_t s) {
    int tiles = std::max(1, (n + kScanTile - 1) / kScanTile);
    cudaMemsetAsync(sb.status, 0, (size_t)(tiles + 1) * sizeof(unsigned long long), s);
    LAUNCH(k_scan_excl<LoadArr>, tiles, kScanBlock, 0, s, LoadArr{in}, n, out, sb.status,
           reinterpret_cast<int*>(sb.status + tiles));
    (void)ctx;
}

static int coop_launch(const char* name, const void* fn, int blocks, int threads, void* arg, cudaStream_t s) {
    void* args[] = {arg};
    prof_pre(name, s);
    cudaError_t e = cudaLaunchCooperativeKernel(fn, dim3(blocks), dim3(threads), args, 0, s);
    prof_post(name, s);
    g_launches++;
    return e == cudaSuccess ? 0 : (int)e;
}

int decimate_run(Context* ctx, const mf_mesh_view* mv, const mf_decimate_config* cfg, cudaStream_t stream,
                 Result** out, mf_status* st) {
    st->code = MF_OK;
    st->mesh_index = -1;
    st->achievable_vertices = 0;
    st->message[0] = 0;
    const int64_t n = mv->n, m = mv->m;
    if (cfg->placement != 0) {
        st->code = MF_ERR_VALUE;
        snprintf(st->message, sizeof(st->message), "placement 'inverse' is not supported by the CUDA path yet");
        return st->code;
    }
    if (n < 0 || m < 0 || n >= (int64_t)INT32_MAX - 1 || 3 * m >= (int64_t)INT32_MAX - 1) {
        st->code = MF_ERR_LIMIT;
        snprintf(st->message, sizeof(st->message), "mesh too large for 32-bit device indices (n=%lld, m=%lld)",
                 (long long)n, (long long)m);
        return st->code;
    }
    const bool alias = (mv->features == nullptr);
    const int64_t C = alias ? 3 : mv->c;
    const int B = mv->vertex_offsets ? (int)mv->n_meshes : 1;
    std::vector<int64_t> voff(B + 1), foff(B + 1);
    if (mv->vertex_offsets) {
        for (int b = 0; b <= B; b++) { voff[b] = mv->vertex_offsets[b]; foff[b] = mv->facet_offsets[b]; }
        bool ok = voff[0] == 0 && foff[0] == 0 && voff[B] == n && foff[B] == m;
        for (int b = 0; b < B && ok; b++) ok = voff[b + 1] >= voff[b] && foff[b + 1] >= foff[b];
        if (!ok) {
            st->code = MF_ERR_STRUCTURAL;
            snprintf(st->message, sizeof(st->message), "vertex/facet offsets must be monotone from 0 to n/m");
            return st->code;
        }
    } else {
        voff[0] = 0; voff[1] = n; foff[0] = 0; foff[1] = m;
    }
    // ---- per-mesh chains and host-side errors, in batch order (decimate.py:363-371)
    const int64_t target = cfg->target_vertices;
    int first_err = B;
    int err_code = MF_OK;
    char err_msg[256] = {0};
    std::vector<std::vector<int64_t>> chains(B);
    for (int b = 0; b < B; b++) {
        int64_t nb = voff[b + 1] - voff[b], mb = foff[b + 1] - foff[b];
        if (target > nb) {
            err_code = MF_ERR_VALUE;
            snprintf(err_msg, sizeof(err_msg), "target_vertices=%lld exceeds the input size %lld", (long long)target,
                     (long long)nb);
        } else if (cfg->rounds == 0 || target == nb) {
            if (target != nb) {
                err_code = MF_ERR_VALUE;
                snprintf(err_msg, sizeof(err_msg), "rounds=0 requires target_vertices == input vertex count");
            }
        } else if (nb < 3 || mb < 1) {
            err_code = MF_ERR_STRUCTURAL;
            snprintf(err_msg, sizeof(err_msg),
                     "decimate_parallel requires a mesh with at least 3 vertices and 1 facet, got %lld vertices / "
                     "%lld facets",
                     (long long)nb, (long long)mb);
        } else {
            round_targets(nb, target, cfg->rounds, chains[b]);
        }
        if (err_code != MF_OK) {
            first_err = b;
            break;
        }
    }
    int R = 0;
    for (int b = 0; b < first_err; b++) R = std::max(R, (int)chains[b].size());

    // ---- per-round host tables: nin, act, budget, voff
    std::vector<int> h_nin((size_t)(R + 1) * B), h_act((size_t)std::max(R, 1) * B, 0),
        h_budget((size_t)std::max(R, 1) * B, 0), h_voff((size_t)(R + 1) * (B + 1));
    for (int b = 0; b < B; b++) h_nin[b] = (int)(voff[b + 1] - voff[b]);
    for (int r = 0; r < R; r++) {
        for (int b = 0; b < B; b++) {
            int nin = h_nin[(size_t)r * B + b];
            bool a = b < first_err && r < (int)chains[b].size();
            h_act[(size_t)r * B + b] = a;
            int tgt = a ? (int)chains[b][r] : nin;
            h_budget[(size_t)r * B + b] = nin - tgt;
            h_nin[(size_t)(r + 1) * B + b] = tgt;
        }
    }
    for (int r = 0; r <= R; r++) {
        int acc = 0;
        h_voff[(size_t)r * (B + 1)] = 0;
        for (int b = 0; b < B; b++) {
            acc += h_nin[(size_t)r * B + b];
            h_voff[(size_t)r * (B + 1) + b + 1] = acc;
        }
    }
    std::vector<int> h_N(R + 1);
    for (int r = 0; r <= R; r++) h_N[r] = h_voff[(size_t)r * (B + 1) + B];
    const int N0 = (int)n, M0 = (int)m;
    const int Nfin = h_N[R];
    const int Mcap = std::max(M0, 1);
    const int Ecap = 3 * Mcap;
    const int N1 = R > 0 ? h_N[1] : N0;

    MF_CUDA_TRY(cudaSetDevice(ctx->device));

    // ---- result allocation (stream ordered)
    Result* res = new Result();
    res->device = ctx->device;
    res->n_in = n;
    res->n_out = Nfin;
    res->c = C;
    res->n_meshes = B;
    res->features_alias = alias;
    {
        Arena ra;
        ra.measuring = true;
        ra.take<double>((size_t)Nfin * 3);
        if (!alias) ra.take<double>((size_t)Nfin * C);
        ra.take<int>((size_t)Mcap * 3);
        ra.take<int>((size_t)N0);
        ra.take<int>((size_t)N0);
        cudaError_t e = cudaMallocAsync(&res->block, ra.off, stream);
        if (e != cudaSuccess) {
            delete res;
            MF_CUDA_TRY(e);
        }
        Arena rb;
        rb.base = (char*)res->block;
        rb.cap = ra.off;
        res->positions = rb.take<double>((size_t)Nfin * 3);
        res->features = alias ? nullptr : rb.take<double>((size_t)Nfin * C);
        res->facets = rb.take<int>((size_t)Mcap * 3);
        res->replace = rb.take<int>((size_t)N0);
        res->mapping = rb.take<int>((size_t)N0);
    }

    // ---- workspace layout (measured, then carved from the context arena)
    const bool seeded = cfg->seeded != 0;
    const int nParamR = std::max(R, 1);
    auto layout = [&](Arena& A, auto& W) {
        W.params = A.template take<int>((size_t)nParamR * B * 3 + (size_t)(R + 1) * (B + 1) + (size_t)(R + 1) * B);
        W.F0 = A.template take<int>((size_t)Mcap * 3);
        W.P0 = A.template take<double>((size_t)N0 * 3);
        W.X0 = alias ? nullptr : A.template take<double>((size_t)N0 * C);
        W.Pa = A.template take<double>((size_t)N1 * 3);
        W.Pb = A.template take<double>((size_t)N1 * 3);
        W.Xa = alias ? nullptr : A.template take<double>((size_t)N1 * C);
        W.Xb = alias ? nullptr : A.template take<double>((size_t)N1 * C);
        W.Fa = A.template take<int>((size_t)Mcap * 3);
        W.Fb = A.template take<int>((size_t)Mcap * 3);
        W.foff_a = A.template take<int>((size_t)B + 1);
        W.foff_b = A.template take<int>((size_t)B + 1);
        W.vmesh = (B > 1) ? A.template take<int>((size_t)N0) : nullptr;
        W.plane = A.template take<Plane>((size_t)Mcap);
        W.deg = A.template take<int>((size_t)N0 + 1);
        W.inc_off = A.template take<int>((size_t)N0 + 1);
        W.cursor = A.template take<int>((size_t)N0 + 1);
        W.inc = A.template take<int>((size_t)Ecap);
        W.inc_tmp = A.template take<int>((size_t)Ecap);
        W.vq = A.template take<double>((size_t)N0 * 10);
        W.nbr = A.template take<int>((size_t)2 * Ecap);
        W.nbr_tmp = A.template take<int>((size_t)2 * Ecap);
        W.adj_eid = A.template take<int>((size_t)2 * Ecap);
        W.ucnt = A.template take<int>((size_t)N0);
        W.upcnt = A.template take<int>((size_t)N0);
        W.eoff = A.template take<int>((size_t)N0 + 1);
        W.heavy = A.template take<int>((size_t)N0);
        W.counters = A.template take<int>(64);
        W.e0 = A.template take<int>((size_t)Ecap);
        W.e1 = A.template take<int>((size_t)Ecap);
        W.cost = A.template take<double>((size_t)Ecap);
        W.key_hi = A.template take<uint64_t>((size_t)Ecap);
        W.key_lo = seeded ? A.template take<uint64_t>((size_t)Ecap) : nullptr;
        W.mlo = A.template take<unsigned long long>((size_t)B);
        W.mhi = A.template take<unsigned long long>((size_t)B);
        W.mate = A.template take<int>((size_t)N0);
        W.best = A.template take<int>((size_t)N0);
        W.front0 = A.template take<int>((size_t)N0);
        W.front1 = A.template take<int>((size_t)N0);
        W.bar = A.template take<unsigned>(64);
        W.chi = A.template take<uint64_t>((size_t)N0);
        W.clo = A.template take<uint64_t>((size_t)N0);
        W.cseg = A.template take<int>((size_t)N0);
        W.cpay = A.template take<int>((size_t)N0);
        W.caux = A.template take<int>((size_t)N0);
        W.seg_cnt = A.template take<int>((size_t)B);
        W.ksel = A.template take<int>((size_t)B);
        W.mode = A.template take<int>((size_t)B);
        W.krem = A.template take<int>((size_t)B);
        W.p_hi = A.template take<uint64_t>((size_t)B);
        W.p_lo = A.template take<uint64_t>((size_t)B);
        W.hist = A.template take<int>((size_t)B * 256);
        W.removed = A.template take<int>((size_t)B);
        W.fail = A.template take<int>((size_t)B * 3 + 8);
        W.absorbed = A.template take<int>((size_t)N0);
        W.minrep = A.template take<int>((size_t)N0);
        W.anchor = A.template take<int>((size_t)N0);
        W.isrep = A.template take<int>((size_t)N0 + 1);
        W.outidx = A.template take<int>((size_t)N0 + 1);
        W.rstep = A.template take<int>((size_t)N0);
        W.ccount = A.template take<int>((size_t)N0 + 1);
        W.coff = A.template take<int>((size_t)N0 + 1);
        W.cmem = A.template take<int>((size_t)N0);
        W.has_live = A.template take<unsigned char>((size_t)N0);
        W.mapped = A.template take<int>((size_t)Mcap * 3);
        W.canon = A.template take<int4>((size_t)Mcap);
        W.slot = A.template take<int>((size_t)Mcap);
        W.keep = A.template take<int>((size_t)Mcap + 1);
        W.kout = A.template take<int>((size_t)Mcap + 1);
        W.tsize = 1u;
        while (W.tsize < (unsigned)(2 * Mcap)) W.tsize <<= 1;
        W.table = A.template take<int>((size_t)W.tsize);
        size_t maxn = (size_t)std::max(N0, Mcap) + 1;
        W.scan.words = maxn / kScanTile + 4;
        W.scan.status = A.template take<unsigned long long>(W.scan.words);
        W.vo64 = A.template take<int64_t>((size_t)B + 1);
        W.fo64 = A.template take<int64_t>((size_t)B + 1);
        W.F64 = A.template take<int64_t>((size_t)Mcap * 3);
        W.Xf32 = A.template take<float>((size_t)N0 * C);
        W.stats = A.template take<int>((size_t)std::max(R, 1) * 4);
    };
    struct WS {
        int* params; int* F0; double* P0; double* X0; double *Pa, *Pb, *Xa, *Xb; int *Fa, *Fb, *foff_a, *foff_b;
        int* vmesh; Plane* plane; int *deg, *inc_off, *cursor, *inc, *inc_tmp; double* vq;
        int *nbr, *nbr_tmp, *adj_eid, *ucnt, *upcnt, *eoff, *heavy, *counters, *e0, *e1;
        double* cost; uint64_t *key_hi, *key_lo; unsigned long long *mlo, *mhi;
        int *mate, *best, *front0, *front1; unsigned* bar;
        uint64_t *chi, *clo; int *cseg, *cpay, *caux, *seg_cnt, *ksel, *mode, *krem; uint64_t *p_hi, *p_lo;
        int *hist, *removed, *fail, *absorbed, *minrep, *anchor, *isrep, *outidx, *rstep, *ccount, *coff, *cmem;
        unsigned char* has_live; int* mapped; int4* canon; int *slot, *keep, *kout; unsigned tsize; int* table;
        ScanBuf scan; int64_t *vo64, *fo64, *F64; float* Xf32; int* stats;
    } W;
    {
        Arena meas;
        meas.measuring = true;
        layout(meas, W);
        if (ctx->arena_bytes < meas.off) {
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
        layout(A, W);
    }
    int* d_abort = W.fail + 3 * B;      // [0] abort, [1] bad facet, [2] bad position, [3] limit
    int* d_fail_ach = W.fail;
    int* d_fail_round = W.fail + B;
    int* d_fail_noedge = W.fail + 2 * B;

    // ---- params upload (one pinned H2D): act | budget | nin(R+1) | voff(R+1)
    size_t pw = (size_t)nParamR * B * 3 + (size_t)(R + 1) * (B + 1) + (size_t)(R + 1) * B;
    size_t pin_need = pw * sizeof(int) + 8 * sizeof(int64_t) * (size_t)(B + 1) + 4096 + (size_t)(B + 1) * 8 +
                      (size_t)B * 12 + (size_t)R * 16 + 64;
    if (ctx->pinned_bytes < pin_need) {
        if (ctx->pinned) cudaFreeHost(ctx->pinned);
        ctx->pinned = nullptr;
        MF_CUDA_TRY(cudaMallocHost(&ctx->pinned, pin_need * 2));
        ctx->pinned_bytes = pin_need * 2;
    }
    int* hp = (int*)ctx->pinned;
    int* h_actp = hp;
    int* h_budp = hp + (size_t)nParamR * B;
    int* h_ninp = hp + (size_t)nParamR * B * 2;
    int* h_voffp = h_ninp + (size_t)(R + 1) * B;
    std::copy(h_act.begin(), h_act.begin() + (size_t)nParamR * B, h_actp);
    std::copy(h_budget.begin(), h_budget.begin() + (size_t)nParamR * B, h_budp);
    std::copy(h_nin.begin(), h_nin.end(), h_ninp);
    std::copy(h_voff.begin(), h_voff.end(), h_voffp);
    // nin table is (R+1)*B; the layout above reserved nParamR*B*3 + ... words in order act, budget, nin, voff.
    int* d_act = W.params;
    int* d_budget = W.params + (size_t)nParamR * B;
    int* d_nin = W.params + (size_t)nParamR * B * 2;
    int* d_voff = d_nin + (size_t)(R + 1) * B;
    MF_CUDA_TRY(cudaMemcpyAsync(W.params, hp, pw * sizeof(int), cudaMemcpyHostToDevice, stream));
    int64_t* h_o64 = (int64_t*)((char*)ctx->pinned + ((pw * sizeof(int) + 255) & ~size_t(255)));
    for (int b = 0; b <= B; b++) { h_o64[b] = voff[b]; h_o64[B + 1 + b] = foff[b]; }
    MF_CUDA_TRY(cudaMemcpyAsync(W.vo64, h_o64, (B + 1) * sizeof(int64_t), cudaMemcpyHostToDevice, stream));
    MF_CUDA_TRY(cudaMemcpyAsync(W.fo64, h_o64 + B + 1, (B + 1) * sizeof(int64_t), cudaMemcpyHostToDevice, stream));
    MF_CUDA_TRY(cudaMemsetAsync(W.fail, 0xFF, (size_t)B * 3 * sizeof(int), stream));
    MF_CUDA_TRY(cudaMemsetAsync(d_abort, 0, 8 * sizeof(int), stream));
    int* d_badf = d_abort + 1;
    int* d_badp = d_abort + 2;
    MF_CUDA_TRY(cudaMemsetAsync(d_badf, 0x7f, sizeof(int), stream));

    // ---- inputs -> device (int64 facets -> int32 with validation)
    const double* dP = mv->positions;
    if (!is_device_ptr(mv->positions)) {
        MF_CUDA_TRY(cudaMemcpyAsync(W.P0, mv->positions, (size_t)n * 3 * sizeof(double), cudaMemcpyHostToDevice,
                                    stream));
        dP = W.P0;
    }
    const int64_t* dF64 = mv->facets;
    if (m > 0 && !is_device_ptr(mv->facets)) {
        MF_CUDA_TRY(cudaMemcpyAsync(W.F64, mv->facets, (size_t)m * 3 * sizeof(int64_t), cudaMemcpyHostToDevice,
                                    stream));
        dF64 = W.F64;
    }
    if (m > 0) LAUNCH(k_facets_in, grid_for(ctx, m), 256, 0, stream, m, dF64, W.F0, B, W.vo64, W.fo64, d_badf);
    if (n > 0) LAUNCH(k_check_finite, grid_for(ctx, 3 * n), 256, 0, stream, 3 * n, dP, d_badp);
    const double* dX = nullptr;
    if (!alias) {
        if (mv->features_dtype == MF_DTYPE_F64) {
            if (is_device_ptr(mv->features)) dX = (const double*)mv->features;
            else {
                MF_CUDA_TRY(cudaMemcpyAsync(W.X0, mv->features, (size_t)n * C * sizeof(double),
                                            cudaMemcpyHostToDevice, stream));
                dX = W.X0;
            }
        } else {
            const float* xf = (const float*)mv->features;
            if (!is_device_ptr(xf)) {
                MF_CUDA_TRY(cudaMemcpyAsync(W.Xf32, xf, (size_t)n * C * sizeof(float), cudaMemcpyHostToDevice,
                                            stream));
                xf = W.Xf32;
            }
            if (n * C > 0) LAUNCH(k_f32_to_f64, grid_for(ctx, n * C), 256, 0, stream, n * C, xf, W.X0);
            dX = W.X0;
        }
    }
    // facet offsets of round 0 (int32)
    {
        std::vector<int> f32(B + 1);
        for (int b = 0; b <= B; b++) f32[b] = (int)foff[b];
        int* hf = (int*)(h_o64 + 2 * (B + 1));
        std::copy(f32.begin(), f32.end(), hf);
        MF_CUDA_TRY(cudaMemcpyAsync(W.foff_a, hf, (B + 1) * sizeof(int), cudaMemcpyHostToDevice, stream));
    }

    // ---- rounds
    const double* Pc = dP;
    const double* Xc = dX;
    const int* Fc = W.F0;
    int* foff_c = W.foff_a;
    int* foff_n = W.foff_b;
    const int order = cfg->einsum_order;
    int* d_ninc = W.counters;       // [0] frontier 0, [1] frontier 1, [2] LD iterations
    int* d_heavy_n = W.counters + 4;
    int* d_ncand = W.counters + 8;
    int* d_heavy_c = W.counters + 12;
    int* d_notdone = W.counters + 16;  // 16 words
    int coop_err = 0;
    for (int r = 0; r < R; r++) {
        const int N = h_N[r];
        const int Nn = h_N[r + 1];
        const int* act = d_act + (size_t)r * B;
        const int* budget = d_budget + (size_t)r * B;
        const int* nin = d_nin + (size_t)r * B;
        const int* voff_r = d_voff + (size_t)r * (B + 1);
        const int* dM = foff_c + B;
        const bool last = (r == R - 1);
        double* Pn = last ? res->positions : ((r & 1) ? W.Pb : W.Pa);
        double* Xn = alias ? nullptr : (last ? res->features : ((r & 1) ? W.Xb : W.Xa));
        int* Fn = last ? res->facets : ((r & 1) ? W.Fb : W.Fa);
        int* vmesh = nullptr;
        if (B > 1) {
            vmesh = W.vmesh;
            LAUNCH(k_vmesh, grid_for(ctx, N), 256, 0, stream, N, voff_r, B, vmesh);
        }
        cudaMemsetAsync(W.deg, 0, (size_t)(N + 1) * sizeof(int), stream);
        cudaMemsetAsync(W.cursor, 0, (size_t)(N + 1) * sizeof(int), stream);
        cudaMemsetAsync(W.counters, 0, 64 * sizeof(int), stream);
        LAUNCH(k_facet_plane, grid_for(ctx, Mcap), 256, 0, stream, Fc, Pc, dM, vmesh, act, W.plane, W.deg, order);
        run_scan(ctx, W.scan, W.deg, W.inc_off, N, stream);
        LAUNCH(k_inc_scatter, grid_for(ctx, Mcap), 256, 0, stream, Fc, dM, Mcap, vmesh, act, W.inc_off, W.cursor,
               W.inc);
        LAUNCH(k_vertex, grid_for(ctx, N, 128), 128, 0, stream, N, W.inc_off, W.inc, Fc, W.plane, Mcap, W.vq, W.nbr,
               W.ucnt, W.upcnt, W.heavy, d_heavy_n);
        LAUNCH(k_vertex_heavy, ctx->sm_count, 256, 0, stream, W.heavy, d_heavy_n, W.inc_off, W.inc, W.inc_tmp, Fc,
               W.plane, Mcap, W.vq, W.nbr, W.nbr_tmp, W.ucnt, W.upcnt);
        run_scan(ctx, W.scan, W.upcnt, W.eoff, N, stream);
        LAUNCH(k_edges, grid_for(ctx, N, 128), 128, 0, stream, N, W.inc_off, W.nbr, W.ucnt, W.upcnt, W.eoff, W.vq, Pc,
               W.e0, W.e1, W.cost, W.key_hi, W.adj_eid, W.mate, W.minrep, W.absorbed, order);
        const int* dE = W.eoff + N;
        if (seeded) {
            cudaMemsetAsync(W.mlo, 0xFF, (size_t)B * sizeof(unsigned long long), stream);
            cudaMemsetAsync(W.mhi, 0, (size_t)B * sizeof(unsigned long long), stream);
            LAUNCH(k_cost_minmax, grid_for(ctx, Ecap), 256, 0, stream, dE, W.cost, W.e0, vmesh, W.mlo, W.mhi);
            LAUNCH(k_seed_keys, grid_for(ctx, (Ecap + kSeedRun - 1) / kSeedRun), 256, 0, stream, dE, W.cost, W.e0,
                   vmesh, W.eoff, voff_r, W.mlo, W.mhi, cfg->pcg_state[0], cfg->pcg_state[1], cfg->pcg_state[2],
                   cfg->pcg_state[3], W.key_hi, W.key_lo);
        }
        // locally-dominant matching
        {
            cudaMemsetAsync(W.bar, 0, 2 * sizeof(unsigned), stream);
            MatchArgs ma{N, W.inc_off, W.ucnt, W.nbr, W.adj_eid, W.e0, W.e1, W.key_hi, seeded ? W.key_lo : nullptr,
                         W.mate, W.best, W.front0, W.front1, d_ninc, W.bar};
            int blocks = std::max(1, std::min(ctx->coop_blocks_match, (N + 255) / 256));
            coop_err |= coop_launch("k_match", (const void*)k_match, blocks, 256, &ma, stream);
        }
        // budget truncation (select the `budget` lowest-ranked matched edges per mesh)
        auto select = [&](const int* removed_in) {
            cudaMemsetAsync(W.bar, 0, 2 * sizeof(unsigned), stream);
            cudaMemsetAsync(d_notdone, 0, 16 * sizeof(int), stream);
            cudaMemsetAsync(W.hist, 0, (size_t)B * 256 * sizeof(int), stream);
            SelectArgs sa{d_ncand, W.chi, W.clo, W.cseg, B, W.seg_cnt, act, budget, removed_in, W.ksel, W.mode,
                          W.p_hi, W.p_lo, W.krem, W.hist, d_notdone, W.bar};
            int blocks = std::max(1, std::min(ctx->coop_blocks_select, (N / 2 + 255) / 256));
            coop_err |= coop_launch("k_select", (const void*)k_select, blocks, 256, &sa, stream);
        };
        cudaMemsetAsync(W.seg_cnt, 0, (size_t)B * sizeof(int), stream);
        LAUNCH(k_trunc_cand, grid_for(ctx, N), 256, 0, stream, N, W.mate, W.e0, W.key_hi, seeded ? W.key_lo : nullptr,
               vmesh, d_ncand, W.chi, W.clo, W.cseg, W.cpay, W.seg_cnt);
        select(nullptr);
        LAUNCH(k_trunc_apply, grid_for(ctx, N / 2 + B), 256, 0, stream, d_ncand, W.chi, W.clo, W.cseg, W.cpay, W.mode,
               W.p_hi, W.p_lo, W.e0, W.e1, W.mate, B, W.ksel, W.removed);
        // absorb leftovers (one pass is exact: the matching is maximal when budget is unmet)
        cudaMemsetAsync(W.seg_cnt, 0, (size_t)B * sizeof(int), stream);
        cudaMemsetAsync(d_ncand, 0, sizeof(int), stream);
        LAUNCH(k_absorb_cand, grid_for(ctx, N), 256, 0, stream, N, W.inc_off, W.ucnt, W.nbr, W.adj_eid, W.cost,
               W.mate, W.e0, vmesh, act, budget, W.removed, d_ncand, W.chi, W.clo, W.cseg, W.cpay, W.caux,
               W.seg_cnt);
        select(W.removed);
        RoundFail rf{d_abort, d_fail_ach, d_fail_round, d_fail_noedge};
        LAUNCH(k_absorb_apply, grid_for(ctx, N / 2 + B), 256, 0, stream, d_ncand, W.chi, W.clo, W.cseg, W.cpay,
               W.caux, W.mode, W.p_hi, W.p_lo, W.absorbed, B, act, budget, nin, W.ksel, W.removed, W.eoff, voff_r, rf,
               r);
        // relabel
        LAUNCH(k_relabel1, grid_for(ctx, N), 256, 0, stream, N, d_abort, W.mate, W.e0, W.absorbed, W.anchor,
               W.minrep);
        LAUNCH(k_relabel2, grid_for(ctx, N), 256, 0, stream, N, d_abort, W.anchor, W.minrep, W.isrep);
        run_scan(ctx, W.scan, W.isrep, W.outidx, N, stream);
        cudaMemsetAsync(W.ccount, 0, (size_t)(Nn + 1) * sizeof(int), stream);
        LAUNCH(k_relabel3, grid_for(ctx, N), 256, 0, stream, N, d_abort, W.anchor, W.minrep, W.outidx, W.rstep,
               W.ccount);
        // cluster CSR + contraction
        run_scan(ctx, W.scan, W.ccount, W.coff, Nn, stream);
        cudaMemsetAsync(W.cursor, 0, (size_t)(Nn + 1) * sizeof(int), stream);
        LAUNCH(k_csr_scatter, grid_for(ctx, N), 256, 0, stream, N, d_abort, W.rstep, W.coff, W.cursor, W.cmem);
        LAUNCH(k_seg_sort_small, grid_for(ctx, Nn), 256, 0, stream, Nn, d_abort, W.coff, W.cmem, W.heavy, d_heavy_c);
        LAUNCH(k_seg_sort_heavy, ctx->sm_count, 256, 0, stream, d_abort, W.coff, W.cmem, W.front0, W.heavy,
               d_heavy_c);
        LAUNCH(k_contract, grid_for(ctx, Nn), 256, 0, stream, Nn, d_abort, W.coff, W.cmem, vmesh, act, Pc, Xc,
               (int)C, Pn, Xn);
        // output facets
        cudaMemsetAsync(W.table, 0xFF, (size_t)W.tsize * sizeof(int), stream);
        cudaMemsetAsync(W.has_live, 0, (size_t)N, stream);
        LAUNCH(k_facet_remap, grid_for(ctx, Mcap), 256, 0, stream, dM, d_abort, Fc, W.rstep, vmesh, act, W.mapped,
               W.canon, W.slot, W.has_live, W.table, W.tsize - 1);
        LAUNCH(k_facet_keep, grid_for(ctx, Mcap), 256, 0, stream, dM, Mcap, d_abort, W.slot, W.table, W.keep);
        run_scan(ctx, W.scan, W.keep, W.kout, Mcap, stream);
        LAUNCH(k_facet_write, grid_for(ctx, Mcap), 256, 0, stream, dM, d_abort, W.keep, W.kout, W.mapped, Fn, B,
               foff_c, foff_n);
        LAUNCH(k_compose, grid_for(ctx, N0), 256, 0, stream, N0, d_abort, W.rstep, W.inc_off, W.has_live, vmesh, act,
               res->replace, res->mapping, r == 0);
        cudaMemcpyAsync(W.stats + 4 * r + 0, foff_c + B, sizeof(int), cudaMemcpyDeviceToDevice, stream);
        cudaMemcpyAsync(W.stats + 4 * r + 1, W.eoff + N, sizeof(int), cudaMemcpyDeviceToDevice, stream);
        cudaMemcpyAsync(W.stats + 4 * r + 2, foff_n + B, sizeof(int), cudaMemcpyDeviceToDevice, stream);
        cudaMemcpyAsync(W.stats + 4 * r + 3, d_ninc + 2, sizeof(int), cudaMemcpyDeviceToDevice, stream);
        Pc = Pn;
        Xc = Xn;
        Fc = Fn;
        std::swap(foff_c, foff_n);
    }
    if (coop_err) {
        st->code = MF_ERR_CUDA;
        snprintf(st->message, sizeof(st->message), "cooperative launch failed (%d)", coop_err);
        cudaFreeAsync(res->block, stream);
        delete res;
        return st->code;
    }
    if (R == 0) {
        // identity (decimate.py:172-174, 367-370): copy inputs, replace = mapping = arange
        MF_CUDA_TRY(cudaMemcpyAsync(res->positions, dP, (size_t)n * 3 * sizeof(double), cudaMemcpyDeviceToDevice,
                                    stream));
        if (!alias && n * C > 0)
            MF_CUDA_TRY(cudaMemcpyAsync(res->features, dX, (size_t)n * C * sizeof(double), cudaMemcpyDeviceToDevice,
                                        stream));
        if (m) MF_CUDA_TRY(cudaMemcpyAsync(res->facets, W.F0, (size_t)m * 3 * sizeof(int), cudaMemcpyDeviceToDevice,
                                           stream));
        LAUNCH(k_identity_index, grid_for(ctx, n), 256, 0, stream, (int)n, res->replace, res->mapping);
    }
    // ---- single readback: status words + final facet offsets + per-mesh failures
    int* h_st = (int*)(h_o64 + 4 * (B + 1));
    MF_CUDA_TRY(cudaMemcpyAsync(h_st, d_abort, 8 * sizeof(int), cudaMemcpyDeviceToHost, stream));
    MF_CUDA_TRY(cudaMemcpyAsync(h_st + 8, foff_c, (B + 1) * sizeof(int), cudaMemcpyDeviceToHost, stream));
    MF_CUDA_TRY(cudaMemcpyAsync(h_st + 8 + B + 1, W.fail, (size_t)B * 3 * sizeof(int), cudaMemcpyDeviceToHost,
                                stream));
    int* h_stats = h_st + 8 + B + 1 + 3 * B;
    if (R > 0)
        MF_CUDA_TRY(cudaMemcpyAsync(h_stats, W.stats, (size_t)R * 4 * sizeof(int), cudaMemcpyDeviceToHost, stream));
    MF_CUDA_TRY(cudaStreamSynchronize(stream));
    MF_CUDA_TRY(cudaGetLastError());
    const int* h_fo = h_st + 8;
    const int* h_fail = h_st + 8 + B + 1;
    if (h_st[1] != 0x7f7f7f7f || h_st[2] != 0) {
        st->code = MF_ERR_STRUCTURAL;
        if (h_st[2]) snprintf(st->message, sizeof(st->message), "positions contain NaN or infinite values");
        else
            snprintf(st->message, sizeof(st->message),
                     "facet %d references an out-of-range vertex (or one outside its batch entry) or repeats a vertex",
                     h_st[1]);
        cudaFreeAsync(res->block, stream);
        delete res;
        return st->code;
    }
    if (h_st[0]) {
        int bf = -1;
        for (int b = 0; b < B; b++)
            if (h_fail[b] >= 0) { bf = b; break; }
        st->code = MF_ERR_INFEASIBLE;
        st->mesh_index = bf;
        if (bf >= 0) {
            st->achievable_vertices = h_fail[bf];
            int rr = h_fail[B + bf];
            st->target_vertices = chains[bf][rr];
            st->no_edges = h_fail[2 * B + bf];
            if (st->no_edges)
                snprintf(st->message, sizeof(st->message),
                         "mesh has no edges; cannot reach %lld vertices (achievable minimum is %d)",
                         (long long)st->target_vertices, h_fail[bf]);
            else
                snprintf(st->message, sizeof(st->message),
                         "cannot reach %lld vertices in one pass; achievable minimum is %d",
                         (long long)st->target_vertices, h_fail[bf]);
        }
        cudaFreeAsync(res->block, stream);
        delete res;
        return st->code;
    }
    if (first_err < B) {
        st->code = err_code;
        st->mesh_index = first_err;
        snprintf(st->message, sizeof(st->message), "%s", err_msg);
        cudaFreeAsync(res->block, stream);
        delete res;
        return st->code;
    }
    res->m_out = (R == 0) ? m : h_fo[B];
    for (int r = 0; r < R; r++) {
        int64_t row[6] = {h_N[r], h_stats[4 * r], h_stats[4 * r + 1], h_N[r + 1], h_stats[4 * r + 2],
                          h_stats[4 * r + 3]};
        res->round_stats.insert(res->round_stats.end(), row, row + 6);
    }
    res->vertex_offsets.resize(B + 1);
    res->facet_offsets.resize(B + 1);
    for (int b = 0; b <= B; b++) {
        res->vertex_offsets[b] = h_voff[(size_t)R * (B + 1) + b];
        res->facet_offsets[b] = (R == 0) ? foff[b] : h_fo[b];
    }
    *out = res;
    return MF_OK;
}

}  // namespace mf
