// mf_pool.cu -- cluster pooling / unpooling over a `replace` tensor (pooling.py:18-77).
//
// The clusters of `replace` become a CSR (counting sort + ascending member
// order, reused from the decimation tiers), then one thread per
// (cluster, channel) folds its members sequentially -- consecutive threads
// walk consecutive channels of the same member row, so every member row is
// one coalesced read (C=64 float32: 256 B per row).  Unpool is a row gather
// with 16-byte vector moves when the row width allows.
#include <algorithm>
#include <cmath>
#include <cstdio>

#include "mf_internal.h"
#include "mf_kernels.cuh"

namespace mf {



static int grid_of(const Context* ctx, int64_t n, int block = 256) {
    int64_t g = (n + block - 1) / block;
    int64_t cap = (int64_t)ctx->sm_count * 16;
    return (int)std::max<int64_t>(1, std::min(g, cap));
}

__global__ void k_replace_in(int64_t n, const int64_t* __restrict__ r64, int64_t n_out, int* __restrict__ r32,
                             int* __restrict__ count, int* __restrict__ bad) {
    MF_PDL_ENTRY;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        int64_t r = r64[i];
        if (r < 0 || r >= n_out) {
            atomicExch(bad, 1);
            r32[i] = 0;
            continue;
        }
        r32[i] = (int)r;
        atomicAdd(count + r, 1);
    }
}
__global__ void k_count_keys(int64_t n, const int* __restrict__ key, int* __restrict__ count) {
    MF_PDL_ENTRY;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        atomicAdd(count + key[i], 1);
}
__global__ void k_check_cover(int64_t n_out, const int* __restrict__ count, int* __restrict__ empty) {
    MF_PDL_ENTRY;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n_out; i += (int64_t)gridDim.x * blockDim.x)
        if (count[i] == 0) atomicExch(empty, 1);
}

// x86 SSE NaN semantics for the folds: a NaN operand propagates with its
// payload (quieted), the first operand winning when both are NaN; NVIDIA FP32
// arithmetic would return the canonical 0x7fffffff instead.
MF_DEV float qnan_of(float a) { return __int_as_float(__float_as_int(a) | 0x00400000); }
MF_DEV double qnan_of(double a) {
    return __longlong_as_double(__double_as_longlong(a) | 0x0008000000000000ll);
}
template <typename T>
MF_DEV T x86_add(T a, T b) {
    if (a != a) return qnan_of(a);
    if (b != b) return qnan_of(b);
    return a + b;
}
template <typename T>
MF_DEV T x86_mul(T a, T b) {
    if (a != a) return qnan_of(a);
    if (b != b) return qnan_of(b);
    return a * b;
}
template <typename T>
MF_DEV T x86_div(T a, T b) {
    if (a != a) return qnan_of(a);
    if (b != b) return qnan_of(b);
    return a / b;
}
// cvtss2sd / cvtsd2ss keep the NaN payload (shifted into the wider mantissa)
MF_DEV double widen(float a) {
    if (a != a) {
        unsigned u = (unsigned)__float_as_int(a);
        unsigned long long d = ((unsigned long long)(u >> 31) << 63) | 0x7FF0000000000000ull |
                               ((unsigned long long)(u & 0x7FFFFF) << 29) | 0x0008000000000000ull;
        return __longlong_as_double((long long)d);
    }
    return (double)a;
}
MF_DEV float narrow(double a) {
    if (a != a) {
        unsigned long long d = (unsigned long long)__double_as_longlong(a);
        unsigned u = ((unsigned)(d >> 63) << 31) | 0x7F800000u | (unsigned)((d >> 29) & 0x7FFFFF) | 0x00400000u;
        return __int_as_float((int)u);
    }
    return (float)a;
}
MF_DEV double to_f64(double a) { return a; }
MF_DEV double to_f64(float a) { return widen(a); }
MF_DEV double avg_div(double acc, int cnt) { return x86_div(acc, (double)cnt); }
MF_DEV float avg_div(float acc, int cnt) { return narrow(x86_div(widen(acc), (double)cnt)); }

// pooling.py:36-71.  max: numpy maximum.at from -inf (later element wins ties,
// NaN sticky); average/sum: sequential fold in the input dtype,
// average divides in float64 and rounds back (in-place `/= int64 counts`);
// weighted: (w*x) folded in dtype over dtype-folded weights.
template <typename T>
__global__ void k_pool(int64_t n_out, int C, const int* __restrict__ off, const int* __restrict__ members,
                       const T* __restrict__ X, const T* __restrict__ w, int mode, T* __restrict__ out,
                       int* __restrict__ zero_weight) {
    MF_PDL_ENTRY;
    const int64_t total = n_out * (int64_t)C;
    for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
         idx += (int64_t)gridDim.x * blockDim.x) {
        int64_t r = idx / C;
        int k = (int)(idx - r * C);
        int s = off[r], e = off[r + 1];
        T acc;
        if (mode == MF_POOL_MAX) {
            acc = -INFINITY;
            for (int i = s; i < e; i++) {
                T v = X[(int64_t)members[i] * C + k];
                acc = (acc != acc || acc > v) ? acc : v;
            }
        } else if (mode == MF_POOL_WEIGHTED) {
            T den = (T)0;
            acc = (T)0;
            for (int i = s; i < e; i++) {
                int m = members[i];
                acc = x86_add(acc, x86_mul(X[(int64_t)m * C + k], w[m]));
                den = x86_add(den, w[m]);
            }
            if (den == (T)0) atomicExch(zero_weight, 1);
            acc = x86_div(acc, den);
        } else {
            acc = (T)0;
            for (int i = s; i < e; i++) acc = x86_add(acc, X[(int64_t)members[i] * C + k]);
            if (mode == MF_POOL_AVERAGE) acc = avg_div(acc, e - s);
        }
        out[idx] = acc;
    }
}

// ---- adjoints (pooling.py:80-102) ----
// sum: grad_in[v] = g[replace[v]];  average: g[replace[v]] / count (numpy promotes to float64);
// weighted: g[replace[v]] * (w[v] / denom[replace[v]]) with w, denom in the feature dtype.
template <typename TG, typename TF, typename TO>
__global__ void k_pool_bwd_gather(int64_t n, int C, const int* __restrict__ rep, const int* __restrict__ off,
                                  const int* __restrict__ members, const TG* __restrict__ g,
                                  const TF* __restrict__ w, int mode, TO* __restrict__ out) {
    MF_PDL_ENTRY;
    const int64_t total = n * (int64_t)C;
    for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
         idx += (int64_t)gridDim.x * blockDim.x) {
        const int64_t v = idx / C;
        const int k = (int)(idx - v * C);
        const int r = rep[v];
        const TG gv = g[(int64_t)r * C + k];
        if (mode == MF_POOL_SUM) {
            out[idx] = (TO)gv;
        } else if (mode == MF_POOL_AVERAGE) {
            out[idx] = (TO)x86_div(to_f64(gv), (double)(off[r + 1] - off[r]));
        } else {  // weighted
            TF den = (TF)0;
            for (int i = off[r]; i < off[r + 1]; i++) den = x86_add(den, w[members[i]]);
            TF q = x86_div(w[v], den);
            out[idx] = (TO)x86_mul((TO)gv, (TO)q);
        }
    }
}

// max: the winner of (cluster, channel) is the lowest member whose value equals the
// forward maximum (== : signed zeros tie, NaN never wins); it receives g, others 0.
template <typename TG, typename TF>
__global__ void k_pool_bwd_max(int64_t n_out, int C, const int* __restrict__ off, const int* __restrict__ members,
                               const TF* __restrict__ X, const TG* __restrict__ g, TF* __restrict__ out,
                               int* __restrict__ no_winner) {
    MF_PDL_ENTRY;
    const int64_t total = n_out * (int64_t)C;
    for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
         idx += (int64_t)gridDim.x * blockDim.x) {
        const int64_t r = idx / C;
        const int k = (int)(idx - r * C);
        TF acc = -INFINITY;
        for (int i = off[r]; i < off[r + 1]; i++) {
            TF v = X[(int64_t)members[i] * C + k];
            acc = (acc != acc || acc > v) ? acc : v;
        }
        int win = -1;
        for (int i = off[r]; i < off[r + 1]; i++)
            if (X[(int64_t)members[i] * C + k] == acc) {
                win = members[i];
                break;
            }
        if (win < 0) {
            atomicExch(no_winner, 1);
            continue;
        }
        out[(int64_t)win * C + k] = x86_add((TF)0, (TF)g[idx]);  // np.add.at into zeros: -0.0 -> +0.0
    }
}

// ---- vectorised forms (C * sizeof(T) a multiple of 16 B): L lanes per row, 16-byte loads ----
// A group of L lanes owns one output row; lane j handles 16-byte vectors j, j+L, ... of it.
// Member loop unrolled by U: the U member ids (broadcast loads) and then their U row vectors are
// in flight together before the in-order fold -- the fold order (ascending member, pooling.py
// np.add.at / maximum.at) is unchanged, only the loads are hoisted.
template <typename T>
struct Vec16;
template <>
struct Vec16<float> {
    static constexpr int E = 4;
    MF_DEV static void split(const uint4& u, float* x) {
        x[0] = __uint_as_float(u.x), x[1] = __uint_as_float(u.y), x[2] = __uint_as_float(u.z),
        x[3] = __uint_as_float(u.w);
    }
    MF_DEV static uint4 join(const float* x) {
        return make_uint4(__float_as_uint(x[0]), __float_as_uint(x[1]), __float_as_uint(x[2]), __float_as_uint(x[3]));
    }
};
template <>
struct Vec16<double> {
    static constexpr int E = 2;
    MF_DEV static void split(const uint4& u, double* x) {
        x[0] = __longlong_as_double(((long long)u.y << 32) | u.x);
        x[1] = __longlong_as_double(((long long)u.w << 32) | u.z);
    }
    MF_DEV static uint4 join(const double* x) {
        const unsigned long long a = (unsigned long long)__double_as_longlong(x[0]);
        const unsigned long long b = (unsigned long long)__double_as_longlong(x[1]);
        return make_uint4((unsigned)a, (unsigned)(a >> 32), (unsigned)b, (unsigned)(b >> 32));
    }
};

template <typename T, int L, int MODE>
__global__ void __launch_bounds__(256) k_pool_vec(int n_out, int row16, const int* __restrict__ off,
                                                  const int* __restrict__ members, const uint4* __restrict__ X,
                                                  const T* __restrict__ w, uint4* __restrict__ out,
                                                  int* __restrict__ zero_weight) {
    MF_PDL_ENTRY;
    constexpr int E = Vec16<T>::E;
    constexpr int U = 4;
    const int lane = threadIdx.x & (L - 1);
    const int G = (int)(((int64_t)gridDim.x * blockDim.x) / L);
    for (int r = (int)(((int64_t)blockIdx.x * blockDim.x + threadIdx.x) / L); r < n_out; r += G) {
        const int s = off[r], e = off[r + 1];
        for (int j = lane; j < row16; j += L) {
            T acc[E], den = (T)0;
#pragma unroll
            for (int k = 0; k < E; k++) acc[k] = MODE == MF_POOL_MAX ? (T)-INFINITY : (T)0;
            for (int i = s; i < e; i += U) {
                int m[U];
                uint4 raw[U];
                T wv[U];
#pragma unroll
                for (int u = 0; u < U; u++) m[u] = i + u < e ? __ldg(members + i + u) : -1;
#pragma unroll
                for (int u = 0; u < U; u++) {
                    if (m[u] >= 0) raw[u] = __ldg(X + (int64_t)m[u] * row16 + j);
                    if (MODE == MF_POOL_WEIGHTED && m[u] >= 0) wv[u] = __ldg(w + m[u]);
                }
#pragma unroll
                for (int u = 0; u < U; u++) {
                    if (m[u] < 0) break;
                    T x[E];
                    Vec16<T>::split(raw[u], x);
#pragma unroll
                    for (int k = 0; k < E; k++) {
                        if (MODE == MF_POOL_MAX) acc[k] = (acc[k] != acc[k] || acc[k] > x[k]) ? acc[k] : x[k];
                        else if (MODE == MF_POOL_WEIGHTED) acc[k] = x86_add(acc[k], x86_mul(x[k], wv[u]));
                        else acc[k] = x86_add(acc[k], x[k]);
                    }
                    if (MODE == MF_POOL_WEIGHTED) den = x86_add(den, wv[u]);
                }
            }
            if (MODE == MF_POOL_WEIGHTED) {
                if (den == (T)0) atomicExch(zero_weight, 1);
#pragma unroll
                for (int k = 0; k < E; k++) acc[k] = x86_div(acc[k], den);
            } else if (MODE == MF_POOL_AVERAGE) {
#pragma unroll
                for (int k = 0; k < E; k++) acc[k] = avg_div(acc[k], e - s);
            }
            out[(int64_t)r * row16 + j] = Vec16<T>::join(acc);
        }
    }
}

// unpool row gather: out[v] = coarse[rep[v]]; a group of L lanes per row, U rows in flight per
// group (rows g, g+G, ... so every store instruction of the grid covers consecutive rows)
template <int L, int U>
__global__ void __launch_bounds__(256) k_unpool_rows(int n, int row16, const int* __restrict__ rep,
                                                     const uint4* __restrict__ coarse, uint4* __restrict__ out) {
    MF_PDL_ENTRY;
    const int lane = threadIdx.x & (L - 1);
    const int G = (int)(((int64_t)gridDim.x * blockDim.x) / L);
    for (int v0 = (int)(((int64_t)blockIdx.x * blockDim.x + threadIdx.x) / L); v0 < n; v0 += G * U) {
        int r[U];
#pragma unroll
        for (int u = 0; u < U; u++) r[u] = v0 + u * G < n ? __ldg(rep + v0 + u * G) : -1;
        for (int j = lane; j < row16; j += L) {
            uint4 x[U];
#pragma unroll
            for (int u = 0; u < U; u++)
                if (r[u] >= 0) x[u] = __ldg(coarse + (int64_t)r[u] * row16 + j);
#pragma unroll
            for (int u = 0; u < U; u++)
                if (r[u] >= 0) __stcs(out + (int64_t)(v0 + u * G) * row16 + j, x[u]);
        }
    }
}

// ---- TMA (bulk-copy engine) form of the row gather: every lane of a warp issues one
// cp.async.bulk global->shared copy of a coarse row (the gather), an mbarrier with a transaction
// count tracks the tile's bytes, and one lane writes the tile's 32 consecutive output rows with a
// single cp.async.bulk shared->global store.  Two tiles per warp double-buffer so the next gather
// overlaps the current store.  The SM issues 33 bulk instructions per 32 rows instead of
// 32 x row16 vector loads + stores.
MF_DEV void bulk_s2g(void* dst, const void* src, unsigned bytes) {
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst), "r"(smem_u32(src)),
                 "r"(bytes)
                 : "memory");
}
MF_DEV void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
MF_DEV void bulk_wait_read0() { asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory"); }
MF_DEV void bulk_wait_read1() { asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory"); }

constexpr int kTmaWarps = 4;
// dynamic smem: per warp 2 buffers x 32 rows x row bytes, then 2 mbarriers per warp
__global__ void __launch_bounds__(kTmaWarps * 32) k_unpool_tma(int n, int row_bytes, const int* __restrict__ rep,
                                                                  const char* __restrict__ coarse, char* __restrict__ out) {
    MF_PDL_ENTRY;
    extern __shared__ __align__(128) unsigned char tma_smem[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const size_t tile_bytes = (size_t)32 * row_bytes;
    unsigned char* buf0 = tma_smem + (size_t)warp * 2 * tile_bytes;
    uint64_t* bars = reinterpret_cast<uint64_t*>(tma_smem + (size_t)kTmaWarps * 2 * tile_bytes) + warp * 2;
    if (lane == 0) {
        mbar_init(bars, 1);
        mbar_init(bars + 1, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncwarp();
    const int tiles = (n + 31) / 32;
    const int gw = blockIdx.x * kTmaWarps + warp, nw = gridDim.x * kTmaWarps;
    unsigned phase[2] = {0u, 0u};
    int k = 0;
    for (int t = gw; t < tiles; t += nw, k ^= 1) {
        unsigned char* buf = buf0 + (size_t)k * tile_bytes;
        const int v0 = t * 32;
        const int rows = min(32, n - v0);
        // the store that last used this buffer (two tiles ago) must have read it
        if (lane == 0) bulk_wait_read1();
        __syncwarp();
        if (lane == 0) mbar_expect_tx(bars + k, (unsigned)(rows * row_bytes));
        __syncwarp();
        if (lane < rows) bulk_g2s(buf + (size_t)lane * row_bytes, coarse + (size_t)__ldg(rep + v0 + lane) * row_bytes,
                                  (unsigned)row_bytes, bars + k);
        mbar_wait(bars + k, phase[k]);
        phase[k] ^= 1u;
        if (lane == 0) {
            bulk_s2g(out + (size_t)v0 * row_bytes, buf, (unsigned)(rows * row_bytes));
            bulk_commit();
        }
    }
    if (lane == 0) bulk_wait_read0();
    __syncwarp();
}

__global__ void k_unpool_vec(int64_t n, int64_t row16, const int* __restrict__ rep, const int4* __restrict__ coarse,
                             int4* __restrict__ out) {
    MF_PDL_ENTRY;
    const int64_t total = n * row16;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    for (; idx + 3 * stride < total; idx += 4 * stride) {  // four rows' gathers in flight
        int4 r[4];
#pragma unroll
        for (int q = 0; q < 4; q++) {
            const int64_t i = idx + q * stride, v = i / row16, j = i - v * row16;
            r[q] = __ldg(coarse + (int64_t)rep[v] * row16 + j);
        }
#pragma unroll
        for (int q = 0; q < 4; q++) out[idx + q * stride] = r[q];
    }
    for (; idx < total; idx += stride) {
        int64_t v = idx / row16, j = idx - v * row16;
        out[idx] = __ldg(coarse + (int64_t)rep[v] * row16 + j);
    }
}
template <typename T>
__global__ void k_unpool(int64_t n, int C, const int* __restrict__ rep, const T* __restrict__ coarse,
                         T* __restrict__ out) {
    MF_PDL_ENTRY;
    const int64_t total = n * (int64_t)C;
    for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
         idx += (int64_t)gridDim.x * blockDim.x) {
        int64_t v = idx / C;
        int k = (int)(idx - v * C);
        out[idx] = coarse[(int64_t)rep[v] * C + k];
    }
}


// Scatter by key into CSR slots, counting each cluster's counter back down to 0 (no cursor
// array to clear); the slot order within a cluster is fixed afterwards by the segment sort.
__global__ void k_csr_scatter_dec(int n, const int* __restrict__ key, const int* __restrict__ off,
                                  int* __restrict__ count, int* __restrict__ members) {
    MF_PDL_ENTRY;
    for (int v = blockIdx.x * blockDim.x + threadIdx.x; v < n; v += gridDim.x * blockDim.x) {
        const int r = key[v];
        members[off[r] + atomicSub(count + r, 1) - 1] = v;
    }
}

// Thread per cluster: <= 4 members sorted in registers (a sorting network: most clusters of a
// decimation are pairs plus a few absorbed vertices), up to kSmallDeg by insertion sort, longer
// ones to the heavy (block-sort) tier.
__global__ void k_seg_sort_small4(int nseg, const int* __restrict__ off, int* __restrict__ members,
                                  int* __restrict__ heavy, int* __restrict__ heavy_count) {
    MF_PDL_ENTRY;
    for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < nseg; r += gridDim.x * blockDim.x) {
        const int s = off[r], d = off[r + 1] - s;
        if (d <= 1) continue;
        if (d <= 4) {
            int a = members[s], b = members[s + 1];
            int c = d > 2 ? members[s + 2] : INT_MAX, e = d > 3 ? members[s + 3] : INT_MAX;
            int t;
#define MF_CSWAP(x, y) if (x > y) t = x, x = y, y = t
            MF_CSWAP(a, b);
            MF_CSWAP(c, e);
            MF_CSWAP(a, c);
            MF_CSWAP(b, e);
            MF_CSWAP(b, c);
#undef MF_CSWAP
            members[s] = a;
            members[s + 1] = b;
            if (d > 2) members[s + 2] = c;
            if (d > 3) members[s + 3] = e;
            continue;
        }
        if (d > kSmallDeg) {
            heavy[append_slot(heavy_count)] = r;
            continue;
        }
        int k[kSmallDeg];
        for (int i = 0; i < d; i++) k[i] = members[s + i];
        isort<kSmallDeg>(k, d);
        for (int i = 0; i < d; i++) members[s + i] = k[i];
    }
}

// One cooperative launch builds the whole cluster CSR: count -> scan -> scatter -> segment
// sort -> heavy segments, phases separated by a grid barrier (one block per SM, co-resident by
// construction of the cooperative launch).  Replaces five launches + a look-back scan whose
// fixed latencies dominated at pooling sizes (cfg3: ~107 us of CSR build per step).
// grid barrier of the cooperative launch (cooperative_groups grid sync)
MF_DEV void coop_bar(unsigned*, unsigned) { cooperative_groups::this_grid().sync(); }

__global__ void __launch_bounds__(1024) k_csr_coop(int n, int n_out, const int* __restrict__ key, int* __restrict__ cnt,
                                                   int* __restrict__ off, int* __restrict__ members,
                                                   int* __restrict__ heavy, int* __restrict__ ctr,
                                                   int* __restrict__ bsum, int* __restrict__ tmp) {
    MF_PDL_ENTRY;
    __shared__ int s_scan[33];
    __shared__ int s_sort[kChunk];
    unsigned* bar = reinterpret_cast<unsigned*>(ctr + 1);
    const unsigned G = gridDim.x;
    const int tid = blockIdx.x * blockDim.x + threadIdx.x, nth = gridDim.x * blockDim.x;
    // 1. cluster sizes
    for (int v = tid; v < n; v += nth) atomicAdd(cnt + key[v], 1);
    coop_bar(bar, 1 * G);
    // 2. exclusive scan: block b owns a contiguous chunk of the clusters
    const int chunk = (n_out + (int)G - 1) / (int)G;
    const int lo = min(n_out, (int)blockIdx.x * chunk), hi = min(n_out, lo + chunk);
    int part = 0;
    for (int i = lo + threadIdx.x; i < hi; i += blockDim.x) part += __ldcg(cnt + i);
    int tot;
    block_excl_scan(part, s_scan, &tot);
    if (threadIdx.x == 0) bsum[blockIdx.x] = tot;
    coop_bar(bar, 2 * G);
    int pre = 0;
    for (int b = threadIdx.x; b < (int)blockIdx.x; b += blockDim.x) pre += __ldcg(bsum + b);
    block_excl_scan(pre, s_scan, &tot);
    int run = tot;
    for (int i0 = lo; i0 < hi; i0 += blockDim.x) {
        const int i = i0 + threadIdx.x;
        const int x = i < hi ? __ldcg(cnt + i) : 0;
        const int ex = block_excl_scan(x, s_scan, &tot);
        if (i < hi) off[i] = run + ex;
        run += tot;
    }
    if (tid == 0) off[n_out] = n;
    coop_bar(bar, 3 * G);
    // 3. scatter (each cluster's counter counts back down to 0)
    for (int v = tid; v < n; v += nth) {
        const int r = key[v];
        members[__ldcg(off + r) + atomicSub(cnt + r, 1) - 1] = v;
    }
    coop_bar(bar, 4 * G);
    // 4. ascending member order: <= 4 in registers, <= kSmallDeg by insertion, longer listed
    for (int r = tid; r < n_out; r += nth) {
        const int s0 = __ldcg(off + r), d = __ldcg(off + r + 1) - s0;
        if (d <= 1) continue;
        if (d <= 4) {
            int a = __ldcg(members + s0), b = __ldcg(members + s0 + 1);
            int c = d > 2 ? __ldcg(members + s0 + 2) : INT_MAX, e = d > 3 ? __ldcg(members + s0 + 3) : INT_MAX;
            int t;
#define MF_CSWAP(x, y) if (x > y) t = x, x = y, y = t
            MF_CSWAP(a, b);
            MF_CSWAP(c, e);
            MF_CSWAP(a, c);
            MF_CSWAP(b, e);
            MF_CSWAP(b, c);
#undef MF_CSWAP
            members[s0] = a;
            members[s0 + 1] = b;
            if (d > 2) members[s0 + 2] = c;
            if (d > 3) members[s0 + 3] = e;
        } else if (d > kSmallDeg) {
            heavy[atomicAdd(ctr, 1)] = r;
        } else {
            int k[kSmallDeg];
            for (int i = 0; i < d; i++) k[i] = __ldcg(members + s0 + i);
            isort<kSmallDeg>(k, d);
            for (int i = 0; i < d; i++) members[s0 + i] = k[i];
        }
    }
    coop_bar(bar, 5 * G);
    // 5. long segments: one block each
    const int H = __ldcg(ctr);
    for (int h = blockIdx.x; h < H; h += gridDim.x) {
        const int r = __ldcg(heavy + h);
        const int s0 = __ldcg(off + r), d = __ldcg(off + r + 1) - s0;
        block_sort_ints(members + s0, tmp + s0, d, s_sort);
    }
}

// vertices per k_csr_coop block (MF_CSR_PER_BLOCK; a huge value = one block, 1 = one per SM)
static int64_t csr_per_block() {
    static int64_t v = -1;
    if (v < 0) {
        const char* e = getenv("MF_CSR_PER_BLOCK");
        v = e ? std::max(1, atoi(e)) : 1;
    }
    return v;
}

// cooperative CSR build available (MF_CSR_COOP=0 forces the five-launch path for A/B runs)
static int g_csr_blocks_per_sm = 1;
static bool csr_coop_ok(const Context* ctx) {
    static int v = -1;
    if (v < 0) {
        const char* e = getenv("MF_CSR_COOP");
        int occ = 0;
        v = (e && e[0] == '0') ? 0 : 1;
        if (v && (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_csr_coop, 1024, 0) != cudaSuccess || occ < 1))
            v = 0;
        cudaGetLastError();
        g_csr_blocks_per_sm = 1;  // one block per SM: fewest barrier arrivals
    }
    (void)ctx;
    return v == 1;
}

// CSR of the clusters of a device int32 replace (every key in [0, n_out)).  Members ascending
// within a cluster.  One clearing memset, then count -> scan -> scatter -> segment sort.
int build_cluster_csr(Context* ctx, const int* d_replace, int64_t n, int64_t n_out, int** d_off, int** d_members,
                      void** block, cudaStream_t stream, mf_status* st) {
    const int scan_tiles = std::max(1, (int)((n_out + kScanTile - 1) / kScanTile));
    const int tiles = std::max(ctx->sm_count * 2, scan_tiles);  // the state words also hold the coop block sums
    Arena me;
    me.measuring = true;
    auto lay = [&](Arena& A, int*& off, int*& mem, int*& cnt, int*& heavy, int*& tmp, int*& ctr,
                   unsigned long long*& sst) {
        off = A.take<int>((size_t)n_out + 1);
        mem = A.take<int>((size_t)n);
        heavy = A.take<int>((size_t)n_out + 1);
        tmp = A.take<int>((size_t)n);
        cnt = A.take<int>((size_t)n_out + 1);  // cnt | ctr | scan state: cleared by one memset
        ctr = A.take<int>(8);
        sst = A.take<unsigned long long>((size_t)tiles + 4);
    };
    int *off, *mem, *cnt, *heavy, *tmp, *ctr;
    unsigned long long* sst;
    lay(me, off, mem, cnt, heavy, tmp, ctr, sst);
    MF_CUDA_TRY(cudaMallocAsync(block, me.off, stream));
    Arena A;
    A.base = (char*)*block;
    A.cap = me.off;
    lay(A, off, mem, cnt, heavy, tmp, ctr, sst);
    MF_CUDA_TRY(cudaMemsetAsync(cnt, 0, (size_t)((char*)(sst + tiles + 4) - (char*)cnt), stream));
    if (csr_coop_ok(ctx)) {
        // bsum reuses the scan-state words (tiles + 4 >= grid blocks is ensured by csr_coop_ok)
        int* bsum = reinterpret_cast<int*>(sst);
        int nn = (int)n, no = (int)n_out;
        void* args[] = {&nn, &no, (void*)&d_replace, &cnt, &off, &mem, &heavy, &ctr, &bsum, &tmp};
        // one block per SM (MF_CSR_PER_BLOCK=n: a block per n vertices -- fewer barrier arrivals
        // for small levels -- measured slower: cfg3 k_csr_coop 0.162 ms at 8192, 0.106 ms at 1)
        const int64_t want = (n + csr_per_block() - 1) / csr_per_block();
        const int blocks = (int)std::max<int64_t>(1, std::min<int64_t>(want, ctx->sm_count * g_csr_blocks_per_sm));
        prof_pre("k_csr_coop", stream);
        cudaError_t e = cudaLaunchCooperativeKernel((const void*)k_csr_coop, dim3(blocks), dim3(1024), args, 0,
                                                    stream);
        prof_post("k_csr_coop", stream);
        g_launches++;
        MF_CUDA_TRY(e);
        *d_off = off;
        *d_members = mem;
        return MF_OK;
    }
    LAUNCH(k_count_keys, grid_of(ctx, n), 256, 0, stream, n, d_replace, cnt);
    LAUNCH(k_scan_excl<LoadArr>, scan_tiles, kScanBlock, 0, stream, LoadArr{cnt}, (int)n_out, off, sst,
           reinterpret_cast<int*>(sst + tiles), (const int*)nullptr, EpiNone(), (unsigned long long*)nullptr, 0);
    LAUNCH(k_csr_scatter_dec, grid_of(ctx, n), 256, 0, stream, (int)n, d_replace, off, cnt, mem);
    LAUNCH(k_seg_sort_small4, grid_of(ctx, n_out), 256, 0, stream, (int)n_out, off, mem, heavy, ctr);
    LAUNCH(k_seg_sort_heavy, ctx->sm_count, 256, 0, stream, nullptr, off, mem, tmp, heavy, ctr);
    MF_CUDA_TRY(cudaGetLastError());
    *d_off = off;
    *d_members = mem;
    return MF_OK;
}

// MF_POOL_SCALAR=1: the thread-per-(cluster, channel) kernels even for 16-byte rows (A/B runs)
static bool pool_scalar_forced() {
    static int v = -1;
    if (v < 0) {
        const char* e = getenv("MF_POOL_SCALAR");
        v = (e && e[0] == '1') ? 1 : 0;
    }
    return v == 1;
}

// MF_UNPOOL_TMA=1: the bulk-copy (TMA) row gather instead of the LSU one (A/B runs)
static bool unpool_tma() {
    static int v = -1;
    if (v < 0) {
        const char* e = getenv("MF_UNPOOL_TMA");
        v = (e && e[0] == '1') ? 1 : 0;
    }
    return v == 1;
}

static int lanes_for(int row16) {  // lanes per row: the row's vectors, 4..32
    int L = 4;
    while (L < row16 && L < 32) L <<= 1;
    return L;
}

template <typename T, int L>
static void launch_pool_vec_l(Context* ctx, int64_t n_out, int row16, const int* off, const int* mem, const void* X,
                              const void* W, int mode, void* O, int* flag, cudaStream_t s) {
    const int grid = grid_of(ctx, n_out * L);
    const uint4* x = (const uint4*)X;
    uint4* o = (uint4*)O;
    const T* w = (const T*)W;
    if (mode == MF_POOL_MAX) LAUNCH((k_pool_vec<T, L, MF_POOL_MAX>), grid, 256, 0, s, (int)n_out, row16, off, mem, x, w, o, flag);
    else if (mode == MF_POOL_WEIGHTED)
        LAUNCH((k_pool_vec<T, L, MF_POOL_WEIGHTED>), grid, 256, 0, s, (int)n_out, row16, off, mem, x, w, o, flag);
    else if (mode == MF_POOL_AVERAGE)
        LAUNCH((k_pool_vec<T, L, MF_POOL_AVERAGE>), grid, 256, 0, s, (int)n_out, row16, off, mem, x, w, o, flag);
    else LAUNCH((k_pool_vec<T, L, MF_POOL_SUM>), grid, 256, 0, s, (int)n_out, row16, off, mem, x, w, o, flag);
}
template <typename T>
static void launch_pool_vec(Context* ctx, int64_t n_out, int row16, const int* off, const int* mem, const void* X,
                            const void* W, int mode, void* O, int* flag, cudaStream_t s) {
    switch (lanes_for(row16)) {
        case 4: launch_pool_vec_l<T, 4>(ctx, n_out, row16, off, mem, X, W, mode, O, flag, s); break;
        case 8: launch_pool_vec_l<T, 8>(ctx, n_out, row16, off, mem, X, W, mode, O, flag, s); break;
        case 16: launch_pool_vec_l<T, 16>(ctx, n_out, row16, off, mem, X, W, mode, O, flag, s); break;
        default: launch_pool_vec_l<T, 32>(ctx, n_out, row16, off, mem, X, W, mode, O, flag, s); break;
    }
}

int pool_run(Context* ctx, const void* features, int dtype, int64_t n, int64_t c, const int* d_replace,
             const int* d_off, const int* d_members, int64_t n_out, int mode, const void* weights, void* out,
             cudaStream_t stream, mf_status* st) {
    const size_t es = dtype == MF_DTYPE_F32 ? 4 : 8;
    const void* dX = features;
    const void* dW = weights;
    void* dO = out;
    void* tmp = nullptr;
    size_t xb = (size_t)(n * c) * es, wb = (mode == MF_POOL_WEIGHTED) ? (size_t)n * es : 0,
           ob = (size_t)(n_out * c) * es;
    bool hx = !is_device_ptr(features), hw = wb && !is_device_ptr(weights), ho = !is_device_ptr(out);
    // device buffers and no data-dependent error to report: stream-ordered, no allocation, no wait
    const bool wait = hx || hw || ho || mode == MF_POOL_WEIGHTED;
    int* d_flag = nullptr;
    char* p = nullptr;
    if (wait) {
        size_t need = (hx ? xb : 0) + (hw ? wb : 0) + (ho ? ob : 0) + 256 * 4;
        MF_CUDA_TRY(cudaMallocAsync(&tmp, need, stream));
        p = (char*)tmp;
        d_flag = (int*)p;
        p += 256;
        MF_CUDA_TRY(cudaMemsetAsync(d_flag, 0, sizeof(int), stream));
    }
    if (hx) {
        MF_CUDA_TRY(cudaMemcpyAsync(p, features, xb, cudaMemcpyHostToDevice, stream));
        dX = p;
        p += (xb + 255) & ~size_t(255);
    }
    if (hw) {
        MF_CUDA_TRY(cudaMemcpyAsync(p, weights, wb, cudaMemcpyHostToDevice, stream));
        dW = p;
        p += (wb + 255) & ~size_t(255);
    }
    if (ho) dO = p;
    if (n_out * c > 0) {
        const size_t row = (size_t)c * es;
        if (row % 16 == 0 && ((uintptr_t)dX % 16) == 0 && ((uintptr_t)dO % 16) == 0 && !pool_scalar_forced()) {
            if (dtype == MF_DTYPE_F32) launch_pool_vec<float>(ctx, n_out, (int)(row / 16), d_off, d_members, dX, dW,
                                                              mode, dO, d_flag, stream);
            else launch_pool_vec<double>(ctx, n_out, (int)(row / 16), d_off, d_members, dX, dW, mode, dO, d_flag,
                                         stream);
        } else if (dtype == MF_DTYPE_F32)
            LAUNCH(k_pool<float>, grid_of(ctx, n_out * c), 256, 0, stream, n_out, (int)c, d_off, d_members,
                   (const float*)dX, (const float*)dW, mode, (float*)dO, d_flag);
        else
            LAUNCH(k_pool<double>, grid_of(ctx, n_out * c), 256, 0, stream, n_out, (int)c, d_off, d_members,
                   (const double*)dX, (const double*)dW, mode, (double*)dO, d_flag);
    }
    if (!wait) {
        MF_CUDA_TRY(cudaGetLastError());
        return MF_OK;
    }
    if (ho) MF_CUDA_TRY(cudaMemcpyAsync(out, dO, ob, cudaMemcpyDeviceToHost, stream));
    int h_flag = 0;
    MF_CUDA_TRY(cudaMemcpyAsync(&h_flag, d_flag, sizeof(int), cudaMemcpyDeviceToHost, stream));
    MF_CUDA_TRY(cudaFreeAsync(tmp, stream));
    MF_CUDA_TRY(cudaStreamSynchronize(stream));
    MF_CUDA_TRY(cudaGetLastError());
    if (h_flag) {
        st->code = MF_ERR_VALUE;
        snprintf(st->message, sizeof(st->message), "weighted pooling: some cluster has zero total weight");
        return st->code;
    }
    return MF_OK;
}

// out dtype: average -> f64; sum -> grad dtype; weighted -> promote(grad, features); max -> features dtype
int pool_backward_run(Context* ctx, const void* grad, int gdtype, const void* features, int fdtype, int64_t n,
                      int64_t c, const int* d_replace, const int* d_off, const int* d_members, int64_t n_out, int mode,
                      const void* weights, void* out, int odtype, cudaStream_t stream, mf_status* st) {
    auto es = [](int d) { return d == MF_DTYPE_F32 ? (size_t)4 : (size_t)8; };
    size_t gb = (size_t)(n_out * c) * es(gdtype), xb = (mode == MF_POOL_MAX) ? (size_t)(n * c) * es(fdtype) : 0,
           wb = (mode == MF_POOL_WEIGHTED) ? (size_t)n * es(fdtype) : 0, ob = (size_t)(n * c) * es(odtype);
    bool hg = !is_device_ptr(grad), hx = xb && !is_device_ptr(features), hw = wb && !is_device_ptr(weights),
         ho = !is_device_ptr(out);
    void* tmp = nullptr;
    MF_CUDA_TRY(cudaMallocAsync(&tmp, 1024 + (hg ? gb : 0) + (hx ? xb : 0) + (hw ? wb : 0) + (ho ? ob : 0), stream));
    char* p = (char*)tmp;
    int* flag = (int*)p;
    p += 256;
    auto stage = [&](bool host, const void* src, size_t bytes) -> const void* {
        if (!host) return src;
        cudaMemcpyAsync(p, src, bytes, cudaMemcpyHostToDevice, stream);
        const void* r = p;
        p += (bytes + 255) & ~size_t(255);
        return r;
    };
    const void* dG = stage(hg, grad, gb);
    const void* dX = xb ? stage(hx, features, xb) : nullptr;
    const void* dW = wb ? stage(hw, weights, wb) : nullptr;
    void* dO = ho ? (void*)p : out;
    MF_CUDA_TRY(cudaMemsetAsync(flag, 0, 4, stream));
    const bool f32g = gdtype == MF_DTYPE_F32, f32f = fdtype == MF_DTYPE_F32, f32o = odtype == MF_DTYPE_F32;
    if (n * c > 0) {
        if (mode == MF_POOL_MAX) {
            MF_CUDA_TRY(cudaMemsetAsync(dO, 0, ob, stream));
#define MFBWD_MAX(TG, TF) \
    LAUNCH((k_pool_bwd_max<TG, TF>), grid_of(ctx, n_out * c), 256, 0, stream, n_out, (int)c, d_off, d_members, \
           (const TF*)dX, (const TG*)dG, (TF*)dO, flag)
            if (f32g && f32f) MFBWD_MAX(float, float);
            else if (f32g) MFBWD_MAX(float, double);
            else if (f32f) MFBWD_MAX(double, float);
            else MFBWD_MAX(double, double);
#undef MFBWD_MAX
        } else {
#define MFBWD_G(TG, TF, TO) \
    LAUNCH((k_pool_bwd_gather<TG, TF, TO>), grid_of(ctx, n * c), 256, 0, stream, n, (int)c, d_replace, d_off, \
           d_members, (const TG*)dG, (const TF*)dW, mode, (TO*)dO)
            if (f32g && f32f && f32o) MFBWD_G(float, float, float);
            else if (f32g && f32f) MFBWD_G(float, float, double);
            else if (f32g && !f32f) MFBWD_G(float, double, double);
            else if (!f32g && f32f) MFBWD_G(double, float, double);
            else MFBWD_G(double, double, double);
#undef MFBWD_G
        }
    }
    if (ho) MF_CUDA_TRY(cudaMemcpyAsync(out, dO, ob, cudaMemcpyDeviceToHost, stream));
    int h_flag = 0;
    MF_CUDA_TRY(cudaMemcpyAsync(&h_flag, flag, 4, cudaMemcpyDeviceToHost, stream));
    MF_CUDA_TRY(cudaFreeAsync(tmp, stream));
    MF_CUDA_TRY(cudaStreamSynchronize(stream));
    MF_CUDA_TRY(cudaGetLastError());
    if (h_flag) {
        st->code = MF_ERR_VALUE;
        snprintf(st->message, sizeof(st->message), "max pooling backward: a cluster's maximum is NaN (no winner row)");
        return st->code;
    }
    return MF_OK;
}

int unpool_run(Context* ctx, const void* coarse, int dtype, int64_t n_out, int64_t c, const int* d_replace, int64_t n,
               void* out, cudaStream_t stream, mf_status* st) {
    const size_t es = dtype == MF_DTYPE_F32 ? 4 : 8;
    size_t cb = (size_t)(n_out * c) * es, ob = (size_t)(n * c) * es;
    bool hc = !is_device_ptr(coarse), ho = !is_device_ptr(out);
    void* tmp = nullptr;
    const bool wait = hc || ho;  // device buffers only: stream-ordered, no allocation, no wait
    size_t need = (hc ? cb + 256 : 0) + (ho ? ob + 256 : 0) + 256;
    if (wait) MF_CUDA_TRY(cudaMallocAsync(&tmp, need, stream));
    char* p = (char*)tmp;
    const void* dC = coarse;
    void* dO = out;
    if (hc) {
        MF_CUDA_TRY(cudaMemcpyAsync(p, coarse, cb, cudaMemcpyHostToDevice, stream));
        dC = p;
        p += (cb + 255) & ~size_t(255);
    }
    if (ho) dO = p;
    const size_t row = (size_t)c * es;
    if (n * c > 0) {
        if (unpool_tma() && row % 16 == 0 && row <= 1024 && ((uintptr_t)dC % 16) == 0 && ((uintptr_t)dO % 16) == 0) {
            const size_t smem = (size_t)kTmaWarps * 2 * 32 * row + kTmaWarps * 2 * 8;
            // per call: the attribute is per device, and calls may come from several threads
            cudaFuncSetAttribute(k_unpool_tma, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
            const int tiles = (int)((n + 31) / 32);
            const int grid = std::max(1, std::min((tiles + kTmaWarps - 1) / kTmaWarps, ctx->sm_count * 8));
            LAUNCH(k_unpool_tma, grid, kTmaWarps * 32, smem, stream, (int)n, (int)row, d_replace, (const char*)dC,
                   (char*)dO);
        } else if (row % 16 == 0 && ((uintptr_t)dC % 16) == 0 && ((uintptr_t)dO % 16) == 0 && !pool_scalar_forced()) {
            const int row16 = (int)(row / 16);
            const int L = lanes_for(row16);
            // up to two waves of groups: one row per group (latency-bound sizes); beyond, 4 rows in
            // flight per group
            const bool deep = (int64_t)n * L > (int64_t)ctx->sm_count * 2048 * 2;
            const int grid = grid_of(ctx, deep ? (n * L + 3) / 4 : n * L);
            const uint4* x = (const uint4*)dC;
            uint4* o = (uint4*)dO;
#define MF_UNPOOL(LL)                                                                                   \
    do {                                                                                               \
        if (deep) LAUNCH((k_unpool_rows<LL, 4>), grid, 256, 0, stream, (int)n, row16, d_replace, x, o); \
        else LAUNCH((k_unpool_rows<LL, 1>), grid, 256, 0, stream, (int)n, row16, d_replace, x, o);      \
    } while (0)
            if (L == 4) MF_UNPOOL(4);
            else if (L == 8) MF_UNPOOL(8);
            else if (L == 16) MF_UNPOOL(16);
            else MF_UNPOOL(32);
#undef MF_UNPOOL
        } else if (row % 16 == 0 && ((uintptr_t)dC % 16) == 0 && ((uintptr_t)dO % 16) == 0) {
            int64_t row16 = (int64_t)(row / 16);
            LAUNCH(k_unpool_vec, grid_of(ctx, n * row16), 256, 0, stream, n, row16, d_replace, (const int4*)dC,
                   (int4*)dO);
        } else if (dtype == MF_DTYPE_F32) {
            LAUNCH(k_unpool<float>, grid_of(ctx, n * c), 256, 0, stream, n, (int)c, d_replace, (const float*)dC,
                   (float*)dO);
        } else {
            LAUNCH(k_unpool<double>, grid_of(ctx, n * c), 256, 0, stream, n, (int)c, d_replace, (const double*)dC,
                   (double*)dO);
        }
    }
    if (!wait) {
        MF_CUDA_TRY(cudaGetLastError());
        return MF_OK;
    }
    if (ho) MF_CUDA_TRY(cudaMemcpyAsync(out, dO, ob, cudaMemcpyDeviceToHost, stream));
    MF_CUDA_TRY(cudaFreeAsync(tmp, stream));
    MF_CUDA_TRY(cudaStreamSynchronize(stream));
    MF_CUDA_TRY(cudaGetLastError());
    return MF_OK;
}

// replace int64 (host or device) -> device int32 with range check + cluster counts.
int upload_replace(Context* ctx, const int64_t* replace, int64_t n, int64_t n_out, int check_cover, int** d_r32,
                   int** d_count, void** block, cudaStream_t stream, mf_status* st) {
    size_t rb = ((size_t)n * 4 + 255) & ~size_t(255), cb = (((size_t)n_out + 1) * 4 + 255) & ~size_t(255);
    size_t hb = is_device_ptr(replace) ? 0 : (((size_t)n * 8 + 255) & ~size_t(255));
    MF_CUDA_TRY(cudaMallocAsync(block, rb + cb + hb + 512, stream));
    char* p = (char*)*block;
    *d_r32 = (int*)p;
    *d_count = (int*)(p + rb);
    int* flags = (int*)(p + rb + cb);
    const int64_t* src = replace;
    if (hb) {
        int64_t* staged = (int64_t*)(p + rb + cb + 512);
        MF_CUDA_TRY(cudaMemcpyAsync(staged, replace, (size_t)n * 8, cudaMemcpyHostToDevice, stream));
        src = staged;
    }
    MF_CUDA_TRY(cudaMemsetAsync(*d_count, 0, ((size_t)n_out + 1) * 4, stream));
    MF_CUDA_TRY(cudaMemsetAsync(flags, 0, 8, stream));
    if (n > 0) LAUNCH(k_replace_in, grid_of(ctx, n), 256, 0, stream, n, src, n_out, *d_r32, *d_count, flags);
    if (n_out > 0 && check_cover) LAUNCH(k_check_cover, grid_of(ctx, n_out), 256, 0, stream, n_out, *d_count, flags + 1);
    int h[2] = {0, 0};
    MF_CUDA_TRY(cudaMemcpyAsync(h, flags, 8, cudaMemcpyDeviceToHost, stream));
    MF_CUDA_TRY(cudaStreamSynchronize(stream));
    if (h[0]) {
        st->code = MF_ERR_VALUE;
        snprintf(st->message, sizeof(st->message), "replace holds indices outside [0, %lld)", (long long)n_out);
        return st->code;
    }
    if (h[1]) {
        st->code = MF_ERR_RUNTIME;
        snprintf(st->message, sizeof(st->message), "replace tensor does not cover every output vertex");
        return st->code;
    }
    return MF_OK;
}

}  // namespace mf
