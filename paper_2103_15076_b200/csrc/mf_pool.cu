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

static void scan_into(const Context* ctx, unsigned long long* status, const int* in, int* out, int n,
                      cudaStream_t s) {
    int tiles = std::max(1, (n + kScanTile - 1) / kScanTile);
    cudaMemsetAsync(status, 0, (size_t)(tiles + 1) * sizeof(unsigned long long), s);
    LAUNCH(k_scan_excl<LoadArr>, tiles, kScanBlock, 0, s, LoadArr{in}, n, out, status,
           reinterpret_cast<int*>(status + tiles), (const int*)nullptr, EpiNone(), (unsigned long long*)nullptr, 0);
    (void)ctx;
}

// CSR of the clusters of a device int32 replace (counts must already be
// known to cover every output vertex).  Members ascending within a cluster.
int build_cluster_csr(Context* ctx, const int* d_replace, int64_t n, int64_t n_out, int** d_off, int** d_members,
                      void** block, cudaStream_t stream, mf_status* st) {
    Arena me;
    me.measuring = true;
    auto lay = [&](Arena& A, int*& off, int*& mem, int*& cnt, int*& cur, int*& heavy, int*& tmp, int*& ctr,
                   unsigned long long*& sst) {
        off = A.take<int>((size_t)n_out + 1);
        mem = A.take<int>((size_t)n);
        cnt = A.take<int>((size_t)n_out + 1);
        cur = A.take<int>((size_t)n_out + 1);
        heavy = A.take<int>((size_t)n_out + 1);
        tmp = A.take<int>((size_t)n);
        ctr = A.take<int>(8);
        sst = A.take<unsigned long long>((size_t)(n_out + 1) / kScanTile + 4);
    };
    int *off, *mem, *cnt, *cur, *heavy, *tmp, *ctr;
    unsigned long long* sst;
    lay(me, off, mem, cnt, cur, heavy, tmp, ctr, sst);
    MF_CUDA_TRY(cudaMallocAsync(block, me.off, stream));
    Arena A;
    A.base = (char*)*block;
    A.cap = me.off;
    lay(A, off, mem, cnt, cur, heavy, tmp, ctr, sst);
    MF_CUDA_TRY(cudaMemsetAsync(cnt, 0, (size_t)(n_out + 1) * sizeof(int), stream));
    MF_CUDA_TRY(cudaMemsetAsync(cur, 0, (size_t)(n_out + 1) * sizeof(int), stream));
    MF_CUDA_TRY(cudaMemsetAsync(ctr, 0, 8 * sizeof(int), stream));
    LAUNCH(k_count_keys, grid_of(ctx, n), 256, 0, stream, n, d_replace, cnt);
    scan_into(ctx, sst, cnt, off, (int)n_out, stream);
    LAUNCH(k_csr_scatter, grid_of(ctx, n), 256, 0, stream, (int)n, nullptr, d_replace, off, cur, mem);
    LAUNCH(k_seg_sort_small, grid_of(ctx, n_out), 256, 0, stream, (int)n_out, nullptr, off, mem, heavy, ctr);
    LAUNCH(k_seg_sort_heavy, ctx->sm_count, 256, 0, stream, nullptr, off, mem, tmp, heavy, ctr);
    MF_CUDA_TRY(cudaGetLastError());
    *d_off = off;
    *d_members = mem;
    return MF_OK;
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
    size_t need = (hx ? xb : 0) + (hw ? wb : 0) + (ho ? ob : 0) + 256 * 4;
    MF_CUDA_TRY(cudaMallocAsync(&tmp, need, stream));
    char* p = (char*)tmp;
    int* d_flag = (int*)p;
    p += 256;
    MF_CUDA_TRY(cudaMemsetAsync(d_flag, 0, sizeof(int), stream));
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
        if (dtype == MF_DTYPE_F32)
            LAUNCH(k_pool<float>, grid_of(ctx, n_out * c), 256, 0, stream, n_out, (int)c, d_off, d_members,
                   (const float*)dX, (const float*)dW, mode, (float*)dO, d_flag);
        else
            LAUNCH(k_pool<double>, grid_of(ctx, n_out * c), 256, 0, stream, n_out, (int)c, d_off, d_members,
                   (const double*)dX, (const double*)dW, mode, (double*)dO, d_flag);
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
    size_t need = (hc ? cb + 256 : 0) + (ho ? ob + 256 : 0) + 256;
    MF_CUDA_TRY(cudaMallocAsync(&tmp, need, stream));
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
        if (row % 16 == 0 && ((uintptr_t)dC % 16) == 0 && ((uintptr_t)dO % 16) == 0) {
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
