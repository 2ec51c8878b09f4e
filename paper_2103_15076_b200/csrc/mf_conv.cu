// mf_conv.cu -- the first network consumer of a decimation: facet2vertex
// evaluated at the cluster representatives (strided facet2vertex,
// conv.py:206-250 with vertex_ids = representative_vertices(result),
// decimate.py:118-123), plus the vertex -> facet adjacency it reads
// (vertex_facet_adjacency, mesh.py:114-122).
//
// Arithmetic follows the reference exactly: effective filter
// eff(f, c, l) = sum_t coeff[f, t] * w[t, c, l] summed sequentially over t
// (numpy einsum 'ft,tcl->fcl', checked bitwise), contribution eff * x[f, c],
// folded from +0.0 over the vertex's facets in ascending facet order
// (np.add.at over the stable-argsort adjacency), then divided by the count.
// float32 features accumulate like np.add.at into a float32 array: each step
// is a float64 add rounded to float32; the final in-place divide by the
// int64 count is a float64 divide rounded to float32.
#include "mf_internal.h"
#include "mf_kernels.cuh"

namespace mf {

// flat incidence index (3 f + corner, ascending within a vertex) -> facet id, widened
__global__ void k_adj_facets(int64_t nnz, const int* __restrict__ members, int64_t* __restrict__ facet_ids) {
    MF_PDL_ENTRY;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nnz; i += (int64_t)gridDim.x * blockDim.x)
        facet_ids[i] = members[i] / 3;
}

// one warp per output row; lanes over (channel, multiplier) pairs
template <typename T>
__global__ void __launch_bounds__(256) k_f2v(int rows, const int64_t* __restrict__ vertex_ids,
                                             const int64_t* __restrict__ offsets,
                                             const int64_t* __restrict__ facet_ids, const T* __restrict__ X, int C,
                                             const double* __restrict__ W, int nt, int L,
                                             const double* __restrict__ coeff, T* __restrict__ out) {
    MF_PDL_ENTRY;
    const int lane = threadIdx.x & 31;
    const int warps = gridDim.x * (blockDim.x >> 5);
    const int CL = C * L;
    for (int r = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); r < rows; r += warps) {
        const int64_t v = vertex_ids ? vertex_ids[r] : r;
        const int64_t a = offsets[v], b = offsets[v + 1];
        for (int j = lane; j < CL; j += 32) {
            const int c = j / L, l = j - c * L;
            double acc = 0.0;
            T acc_t = (T)0;
            for (int64_t i = a; i < b; i++) {
                const int64_t f = facet_ids[i];
                const double* cf = coeff + (size_t)f * nt;
                double eff = 0.0;
                for (int t = 0; t < nt; t++) eff = eff + cf[t] * W[((size_t)t * C + c) * L + l];
                const double contrib = eff * (double)X[(size_t)f * C + c];
                if (sizeof(T) == 8) acc = acc + contrib;
                else acc_t = (T)((double)acc_t + contrib);
            }
            const int64_t cnt = b - a;
            T o;
            if (sizeof(T) == 8) o = (T)(cnt ? acc / (double)cnt : acc);
            else o = cnt ? (T)((double)acc_t / (double)cnt) : acc_t;
            out[(size_t)r * CL + j] = o;
        }
    }
}

static int grid_rows(const Context* ctx, int64_t rows) {
    int64_t g = (rows + 7) / 8;
    int64_t cap = (int64_t)ctx->sm_count * 32;
    return (int)std::max<int64_t>(1, std::min(g, cap));
}

int adjacency_run(Context* ctx, const int64_t* facets, int64_t m, int64_t n, int64_t* offsets, int64_t* facet_ids,
                  cudaStream_t stream, mf_status* st) {
    if (3 * m >= (int64_t)INT32_MAX - 1 || n >= (int64_t)INT32_MAX - 1) {
        st->code = MF_ERR_LIMIT;
        snprintf(st->message, sizeof(st->message), "mesh too large for 32-bit device indices");
        return st->code;
    }
    int *k32 = nullptr, *cnt = nullptr, *off = nullptr, *mem = nullptr;
    void *blk_k = nullptr, *blk_csr = nullptr, *blk_o = nullptr;
    int rc = upload_replace(ctx, facets, 3 * m, n, 0, &k32, &cnt, &blk_k, stream, st);
    if (rc == MF_ERR_VALUE) snprintf(st->message, sizeof(st->message), "facets reference vertices outside [0, %lld)",
                                     (long long)n);
    if (rc == MF_OK) rc = build_cluster_csr(ctx, k32, 3 * m, n, &off, &mem, &blk_csr, stream, st);
    if (rc == MF_OK) {
        const bool ho = !is_device_ptr(offsets), hf = !is_device_ptr(facet_ids);
        const size_t ob = (size_t)(n + 1) * 8, fb = (size_t)(3 * m) * 8;
        cudaError_t e = cudaMallocAsync(&blk_o, ob + fb + 512, stream);
        if (e == cudaSuccess) {
            int64_t* d_off = ho ? (int64_t*)blk_o : offsets;
            int64_t* d_fid = hf ? (int64_t*)((char*)blk_o + ((ob + 255) & ~size_t(255))) : facet_ids;
            LAUNCH(k_i32_to_i64, grid_of(ctx, n + 1), 256, 0, stream, n + 1, off, d_off, 0);
            if (m) LAUNCH(k_adj_facets, grid_of(ctx, 3 * m), 256, 0, stream, 3 * m, mem, d_fid);
            e = cudaGetLastError();
            if (e == cudaSuccess && ho) e = cudaMemcpyAsync(offsets, d_off, ob, cudaMemcpyDeviceToHost, stream);
            if (e == cudaSuccess && hf && m) e = cudaMemcpyAsync(facet_ids, d_fid, fb, cudaMemcpyDeviceToHost, stream);
            if (e == cudaSuccess) e = cudaStreamSynchronize(stream);
        }
        if (e != cudaSuccess) {
            st->code = rc = MF_ERR_CUDA;
            snprintf(st->message, sizeof(st->message), "%s", cudaGetErrorString(e));
        }
    }
    if (blk_k) cudaFreeAsync(blk_k, stream);
    if (blk_csr) cudaFreeAsync(blk_csr, stream);
    if (blk_o) cudaFreeAsync(blk_o, stream);
    return rc;
}

// host or device inputs; every host array is staged once
int f2v_run(Context* ctx, const int64_t* offsets, int64_t n, const int64_t* facet_ids, const void* X, int dtype,
            int64_t m, int64_t C, const double* W, int64_t nt, int64_t L, const double* coeff,
            const int64_t* vertex_ids, int64_t rows, void* out, cudaStream_t stream, mf_status* st) {
    const size_t es = dtype == MF_DTYPE_F32 ? 4 : 8;
    const int64_t nnz = 3 * m;
    struct Arr {
        const void* src;
        size_t bytes;
        const void* dev;
    } arrs[6] = {{offsets, (size_t)(n + 1) * 8, nullptr}, {facet_ids, (size_t)nnz * 8, nullptr},
                 {X, (size_t)(m * C) * es, nullptr},        {W, (size_t)(nt * C * L) * 8, nullptr},
                 {coeff, (size_t)(m * nt) * 8, nullptr},    {vertex_ids, (size_t)rows * 8, nullptr}};
    size_t need = 256;
    for (auto& a : arrs)
        if (a.src && a.bytes && !is_device_ptr(a.src)) need += (a.bytes + 255) & ~size_t(255);
    const bool ho = !is_device_ptr(out);
    const size_t ob = (size_t)(rows * C * L) * es;
    if (ho) need += (ob + 255) & ~size_t(255);
    void* blk = nullptr;
    MF_CUDA_TRY(cudaMallocAsync(&blk, need, stream));
    char* p = (char*)blk;
    for (auto& a : arrs) {
        a.dev = a.src;
        if (a.src && a.bytes && !is_device_ptr(a.src)) {
            cudaError_t e = cudaMemcpyAsync(p, a.src, a.bytes, cudaMemcpyHostToDevice, stream);
            if (e != cudaSuccess) {
                cudaFreeAsync(blk, stream);
                MF_CUDA_TRY(e);
            }
            a.dev = p;
            p += (a.bytes + 255) & ~size_t(255);
        }
    }
    void* d_out = ho ? (void*)p : out;
    if (rows > 0 && C * L > 0) {
        if (dtype == MF_DTYPE_F32)
            LAUNCH(k_f2v<float>, grid_rows(ctx, rows), 256, 0, stream, (int)rows, (const int64_t*)arrs[5].dev,
                   (const int64_t*)arrs[0].dev, (const int64_t*)arrs[1].dev, (const float*)arrs[2].dev, (int)C,
                   (const double*)arrs[3].dev, (int)nt, (int)L, (const double*)arrs[4].dev, (float*)d_out);
        else
            LAUNCH(k_f2v<double>, grid_rows(ctx, rows), 256, 0, stream, (int)rows, (const int64_t*)arrs[5].dev,
                   (const int64_t*)arrs[0].dev, (const int64_t*)arrs[1].dev, (const double*)arrs[2].dev, (int)C,
                   (const double*)arrs[3].dev, (int)nt, (int)L, (const double*)arrs[4].dev, (double*)d_out);
    }
    cudaError_t e = cudaGetLastError();
    if (e == cudaSuccess && ho && ob) e = cudaMemcpyAsync(out, d_out, ob, cudaMemcpyDeviceToHost, stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(stream);
    cudaFreeAsync(blk, stream);
    MF_CUDA_TRY(e);
    return MF_OK;
}

}  // namespace mf
