// mf_api.cu -- extern "C" entry points of libmfgpu.so (declared in include/mfgpu.h).
#include <cstdio>
#include <cstring>
#include <vector>

#include "mf_internal.h"
#include "mf_kernels.cuh"

struct mf_context {
    mf::Context c;
};
struct mf_decimation {
    mf::Result r;
};

namespace mf {

bool is_device_ptr(const void* p) {
    if (!p) return false;
    cudaPointerAttributes a;
    cudaError_t e = cudaPointerGetAttributes(&a, p);
    if (e != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged;
}

static int grid_n(int64_t n) {
    int64_t g = (n + 255) / 256;
    if (g > 148 * 16) g = 148 * 16;
    return (int)(g < 1 ? 1 : g);
}

// int32 device array -> int64 destination (host or device), adding `add`.
static int copy_i32_as_i64(const int* src, int64_t n, int64_t* dst, cudaStream_t s, mf_status* st) {
    if (!dst || n <= 0) return MF_OK;
    if (is_device_ptr(dst)) {
        LAUNCH(k_i32_to_i64, grid_n(n), 256, 0, s, n, src, dst, 0);
        MF_CUDA_TRY(cudaGetLastError());
        return MF_OK;
    }
    int64_t* tmp = nullptr;
    MF_CUDA_TRY(cudaMallocAsync(&tmp, (size_t)n * 8, s));
    LAUNCH(k_i32_to_i64, grid_n(n), 256, 0, s, n, src, tmp, 0);
    MF_CUDA_TRY(cudaMemcpyAsync(dst, tmp, (size_t)n * 8, cudaMemcpyDeviceToHost, s));
    MF_CUDA_TRY(cudaFreeAsync(tmp, s));
    return MF_OK;
}

// Destination the device can write: device memory as is, pinned host memory through its
// mapped device address; nullptr for pageable host memory.
void* device_writable(void* p) {
    cudaPointerAttributes a;
    if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
        cudaGetLastError();
        return nullptr;
    }
    if (a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged) return p;
    if (a.type == cudaMemoryTypeHost && a.devicePointer) return a.devicePointer;
    return nullptr;
}

static int copy_f64_as(const double* src, int64_t n, void* dst, int dtype, cudaStream_t s, mf_status* st) {
    if (!dst || n <= 0) return MF_OK;
    if (dtype == MF_DTYPE_F64) {
        MF_CUDA_TRY(cudaMemcpyAsync(dst, src, (size_t)n * 8, cudaMemcpyDefault, s));
        return MF_OK;
    }
    if (is_device_ptr(dst)) {
        LAUNCH(k_f64_to_f32, grid_n(n), 256, 0, s, n, src, (float*)dst);
        return MF_OK;
    }
    float* tmp = nullptr;
    MF_CUDA_TRY(cudaMallocAsync(&tmp, (size_t)n * 4, s));
    LAUNCH(k_f64_to_f32, grid_n(n), 256, 0, s, n, src, tmp);
    MF_CUDA_TRY(cudaMemcpyAsync(dst, tmp, (size_t)n * 4, cudaMemcpyDeviceToHost, s));
    MF_CUDA_TRY(cudaFreeAsync(tmp, s));
    return MF_OK;
}

}  // namespace mf

using namespace mf;

static void clear_status(mf_status* st) {
    if (!st) return;
    memset(st, 0, sizeof(*st));
    st->mesh_index = -1;
}

extern "C" {

int mf_context_create(int device, mf_context** out) {
    mf_context* c = new mf_context();
    c->c.device = device;
    if (cudaSetDevice(device) != cudaSuccess) {
        delete c;
        return MF_ERR_CUDA;
    }
    cudaDeviceProp prop;
    if (cudaGetDeviceProperties(&prop, device) != cudaSuccess) {
        delete c;
        return MF_ERR_CUDA;
    }
    c->c.sm_count = prop.multiProcessorCount;
    cudaFuncSetAttribute(k_adj_rank_tiled, cudaFuncAttributeMaxDynamicSharedMemorySize, kRankSmem);
    cudaFuncSetAttribute(k_select<1024>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         kSelBins * 4 + 8 * std::max(2 * kSelCapMax, kSelChiCap));
    cudaFuncSetAttribute(k_select<512>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         kSelBins * 4 + 8 * std::max(2 * kSelCapMax, kSelChiCap));
    cudaFuncSetAttribute(k_select_cl, cudaFuncAttributeMaxDynamicSharedMemorySize, kClSmem);
    // keep freed stream-ordered allocations cached in the device pool
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, device) == cudaSuccess) {
        uint64_t thr = UINT64_MAX;
        cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
    }
    cudaGetLastError();
    *out = c;
    return MF_OK;
}

void mf_context_destroy(mf_context* ctx) {
    if (!ctx) return;
    cudaSetDevice(ctx->c.device);
    drop_graphs(&ctx->c);
    delete ctx->c.pending;
    if (ctx->c.arena) cudaFree(ctx->c.arena);
    if (ctx->c.pinned) cudaFreeHost(ctx->c.pinned);
    if (ctx->c.aux) cudaStreamDestroy(ctx->c.aux);
    for (cudaEvent_t e : ctx->c.aux_ev)
        if (e) cudaEventDestroy(e);
    delete ctx;
}

int mf_decimate(mf_context* ctx, const mf_mesh_view* mesh, const mf_decimate_config* cfg, void* stream,
                mf_decimation** out, mf_status* status) {
    mf_status local;
    mf_status* st = status ? status : &local;
    clear_status(st);
    if (!ctx || !mesh || !cfg || !out) {
        st->code = MF_ERR_VALUE;
        snprintf(st->message, sizeof(st->message), "null argument");
        return st->code;
    }
    *out = nullptr;
    Result* r = nullptr;
    int rc = decimate_run(&ctx->c, mesh, cfg, (cudaStream_t)stream, &r, st);
    if (rc != MF_OK) return rc;
    mf_decimation* d = new mf_decimation();
    d->r = *r;
    delete r;
    *out = d;
    return MF_OK;
}

int mf_decimate_into(mf_context* ctx, const mf_mesh_view* mesh, const mf_decimate_config* cfg, void* stream,
                     const mf_outputs* outputs, mf_decimation** out, mf_status* status) {
    mf_status local;
    mf_status* st = status ? status : &local;
    clear_status(st);
    if (!ctx || !mesh || !cfg || !out || !outputs) {
        st->code = MF_ERR_VALUE;
        snprintf(st->message, sizeof(st->message), "null argument");
        return st->code;
    }
    *out = nullptr;
    Result* r = nullptr;
    int rc = decimate_run(&ctx->c, mesh, cfg, (cudaStream_t)stream, &r, st, false, outputs);
    if (rc != MF_OK) return rc;
    mf_decimation* d = new mf_decimation();
    d->r = *r;
    delete r;
    *out = d;
    return MF_OK;
}

int mf_decimate_begin(mf_context* ctx, const mf_mesh_view* mesh, const mf_decimate_config* cfg, void* stream,
                      mf_status* status) {
    mf_status local;
    mf_status* st = status ? status : &local;
    clear_status(st);
    if (!ctx || !mesh || !cfg) {
        st->code = MF_ERR_VALUE;
        snprintf(st->message, sizeof(st->message), "null argument");
        return st->code;
    }
    if (!ctx->c.pending) ctx->c.pending = new DecCall();
    if (ctx->c.pending->active) {  // a begun call its caller abandoned: finish and discard it
        mf_status drop;
        clear_status(&drop);
        Result* r = nullptr;
        if (decimate_end(&ctx->c, *ctx->c.pending, nullptr, &r, &drop) == MF_OK && r) {
            if (r->block) cudaFree(r->block);
            delete r;
        }
        clear_status(st);
    }
    return decimate_begin(&ctx->c, mesh, cfg, (cudaStream_t)stream, st, false, *ctx->c.pending);
}

int mf_decimate_end(mf_context* ctx, const mf_outputs* outputs, mf_decimation** out, mf_status* status) {
    mf_status local;
    mf_status* st = status ? status : &local;
    clear_status(st);
    if (!ctx || !out || !ctx->c.pending || !ctx->c.pending->active) {
        st->code = MF_ERR_VALUE;
        snprintf(st->message, sizeof(st->message), "mf_decimate_end: no begun call on this context");
        return st->code;
    }
    *out = nullptr;
    Result* r = nullptr;
    int rc = decimate_end(&ctx->c, *ctx->c.pending, outputs, &r, st);
    if (rc != MF_OK) return rc;
    mf_decimation* d = new mf_decimation();
    d->r = *r;
    delete r;
    *out = d;
    return MF_OK;
}

int mf_decimation_sizes(const mf_decimation* res, int64_t* n_in, int64_t* n_out, int64_t* m_out, int64_t* c,
                        int64_t* n_meshes) {
    if (!res) return MF_ERR_VALUE;
    if (n_in) *n_in = res->r.n_in;
    if (n_out) *n_out = res->r.n_out;
    if (m_out) *m_out = res->r.m_out;
    if (c) *c = res->r.c;
    if (n_meshes) *n_meshes = res->r.n_meshes;
    return MF_OK;
}

int mf_decimation_copy(const mf_decimation* res, double* positions, int64_t* facets, void* features,
                       int32_t features_dtype, int64_t* replace, int64_t* mapping, int64_t* vertex_offsets,
                       int64_t* facet_offsets, void* stream, mf_status* status) {
    mf_status local;
    mf_status* st = status ? status : &local;
    clear_status(st);
    if (!res) return MF_ERR_VALUE;
    const Result& r = res->r;
    cudaStream_t s = (cudaStream_t)stream;
    MF_CUDA_TRY(cudaSetDevice(r.device));
    // Every output whose destination the device can write (device memory, or pinned host
    // memory through its mapped address) is emitted by ONE kernel: int32 -> int64 widening
    // and float64 copies fused, host-bound bytes written over the bus directly -- no staging
    // buffers, no per-array copies.  Pageable destinations take the staged path.
    const double* fsrc = r.features_alias ? r.positions : r.features;
    EmitJobs jobs;
    auto add = [&](int kind, const void* src, void* dst, int64_t n) -> bool {
        if (!dst || n <= 0) return true;
        void* d = device_writable(dst);
        if (!d) return false;
        jobs.add(kind, src, d, n);
        return true;
    };
    const bool pos_ok = add(kEmitF64, r.positions, positions, r.n_out * 3);
    const bool fac_ok = add(kEmitI32, r.facets, facets, r.m_out * 3);
    const bool fea_ok = features_dtype == MF_DTYPE_F64 ? add(kEmitF64, fsrc, features, r.n_out * r.c)
                                                       : add(kEmitF32, fsrc, features, r.n_out * r.c);
    const bool rep_ok = add(kEmitI32, r.replace, replace, r.n_in);
    const bool map_ok = add(kEmitI32, r.mapping, mapping, r.n_in);
    if (jobs.count) {
        LAUNCH(k_emit, grid_n(jobs.total()), 256, 0, s, jobs);
        MF_CUDA_TRY(cudaGetLastError());
    }
    if (!pos_ok && positions && r.n_out)
        MF_CUDA_TRY(cudaMemcpyAsync(positions, r.positions, (size_t)r.n_out * 24, cudaMemcpyDefault, s));
    int rc;
    if (!fac_ok && (rc = copy_i32_as_i64(r.facets, r.m_out * 3, facets, s, st))) return rc;
    if (!fea_ok && features) {
        if ((rc = copy_f64_as(fsrc, r.n_out * r.c, features, features_dtype, s, st))) return rc;
    }
    if (!rep_ok && (rc = copy_i32_as_i64(r.replace, r.n_in, replace, s, st))) return rc;
    if (!map_ok && (rc = copy_i32_as_i64(r.mapping, r.n_in, mapping, s, st))) return rc;
    for (int which = 0; which < 2; which++) {
        int64_t* dst = which ? facet_offsets : vertex_offsets;
        const std::vector<int64_t>& src = which ? r.facet_offsets : r.vertex_offsets;
        if (!dst) continue;
        MF_CUDA_TRY(cudaMemcpyAsync(dst, src.data(), src.size() * 8, cudaMemcpyDefault, s));
    }
    MF_CUDA_TRY(cudaStreamSynchronize(s));
    MF_CUDA_TRY(cudaGetLastError());
    return MF_OK;
}

int mf_decimation_device_arrays(const mf_decimation* res, const double** positions, const int32_t** facets,
                                int32_t* features_alias) {
    if (!res) return MF_ERR_VALUE;
    if (positions) *positions = res->r.positions;
    if (facets) *facets = res->r.facets;
    if (features_alias) *features_alias = res->r.features_alias;
    return MF_OK;
}

void mf_decimation_free(mf_decimation* res) {
    if (!res) return;
    cudaSetDevice(res->r.device);
    if (res->r.block) cudaFree(res->r.block);
    if (res->r.csr_block) cudaFree(res->r.csr_block);
    delete res;
}

int mf_pool(mf_context* ctx, const mf_decimation* res, const int64_t* replace, int64_t n, int64_t n_out,
            const void* features, int32_t dtype, int64_t c, int32_t mode, const void* weights, void* out,
            void* stream, mf_status* status) {
    mf_status local;
    mf_status* st = status ? status : &local;
    clear_status(st);
    if (!ctx || mode < 0 || mode > 3) {
        st->code = MF_ERR_VALUE;
        snprintf(st->message, sizeof(st->message), "mode must be one of ('average', 'max', 'weighted', 'sum')");
        return st->code;
    }
    cudaStream_t s = (cudaStream_t)stream;
    MF_CUDA_TRY(cudaSetDevice(ctx->c.device));
    const int* d_off = nullptr;
    const int* d_mem = nullptr;
    void* blk_r = nullptr;
    void* blk_csr = nullptr;
    int rc = MF_OK;
    if (res) {
        Result& r = const_cast<mf_decimation*>(res)->r;
        n = r.n_in;
        n_out = r.n_out;
        if (!r.csr_block) {
            int *o, *mm;
            if ((rc = build_cluster_csr(&ctx->c, r.replace, r.n_in, r.n_out, &o, &mm, &r.csr_block, s, st)))
                return rc;
            r.csr_off = o;
            r.csr_members = mm;
        }
        d_off = r.csr_off;
        d_mem = r.csr_members;
    } else {
        int *r32, *cnt;
        if ((rc = upload_replace(&ctx->c, replace, n, n_out, 1, &r32, &cnt, &blk_r, s, st))) goto done;
        int *o, *mm;
        if ((rc = build_cluster_csr(&ctx->c, r32, n, n_out, &o, &mm, &blk_csr, s, st))) goto done;
        d_off = o;
        d_mem = mm;
    }
    if (mode == MF_POOL_WEIGHTED && !weights) {
        st->code = rc = MF_ERR_VALUE;
        snprintf(st->message, sizeof(st->message), "weighted pooling requires per-input-vertex weights");
        goto done;
    }
    rc = pool_run(&ctx->c, features, dtype, n, c, nullptr, d_off, d_mem, n_out, mode, weights, out, s, st);
done:
    if (blk_r) cudaFreeAsync(blk_r, s);
    if (blk_csr) cudaFreeAsync(blk_csr, s);
    return rc;
}

/* pooling.pool_backward (pooling.py:80-97); unpool_backward = mf_pool(..., MF_POOL_SUM) (pooling.py:100-102). */
int mf_pool_backward(mf_context* ctx, const mf_decimation* res, const int64_t* replace, int64_t n, int64_t n_out,
                     const void* grad_output, int32_t grad_dtype, const void* features, int32_t features_dtype,
                     int64_t c, int32_t mode, const void* weights, void* out, int32_t out_dtype, void* stream,
                     mf_status* status) {
    mf_status local;
    mf_status* st = status ? status : &local;
    clear_status(st);
    if (!ctx || mode < 0 || mode > 3) {
        st->code = MF_ERR_VALUE;
        snprintf(st->message, sizeof(st->message), "mode must be one of ('average', 'max', 'weighted', 'sum')");
        return st->code;
    }
    cudaStream_t s = (cudaStream_t)stream;
    MF_CUDA_TRY(cudaSetDevice(ctx->c.device));
    const int *d_off = nullptr, *d_mem = nullptr, *d_rep = nullptr;
    void *blk_r = nullptr, *blk_csr = nullptr;
    int rc = MF_OK;
    if (res) {
        Result& r = const_cast<mf_decimation*>(res)->r;
        n = r.n_in;
        n_out = r.n_out;
        if (!r.csr_block) {
            int *o, *mm;
            if ((rc = build_cluster_csr(&ctx->c, r.replace, r.n_in, r.n_out, &o, &mm, &r.csr_block, s, st)))
                return rc;
            r.csr_off = o;
            r.csr_members = mm;
        }
        d_off = r.csr_off;
        d_mem = r.csr_members;
        d_rep = r.replace;
    } else {
        int *r32, *cnt;
        if ((rc = upload_replace(&ctx->c, replace, n, n_out, 1, &r32, &cnt, &blk_r, s, st))) goto done;
        int *o, *mm;
        if ((rc = build_cluster_csr(&ctx->c, r32, n, n_out, &o, &mm, &blk_csr, s, st))) goto done;
        d_off = o;
        d_mem = mm;
        d_rep = r32;
    }
    if (mode == MF_POOL_WEIGHTED && !weights) {
        st->code = rc = MF_ERR_VALUE;
        snprintf(st->message, sizeof(st->message), "weighted pooling requires per-input-vertex weights");
        goto done;
    }
    rc = pool_backward_run(&ctx->c, grad_output, grad_dtype, features, features_dtype, n, c, d_rep, d_off, d_mem,
                           n_out, mode, weights, out, out_dtype, s, st);
done:
    if (blk_r) cudaFreeAsync(blk_r, s);
    if (blk_csr) cudaFreeAsync(blk_csr, s);
    return rc;
}

int mf_unpool(mf_context* ctx, const mf_decimation* res, const int64_t* replace, int64_t n, int64_t n_out,
              const void* coarse, int32_t dtype, int64_t c, void* out, void* stream, mf_status* status) {
    mf_status local;
    mf_status* st = status ? status : &local;
    clear_status(st);
    if (!ctx) return MF_ERR_VALUE;
    cudaStream_t s = (cudaStream_t)stream;
    MF_CUDA_TRY(cudaSetDevice(ctx->c.device));
    int rc;
    if (res) {
        const Result& r = res->r;
        return unpool_run(&ctx->c, coarse, dtype, r.n_out, c, r.replace, r.n_in, out, s, st);
    }
    int *r32, *cnt;
    void* blk = nullptr;
    rc = upload_replace(&ctx->c, replace, n, n_out, 0, &r32, &cnt, &blk, s, st);
    if (rc == MF_OK) rc = unpool_run(&ctx->c, coarse, dtype, n_out, c, r32, n, out, s, st);
    if (blk) cudaFreeAsync(blk, s);
    return rc;
}

/* binary PLY bodies (io.py:226-431) */
int mf_ply_decode(mf_context* ctx, const uint8_t* body, int64_t body_len, int64_t n_vertices,
                  const mf_ply_vertex_spec* vspec, int64_t face_offset, int64_t n_faces, int32_t arity,
                  int32_t index_type, double* positions, double* features, int32_t n_channels, int64_t* facets,
                  void* stream, mf_status* status) {
    mf_status local;
    mf_status* st = status ? status : &local;
    clear_status(st);
    bool ok = ctx && vspec && n_vertices >= 0 && n_faces >= 0 && body_len >= 0 && (n_channels == 3 || n_channels == 6);
    if (ok && n_vertices) ok = vspec->record_size > 0 && (int64_t)vspec->record_size * n_vertices <= body_len;
    if (ok && n_faces) {
        const int isz = index_type <= MF_PLY_U1 ? 1 : (index_type <= MF_PLY_U2 ? 2 : (index_type <= MF_PLY_U4 ? 4 : 8));
        ok = arity >= 3 && index_type >= MF_PLY_I1 && index_type <= MF_PLY_U4 && face_offset >= 0 &&
             face_offset + (int64_t)(1 + arity * isz) * n_faces <= body_len;
    }
    if (ok)
        for (int k = 0; k < 6; k++) {
            const int o = vspec->offset[k], t = vspec->type[k];
            if ((k < 3 || n_channels == 6) && (o < 0 || t < MF_PLY_I1 || t > MF_PLY_F8 || o >= vspec->record_size)) ok = false;
        }
    if (!ok) {
        st->code = MF_ERR_VALUE;
        snprintf(st->message, sizeof(st->message), "invalid PLY layout (record sizes / offsets exceed the body)");
        return st->code;
    }
    MF_CUDA_TRY(cudaSetDevice(ctx->c.device));
    PlyVertexSpec vs;
    vs.record = vspec->record_size;
    for (int k = 0; k < 6; k++) {
        vs.off[k] = (k < 3 || n_channels == 6) ? vspec->offset[k] : -1;
        vs.type[k] = vspec->type[k];
    }
    return ply_decode_run(&ctx->c, body, body_len, n_vertices, vs, face_offset, n_faces, arity, index_type,
                          positions, features, n_channels, facets, (cudaStream_t)stream, st);
}

int mf_ply_encode(mf_context* ctx, const double* positions, int64_t n, const double* features, int64_t c,
                  const int64_t* facets, int64_t m, uint8_t* body, void* stream, mf_status* status) {
    mf_status local;
    mf_status* st = status ? status : &local;
    clear_status(st);
    if (!ctx || n < 0 || m < 0 || (n && !positions) || (m && !facets) || (n + m && !body)) {
        st->code = MF_ERR_VALUE;
        snprintf(st->message, sizeof(st->message), "invalid PLY encode arguments");
        return st->code;
    }
    MF_CUDA_TRY(cudaSetDevice(ctx->c.device));
    return ply_encode_run(&ctx->c, positions, n, c >= 6 ? features : nullptr, c, facets, m, body,
                          (cudaStream_t)stream, st);
}

/* vertex_facet_adjacency (mesh.py:114-122) */
int mf_vertex_facet_adjacency(mf_context* ctx, const int64_t* facets, int64_t m, int64_t n, int64_t* offsets,
                              int64_t* facet_ids, void* stream, mf_status* status) {
    mf_status local;
    mf_status* st = status ? status : &local;
    clear_status(st);
    if (!ctx || m < 0 || n < 0 || (m && !facets) || !offsets || (m && !facet_ids)) {
        st->code = MF_ERR_VALUE;
        snprintf(st->message, sizeof(st->message), "invalid adjacency arguments");
        return st->code;
    }
    MF_CUDA_TRY(cudaSetDevice(ctx->c.device));
    return adjacency_run(&ctx->c, facets, m, n, offsets, facet_ids, (cudaStream_t)stream, st);
}

/* facet2vertex_forward (conv.py:222-250) */
int mf_facet2vertex(mf_context* ctx, const int64_t* offsets, int64_t n, const int64_t* facet_ids, const void* features,
                    int32_t dtype, int64_t m, int64_t c, const double* weights, int64_t t, int64_t multiplier,
                    const double* coeff, const int64_t* vertex_ids, int64_t rows, void* out, void* stream,
                    mf_status* status) {
    mf_status local;
    mf_status* st = status ? status : &local;
    clear_status(st);
    if (!ctx || n < 0 || m < 0 || c < 0 || t < 0 || multiplier < 0 || rows < 0 ||
        (dtype != MF_DTYPE_F32 && dtype != MF_DTYPE_F64)) {
        st->code = MF_ERR_VALUE;
        snprintf(st->message, sizeof(st->message), "invalid facet2vertex arguments");
        return st->code;
    }
    MF_CUDA_TRY(cudaSetDevice(ctx->c.device));
    return f2v_run(&ctx->c, offsets, n, facet_ids, features, dtype, m, c, weights, t, multiplier, coeff, vertex_ids,
                   rows, out, (cudaStream_t)stream, st);
}

/* quality_report errors (decimate.py:580-602) */
int mf_quality_errors(mf_context* ctx, const mf_mesh_view* original, const mf_decimation* res, const int64_t* replace,
                      int64_t n_out, const double* positions_out, int32_t einsum_order, double* errors, void* stream,
                      mf_status* status) {
    mf_status local;
    mf_status* st = status ? status : &local;
    clear_status(st);
    if (!ctx || !original || original->facets_i32) {
        st->code = MF_ERR_VALUE;
        snprintf(st->message, sizeof(st->message), "context and an int64-facet original mesh are required");
        return st->code;
    }
    cudaStream_t s = (cudaStream_t)stream;
    MF_CUDA_TRY(cudaSetDevice(ctx->c.device));
    const int64_t n = original->n;
    const int* d_off = nullptr;
    const int* d_mem = nullptr;
    void* blk_r = nullptr;
    void* blk_csr = nullptr;
    int rc = MF_OK;
    if (res) {
        Result& r = const_cast<mf_decimation*>(res)->r;
        if (r.n_in != n || r.n_out != n_out) {
            st->code = MF_ERR_VALUE;
            snprintf(st->message, sizeof(st->message), "result does not belong to this mesh (%lld -> %lld vertices)",
                     (long long)r.n_in, (long long)r.n_out);
            return st->code;
        }
        if (!r.csr_block) {
            int *o, *mm;
            if ((rc = build_cluster_csr(&ctx->c, r.replace, r.n_in, r.n_out, &o, &mm, &r.csr_block, s, st)))
                return rc;
            r.csr_off = o;
            r.csr_members = mm;
        }
        d_off = r.csr_off;
        d_mem = r.csr_members;
    } else {
        int *r32, *cnt;
        if ((rc = upload_replace(&ctx->c, replace, n, n_out, 1, &r32, &cnt, &blk_r, s, st))) goto done;
        int *o, *mm;
        if ((rc = build_cluster_csr(&ctx->c, r32, n, n_out, &o, &mm, &blk_csr, s, st))) goto done;
        d_off = o;
        d_mem = mm;
    }
    rc = quality_run(&ctx->c, original, d_off, d_mem, n_out, positions_out, einsum_order, errors, s, st);
done:
    if (blk_r) cudaFreeAsync(blk_r, s);
    if (blk_csr) cudaFreeAsync(blk_csr, s);
    return rc;
}

int32_t mf_decimation_round_stats(const mf_decimation* res, int64_t* out, int32_t cap_rounds) {
    if (!res) return -1;
    int32_t R = (int32_t)(res->r.round_stats.size() / 6);
    for (int32_t i = 0; i < R && i < cap_rounds; i++)
        for (int k = 0; k < 6; k++) out[6 * i + k] = res->r.round_stats[6 * i + k];
    return R;
}

/* TriMesh re-validation on the device (validation.py:8-41), + optional facet-set uniqueness. */
int mf_validate_mesh(mf_context* ctx, const double* positions, int64_t n, const int64_t* facets, int64_t m,
                     const int64_t* vertex_offsets, const int64_t* facet_offsets, int64_t n_meshes,
                     int32_t check_duplicates, void* stream, mf_status* status) {
    mf_status local;
    mf_status* st = status ? status : &local;
    clear_status(st);
    if (!ctx || n < 0 || m < 0 || (n > 0 && !positions) || (m > 0 && !facets)) {
        st->code = MF_ERR_VALUE;
        snprintf(st->message, sizeof(st->message), "null argument");
        return st->code;
    }
    cudaStream_t s = (cudaStream_t)stream;
    MF_CUDA_TRY(cudaSetDevice(ctx->c.device));
    const bool hp = n > 0 && !is_device_ptr(positions), hf = m > 0 && !is_device_ptr(facets);
    const size_t pb = ((size_t)n * 24 + 255) & ~size_t(255), fb = ((size_t)m * 24 + 255) & ~size_t(255);
    void* tmp = nullptr;
    if (hp || hf) MF_CUDA_TRY(cudaMallocAsync(&tmp, (hp ? pb : 0) + (hf ? fb : 0), s));
    const double* dP = positions;
    const int64_t* dF = facets;
    char* q = (char*)tmp;
    if (hp) {
        MF_CUDA_TRY(cudaMemcpyAsync(q, positions, (size_t)n * 24, cudaMemcpyHostToDevice, s));
        dP = (const double*)q;
        q += pb;
    }
    if (hf) {
        MF_CUDA_TRY(cudaMemcpyAsync(q, facets, (size_t)m * 24, cudaMemcpyHostToDevice, s));
        dF = (const int64_t*)q;
    }
    int rc = validate_mesh_run<int64_t>(&ctx->c, dP, n, dF, m, vertex_offsets, facet_offsets,
                                        vertex_offsets ? (int)n_meshes : 1, check_duplicates != 0, nullptr, nullptr,
                                        0, s, st);
    if (tmp) {
        cudaFreeAsync(tmp, s);
        cudaStreamSynchronize(s);
    }
    return rc;
}

int64_t mf_round_targets(int64_t n_in, int64_t target, int32_t rounds, int64_t* chain, int64_t cap) {
    std::vector<int64_t> v;
    round_targets(n_in, target, rounds, v);
    for (int64_t i = 0; i < (int64_t)v.size() && i < cap; i++) chain[i] = v[i];
    return (int64_t)v.size();
}

int64_t mf_kernel_launch_count(int32_t reset) {
    int64_t v = g_launches;
    if (reset) g_launches = 0;
    return v;
}

const char* mf_version(void) { return "mfgpu 0.1.0 (sm_100a)"; }

/* Per-kernel CUDA-event timing on the launching stream.  mode 0 = off,
 * 1 = every kernel, 2 = only the kernel named `only` (e.g. "k_suitor").
 * Enabling clears earlier records.  Graph replays are timed through event
 * nodes captured with the graph. */
void mf_profile(int32_t mode, const char* only) {
    cudaDeviceSynchronize();
    prof_collect_pending();
    g_prof_mode = mode;
    g_prof_only = only ? only : "";
    g_prof_recs.clear();
    g_prof_done.clear();
}
/* Aggregate the timed launches (synchronises the device): fills up to `cap`
 * rows of names / total milliseconds / launch counts, returns the number of
 * distinct kernels. */
int32_t mf_profile_read(char* names, int32_t name_cap, double* total_ms, int64_t* launches, int32_t cap) {
    cudaDeviceSynchronize();
    prof_collect_pending();
    std::vector<std::string> keys;
    std::vector<double> ms;
    std::vector<int64_t> cnt;
    for (const auto& r : g_prof_done) {
        size_t k = 0;
        while (k < keys.size() && keys[k] != r.first) k++;
        if (k == keys.size()) {
            keys.push_back(r.first);
            ms.push_back(0.0);
            cnt.push_back(0);
        }
        ms[k] += r.second;
        cnt[k]++;
    }
    for (size_t k = 0; k < keys.size() && (int32_t)k < cap; k++) {
        snprintf(names + k * name_cap, name_cap, "%s", keys[k].c_str());
        total_ms[k] = ms[k];
        launches[k] = cnt[k];
    }
    return (int32_t)keys.size();
}

}  // extern "C"
