// mf_internal.h -- host-side declarations shared by the library's translation units.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <string>
#include <vector>

#include "../../include/mfgpu.h"

namespace mf {

// Status words the device writes and the host reads back once per call.
struct DevStatus {
    int abort;            // a round failed (infeasible) -> later kernels exit early
    int fail_round;       // first failing round
    int limit_exceeded;   // a per-vertex / per-cluster size exceeded the heavy-tier capacity
    int pad;
};

struct DecCall;  // mf_decimate.cu: a call between mf_decimate_begin and mf_decimate_end

struct Context {
    int device = 0;
    DecCall* pending = nullptr;  // the begun, not yet ended call of this context
    int sm_count = 148;
    // workspace arena (grown on demand, kept across calls)
    void* arena = nullptr;
    size_t arena_bytes = 0;
    // pinned host staging for params / status
    void* pinned = nullptr;
    size_t pinned_bytes = 0;
    cudaEvent_t done_event = nullptr;
    // side stream + events: uploads that overlap the round chain (features check)
    cudaStream_t aux = nullptr;
    cudaEvent_t aux_ev[2] = {nullptr, nullptr};
    std::string last_error;
};

// Bump allocator over the context arena (256-byte aligned carving).
struct Arena {
    char* base = nullptr;
    size_t cap = 0, off = 0;
    bool measuring = false;
    template <typename T>
    T* take(size_t count) {
        size_t bytes = (count * sizeof(T) + 255) & ~size_t(255);
        if (bytes == 0) bytes = 256;
        size_t at = off;
        off += bytes;
        if (measuring || base == nullptr) return nullptr;
        return reinterpret_cast<T*>(base + at);
    }
};

// Device-resident decimation result (owned by mf_decimation).
struct Result {
    int device = 0;
    int64_t n_in = 0, n_out = 0, m_out = 0, c = 0, n_meshes = 1;
    int features_alias = 0;  // features == positions bitwise (features omitted on input)
    double* positions = nullptr;  // n_out*3
    int* facets = nullptr;        // m_out*3 (int32 on device)
    double* features = nullptr;   // n_out*c (nullptr when aliasing positions)
    int* replace = nullptr;       // n_in
    int* mapping = nullptr;       // n_in
    std::vector<int64_t> vertex_offsets, facet_offsets;
    std::vector<int64_t> round_stats;  // per round: N, M, E, N', M', LD iterations
    void* block = nullptr;        // single allocation backing all arrays
    // cluster CSR of `replace` for pooling (built lazily)
    int* csr_off = nullptr;
    int* csr_members = nullptr;
    void* csr_block = nullptr;
};

int decimate_run(Context* ctx, const mf_mesh_view* mesh, const mf_decimate_config* cfg, cudaStream_t stream,
                 Result** out, mf_status* st, bool force_carry = false, const mf_outputs* outs = nullptr);
int decimate_begin(Context* ctx, const mf_mesh_view* mv, const mf_decimate_config* cfg, cudaStream_t stream,
                   mf_status* st, bool force_carry, DecCall& call);
int decimate_end(Context* ctx, DecCall& call, const mf_outputs* outs, Result** out, mf_status* st);
// device address the GPU can write for p (device memory, or pinned host memory's mapped
// address); nullptr for pageable host memory
void* device_writable(void* p);
int pool_run(Context* ctx, const void* features, int dtype, int64_t n, int64_t c, const int* d_replace,
             const int* d_off, const int* d_members, int64_t n_out, int mode, const void* weights, void* out,
             cudaStream_t stream, mf_status* st);
int build_cluster_csr(Context* ctx, const int* d_replace, int64_t n, int64_t n_out, int** d_off, int** d_members,
                      void** block, cudaStream_t stream, mf_status* st);
struct PlyVertexSpec;
int ply_decode_run(Context* ctx, const unsigned char* body, int64_t body_len, int64_t nv, const PlyVertexSpec& vs,
                   int64_t face_off, int64_t nf, int arity, int itype, double* P, double* X, int C, int64_t* F,
                   cudaStream_t stream, mf_status* st);
int ply_encode_run(Context* ctx, const double* P, int64_t n, const double* X, int64_t C, const int64_t* F, int64_t m,
                   unsigned char* out, cudaStream_t stream, mf_status* st);
int adjacency_run(Context* ctx, const int64_t* facets, int64_t m, int64_t n, int64_t* offsets, int64_t* facet_ids,
                  cudaStream_t stream, mf_status* st);
int f2v_run(Context* ctx, const int64_t* offsets, int64_t n, const int64_t* facet_ids, const void* X, int dtype,
            int64_t m, int64_t C, const double* W, int64_t nt, int64_t L, const double* coeff,
            const int64_t* vertex_ids, int64_t rows, void* out, cudaStream_t stream, mf_status* st);
int quality_run(Context* ctx, const mf_mesh_view* mv, const int* d_off, const int* d_mem, int64_t n_out,
                const double* positions_out, int order, double* errors, cudaStream_t stream, mf_status* st);

// memory-space helper: true when p is device (or managed) memory on any device
bool is_device_ptr(const void* p);

#define MF_CUDA_TRY(expr)                                                              \
    do {                                                                               \
        cudaError_t _e = (expr);                                                       \
        if (_e != cudaSuccess) {                                                       \
            if (st) {                                                                  \
                st->code = MF_ERR_CUDA;                                                \
                snprintf(st->message, sizeof(st->message), "%s: %s (%s:%d)", #expr,   \
                         cudaGetErrorString(_e), __FILE__, __LINE__);                  \
            }                                                                          \
            return MF_ERR_CUDA;                                                        \
        }                                                                              \
    } while (0)

}  // namespace mf

namespace mf {
int upload_replace(Context* ctx, const int64_t* replace, int64_t n, int64_t n_out, int check_cover, int** d_r32,
                   int** d_count, void** block, cudaStream_t stream, mf_status* st);
int unpool_run(Context* ctx, const void* coarse, int dtype, int64_t n_out, int64_t c, const int* d_replace, int64_t n,
               void* out, cudaStream_t stream, mf_status* st);
int64_t round_targets(int64_t n_in, int64_t target, int rounds, std::vector<int64_t>& chain);
int pool_backward_run(Context* ctx, const void* grad, int gdtype, const void* features, int fdtype, int64_t n,
                      int64_t c, const int* d_replace, const int* d_off, const int* d_members, int64_t n_out, int mode,
                      const void* weights, void* out, int odtype, cudaStream_t stream, mf_status* st);
extern thread_local int64_t g_launches;
bool debug_validate();
int validate_result(Context* ctx, const Result* r, cudaStream_t s, mf_status* st);
template <typename I>
int validate_mesh_run(Context* ctx, const double* P, int64_t n, const I* F, int64_t m, const int64_t* h_voff,
                      const int64_t* h_foff, int B, bool check_dup, const int* rep, const int* map, int64_t n_rep,
                      cudaStream_t s, mf_status* st);
void drop_graphs(const Context* ctx);
void prof_collect_pending();
}  // namespace mf
