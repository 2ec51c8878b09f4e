// mf_validate.cu -- device re-validation of a mesh.
//
// The reference re-validates every output mesh when it builds the result
// TriMesh (mesh.py:25-31 -> validation.py:8-41): finite positions, facet
// indices in range, no facet repeating a vertex.  The decimation guarantees
// those by construction, so the library skips them on the hot path; this is
// the debug-mode check that proves it: `mf_validate_mesh` (any mesh, host or
// device arrays) and MF_DEBUG=1, which runs it on every mf_decimate result
// (plus facet uniqueness -- the dedupe invariant of decimate.py:153-157 -- and
// the replace / mapping ranges) before the call returns.
//
// Errors carry the reference's messages (validation.py:13-40) and its check
// order: positions first, then the lowest out-of-range facet, then the lowest
// facet repeating a vertex.
#include <algorithm>
#include <cstdio>

#include "mf_internal.h"
#include "mf_kernels.cuh"

namespace mf {

__global__ void k_validate_positions(int64_t n3, const double* __restrict__ P, int* __restrict__ bad) {
    MF_PDL_ENTRY;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n3; i += (int64_t)gridDim.x * blockDim.x)
        if (!isfinite(P[i])) atomicExch(bad, 1);
}

MF_DEV unsigned triple_hash(long long a, long long b, long long c) {
    unsigned long long h = (unsigned long long)a * 0x9E3779B97F4A7C15ull;
    h ^= (unsigned long long)b * 0xC2B2AE3D27D4EB4Full + (h >> 29);
    h ^= (unsigned long long)c * 0x165667B19E3779F9ull + (h >> 32);
    return (unsigned)(h ^ (h >> 31));
}

template <typename I>
MF_DEV void sorted3(const I* __restrict__ F, int64_t f, long long& a, long long& b, long long& c) {
    a = (long long)F[3 * f];
    b = (long long)F[3 * f + 1];
    c = (long long)F[3 * f + 2];
    long long t;
    if (a > b) t = a, a = b, b = t;
    if (b > c) t = b, b = c, c = t;
    if (a > b) t = a, a = b, b = t;
}

// One thread per facet.  range: the lowest facet with an index outside [0, n) (the reference's
// check) or outside its own batch entry; repeat: the lowest facet repeating a vertex; dup: the
// lowest (later facet << 32 | earlier facet) pair with the same vertex set (hash table of facet
// ids; a collision compares the stored facet's triple, which the producer kernel wrote before).
template <typename I>
__global__ void k_validate_facets(int64_t m, const I* __restrict__ F, int64_t n, int B,
                                  const int64_t* __restrict__ voff, const int64_t* __restrict__ foff,
                                  int* __restrict__ range, int* __restrict__ repeat, unsigned* __restrict__ table,
                                  unsigned tmask, unsigned long long* __restrict__ dup) {
    MF_PDL_ENTRY;
    for (int64_t f = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; f < m; f += (int64_t)gridDim.x * blockDim.x) {
        int64_t vlo = 0, vhi = n;
        if (B > 1) {
            int lo = 0, hi = B;
            while (hi - lo > 1) {
                int mid = (lo + hi) >> 1;
                if (foff[mid] <= f) lo = mid; else hi = mid;
            }
            vlo = voff[lo];
            vhi = voff[lo + 1];
        }
        const long long x = (long long)F[3 * f], y = (long long)F[3 * f + 1], z = (long long)F[3 * f + 2];
        if (x < vlo || x >= vhi || y < vlo || y >= vhi || z < vlo || z >= vhi) {
            atomicMin(range, (int)min(f, (int64_t)0x7ffffffe));
            continue;
        }
        if (x == y || y == z || x == z) {
            atomicMin(repeat, (int)min(f, (int64_t)0x7ffffffe));
            continue;
        }
        if (!table) continue;
        long long a, b, c;
        sorted3(F, f, a, b, c);
        unsigned h = triple_hash(a, b, c) & tmask;
        for (unsigned probe = 0; probe <= tmask; probe++, h = (h + 1) & tmask) {
            const unsigned cur = atomicCAS(table + h, 0xffffffffu, (unsigned)f);
            if (cur == 0xffffffffu) break;
            long long a2, b2, c2;
            sorted3(F, (int64_t)cur, a2, b2, c2);
            if (a2 == a && b2 == b && c2 == c) {
                const unsigned long long lo = (unsigned long long)min((int64_t)cur, f);
                const unsigned long long hi = (unsigned long long)max((int64_t)cur, f);
                atomicMin(dup, (hi << 32) | lo);
                break;
            }
        }
    }
}

// replace in [0, n_out); mapping = replace or -1 (decimate.py:159-167)
__global__ void k_validate_index(int64_t n, const int* __restrict__ rep, const int* __restrict__ map, int64_t n_out,
                                 int* __restrict__ bad) {
    MF_PDL_ENTRY;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const int r = rep[i], mp = map[i];
        if (r < 0 || r >= n_out || (mp != -1 && mp != r)) atomicMin(bad, (int)min(i, (int64_t)0x7ffffffe));
    }
}

static int vgrid(const Context* ctx, int64_t n) {
    int64_t g = (n + 255) / 256, cap = (int64_t)ctx->sm_count * 16;
    return (int)std::max<int64_t>(1, std::min(g, cap));
}

// Device arrays in; host offsets ([B+1] each, B <= 1 = one mesh).  rep/map may be null.
template <typename I>
int validate_mesh_run(Context* ctx, const double* P, int64_t n, const I* F, int64_t m, const int64_t* h_voff,
                      const int64_t* h_foff, int B, bool check_dup, const int* rep, const int* map, int64_t n_rep,
                      cudaStream_t s, mf_status* st) {
    const bool batch = B > 1 && h_voff && h_foff;
    unsigned tsize = 1;
    while (check_dup && tsize < (unsigned)std::min<int64_t>(2 * std::max<int64_t>(m, 1), 1u << 31)) tsize <<= 1;
    const size_t offb = batch ? (size_t)(B + 1) * 8 : 0;
    const size_t tb = check_dup ? (size_t)tsize * 4 : 0;
    void* blk = nullptr;
    MF_CUDA_TRY(cudaMallocAsync(&blk, 256 + 2 * ((offb + 255) & ~size_t(255)) + tb, s));
    char* p = (char*)blk;
    int* flags = (int*)p;  // [0] positions, [1] range, [2] repeat, [3] index, [4..5] dup (u64)
    unsigned long long* dup = (unsigned long long*)(p + 32);
    p += 256;
    int64_t *d_voff = nullptr, *d_foff = nullptr;
    int h0[8] = {0, 0x7fffffff, 0x7fffffff, 0x7fffffff, 0, 0, 0, 0};
    unsigned long long hdup = ~0ull;
    MF_CUDA_TRY(cudaMemcpyAsync(flags, h0, sizeof(h0), cudaMemcpyHostToDevice, s));
    MF_CUDA_TRY(cudaMemcpyAsync(dup, &hdup, 8, cudaMemcpyHostToDevice, s));
    if (batch) {
        d_voff = (int64_t*)p;
        p += (offb + 255) & ~size_t(255);
        d_foff = (int64_t*)p;
        p += (offb + 255) & ~size_t(255);
        MF_CUDA_TRY(cudaMemcpyAsync(d_voff, h_voff, offb, cudaMemcpyHostToDevice, s));
        MF_CUDA_TRY(cudaMemcpyAsync(d_foff, h_foff, offb, cudaMemcpyHostToDevice, s));
    }
    unsigned* table = check_dup ? (unsigned*)p : nullptr;
    if (table) MF_CUDA_TRY(cudaMemsetAsync(table, 0xff, tb, s));
    if (n > 0) LAUNCH(k_validate_positions, vgrid(ctx, 3 * n), 256, 0, s, 3 * n, P, flags);
    if (m > 0)
        LAUNCH(k_validate_facets<I>, vgrid(ctx, m), 256, 0, s, m, F, n, batch ? B : 1, d_voff, d_foff, flags + 1,
               flags + 2, table, tsize - 1, dup);
    if (rep && n_rep > 0) LAUNCH(k_validate_index, vgrid(ctx, n_rep), 256, 0, s, n_rep, rep, map, n, flags + 3);
    int h[8];
    MF_CUDA_TRY(cudaMemcpyAsync(h, flags, sizeof(h), cudaMemcpyDeviceToHost, s));
    MF_CUDA_TRY(cudaMemcpyAsync(&hdup, dup, 8, cudaMemcpyDeviceToHost, s));
    MF_CUDA_TRY(cudaFreeAsync(blk, s));
    MF_CUDA_TRY(cudaStreamSynchronize(s));
    MF_CUDA_TRY(cudaGetLastError());
    auto facet_row = [&](int f, int64_t out[3]) -> int {
        I row[3];
        MF_CUDA_TRY(cudaMemcpy(row, F + 3 * (int64_t)f, sizeof(row), cudaMemcpyDeviceToHost));
        for (int k = 0; k < 3; k++) out[k] = (int64_t)row[k];
        return MF_OK;
    };
    st->code = MF_ERR_STRUCTURAL;
    if (h[0]) {  // validation.py:13-14
        snprintf(st->message, sizeof(st->message), "positions contain NaN or infinite values");
        return st->code;
    }
    if (h[1] != 0x7fffffff) {  // validation.py:27-33
        int64_t r[3];
        if (facet_row(h[1], r)) return MF_ERR_CUDA;
        const int64_t mx = std::max(r[0], std::max(r[1], r[2]));
        const bool global = r[0] >= 0 && r[1] >= 0 && r[2] >= 0 && mx < n;
        if (global)  // in range of the whole mesh but outside its own batch entry
            snprintf(st->message, sizeof(st->message), "facet %d references vertex %lld outside its batch entry",
                     h[1], (long long)mx);
        else
            snprintf(st->message, sizeof(st->message), "facet %d references vertex %lld but the mesh has %lld vertices",
                     h[1], (long long)mx, (long long)n);
        return st->code;
    }
    if (h[2] != 0x7fffffff) {  // validation.py:34-39
        int64_t r[3];
        if (facet_row(h[2], r)) return MF_ERR_CUDA;
        // f"{tuple(arr[f])}" of numpy int64 scalars (numpy >= 2 repr)
        snprintf(st->message, sizeof(st->message),
                 "facet %d (np.int64(%lld), np.int64(%lld), np.int64(%lld)) repeats a vertex index", h[2],
                 (long long)r[0], (long long)r[1], (long long)r[2]);
        return st->code;
    }
    if (hdup != ~0ull) {  // decimate.py:153-157 keeps one facet per vertex set
        snprintf(st->message, sizeof(st->message), "facet %u repeats the vertex set of facet %u",
                 (unsigned)(hdup >> 32), (unsigned)(hdup & 0xffffffffu));
        return st->code;
    }
    if (h[3] != 0x7fffffff) {
        snprintf(st->message, sizeof(st->message),
                 "replace / mapping of input vertex %d is outside [0, %lld) or disagrees", h[3], (long long)n);
        return st->code;
    }
    st->code = MF_OK;
    return MF_OK;
}

template int validate_mesh_run<int>(Context*, const double*, int64_t, const int*, int64_t, const int64_t*,
                                    const int64_t*, int, bool, const int*, const int*, int64_t, cudaStream_t,
                                    mf_status*);
template int validate_mesh_run<int64_t>(Context*, const double*, int64_t, const int64_t*, int64_t, const int64_t*,
                                        const int64_t*, int, bool, const int*, const int*, int64_t, cudaStream_t,
                                        mf_status*);

// MF_DEBUG=1: every mf_decimate result is re-validated on the device before the call returns.
bool debug_validate() {
    static int v = -1;
    if (v < 0) {
        const char* e = getenv("MF_DEBUG");
        v = (e && e[0] == '1') ? 1 : 0;
    }
    return v == 1;
}

int validate_result(Context* ctx, const Result* r, cudaStream_t s, mf_status* st) {
    const int B = (int)r->n_meshes;
    int rc = validate_mesh_run<int>(ctx, r->positions, r->n_out, r->facets, r->m_out, r->vertex_offsets.data(),
                                    r->facet_offsets.data(), B, true, r->replace, r->mapping, r->n_in, s, st);
    if (rc != MF_OK) {
        char buf[sizeof(st->message)];
        snprintf(buf, sizeof(buf), "output re-validation (MF_DEBUG=1): %.200s", st->message);
        memcpy(st->message, buf, sizeof(buf));
    }
    return rc;
}

}  // namespace mf
