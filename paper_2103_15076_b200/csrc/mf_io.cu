// mf_io.cu -- binary little-endian PLY bodies decoded / encoded on the device
// (the on-disk format either side of the decimation step, io.py:226-431).
//
// Decode (the reference's vectorised fast path, io.py:277-306 + 329-344):
// fixed-size vertex records -> float64 positions (+ uchar colours rescaled
// c / 255 * 2 - 1 as extra feature channels, io.py:390-392); uniform-arity
// face records (uchar count + `arity` indices) -> int64 triangles, fanned as
// (v0, v[k], v[k+1]) like _fan_triangulate (io.py:92-93).  Encode (io.py:
// 404-431): float32 xyz (+ uchar rgb = clip(rint((f + 1) * 127.5))) and
// (uchar 3, int32 x3) face records, packed little-endian.  Pure byte work:
// one thread per record, unaligned fields assembled from bytes.
#include "mf_internal.h"
#include "mf_kernels.cuh"

namespace mf {

enum PlyType { kPlyI1 = 0, kPlyU1, kPlyI2, kPlyU2, kPlyI4, kPlyU4, kPlyF4, kPlyF8 };

MF_DEV uint64_t ply_bytes(const unsigned char* p, int n) {
    uint64_t v = 0;
    for (int i = 0; i < n; i++) v |= (uint64_t)p[i] << (8 * i);
    return v;
}
MF_DEV int ply_size(int t) { return t <= kPlyU1 ? 1 : (t <= kPlyU2 ? 2 : (t <= kPlyF4 ? 4 : 8)); }
MF_DEV double ply_f64(const unsigned char* p, int t) {  // field.astype(np.float64)
    const uint64_t b = ply_bytes(p, ply_size(t));
    switch (t) {
        case kPlyI1: return (double)(int8_t)b;
        case kPlyU1: return (double)(uint8_t)b;
        case kPlyI2: return (double)(int16_t)b;
        case kPlyU2: return (double)(uint16_t)b;
        case kPlyI4: return (double)(int32_t)b;
        case kPlyU4: return (double)(uint32_t)b;
        case kPlyF4: return (double)__int_as_float((int)(uint32_t)b);
        default: return __longlong_as_double((long long)b);
    }
}
MF_DEV int64_t ply_i64(const unsigned char* p, int t) {  // index.astype(np.int64)
    const uint64_t b = ply_bytes(p, ply_size(t));
    switch (t) {
        case kPlyI1: return (int8_t)b;
        case kPlyU1: return (uint8_t)b;
        case kPlyI2: return (int16_t)b;
        case kPlyU2: return (uint16_t)b;
        case kPlyI4: return (int32_t)b;
        case kPlyU4: return (uint32_t)b;
        default: return (int64_t)b;
    }
}

struct PlyVertexSpec {
    int record;
    int off[6];   // x y z red green blue (-1: absent)
    int type[6];
};

__global__ void k_ply_vertices(int64_t nv, const unsigned char* __restrict__ body, PlyVertexSpec sp,
                               double* __restrict__ P, double* __restrict__ X, int C) {
    MF_PDL_ENTRY;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nv; i += (int64_t)gridDim.x * blockDim.x) {
        const unsigned char* r = body + i * sp.record;
        double v[6];
#pragma unroll
        for (int k = 0; k < 6; k++) v[k] = sp.off[k] >= 0 ? ply_f64(r + sp.off[k], sp.type[k]) : 0.0;
        P[3 * i] = v[0];
        P[3 * i + 1] = v[1];
        P[3 * i + 2] = v[2];
        double* x = X + i * C;
        x[0] = v[0];
        x[1] = v[1];
        x[2] = v[2];
        if (C == 6)
            for (int k = 3; k < 6; k++) x[k] = (v[k] / 255.0) * 2.0 - 1.0;
    }
}

__global__ void k_ply_faces(int64_t nf, const unsigned char* __restrict__ body, int arity, int itype,
                            int64_t* __restrict__ F, int* __restrict__ bad) {
    MF_PDL_ENTRY;
    const int isz = ply_size(itype), rec = 1 + arity * isz, tri = arity - 2;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nf; i += (int64_t)gridDim.x * blockDim.x) {
        const unsigned char* r = body + i * rec;
        if (r[0] != arity) {
            atomicExch(bad, 1);
            continue;
        }
        const int64_t v0 = ply_i64(r + 1, itype);
        int64_t prev = ply_i64(r + 1 + isz, itype);
        for (int t = 0; t < tri; t++) {
            const int64_t nx = ply_i64(r + 1 + (t + 2) * isz, itype);
            int64_t* o = F + 3 * (i * tri + t);
            o[0] = v0;
            o[1] = prev;
            o[2] = nx;
            prev = nx;
        }
    }
}

MF_DEV void put_bytes(unsigned char* p, uint64_t v, int n) {
    for (int i = 0; i < n; i++) p[i] = (unsigned char)(v >> (8 * i));
}

__global__ void k_ply_encode_vertices(int64_t n, const double* __restrict__ P, const double* __restrict__ X, int C,
                                      unsigned char* __restrict__ out) {
    MF_PDL_ENTRY;
    const int rec = X ? 15 : 12;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        unsigned char* o = out + i * rec;
        for (int k = 0; k < 3; k++) put_bytes(o + 4 * k, (uint32_t)__float_as_int(__double2float_rn(P[3 * i + k])), 4);
        if (X)
            for (int k = 0; k < 3; k++) {
                double t = rint((X[i * C + 3 + k] + 1.0) * 127.5);  // np.round: half to even
                t = t < 0.0 ? 0.0 : (t > 255.0 ? 255.0 : t);
                o[12 + k] = (unsigned char)(int)t;
            }
    }
}

__global__ void k_ply_encode_faces(int64_t m, const int64_t* __restrict__ F, unsigned char* __restrict__ out) {
    MF_PDL_ENTRY;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m; i += (int64_t)gridDim.x * blockDim.x) {
        unsigned char* o = out + i * 13;
        o[0] = 3;
        for (int k = 0; k < 3; k++) put_bytes(o + 1 + 4 * k, (uint32_t)(int32_t)F[3 * i + k], 4);  // astype('<i4')
    }
}

int ply_decode_run(Context* ctx, const unsigned char* body, int64_t body_len, int64_t nv, const PlyVertexSpec& vs,
                   int64_t face_off, int64_t nf, int arity, int itype, double* P, double* X, int C, int64_t* F,
                   cudaStream_t stream, mf_status* st) {
    const int64_t ntri = nf * (arity - 2);
    const size_t pb = (size_t)nv * 24, xb = (size_t)(nv * C) * 8, fb = (size_t)ntri * 24;
    auto al = [](size_t b) { return (b + 255) & ~size_t(255); };
    void* blk = nullptr;
    MF_CUDA_TRY(cudaMallocAsync(&blk, al((size_t)body_len) + al(pb) + al(xb) + al(fb) + 256, stream));
    char* p = (char*)blk;
    unsigned char* d_body = (unsigned char*)p;
    p += al((size_t)body_len);
    double* d_P = (double*)p;
    p += al(pb);
    double* d_X = (double*)p;
    p += al(xb);
    int64_t* d_F = (int64_t*)p;
    p += al(fb);
    int* d_bad = (int*)p;
    cudaError_t e = cudaMemsetAsync(d_bad, 0, 4, stream);
    if (e == cudaSuccess && body_len) e = cudaMemcpyAsync(d_body, body, (size_t)body_len, cudaMemcpyDefault, stream);
    if (e == cudaSuccess) {
        if (nv) LAUNCH(k_ply_vertices, grid_of(ctx, nv), 256, 0, stream, nv, d_body, vs, d_P, d_X, C);
        if (nf) LAUNCH(k_ply_faces, grid_of(ctx, nf), 256, 0, stream, nf, d_body + face_off, arity, itype, d_F, d_bad);
        e = cudaGetLastError();
    }
    int bad = 0;
    if (e == cudaSuccess && pb) e = cudaMemcpyAsync(P, d_P, pb, cudaMemcpyDefault, stream);
    if (e == cudaSuccess && xb) e = cudaMemcpyAsync(X, d_X, xb, cudaMemcpyDefault, stream);
    if (e == cudaSuccess && fb) e = cudaMemcpyAsync(F, d_F, fb, cudaMemcpyDefault, stream);
    if (e == cudaSuccess) e = cudaMemcpyAsync(&bad, d_bad, 4, cudaMemcpyDeviceToHost, stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(stream);
    cudaFreeAsync(blk, stream);
    MF_CUDA_TRY(e);
    if (bad) {
        st->code = MF_ERR_STRUCTURAL;
        snprintf(st->message, sizeof(st->message), "face records do not all have %d vertices", arity);
        return st->code;
    }
    return MF_OK;
}

int ply_encode_run(Context* ctx, const double* P, int64_t n, const double* X, int64_t C, const int64_t* F, int64_t m,
                   unsigned char* out, cudaStream_t stream, mf_status* st) {
    const bool color = X != nullptr && C >= 6;
    const size_t vb = (size_t)n * (color ? 15 : 12), fb = (size_t)m * 13;
    const size_t pb = (size_t)n * 24, xb = color ? (size_t)(n * C) * 8 : 0, f64b = (size_t)m * 24;
    auto al = [](size_t b) { return (b + 255) & ~size_t(255); };
    void* blk = nullptr;
    MF_CUDA_TRY(cudaMallocAsync(&blk, al(vb + fb) + al(pb) + al(xb) + al(f64b) + 256, stream));
    char* p = (char*)blk;
    unsigned char* d_out = (unsigned char*)p;
    p += al(vb + fb);
    const double* d_P = P;
    const double* d_X = color ? X : nullptr;
    const int64_t* d_F = F;
    cudaError_t e = cudaSuccess;
    if (pb && !is_device_ptr(P)) {
        e = cudaMemcpyAsync(p, P, pb, cudaMemcpyHostToDevice, stream);
        d_P = (const double*)p;
    }
    p += al(pb);
    if (e == cudaSuccess && xb && !is_device_ptr(X)) {
        e = cudaMemcpyAsync(p, X, xb, cudaMemcpyHostToDevice, stream);
        d_X = (const double*)p;
    }
    p += al(xb);
    if (e == cudaSuccess && f64b && !is_device_ptr(F)) {
        e = cudaMemcpyAsync(p, F, f64b, cudaMemcpyHostToDevice, stream);
        d_F = (const int64_t*)p;
    }
    if (e == cudaSuccess) {
        if (n) LAUNCH(k_ply_encode_vertices, grid_of(ctx, n), 256, 0, stream, n, d_P, d_X, (int)C, d_out);
        if (m) LAUNCH(k_ply_encode_faces, grid_of(ctx, m), 256, 0, stream, m, d_F, d_out + vb);
        e = cudaGetLastError();
    }
    if (e == cudaSuccess && vb + fb) e = cudaMemcpyAsync(out, d_out, vb + fb, cudaMemcpyDefault, stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(stream);
    cudaFreeAsync(blk, stream);
    MF_CUDA_TRY(e);
    return MF_OK;
}

}  // namespace mf
