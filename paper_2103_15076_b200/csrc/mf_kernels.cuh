// mf_kernels.cuh -- device kernels of one decimation round and of cluster pooling.
//
// Kernel map (reference call site -> kernel), SURVEY.md §8(a):
//   mesh.py:72-88 + quadrics.py:36-45    k_facet_plane        facet plane (n, d), incidence degrees
//   quadrics.py:69-77 (np.add.at order)  k_inc_scatter + k_vertex_t / k_vertex_tiers: incidence CSR,
//                                         sequential per-vertex quadric fold, unique neighbour lists
//   mesh.py:125-134 + quadrics.py:117-132 k_edges             lexicographic edge ids, pair cost, rank keys
//   decimate.py:181-191 (seeded)         k_cost_minmax + k_seed_keys  PCG64 jump-ahead keys, buckets
//   decimate.py:248-263 (greedy)         k_suitor + k_mates    proposal (Suitor) greedy matching, CAS only
//   decimate.py:256-263 (budget stop)    k_select + k_trunc_absorb  per-mesh radix select of the lowest ranks
//   decimate.py:194-226 (absorb)         k_trunc_absorb + k_select + k_absorb_apply  one-pass absorption
//   decimate.py:130-137, 275-278         k_scan<rep> + k_relabel3  min-member flags + exclusive scan
//   decimate.py:142-145, 280-283         k_contract{,_heavy}   ascending-member fold from +0.0, / count
//   decimate.py:147-167                  k_facet_remap / keep / write   remap, degenerate drop, hash dedupe
//   decimate.py:380-381                  k_compose             replace / mapping chaining (-1 sticky)
//   pooling.py:36-77                     k_pool / k_unpool
//
// All float64 arithmetic is compiled with --fmad=false: numpy never fuses
// multiply-add, and bit-exact positions are required for multi-round
// topology parity.
#pragma once

#include <cooperative_groups.h>
#include <type_traits>

#include "mf_common.cuh"
#include "mf_inverse.cuh"

namespace mf {

struct __align__(32) Plane {
    double n0, n1, n2, d;
};

constexpr int kSmallDeg = 32;       // thread-tier bound for per-vertex incidence lists / clusters
constexpr int kChunk = 2048;        // smem chunk of the heavy-tier block sort

// ------------------------------------------------------------------------
// Block-cooperative sort of vals[0..n) (ascending) for the heavy tier:
// chunks of kChunk sorted in shared memory (bitonic), then bottom-up
// merge-path merges ping-ponging through tmp[0..n).  Any n.
MF_DEV int merge_path_split(const int* a, int na, const int* b, int nb, int diag) {
    int lo = diag > nb ? diag - nb : 0, hi = diag < na ? diag : na;
    while (lo < hi) {
        int mid = (lo + hi) >> 1;
        if (a[mid] <= b[diag - 1 - mid]) lo = mid + 1;  // stable: a before equal b
        else hi = mid;
    }
    return lo;
}

MF_DEV void block_sort_ints(int* vals, int* tmp, int n, int* smem /* kChunk ints */) {
    for (int c0 = 0; c0 < n; c0 += kChunk) {
        int len = min(kChunk, n - c0);
        int p2 = 1;
        while (p2 < len) p2 <<= 1;
        for (int i = threadIdx.x; i < p2; i += blockDim.x) smem[i] = (i < len) ? vals[c0 + i] : 0x7fffffff;
        __syncthreads();
        block_bitonic(smem, p2);
        for (int i = threadIdx.x; i < len; i += blockDim.x) vals[c0 + i] = smem[i];
        __syncthreads();
    }
    int* src = vals;
    int* dst = tmp;
    for (int w = kChunk; w < n; w <<= 1) {
        for (int a0 = 0; a0 < n; a0 += 2 * w) {
            int na = min(w, n - a0);
            int nb = max(0, min(w, n - a0 - na));
            const int* A = src + a0;
            const int* Bp = src + a0 + na;
            int tot = na + nb;
            int per = (tot + blockDim.x - 1) / blockDim.x;
            int d0 = min(tot, (int)threadIdx.x * per), d1 = min(tot, d0 + per);
            if (d0 < d1) {
                int i = merge_path_split(A, na, Bp, nb, d0);
                int j = d0 - i;
                for (int d = d0; d < d1; d++) {
                    bool takeA = (j >= nb) || (i < na && A[i] <= Bp[j]);
                    dst[a0 + d] = takeA ? A[i++] : Bp[j++];
                }
            }
        }
        __syncthreads();
        int* t = src; src = dst; dst = t;
    }
    if (src != vals)
        for (int i = threadIdx.x; i < n; i += blockDim.x) vals[i] = src[i];
    __syncthreads();
}

// Block-wide exclusive scan helper (blockDim.x <= 1024), returns total.
MF_DEV int block_excl_scan(int v, int* s_tmp /* 33 ints */, int* total) {
    int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    int incl = warp_incl_scan(v);
    if (lane == 31) s_tmp[warp] = incl;
    __syncthreads();
    if (warp == 0) {
        int nw = (blockDim.x + 31) >> 5;
        int w = lane < nw ? s_tmp[lane] : 0;
        int wi = warp_incl_scan(w);
        if (lane < nw) s_tmp[lane] = wi - w;
        if (lane == 31) s_tmp[32] = wi;
    }
    __syncthreads();
    int r = s_tmp[warp] + incl - v;
    *total = s_tmp[32];
    __syncthreads();
    return r;
}

// ------------------------------------------------------------------------
// small helpers
MF_DEV double dot3(double u0, double u1, double u2, double v0, double v1, double v2, int order) {
    // numpy einsum('ij,ij->i') on AVX-512: (u0v0 + u2v2) + u1v1; else sequential.
    if (order == 0) return (u0 * v0 + u2 * v2) + u1 * v1;
    return (u0 * v0 + u1 * v1) + u2 * v2;
}

MF_DEV int mesh_of(const int* __restrict__ vmesh, int v) { return vmesh ? vmesh[v] : 0; }

// ------------------------------------------------------------------------
// K0: batch bookkeeping -- owning mesh of every vertex of this round.
__global__ void k_vmesh(const int* __restrict__ abort_flag, int N, const int* __restrict__ voff, int B, int* __restrict__ vmesh) {
    MF_PDL_ENTRY;
    if (*abort_flag) return;
    for (int v = blockIdx.x * blockDim.x + threadIdx.x; v < N; v += gridDim.x * blockDim.x) {
        int lo = 0, hi = B;  // find b with voff[b] <= v < voff[b+1]
        while (hi - lo > 1) {
            int mid = (lo + hi) >> 1;
            if (voff[mid] <= v) lo = mid; else hi = mid;
        }
        vmesh[v] = lo;
    }
}

// K1: facet plane (mesh.py:77-87) + incidence degrees.
MF_DEV Plane facet_plane_of(const int* __restrict__ F, const double* __restrict__ P, int f, int order) {
    const int ia = F[3 * f], ib = F[3 * f + 1], ic = F[3 * f + 2];
    const double x0 = P[3 * ia], y0 = P[3 * ia + 1], z0 = P[3 * ia + 2];
    const double ax = P[3 * ib] - x0, ay = P[3 * ib + 1] - y0, az = P[3 * ib + 2] - z0;
    const double bx = P[3 * ic] - x0, by = P[3 * ic + 1] - y0, bz = P[3 * ic + 2] - z0;
    const double cx = ay * bz - az * by;
    const double cy = az * bx - ax * bz;
    const double cz = ax * by - ay * bx;
    const double nrm = sqrt((cx * cx + cy * cy) + cz * cz);
    Plane p;
    if (nrm == 0.0) {
        p.n0 = 0.0; p.n1 = 0.0; p.n2 = 0.0;
    } else {
        p.n0 = cx / nrm; p.n1 = cy / nrm; p.n2 = cz / nrm;
    }
    p.d = -dot3(p.n0, p.n1, p.n2, x0, y0, z0, order);
    return p;
}
// Where the vertex fold gets a facet's plane: the materialised array (k_facet_plane wrote it), or
// recomputed from the facet's corners (plane == nullptr: the planes are never written -- the
// same arithmetic, so the same bits)
struct PlaneSrc {
    const Plane* plane;
    const int* F;
    const double* P;
    int order;
    MF_DEV Plane get(int f) const { return plane ? plane[f] : facet_plane_of(F, P, f, order); }
};
// compile-time form for the hot kernels (the recompute path would otherwise cost the gather form
// ~24 registers)
template <bool RC>
struct PlaneSrcT {
    const Plane* plane;
    const int* F;
    const double* P;
    int order;
    MF_DEV Plane get(int f) const {
        if constexpr (RC) return facet_plane_of(F, P, f, order);
        else return plane[f];
    }
};
template <bool RC>
MF_DEV PlaneSrcT<RC> plane_src(const PlaneSrc& p) {
    return PlaneSrcT<RC>{p.plane, p.F, p.P, p.order};
}
MF_DEV void facet_plane_body(int M, const int* __restrict__ F, const double* __restrict__ P,
                             const int* __restrict__ vmesh, const int* __restrict__ act, Plane* __restrict__ plane,
                             int* __restrict__ deg, int order, int tid, int nth) {
    for (int f = tid; f < M; f += nth) {
        int ia = F[3 * f], ib = F[3 * f + 1], ic = F[3 * f + 2];
        if (!act[mesh_of(vmesh, ia)]) continue;
        if (plane) plane[f] = facet_plane_of(F, P, f, order);  // nullptr: degrees only (planes recomputed)
        atomicAdd(deg + ia, 1);
        atomicAdd(deg + ib, 1);
        atomicAdd(deg + ic, 1);
    }
}
__global__ void k_facet_plane(const int* __restrict__ abort_flag, const int* __restrict__ F, const double* __restrict__ P, const int* __restrict__ dM,
                              const int* __restrict__ vmesh, const int* __restrict__ act, Plane* __restrict__ plane,
                              int* __restrict__ deg, int order) {
    MF_PDL_ENTRY;
    if (*abort_flag) return;
    facet_plane_body(*dM, F, P, vmesh, act, plane, deg, order, blockIdx.x * blockDim.x + threadIdx.x,
                     gridDim.x * blockDim.x);
}

// K2: corner-major incidence scatter; key k = corner*Mcap + f keeps the
// np.add.at order (corner 0 facets ascending, then corner 1, then 2).
__global__ void k_inc_scatter(const int* __restrict__ abort_flag, const int* __restrict__ F, const int* __restrict__ dM, int Mcap,
                              const int* __restrict__ vmesh, const int* __restrict__ act,
                              const int* __restrict__ inc_off, int* __restrict__ cursor, int* __restrict__ inc) {
    MF_PDL_ENTRY;
    if (*abort_flag) return;
    const int M = *dM;
    for (int f = blockIdx.x * blockDim.x + threadIdx.x; f < M; f += gridDim.x * blockDim.x) {
        int t[3] = {F[3 * f], F[3 * f + 1], F[3 * f + 2]};
        if (!act[mesh_of(vmesh, t[0])]) continue;
        // the three cursor atomics and offset loads are independent: all in flight before any store
        int slot[3], base[3];
#pragma unroll
        for (int c = 0; c < 3; c++) {
            slot[c] = atomicAdd(cursor + t[c], 1);
            base[c] = inc_off[t[c]];
        }
#pragma unroll
        for (int c = 0; c < 3; c++) inc[base[c] + slot[c]] = c * Mcap + f;
    }
}

// Quadric accumulation of one facet plane (quadrics.py:42-44 products, 74-76 sums).
struct Q10 {
    double a00, a01, a02, a11, a12, a22, b0, b1, b2, c;
};
MF_DEV void q_zero(Q10& q) { q.a00 = q.a01 = q.a02 = q.a11 = q.a12 = q.a22 = q.b0 = q.b1 = q.b2 = q.c = 0.0; }
MF_DEV void q_add_plane(Q10& q, const Plane& p) {
    q.a00 = q.a00 + p.n0 * p.n0; q.a01 = q.a01 + p.n0 * p.n1; q.a02 = q.a02 + p.n0 * p.n2;
    q.a11 = q.a11 + p.n1 * p.n1; q.a12 = q.a12 + p.n1 * p.n2; q.a22 = q.a22 + p.n2 * p.n2;
    q.b0 = q.b0 + p.d * p.n0; q.b1 = q.b1 + p.d * p.n1; q.b2 = q.b2 + p.d * p.n2;
    q.c = q.c + p.d * p.d;  // degenerate facets: n = 0, d = -0*.. -> d*d == +0 == forced 0 (quadrics.py:65)
}
MF_DEV void q_store(double* __restrict__ vq, int v, const Q10& q) {
    double2* o = reinterpret_cast<double2*>(vq + 10 * (size_t)v);  // 80-byte rows: 16-byte aligned
    o[0] = make_double2(q.a00, q.a01);
    o[1] = make_double2(q.a02, q.a11);
    o[2] = make_double2(q.a12, q.a22);
    o[3] = make_double2(q.b0, q.b1);
    o[4] = make_double2(q.b2, q.c);
}
MF_DEV void q_load(const double* __restrict__ vq, int v, Q10& q) {
    const double2* o = reinterpret_cast<const double2*>(vq + 10 * (size_t)v);
    double2 t0 = o[0], t1 = o[1], t2 = o[2], t3 = o[3], t4 = o[4];
    q.a00 = t0.x; q.a01 = t0.y; q.a02 = t1.x; q.a11 = t1.y; q.a12 = t2.x;
    q.a22 = t2.y; q.b0 = t3.x; q.b1 = t3.y; q.b2 = t4.x; q.c = t4.y;
}

MF_DEV void decode_inc(int k, int Mcap, int& corner, int& f) {
    corner = (k >= 2 * Mcap) ? 2 : (k >= Mcap ? 1 : 0);
    f = k - corner * Mcap;
}

MF_DEV void other_two(const int* __restrict__ F, int f, int corner, int& a, int& b) {
    int x = F[3 * f], y = F[3 * f + 1], z = F[3 * f + 2];
    a = corner == 0 ? y : (corner == 1 ? z : x);
    b = corner == 0 ? z : (corner == 1 ? x : y);
}


// Pair cost (quadrics.py:117-132 + evaluate 53-58) for 'average' placement.
template <int PLACEMENT>
MF_DEV double pair_cost(const Q10& qi, const Q10& qj, double pix, double piy, double piz, double pjx, double pjy,
                        double pjz, int order) {
    double a00 = qi.a00 + qj.a00, a01 = qi.a01 + qj.a01, a02 = qi.a02 + qj.a02;
    double a11 = qi.a11 + qj.a11, a12 = qi.a12 + qj.a12, a22 = qi.a22 + qj.a22;
    double b0 = qi.b0 + qj.b0, b1 = qi.b1 + qj.b1, b2 = qi.b2 + qj.b2, c = qi.c + qj.c;
    double x0 = 0.5 * (pix + pjx), x1 = 0.5 * (piy + pjy), x2 = 0.5 * (piz + pjz);
    if (PLACEMENT) {  // optimal_positions(q, midpoints, 'inverse'), quadrics.py:131
        const double a6[6] = {a00, a01, a02, a11, a12, a22}, bb[3] = {b0, b1, b2}, mid[3] = {x0, x1, x2};
        double t[3];
        mf_optimal_position(a6, bb, mid, t);
        x0 = t[0]; x1 = t[1]; x2 = t[2];
    }
    double quad = 0.0;
    quad = quad + (x0 * a00) * x0;
    quad = quad + (x0 * a01) * x1;
    quad = quad + (x0 * a02) * x2;
    quad = quad + (x1 * a01) * x0;
    quad = quad + (x1 * a11) * x1;
    quad = quad + (x1 * a12) * x2;
    quad = quad + (x2 * a02) * x0;
    quad = quad + (x2 * a12) * x1;
    quad = quad + (x2 * a22) * x2;
    double lin = 2.0 * dot3(b0, b1, b2, x0, x1, x2, order);
    return (quad + lin) + c;
}

// ------------------------------------------------------------------------
// Group-cooperative tier: 16 lanes per vertex (two vertices per warp).  The
// incidence list (deg <= 16) is spread over the lanes, sorted with a shuffle
// bitonic network, every lane gathers its facet's plane and corner vertices
// in parallel, the ten quadric products are staged in shared memory and
// folded by ten lanes (one component each) in incidence order, and the
// 2*deg neighbour candidates are sorted / de-duplicated in shared memory.
// Neighbours are written sorted & unique to nbr[2*inc_off[v] ...]; ucnt = count,
// upcnt = count of neighbours > v (the vertex's lexicographic edges).
constexpr int kGrp = 16;
constexpr int kGrpWarps = 8;  // 256-thread blocks

MF_DEV unsigned grp_mask() { return 0xFFFFu << (threadIdx.x & 16); }

MF_DEV int grp_bitonic16(int x, unsigned mask) {
    const int l = threadIdx.x & 15;
#pragma unroll
    for (int k = 2; k <= 16; k <<= 1) {
#pragma unroll
        for (int j = k >> 1; j > 0; j >>= 1) {
            int y = __shfl_xor_sync(mask, x, j, kGrp);
            bool up = ((l & k) == 0);
            bool lower = ((l & j) == 0);
            x = (lower == up) ? min(x, y) : max(x, y);
        }
    }
    return x;
}

// In-register bitonic network (fully unrolled: the array stays in registers).
template <int L>
MF_DEV void reg_sort(int (&a)[L]) {
#pragma unroll
    for (int k = 2; k <= L; k <<= 1) {
#pragma unroll
        for (int j = k >> 1; j > 0; j >>= 1) {
#pragma unroll
            for (int i = 0; i < L; i++) {
                int ixj = i ^ j;
                if (ixj > i) {
                    int x = a[i], y = a[ixj];
                    bool up = ((i & k) == 0);
                    int lo = min(x, y), hi = max(x, y);
                    a[i] = up ? lo : hi;
                    a[ixj] = up ? hi : lo;
                }
            }
        }
    }
}

// K3 thread tier (deg <= 8): one thread per vertex, incidences and the 16
// neighbour candidates sorted by register networks, every plane / facet gather
// issued before the ordered fold.  Degree 9..32 goes to the warp-per-vertex
// kernel (list `mid`), larger to the block tier (list `heavy`).
constexpr int kThreadDeg = 8;
constexpr int kMid = 32;
constexpr int kVtStage = 4096;  // k_vertex_t neighbour-list stage (ints): 128 vertices of mean degree <= 16
// One vertex of the thread tier: its DEG-padded incidence list sorted in registers (corner-major
// key = np.add.at order), the planes folded from +0.0 in that order, the 2*DEG neighbour candidates
// sorted and de-duplicated into `out`.  DEG = 8 for nearly all vertices; degrees 9..16 take the
// DEG = 16 instance (a divergent branch of the same warp) instead of the warp-per-vertex tier.
template <int DEG, class PS>
MF_DEV void vertex_thread_tier(int v, int s, int d, const int* __restrict__ inc, const int* __restrict__ F,
                               PS plane, int Mcap, double* __restrict__ vq, int* out,
                               int* __restrict__ ucnt, int* __restrict__ upcnt) {
    int k[DEG];
#pragma unroll
    for (int i = 0; i < DEG; i++) k[i] = (i < d) ? inc[s + i] : 0x7fffffff;
    reg_sort(k);
    Q10 q;
    q_zero(q);
    int c[2 * DEG];
#pragma unroll
    for (int i = 0; i < DEG; i++) {
        c[2 * i] = 0x7fffffff;
        c[2 * i + 1] = 0x7fffffff;
        if (i < d) {
            int corner, f;
            decode_inc(k[i], Mcap, corner, f);
            Plane p = plane.get(f);
            q_add_plane(q, p);
            other_two(F, f, corner, c[2 * i], c[2 * i + 1]);
        }
    }
    q_store(vq, v, q);
    reg_sort(c);
    int nu = 0, nup = 0;
#pragma unroll
    for (int i = 0; i < 2 * DEG; i++) {
        const int x = c[i];
        const bool keep = (x != 0x7fffffff) && (i == 0 || x != c[i > 0 ? i - 1 : 0]);
        if (keep) {
            out[nu++] = x;
            nup += x > v;
        }
    }
    ucnt[v] = nu;
    upcnt[v] = nup;
}
// TMAX: largest degree of the thread tier (8: 62 registers, for the bandwidth-bound large rounds;
// 16: 90 registers, degrees 9..16 in-thread instead of the warp tier -- latency-bound rounds)
template <int TMAX, bool RC>
__global__ void __launch_bounds__(128) k_vertex_t(const int* __restrict__ abort_flag, int N,
                                                  const int* __restrict__ inc_off, const int* __restrict__ inc,
                                                  const int* __restrict__ F, PlaneSrc plane,
                                                  int Mcap, double* __restrict__ vq, int* __restrict__ nbr,
                                                  int* __restrict__ ucnt, int* __restrict__ upcnt,
                                                  int* __restrict__ mid, int* __restrict__ mid_count,
                                                  int* __restrict__ heavy, int* __restrict__ heavy_count) {
    MF_PDL_ENTRY;
    if (*abort_flag) return;
    // The neighbour lists of a block's 128 consecutive vertices form one contiguous range
    // (2 * inc_off layout); they are assembled in shared memory and written out coalesced
    // (per-thread stores of a few ints at 2*deg strides touch a sector each).  Slots of
    // mid / heavy vertices and the unused tail of each list get whatever the stage holds:
    // k_vertex_tiers writes the former afterwards, nothing reads the latter.
    __shared__ int s_nb[kVtStage];
    for (int base = blockIdx.x * blockDim.x; base < N; base += gridDim.x * blockDim.x) {
        const int v = base + threadIdx.x;
        const int r0 = inc_off[base], r1 = inc_off[min(N, base + (int)blockDim.x)];
        const bool staged = 2 * (r1 - r0) <= kVtStage;  // block-uniform
        bool work = false;
        int s = 0, d = 0;
        if (v < N) {
            s = inc_off[v];
            d = inc_off[v + 1] - s;
            if (d > TMAX) {
                if (d <= kMid) mid[append_slot(mid_count)] = v;
                else heavy[append_slot(heavy_count)] = v;
            } else {
                work = true;
            }
        }
        if (work) {
            int* out = staged ? s_nb + 2 * (s - r0) : nbr + 2 * (size_t)s;
            if (TMAX == kThreadDeg || d <= kThreadDeg)
                vertex_thread_tier<kThreadDeg>(v, s, d, inc, F, plane_src<RC>(plane), Mcap, vq, out, ucnt, upcnt);
            else vertex_thread_tier<TMAX>(v, s, d, inc, F, plane_src<RC>(plane), Mcap, vq, out, ucnt, upcnt);
        }
        if (staged) {
            __syncthreads();
            int* dst = nbr + 2 * (size_t)r0;
            for (int i = threadIdx.x; i < 2 * (r1 - r0); i += blockDim.x) dst[i] = s_nb[i];
            __syncthreads();
        }
    }
}

// Mid tier (degree 9..32): one full warp per vertex, one incidence per lane.
template <class PS>
MF_DEV void vertex_mid_body(const int* __restrict__ list,
                                                const int* __restrict__ list_count, const int* __restrict__ inc_off,
                                                const int* __restrict__ inc, const int* __restrict__ F,
                                                PS plane, int Mcap, double* __restrict__ vq,
                                                int* __restrict__ nbr, int* __restrict__ ucnt,
                                                int* __restrict__ upcnt, int* __restrict__ heavy,
                                                int* __restrict__ heavy_count) {
    __shared__ double s_q[8][kMid][10];
    __shared__ int s_c[8][2 * kMid];
    const int g = threadIdx.x >> 5;  // warp within block
    const int l = threadIdx.x & 31;
    const unsigned mask = 0xffffffffu;
    const int groups = gridDim.x * (blockDim.x >> 5);
    const int N = *list_count;
    for (int vi = blockIdx.x * (blockDim.x >> 5) + g; vi < N; vi += groups) {
        const int v = list[vi];
        const int s = inc_off[v], d = inc_off[v + 1] - s;
        int k = (l < d) ? inc[s + l] : 0x7fffffff;
#pragma unroll
        for (int kk = 2; kk <= kMid; kk <<= 1) {
#pragma unroll
            for (int j = kk >> 1; j > 0; j >>= 1) {
                int y = __shfl_xor_sync(mask, k, j);
                bool up = ((l & kk) == 0), lower = ((l & j) == 0);
                k = (lower == up) ? min(k, y) : max(k, y);
            }
        }
        int a = 0x7fffffff, b = 0x7fffffff;
        if (l < d) {
            int corner, f;
            decode_inc(k, Mcap, corner, f);
            Plane p = plane.get(f);
            other_two(F, f, corner, a, b);
            double* q = s_q[g][l];
            q[0] = p.n0 * p.n0; q[1] = p.n0 * p.n1; q[2] = p.n0 * p.n2;
            q[3] = p.n1 * p.n1; q[4] = p.n1 * p.n2; q[5] = p.n2 * p.n2;
            q[6] = p.d * p.n0; q[7] = p.d * p.n1; q[8] = p.d * p.n2;
            q[9] = p.d * p.d;
        }
        s_c[g][2 * l] = a;
        s_c[g][2 * l + 1] = b;
        __syncwarp(mask);
        if (l < 10) {  // quadrics.py:72-76: fold each component in incidence order from +0.0
            double acc = 0.0;
            for (int i = 0; i < d; i++) acc = acc + s_q[g][i][l];
            vq[10 * (size_t)v + l] = acc;
        }
        // bitonic sort of the 64 candidates (32 lanes, one compare-exchange each per stage)
        int* c = s_c[g];
        for (int kk = 2; kk <= 2 * kMid; kk <<= 1) {
            for (int j = kk >> 1; j > 0; j >>= 1) {
                int i = ((l & ~(j - 1)) << 1) | (l & (j - 1));  // l-th pair (i, i + j)
                int x = c[i], y = c[i + j];
                bool up = ((i & kk) == 0);
                if ((x > y) == up) { c[i] = y; c[i + j] = x; }
                __syncwarp(mask);
            }
        }
        // unique (keep first of each run), order preserving, among the 2d real values
        int x0 = c[2 * l], x1 = c[2 * l + 1];
        int prev = (l == 0) ? -1 : c[2 * l - 1];
        bool k0 = (2 * l < 2 * d) && x0 != prev;
        bool k1 = (2 * l + 1 < 2 * d) && x1 != x0;
        unsigned b0 = __ballot_sync(mask, k0), b1 = __ballot_sync(mask, k1);
        unsigned u0 = __ballot_sync(mask, k0 && x0 > v), u1 = __ballot_sync(mask, k1 && x1 > v);
        unsigned below = (1u << l) - 1u;
        int pos = __popc(b0 & below) + __popc(b1 & below);
        int* out = nbr + 2 * (size_t)s;
        if (k0) out[pos++] = x0;
        if (k1) out[pos] = x1;
        if (l == 0) {
            ucnt[v] = __popc(b0) + __popc(b1);
            upcnt[v] = __popc(u0) + __popc(u1);
        }
        __syncwarp(mask);
    }
}

// K4: lexicographic edge list + pair cost + rank key + adjacency slots.
// Edge id of (v, u>v) = eoff[v] + rank of u among v's upper neighbours, which
// is exactly np.unique(axis=0)'s lexicographic order (mesh.py:131-134).  Only
// the upper end evaluates an edge (4 lanes per vertex, one upper neighbour
// per lane): it stores the edge (e0, e1, key or cost), fills its own slot and
// appends the edge into a free lower slot of the other end (one atomic per
// edge on that vertex's fill counter) -- slot order inside a vertex is free,
// k_adj_rank orders every vertex's slots by rank afterwards, so no lane ever
// searches another vertex's list.
MF_DEV void sort8_by_key(uint64_t& h, uint64_t& lo, int& u, int& e, unsigned mask) {
    const int l = threadIdx.x & 7;
#pragma unroll
    for (int k = 2; k <= 8; k <<= 1) {
#pragma unroll
        for (int j = k >> 1; j > 0; j >>= 1) {
            const uint64_t ph = __shfl_xor_sync(mask, h, j, 8), pl = __shfl_xor_sync(mask, lo, j, 8);
            const int pu = __shfl_xor_sync(mask, u, j, 8), pe = __shfl_xor_sync(mask, e, j, 8);
            const bool want_min = (((l & k) == 0) == ((l & j) == 0));
            const bool take = want_min ? key_lt(ph, pl, h, lo) : key_lt(h, lo, ph, pl);
            if (take) { h = ph; lo = pl; u = pu; e = pe; }
        }
    }
}

struct EdgeOut {
    int* e0;
    int* e1;
    double* cost;        // seeded rounds only (else nullptr)
    uint64_t* key_hi;    // unseeded: f64_key(cost)
    int* snbr;           // adjacency slots: neighbour, edge id, rank key (unseeded)
    int* seid;
    uint64_t* skey;
    int* lowfill;        // per vertex: lower slots filled so far (zeroed by k_vertex_t)
    int* mate;
    int* minrep;
    int* absorbed;
    int* abshead;
    unsigned long long* suitor;
    unsigned long long* mlo;
    unsigned long long* mhi;
    int* seg_cnt;
    int* ldc;
    int* seg_cnt2;  // absorb-candidate segments (appended while the truncation runs)
    int lite;       // unseeded two-pass form: only the edge arrays (e0, e1 / key_hi at the edge id);
                    // k_adj_build assembles the rank-ordered adjacency (no lower-slot atomics)
};

constexpr int kEdgeLanes = 4;
template <int PLACEMENT>
__global__ void __launch_bounds__(256, PLACEMENT ? 1 : 4) k_edges(const int* __restrict__ abort_flag, int N,
                                               const int* __restrict__ inc_off, const int* __restrict__ nbr,
                                               const int* __restrict__ ucnt, const int* __restrict__ upcnt,
                                               const int* __restrict__ aoff, const int* __restrict__ eoff,
                                               const double* __restrict__ vq, const double* __restrict__ P, EdgeOut o,
                                               int order, int B) {
    MF_PDL_ENTRY;
    if (*abort_flag) return;
    const bool seeded = o.cost != nullptr;
    for (int b = blockIdx.x * blockDim.x + threadIdx.x; b < B; b += gridDim.x * blockDim.x) {
        o.mlo[b] = ~0ull;
        o.mhi[b] = 0ull;
        o.seg_cnt[b] = 0;  // truncation-candidate segments (k_mates appends)
        o.seg_cnt2[b] = 0;
    }
    if (blockIdx.x == 0 && threadIdx.x < 8) o.ldc[threadIdx.x] = 0;  // LD round counters
    const int l = threadIdx.x % kEdgeLanes;
    const int groups = gridDim.x * (blockDim.x / kEdgeLanes);
    for (int v = blockIdx.x * (blockDim.x / kEdgeLanes) + threadIdx.x / kEdgeLanes; v < N; v += groups) {
        if (l == 0) {
            o.mate[v] = -1;
            o.minrep[v] = v;
            o.absorbed[v] = -1;
            o.abshead[v] = -1;
            o.suitor[v] = ~0ull;
        }
        // every per-vertex word is loaded up front (one latency), the neighbour list's offset
        // included -- loaded after the nup branch it cost a dependent round trip (ncu stalls)
        const int nu = ucnt[v], nup = upcnt[v];
        const size_t s2 = (size_t)aoff[v];  // compact adjacency slots
        const size_t sn = 2 * (size_t)inc_off[v];  // neighbour list (k_vertex layout)
        // unseeded: an edge's id is its lower end's slot, so e0 is the slot owner -- written
        // for every slot of v (full sectors; only the lower end's slots are ever read as e0)
        if (!seeded)
            for (int j = l; j < nu; j += kEdgeLanes) o.e0[s2 + j] = v;
        if (l >= nup) continue;
        const int nlow = nu - nup;
        // unseeded: edge id = slot index of the upper end (aoff[v] + j), which orders edges
        // lexicographically like the dense index; seeded: the dense index (PCG stream position)
        const int eb = seeded ? eoff[v] : aoff[v] + nlow;
        Q10 qv;
        q_load(vq, v, qv);
        const double px = P[3 * v], py = P[3 * v + 1], pz = P[3 * v + 2];
        for (int k = l; k < nup; k += kEdgeLanes) {
            const int j = nlow + k;
            const int u = nbr[sn + j];
            const int eid = eb + k;
            Q10 qu;
            q_load(vq, u, qu);
            const double ux = P[3 * u], uy = P[3 * u + 1], uz = P[3 * u + 2];
            // the other end's slot: its atomic and the key-independent stores go out while the
            // quadric gathers are in flight
            size_t su = 0;
            if (!o.lite) {
                su = (size_t)aoff[u] + atomicAdd(o.lowfill + u, 1);
                o.seid[s2 + j] = eid;
                o.snbr[su] = v;
                o.seid[su] = eid;
            }
            o.snbr[s2 + j] = u;
            const double c = pair_cost<PLACEMENT>(qv, qu, px, py, pz, ux, uy, uz, order);
            // unseeded: the rank key IS the order-preserving cost (f64_key is invertible, so no
            // cost array), and the slot arrays double as e1 / key_hi (o.snbr = e1, o.skey = key_hi:
            // the own slot s2 + j is the edge id); seeded: dense ids, the cost feeds k_seed_keys
            const uint64_t key = f64_key(c);
            if (seeded) {
                o.e0[eid] = v;
                o.e1[eid] = u;
                o.cost[eid] = c;
            }
            if (!seeded) {
                o.skey[s2 + j] = key;
                if (!o.lite) o.skey[su] = key;
            }
        }
    }
}

// K4 fused (unseeded rounds): edges, pair costs and the RANK-ORDERED adjacency in one pass,
// no atomics.  Every vertex evaluates all of its incident edges itself -- 8 lanes per vertex,
// lane j owns slot j -- with the pair cost taken in (lower, upper) argument order, so both ends
// produce the same bits; the edge id is the lower end's slot (aoff[lower] + position of the
// upper end in the lower end's sorted neighbour list; a lower neighbour is found by a binary
// search of its list).  A vertex of degree <= 8 then sorts its slots across the lanes by the
// rank key (cost key, edge id) and writes them in rank order; larger degrees keep neighbour
// order (acur = -1, scanned in full) with the argmin as the LD round-0 pick.  The lower end
// also writes the edge arrays (e0 = owner of every slot, e1 / key_hi at the edge id).  This
// replaces k_edges' lower-slot atomics + scattered slot writes AND the k_adj_rank_tiled pass
// that re-read and re-sorted them; the price is evaluating each pair cost twice (FP64 is
// idle here) and a second gather of each neighbour's quadric (L2-resident).
struct EdgeRankOut {
    int* e0;
    int* e1;
    uint64_t* key_hi;
    int* snbr;          // rank-ordered slots: neighbour, edge id, 32-bit key prefix
    int* adj_eid;
    unsigned* adj_k32;
    int* acur;
    int* best;          // LD round-0 picks (nullptr when no LD rounds)
    int* bestu;
    int* mate;
    int* minrep;
    int* absorbed;
    int* abshead;
    unsigned long long* suitor;
    unsigned long long* mlo;
    unsigned long long* mhi;
    int* seg_cnt;
    int* ldc;
    int* seg_cnt2;
};

template <int PLACEMENT>
__global__ void __launch_bounds__(256, PLACEMENT ? 1 : 4) k_edges_rank(const int* __restrict__ abort_flag, int N,
                                                    const int* __restrict__ inc_off, const int* __restrict__ nbr,
                                                    const int* __restrict__ ucnt, const int* __restrict__ aoff,
                                                    const double* __restrict__ vq, const double* __restrict__ P,
                                                    EdgeRankOut o, int order, int B) {
    MF_PDL_ENTRY;
    if (*abort_flag) return;
    for (int b = blockIdx.x * blockDim.x + threadIdx.x; b < B; b += gridDim.x * blockDim.x) {
        o.mlo[b] = ~0ull;
        o.mhi[b] = 0ull;
        o.seg_cnt[b] = 0;
        o.seg_cnt2[b] = 0;
    }
    if (blockIdx.x == 0 && threadIdx.x < 8) o.ldc[threadIdx.x] = 0;
    const int l = threadIdx.x & 7;
    const unsigned mask = 0xFFu << (threadIdx.x & 24);
    const int groups = gridDim.x * (blockDim.x >> 3);
    for (int v = blockIdx.x * (blockDim.x >> 3) + (threadIdx.x >> 3); v < N; v += groups) {
        if (l == 0) {
            o.mate[v] = -1;
            o.minrep[v] = v;
            o.absorbed[v] = -1;
            o.abshead[v] = -1;
            o.suitor[v] = ~0ull;
        }
        const int nu = ucnt[v];
        const size_t s2 = (size_t)aoff[v];
        const size_t sn = 2 * (size_t)inc_off[v];
        Q10 qv;
        q_load(vq, v, qv);
        const double px = P[3 * v], py = P[3 * v + 1], pz = P[3 * v + 2];
        uint64_t bh = ~0ull, bl = ~0ull;  // this lane's best slot (degree > 8: argmin over its slots)
        int bu = -1, be = -1;
        for (int j0 = 0; j0 < nu; j0 += 8) {  // group-uniform trip count
            const int j = j0 + l;
            uint64_t h = ~0ull, lo = ~0ull;
            int u = -1, e = -1;
            if (j < nu) {
                u = nbr[sn + j];
                Q10 qu;
                q_load(vq, u, qu);
                const double ux = P[3 * u], uy = P[3 * u + 1], uz = P[3 * u + 2];
                o.e0[s2 + j] = v;  // slot owner (read as e0 only at the lower end's slots)
                double c;
                if (u > v) {
                    c = pair_cost<PLACEMENT>(qv, qu, px, py, pz, ux, uy, uz, order);
                    e = (int)(s2 + j);
                } else {
                    c = pair_cost<PLACEMENT>(qu, qv, ux, uy, uz, px, py, pz, order);
                    const int* lu = nbr + 2 * (size_t)inc_off[u];
                    int a = 0, z = ucnt[u];  // lower_bound of v in u's sorted neighbour list
                    while (a < z) {
                        const int m = (a + z) >> 1;
                        if (lu[m] < v) a = m + 1; else z = m;
                    }
                    e = aoff[u] + a;
                }
                h = f64_key(c);
                lo = (uint64_t)(unsigned)e;
                if (u > v) {
                    o.e1[e] = u;
                    o.key_hi[e] = h;
                }
            }
            if (nu <= 8) {
                sort8_by_key(h, lo, u, e, mask);
                if (l < nu) {
                    o.snbr[s2 + l] = u;
                    o.adj_eid[s2 + l] = e;
                    o.adj_k32[s2 + l] = (unsigned)(h >> 32);
                }
                bh = h, bl = lo, bu = u, be = e;  // lane 0 holds the lowest-ranked slot
            } else {
                if (j < nu) {
                    o.snbr[s2 + j] = u;
                    o.adj_eid[s2 + j] = e;
                    o.adj_k32[s2 + j] = (unsigned)(h >> 32);
                    if (key_lt(h, lo, bh, bl)) bh = h, bl = lo, bu = u, be = e;
                }
            }
        }
        if (nu > 8) {
#pragma unroll
            for (int off = 4; off > 0; off >>= 1) {
                const uint64_t ph = __shfl_xor_sync(mask, bh, off, 8), pl = __shfl_xor_sync(mask, bl, off, 8);
                const int pu = __shfl_xor_sync(mask, bu, off, 8), pe = __shfl_xor_sync(mask, be, off, 8);
                if (key_lt(ph, pl, bh, bl)) bh = ph, bl = pl, bu = pu, be = pe;
            }
        }
        if (l == 0) {
            o.acur[v] = nu > 8 ? -1 : 0;
            if (o.best) {
                o.best[v] = nu ? be : -1;
                o.bestu[v] = nu ? bu : -1;
            }
        }
    }
}

// K4b (unseeded two-pass form): the rank-ordered adjacency assembled from the edge arrays k_edges
// wrote in its lite form.  Thread per vertex: an upper neighbour's edge id is the vertex's own
// slot; a lower neighbour u's is u's slot of this vertex (aoff[u] + the position of v in u's
// sorted neighbour list -- a binary search of a few L1/L2-resident ints); the rank key is
// key_hi[edge].  Degree <= 8 is sorted in registers by (key, edge id); larger degrees keep
// neighbour order (acur = -1) with the argmin as the LD round-0 pick.  A block's 256 vertices'
// slots are staged in shared memory and written out coalesced.  Replaces the lower-slot atomics
// and scattered slot writes of k_edges and the re-read of k_adj_rank_tiled.
constexpr int kBuildCap = 2048;  // staged slots per block (256 vertices of mean degree <= 8)
MF_DEV int slot_of_lower(const int* __restrict__ nbr, const int* __restrict__ inc_off, const int* __restrict__ ucnt,
                         const int* __restrict__ aoff, int u, int v) {
    const int* lu = nbr + 2 * (size_t)inc_off[u];
    int a = 0, z = ucnt[u];
    while (a < z) {
        const int m = (a + z) >> 1;
        if (lu[m] < v) a = m + 1; else z = m;
    }
    return aoff[u] + a;
}

__global__ void __launch_bounds__(256) k_adj_build(const int* __restrict__ abort_flag, int N,
                                                   const int* __restrict__ inc_off, const int* __restrict__ nbr,
                                                   const int* __restrict__ ucnt, const int* __restrict__ upcnt,
                                                   const int* __restrict__ aoff, const uint64_t* __restrict__ key_hi,
                                                   int* __restrict__ snbr, int* __restrict__ seid,
                                                   unsigned* __restrict__ adj_k32, int* __restrict__ acur,
                                                   int* __restrict__ best, int* __restrict__ bestu) {
    MF_PDL_ENTRY;
    if (*abort_flag) return;
    __shared__ int s_n[kBuildCap];
    __shared__ int s_e[kBuildCap];
    __shared__ unsigned s_32[kBuildCap];
    const int T = blockDim.x;
    for (int v0 = blockIdx.x * T; v0 < N; v0 += gridDim.x * T) {
        const int v1 = min(N, v0 + T);
        const int base = aoff[v0], cnt = aoff[v1] - base;
        const bool staged = cnt <= kBuildCap;  // block-uniform
        const int v = v0 + threadIdx.x;
        if (v < v1) {
            const int nu = ucnt[v], nlow = nu - upcnt[v];
            const int s2 = aoff[v];
            const size_t sn = 2 * (size_t)inc_off[v];
            int* on = staged ? s_n + (s2 - base) : snbr + s2;
            int* oe = staged ? s_e + (s2 - base) : seid + s2;
            unsigned* ok = staged ? s_32 + (s2 - base) : adj_k32 + s2;
            if (nu <= 8) {
                uint64_t h[8];
                unsigned lo[8];
                int u[8];
#pragma unroll
                for (int i = 0; i < 8; i++) {
                    h[i] = ~0ull;
                    lo[i] = ~0u;
                    u[i] = -1;
                    if (i < nu) {
                        u[i] = nbr[sn + i];
                        const int e = i >= nlow ? s2 + i : slot_of_lower(nbr, inc_off, ucnt, aoff, u[i], v);
                        lo[i] = (unsigned)e;
                    }
                }
#pragma unroll
                for (int i = 0; i < 8; i++)
                    if (i < nu) h[i] = key_hi[lo[i]];
#pragma unroll
                for (int k = 2; k <= 8; k <<= 1) {
#pragma unroll
                    for (int j = k >> 1; j > 0; j >>= 1) {
#pragma unroll
                        for (int i = 0; i < 8; i++) {
                            const int ixj = i ^ j;
                            if (ixj > i) {
                                const bool up = ((i & k) == 0);
                                const bool gt = h[i] > h[ixj] || (h[i] == h[ixj] && lo[i] > lo[ixj]);
                                if (gt == up) {
                                    uint64_t th = h[i]; h[i] = h[ixj]; h[ixj] = th;
                                    unsigned tl = lo[i]; lo[i] = lo[ixj]; lo[ixj] = tl;
                                    int tu = u[i]; u[i] = u[ixj]; u[ixj] = tu;
                                }
                            }
                        }
                    }
                }
#pragma unroll
                for (int i = 0; i < 8; i++)
                    if (i < nu) {
                        on[i] = u[i];
                        oe[i] = (int)lo[i];
                        ok[i] = (unsigned)(h[i] >> 32);
                    }
                acur[v] = 0;
                if (best) {
                    best[v] = nu ? (int)lo[0] : -1;
                    bestu[v] = nu ? u[0] : -1;
                }
            } else {
                uint64_t bh = ~0ull, bl = ~0ull;
                int be = -1, bu = -1;
                for (int i = 0; i < nu; i++) {
                    const int ui = nbr[sn + i];
                    const int e = i >= nlow ? s2 + i : slot_of_lower(nbr, inc_off, ucnt, aoff, ui, v);
                    const uint64_t hk = key_hi[e];
                    on[i] = ui;
                    oe[i] = e;
                    ok[i] = (unsigned)(hk >> 32);
                    if (key_lt(hk, (uint64_t)(unsigned)e, bh, bl)) bh = hk, bl = (uint64_t)(unsigned)e, be = e, bu = ui;
                }
                acur[v] = -1;
                if (best) {
                    best[v] = be;
                    bestu[v] = bu;
                }
            }
        }
        if (staged) {
            __syncthreads();
            for (int i = threadIdx.x; i < cnt; i += T) {
                snbr[base + i] = s_n[i];
                seid[base + i] = s_e[i];
                adj_k32[base + i] = s_32[i];
            }
            __syncthreads();
        }
    }
}

// K4b: rank-ordered adjacency.  Every vertex of degree <= 8 has its slots
// sorted in place by the full rank key of their edge -- one thread per vertex,
// register bitonic network on (key_hi, key_lo | edge id) -- so the matching
// kernels find a vertex's best live edge as the FIRST live slot from a
// per-vertex cursor that only moves forward: a slot whose neighbour is
// matched, or whose neighbour already holds a better proposal, stays dead.
// Higher degrees keep their order (acur = -1) and are scanned in full.  The
// 32-bit rank-key prefix of every slot is stored beside it (adj_k32) so the
// scans compare prefixes and gather the full keys only on prefix ties.
// Unseeded keys come from the slots (skey, secondary = edge id); seeded keys
// are gathered once k_seed_keys has run.
// Slots of one vertex at sn / se / sk / k32 (global or shared memory).
template <bool SEEDED>
MF_DEV void rank_one(int v, int nu, const int* sn, const int* se, const uint64_t* sk, int* sn_out, int* se_out,
                     const uint64_t* __restrict__ key_hi, const uint64_t* __restrict__ key_lo, unsigned* k32,
                     int* __restrict__ acur, int* __restrict__ best, int* __restrict__ bestu) {
    typedef typename std::conditional<SEEDED, uint64_t, unsigned>::type Lo;
    if (nu > 8) {
        uint64_t bh = ~0ull, bl = ~0ull;
        int be = -1, bu = -1;
        for (int j = 0; j < nu; j++) {
            const int e = se[j];
            const uint64_t h = SEEDED ? key_hi[e] : sk[j];
            const uint64_t l = SEEDED ? key_lo[e] : (uint64_t)(unsigned)e;
            const int u = sn[j];
            k32[j] = (unsigned)(h >> 32);
            sn_out[j] = u;
            se_out[j] = e;
            if (key_lt(h, l, bh, bl)) { bh = h; bl = l; be = e; bu = u; }
        }
        acur[v] = -1;
        if (best) {
            best[v] = be;
            bestu[v] = bu;
        }
        return;
    }
    uint64_t h[8];
    Lo lo[8];
    int u[8];
#pragma unroll
    for (int i = 0; i < 8; i++) {
        h[i] = ~0ull;
        lo[i] = (Lo)~0ull;
        u[i] = -1;
        if (i < nu) {
            u[i] = sn[i];
            const int e = se[i];
            if (SEEDED) {
                h[i] = key_hi[e];
                lo[i] = (Lo)key_lo[e];
            } else {
                h[i] = sk[i];
                lo[i] = (Lo)(unsigned)e;
            }
        }
    }
    // bitonic network over 8 register entries (keys are unique; padding sorts last)
#pragma unroll
    for (int k = 2; k <= 8; k <<= 1) {
#pragma unroll
        for (int j = k >> 1; j > 0; j >>= 1) {
#pragma unroll
            for (int i = 0; i < 8; i++) {
                const int ixj = i ^ j;
                if (ixj > i) {
                    const bool up = ((i & k) == 0);
                    const bool gt = h[i] > h[ixj] || (h[i] == h[ixj] && lo[i] > lo[ixj]);
                    if (gt == up) {
                        uint64_t th = h[i]; h[i] = h[ixj]; h[ixj] = th;
                        Lo tl = lo[i]; lo[i] = lo[ixj]; lo[ixj] = tl;
                        int tu = u[i]; u[i] = u[ixj]; u[ixj] = tu;
                    }
                }
            }
        }
    }
#pragma unroll
    for (int i = 0; i < 8; i++)
        if (i < nu) {
            sn_out[i] = u[i];
            se_out[i] = (int)(unsigned)lo[i];  // seeded key_lo carries the edge id in its low bits
            k32[i] = (unsigned)(h[i] >> 32);
        }
    acur[v] = 0;
    if (best) {
        best[v] = nu ? (int)(unsigned)lo[0] : -1;
        bestu[v] = nu ? u[0] : -1;
    }
}

// best / bestu (locally-dominant rounds only): every vertex's round-0 pick, i.e. its
// lowest-ranked edge -- nothing is matched yet, so the first LD pick pass is not needed.
template <bool SEEDED>
__global__ void __launch_bounds__(256) k_adj_rank(const int* __restrict__ abort_flag, int N,
                                                  const int* __restrict__ aoff, const int* __restrict__ ucnt,
                                                  int* __restrict__ snbr, int* __restrict__ seid,
                                                  const uint64_t* __restrict__ skey,
                                                  const uint64_t* __restrict__ key_hi,
                                                  const uint64_t* __restrict__ key_lo, unsigned* __restrict__ adj_k32,
                                                  int* __restrict__ acur, int* __restrict__ best,
                                                  int* __restrict__ bestu) {
    MF_PDL_ENTRY;
    if (*abort_flag) return;
    for (int v = blockIdx.x * blockDim.x + threadIdx.x; v < N; v += gridDim.x * blockDim.x) {
        const size_t s = (size_t)aoff[v];
        rank_one<SEEDED>(v, ucnt[v], snbr + s, seid + s, SEEDED ? nullptr : skey + s, snbr + s, seid + s, key_hi,
                         key_lo, adj_k32 + s, acur, best, bestu);
    }
}

// Unseeded rounds: the same sort with the slots of 256 consecutive vertices (one
// contiguous range of the compact adjacency) staged through shared memory, so
// every global load / store is coalesced; a tile whose range exceeds the stage
// (high-degree vertices) sorts straight from / to global memory.  Out of place:
// the unsorted slots (in_nbr, in_eid, in_key) double as the edge arrays e1 /
// key_hi (an edge's id is its lower end's slot), so they must survive.
constexpr int kRankCap = 2048;
constexpr int kRankSmem = 2 * kRankCap * (4 + 4 + 8) + kRankCap * 4;  // double-buffered inputs + k32 (72 KiB)
MF_DEV void cp_async4(void* s, const void* g) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"((unsigned)__cvta_generic_to_shared(s)), "l"(g));
}
MF_DEV void cp_async8(void* s, const void* g) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"((unsigned)__cvta_generic_to_shared(s)), "l"(g));
}
MF_DEV void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
MF_DEV void cp_async_wait1() { asm volatile("cp.async.wait_group 1;\n" ::); }
// The next tile's slots are fetched with cp.async into the other buffer while the
// current tile sorts, so the load phase of one tile overlaps the compute of the last.
__global__ void __launch_bounds__(256) k_adj_rank_tiled(const int* __restrict__ abort_flag, int N,
                                                        const int* __restrict__ aoff, const int* __restrict__ ucnt,
                                                        const int* __restrict__ in_nbr, const int* __restrict__ in_eid,
                                                        const uint64_t* __restrict__ skey, int* __restrict__ snbr,
                                                        int* __restrict__ seid, unsigned* __restrict__ adj_k32,
                                                        int* __restrict__ acur,
                                                        int* __restrict__ best, int* __restrict__ bestu) {
    MF_PDL_ENTRY;
    if (*abort_flag) return;
    extern __shared__ __align__(16) unsigned char rank_smem[];
    uint64_t* s_kb = reinterpret_cast<uint64_t*>(rank_smem);         // [2][cap]
    int* s_nb = reinterpret_cast<int*>(s_kb + 2 * kRankCap);           // [2][cap]
    int* s_eb = s_nb + 2 * kRankCap;                                   // [2][cap]
    unsigned* s_32 = reinterpret_cast<unsigned*>(s_eb + 2 * kRankCap);  // [cap]
    const int T = blockDim.x;
    const int stride = gridDim.x * T;
    // issue the cp.async group of the tile starting at v0 into buffer `buf` (empty group past the end)
    auto prefetch = [&](int v0, int buf) {
        if (v0 < N) {
            const int v1 = min(N, v0 + T);
            const int base = aoff[v0], cnt = aoff[v1] - base;
            if (cnt <= kRankCap) {
                int* dn = s_nb + buf * kRankCap;
                int* de = s_eb + buf * kRankCap;
                uint64_t* dk = s_kb + buf * kRankCap;
                for (int i = threadIdx.x; i < cnt; i += T) {
                    cp_async4(dn + i, in_nbr + base + i);
                    cp_async4(de + i, in_eid + base + i);
                    cp_async8(dk + i, skey + base + i);
                }
            }
        }
        cp_async_commit();
    };
    int buf = 0;
    prefetch(blockIdx.x * T, 0);
    for (int v0 = blockIdx.x * T; v0 < N; v0 += stride, buf ^= 1) {
        prefetch(v0 + stride, buf ^ 1);
        const int v1 = min(N, v0 + T);
        const int base = aoff[v0], cnt = aoff[v1] - base;
        const int v = v0 + threadIdx.x;
        cp_async_wait1();  // this tile's group has landed (the next one may still fly)
        __syncthreads();
        if (cnt > kRankCap) {
            if (v < v1) {
                const size_t s = (size_t)aoff[v];
                rank_one<false>(v, ucnt[v], in_nbr + s, in_eid + s, skey + s, snbr + s, seid + s, nullptr, nullptr,
                                adj_k32 + s, acur, best, bestu);
            }
            __syncthreads();
            continue;  // block-uniform
        }
        int* s_n = s_nb + buf * kRankCap;
        int* s_e = s_eb + buf * kRankCap;
        uint64_t* s_k = s_kb + buf * kRankCap;
        if (v < v1) {
            const int o = aoff[v] - base;
            rank_one<false>(v, ucnt[v], s_n + o, s_e + o, s_k + o, s_n + o, s_e + o, nullptr, nullptr, s_32 + o, acur,
                            best, bestu);
        }
        __syncthreads();
        for (int i = threadIdx.x; i < cnt; i += T) {
            snbr[base + i] = s_n[i];
            seid[base + i] = s_e[i];
            adj_k32[base + i] = s_32[i];
        }
        __syncthreads();  // buffers free before the next prefetch overwrites them
    }
    asm volatile("cp.async.wait_all;\n" ::);
}

// K3h: heavy tier -- one block per high-degree vertex (any degree).
template <class PS>
MF_DEV void vertex_heavy_body(const int* __restrict__ heavy, const int* __restrict__ heavy_count,
                                                      const int* __restrict__ inc_off, int* __restrict__ inc,
                                                      int* __restrict__ inc_tmp, const int* __restrict__ F,
                                                      PS plane, int Mcap, double* __restrict__ vq,
                                                      int* __restrict__ nbr, int* __restrict__ nbr_tmp,
                                                      int* __restrict__ ucnt, int* __restrict__ upcnt) {
    __shared__ int smem[kChunk];
    __shared__ Plane s_pl[256];
    __shared__ int s_scan[33];
    const int H = *heavy_count;
    for (int h = blockIdx.x; h < H; h += gridDim.x) {
        int v = heavy[h];
        int s = inc_off[v], d = inc_off[v + 1] - s;
        block_sort_ints(inc + s, inc_tmp + s, d, smem);
        // sequential fold (thread 0) over planes staged 256 at a time
        Q10 q;
        q_zero(q);
        for (int c0 = 0; c0 < d; c0 += 256) {
            int len = min(256, d - c0);
            if ((int)threadIdx.x < len) {
                int corner, f;
                decode_inc(inc[s + c0 + threadIdx.x], Mcap, corner, f);
                s_pl[threadIdx.x] = plane.get(f);
            }
            __syncthreads();
            if (threadIdx.x == 0)
                for (int i = 0; i < len; i++) q_add_plane(q, s_pl[i]);
            __syncthreads();
        }
        if (threadIdx.x == 0) q_store(vq, v, q);
        // candidates -> nbr[2s .. 2s+2d)
        int* cand = nbr + 2 * (size_t)s;
        for (int i = threadIdx.x; i < d; i += blockDim.x) {
            int corner, f, a, b;
            decode_inc(inc[s + i], Mcap, corner, f);
            other_two(F, f, corner, a, b);
            cand[2 * i] = a;
            cand[2 * i + 1] = b;
        }
        __syncthreads();
        block_sort_ints(cand, nbr_tmp + 2 * (size_t)s, 2 * d, smem);
        // unique compaction (order preserving) through nbr_tmp
        int* tmpo = nbr_tmp + 2 * (size_t)s;
        int base = 0, nup = 0;
        for (int c0 = 0; c0 < 2 * d; c0 += blockDim.x) {
            int i = c0 + threadIdx.x;
            int keep = 0, x = 0;
            if (i < 2 * d) {
                x = cand[i];
                keep = (i == 0) || (x != cand[i - 1]);
            }
            int tot;
            int pos = block_excl_scan(keep, s_scan, &tot);
            if (keep) tmpo[base + pos] = x;
            int upk = keep && x > v;
            int totu;
            block_excl_scan(upk, s_scan, &totu);
            base += tot;
            nup += totu;
        }
        __syncthreads();
        for (int i = threadIdx.x; i < base; i += blockDim.x) cand[i] = tmpo[i];
        if (threadIdx.x == 0) {
            ucnt[v] = base;
            upcnt[v] = nup;
        }
        __syncthreads();
    }
}



// Mid (degree 9..32, a warp per vertex) and heavy (a block per vertex) tiers in one
// launch: both lists are complete once k_vertex_t has run, and they are disjoint.
template <bool RC>
__global__ void __launch_bounds__(256) k_vertex_tiers(const int* __restrict__ abort_flag, const int* __restrict__ mid,
                                                      const int* __restrict__ mid_count, const int* __restrict__ heavy,
                                                      const int* __restrict__ heavy_count,
                                                      const int* __restrict__ inc_off, int* __restrict__ inc,
                                                      int* __restrict__ inc_tmp, const int* __restrict__ F,
                                                      PlaneSrc plane, int Mcap, double* __restrict__ vq,
                                                      int* __restrict__ nbr, int* __restrict__ nbr_tmp,
                                                      int* __restrict__ ucnt, int* __restrict__ upcnt) {
    MF_PDL_ENTRY;
    if (*abort_flag) return;
    vertex_heavy_body(heavy, heavy_count, inc_off, inc, inc_tmp, F, plane_src<RC>(plane), Mcap, vq, nbr, nbr_tmp,
                      ucnt, upcnt);
    vertex_mid_body(mid, mid_count, inc_off, inc, F, plane_src<RC>(plane), Mcap, vq, nbr, ucnt, upcnt, nullptr,
                    nullptr);
}

// ------------------------------------------------------------------------
// K3 fused: every tier of the vertex fold + the adjacency-offset scans in ONE launch.
// A block owns a tile of 128 consecutive vertices (tickets in launch order): thread tier
// (deg <= 8) as k_vertex_t; the tile's degree 9..32 vertices one warp each (mid body), any
// larger one by the whole block (heavy body); then the tile's ucnt / upcnt totals are chained
// through a decoupled look-back (one 64-bit word carries both sums) and the block writes the
// compact adjacency offsets aoff (and the dense lexicographic edge offsets eoff) itself --
// replacing k_vertex_tiers and the k_scan<adj> (+ k_scan<edges>) launches.
constexpr unsigned long long kVsAgg = 1ull << 62, kVsPre = 2ull << 62;
constexpr int kVsTile = 128;
MF_DEV unsigned long long vs_pack(int u, int up) { return ((unsigned long long)(unsigned)u << 31) | (unsigned)up; }
MF_DEV int vs_u(unsigned long long w) { return (int)((w >> 31) & 0x7fffffffull); }
MF_DEV int vs_up(unsigned long long w) { return (int)(w & 0x7fffffffull); }

// one degree-9..32 vertex by warp g of the block (vertex_mid_body's per-vertex step); the
// unique neighbour list goes to `out`, the counts to ucnt / upcnt
template <class PS>
MF_DEV void vertex_mid_one(int v, int s, int d, const int* __restrict__ inc, const int* __restrict__ F,
                           PS plane, int Mcap, double* __restrict__ vq, int* out,
                           int* __restrict__ ucnt, int* __restrict__ upcnt, double (*s_q)[10], int* s_c) {
    const int l = threadIdx.x & 31;
    const unsigned mask = 0xffffffffu;
    int k = (l < d) ? inc[s + l] : 0x7fffffff;
#pragma unroll
    for (int kk = 2; kk <= kMid; kk <<= 1) {
#pragma unroll
        for (int j = kk >> 1; j > 0; j >>= 1) {
            int y = __shfl_xor_sync(mask, k, j);
            bool up = ((l & kk) == 0), lower = ((l & j) == 0);
            k = (lower == up) ? min(k, y) : max(k, y);
        }
    }
    int a = 0x7fffffff, b = 0x7fffffff;
    if (l < d) {
        int corner, f;
        decode_inc(k, Mcap, corner, f);
        Plane p = plane.get(f);
        other_two(F, f, corner, a, b);
        double* q = s_q[l];
        q[0] = p.n0 * p.n0; q[1] = p.n0 * p.n1; q[2] = p.n0 * p.n2;
        q[3] = p.n1 * p.n1; q[4] = p.n1 * p.n2; q[5] = p.n2 * p.n2;
        q[6] = p.d * p.n0; q[7] = p.d * p.n1; q[8] = p.d * p.n2;
        q[9] = p.d * p.d;
    }
    s_c[2 * l] = a;
    s_c[2 * l + 1] = b;
    __syncwarp(mask);
    if (l < 10) {  // quadrics.py:72-76: fold each component in incidence order from +0.0
        double acc = 0.0;
        for (int i = 0; i < d; i++) acc = acc + s_q[i][l];
        vq[10 * (size_t)v + l] = acc;
    }
    for (int kk = 2; kk <= 2 * kMid; kk <<= 1) {
        for (int j = kk >> 1; j > 0; j >>= 1) {
            int i = ((l & ~(j - 1)) << 1) | (l & (j - 1));
            int x = s_c[i], y = s_c[i + j];
            bool up = ((i & kk) == 0);
            if ((x > y) == up) { s_c[i] = y; s_c[i + j] = x; }
            __syncwarp(mask);
        }
    }
    int x0 = s_c[2 * l], x1 = s_c[2 * l + 1];
    int prev = (l == 0) ? -1 : s_c[2 * l - 1];
    bool k0 = (2 * l < 2 * d) && x0 != prev;
    bool k1 = (2 * l + 1 < 2 * d) && x1 != x0;
    unsigned b0 = __ballot_sync(mask, k0), b1 = __ballot_sync(mask, k1);
    unsigned u0 = __ballot_sync(mask, k0 && x0 > v), u1 = __ballot_sync(mask, k1 && x1 > v);
    unsigned below = (1u << l) - 1u;
    int pos = __popc(b0 & below) + __popc(b1 & below);
    if (k0) out[pos++] = x0;
    if (k1) out[pos] = x1;
    if (l == 0) {
        ucnt[v] = __popc(b0) + __popc(b1);
        upcnt[v] = __popc(u0) + __popc(u1);
    }
    __syncwarp(mask);
}

// one vertex of any degree by the whole block (vertex_heavy_body's per-vertex step): the
// incidences sorted in place, the fold staged kVsTile planes at a time, the neighbour
// candidates sorted / de-duplicated in nbr (scratch nbr_tmp)
template <class PS>
MF_DEV void vertex_heavy_one(int v, int s, int d, int* __restrict__ inc, int* __restrict__ inc_tmp,
                             const int* __restrict__ F, PS plane, int Mcap,
                             double* __restrict__ vq, int* __restrict__ nbr, int* __restrict__ nbr_tmp,
                             int* __restrict__ ucnt, int* __restrict__ upcnt, int* smem, Plane* s_pl, int* s_scan) {
    block_sort_ints(inc + s, inc_tmp + s, d, smem);
    Q10 q;
    q_zero(q);
    for (int c0 = 0; c0 < d; c0 += kVsTile) {
        const int len = min(kVsTile, d - c0);
        for (int i = threadIdx.x; i < len; i += blockDim.x) {
            int corner, f;
            decode_inc(inc[s + c0 + i], Mcap, corner, f);
            s_pl[i] = plane.get(f);
        }
        __syncthreads();
        if (threadIdx.x == 0)
            for (int i = 0; i < len; i++) q_add_plane(q, s_pl[i]);
        __syncthreads();
    }
    if (threadIdx.x == 0) q_store(vq, v, q);
    int* cand = nbr + 2 * (size_t)s;
    for (int i = threadIdx.x; i < d; i += blockDim.x) {
        int corner, f, a, b;
        decode_inc(inc[s + i], Mcap, corner, f);
        other_two(F, f, corner, a, b);
        cand[2 * i] = a;
        cand[2 * i + 1] = b;
    }
    __syncthreads();
    block_sort_ints(cand, nbr_tmp + 2 * (size_t)s, 2 * d, smem);
    int* tmpo = nbr_tmp + 2 * (size_t)s;
    int base = 0, nup = 0;
    for (int c0 = 0; c0 < 2 * d; c0 += blockDim.x) {
        int i = c0 + threadIdx.x;
        int keep = 0, x = 0;
        if (i < 2 * d) {
            x = cand[i];
            keep = (i == 0) || (x != cand[i - 1]);
        }
        int tot;
        int pos = block_excl_scan(keep, s_scan, &tot);
        if (keep) tmpo[base + pos] = x;
        int upk = keep && x > v;
        int totu;
        block_excl_scan(upk, s_scan, &totu);
        base += tot;
        nup += totu;
    }
    __syncthreads();
    for (int i = threadIdx.x; i < base; i += blockDim.x) cand[i] = tmpo[i];
    if (threadIdx.x == 0) {
        ucnt[v] = base;
        upcnt[v] = nup;
    }
    __syncthreads();
}

struct VertexScanArgs {
    const int* abort_flag;
    int N;
    const int* inc_off;
    int* inc;
    int* inc_tmp;
    const int* F;
    PlaneSrc plane;
    int Mcap;
    double* vq;
    int* nbr;
    int* nbr_tmp;
    int* ucnt;
    int* upcnt;
    int* aoff;  // compact adjacency offsets (exclusive scan of ucnt), [N+1]
    int* eoff;  // dense edge offsets (exclusive scan of upcnt), [N+1]
    unsigned long long* state;  // look-back words, zero on entry; the ticket follows them
    int* ticket;
    unsigned long long* clear;  // the other round's look-back buffer, cleared here for the next round
    int clear_words;
};

// THREADS = 128 or 256 per block for a tile of 128 vertices: the extra warps only share the
// tile's mid-degree vertices (one warp each) and the heavy / scan / write-out phases.
template <int THREADS>
__global__ void __launch_bounds__(THREADS) k_vertex_scan(VertexScanArgs a) {
    MF_PDL_ENTRY;
    __shared__ int s_nb[kVtStage];
    __shared__ union {
        struct {
            double q[THREADS / 32][kMid][10];
            int c[THREADS / 32][2 * kMid];
        } mid;
        struct {
            int sort[kChunk];
            Plane pl[kVsTile];
        } heavy;
    } sc;
    __shared__ int s_list[kVsTile];
    __shared__ int s_nmid, s_nheavy, s_tile;
    __shared__ int s_scan[33];
    __shared__ int s_pre[2];
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < a.clear_words; i += gridDim.x * blockDim.x)
        a.clear[i] = 0ull;
    if (*a.abort_flag) return;
    const int N = a.N;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    while (true) {
        if (tid == 0) {
            s_tile = atomicAdd(a.ticket, 1);
            s_nmid = 0;
            s_nheavy = 0;
        }
        __syncthreads();
        const int tile = s_tile;
        const int base = tile * kVsTile;
        if (base >= N) break;
        const int v = base + tid;
        const bool mine = tid < kVsTile && v < N;  // the thread-tier owner of vertex v
        const int r0 = a.inc_off[base], r1 = a.inc_off[min(N, base + kVsTile)];
        const bool staged = 2 * (r1 - r0) <= kVtStage;  // block-uniform
        int s = 0, d = 0, nu = 0, nup = 0;
        if (mine) {
            s = a.inc_off[v];
            d = a.inc_off[v + 1] - s;
            if (d > kThreadDeg) {
                if (d <= kMid) s_list[atomicAdd(&s_nmid, 1)] = v;
                else s_list[kVsTile - 1 - atomicAdd(&s_nheavy, 1)] = v;
            } else {
                int k[kThreadDeg];
#pragma unroll
                for (int i = 0; i < kThreadDeg; i++) k[i] = (i < d) ? a.inc[s + i] : 0x7fffffff;
                reg_sort(k);
                Q10 q;
                q_zero(q);
                int c[2 * kThreadDeg];
#pragma unroll
                for (int i = 0; i < kThreadDeg; i++) {
                    c[2 * i] = 0x7fffffff;
                    c[2 * i + 1] = 0x7fffffff;
                    if (i < d) {
                        int corner, f;
                        decode_inc(k[i], a.Mcap, corner, f);
                        Plane p = a.plane.plane[f];  // materialised planes (no recompute here)
                        q_add_plane(q, p);
                        other_two(a.F, f, corner, c[2 * i], c[2 * i + 1]);
                    }
                }
                q_store(a.vq, v, q);
                reg_sort(c);
                int* out = staged ? s_nb + 2 * (s - r0) : a.nbr + 2 * (size_t)s;
#pragma unroll
                for (int i = 0; i < 2 * kThreadDeg; i++) {
                    const int x = c[i];
                    const bool keep = (x != 0x7fffffff) && (i == 0 || x != c[i > 0 ? i - 1 : 0]);
                    if (keep) {
                        out[nu++] = x;
                        nup += x > v;
                    }
                }
                a.ucnt[v] = nu;
                a.upcnt[v] = nup;
            }
        }
        __syncthreads();
        const int nmid = s_nmid, nheavy = s_nheavy;
        for (int i = warp; i < nmid; i += THREADS / 32) {
            const int w = s_list[i];
            const int ws = a.inc_off[w], wd = a.inc_off[w + 1] - ws;
            int* out = staged ? s_nb + 2 * (ws - r0) : a.nbr + 2 * (size_t)ws;
            vertex_mid_one(w, ws, wd, a.inc, a.F, plane_src<false>(a.plane), a.Mcap, a.vq, out, a.ucnt, a.upcnt, sc.mid.q[warp],
                           sc.mid.c[warp]);
        }
        __syncthreads();
        for (int i = 0; i < nheavy; i++) {
            const int w = s_list[kVsTile - 1 - i];
            const int ws = a.inc_off[w], wd = a.inc_off[w + 1] - ws;
            vertex_heavy_one(w, ws, wd, a.inc, a.inc_tmp, a.F, plane_src<false>(a.plane), a.Mcap, a.vq, a.nbr, a.nbr_tmp, a.ucnt,
                             a.upcnt, sc.heavy.sort, sc.heavy.pl, s_scan);
            if (staged) {  // the heavy list lives in global memory: copy it into the stage
                const int cnt = a.ucnt[w];
                for (int j = tid; j < cnt; j += THREADS) s_nb[2 * (ws - r0) + j] = a.nbr[2 * (size_t)ws + j];
            }
            __syncthreads();
        }
        // this tile's counts (mid / heavy ones were written by other threads of the block)
        if (mine && d > kThreadDeg) {
            nu = a.ucnt[v];
            nup = a.upcnt[v];
        }
        int tot_u, tot_up;
        const int ex_u = block_excl_scan(nu, s_scan, &tot_u);
        const int ex_up = block_excl_scan(nup, s_scan, &tot_up);
        if (warp == 0) {  // decoupled look-back over the tiles before this one
            if (lane == 0) {
                const unsigned long long word = (tile == 0 ? kVsPre : kVsAgg) | vs_pack(tot_u, tot_up);
                __threadfence();
                atomicExch(a.state + tile, word);
            }
            int pu = 0, pup = 0;
            if (tile > 0) {
                int pred = tile - 1;
                while (true) {
                    const int idx = pred - lane;
                    unsigned long long w = idx >= 0 ? ld_volatile(a.state + idx) : kVsPre;
                    while (__any_sync(0xffffffffu, (w >> 62) == 0ull))
                        if ((w >> 62) == 0ull) w = ld_volatile(a.state + idx);
                    const unsigned pmask = __ballot_sync(0xffffffffu, (w >> 62) == 2ull);
                    const int first = pmask ? (__ffs(pmask) - 1) : 32;
                    pu += warp_sum(lane <= first ? vs_u(w) : 0);
                    pup += warp_sum(lane <= first ? vs_up(w) : 0);
                    if (pmask) break;
                    pred -= 32;
                }
                if (lane == 0) {
                    __threadfence();
                    atomicExch(a.state + tile, kVsPre | vs_pack(pu + tot_u, pup + tot_up));
                }
            }
            if (lane == 0) {
                s_pre[0] = pu;
                s_pre[1] = pup;
            }
        }
        __syncthreads();
        if (mine) {
            a.aoff[v] = s_pre[0] + ex_u;
            if (a.eoff) a.eoff[v] = s_pre[1] + ex_up;
            if (v == N - 1) {
                a.aoff[N] = s_pre[0] + tot_u;
                if (a.eoff) a.eoff[N] = s_pre[1] + tot_up;
            }
        }
        if (staged) {
            int* dst = a.nbr + 2 * (size_t)r0;
            for (int i = tid; i < 2 * (r1 - r0); i += THREADS) dst[i] = s_nb[i];
        }
        __syncthreads();
    }
    if (N == 0 && blockIdx.x == 0 && tid == 0) {
        a.aoff[0] = 0;
        if (a.eoff) a.eoff[0] = 0;
    }
}

// ------------------------------------------------------------------------
// Seeded shuffle keys (decimate.py:184-191).
__global__ void k_cost_minmax(const int* __restrict__ abort_flag, const int* __restrict__ dE, const double* __restrict__ cost, const int* __restrict__ e0,
                              const int* __restrict__ vmesh, unsigned long long* __restrict__ mlo,
                              unsigned long long* __restrict__ mhi) {
    MF_PDL_ENTRY;
    if (*abort_flag) return;
    const int E = *dE;
    uint64_t lo = ~0ull, hi = 0ull;
    for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < E; e += gridDim.x * blockDim.x) {
        int b = mesh_of(vmesh, e0[e]);
        uint64_t k = f64_key(cost[e]);
        if (vmesh) {
            atomicMin(mlo + b, (unsigned long long)k);
            atomicMax(mhi + b, (unsigned long long)k);
        } else {
            lo = k < lo ? k : lo;
            hi = k > hi ? k : hi;
        }
    }
    if (!vmesh) {
        for (int o = 16; o > 0; o >>= 1) {
            uint64_t a = __shfl_xor_sync(0xffffffffu, lo, o), b = __shfl_xor_sync(0xffffffffu, hi, o);
            lo = a < lo ? a : lo;
            hi = b > hi ? b : hi;
        }
        if ((threadIdx.x & 31) == 0) {
            atomicMin(mlo, (unsigned long long)lo);
            atomicMax(mhi, (unsigned long long)hi);
        }
    }
}

typedef unsigned __int128 u128;
MF_DEV u128 pcg_mult() { return ((u128)0x2360ED051FC65DA4ull << 64) | 0x4385DF649FCCF645ull; }

// state after `delta` LCG steps: s' = A s + C with (A, C) from square-and-multiply.
MF_DEV u128 pcg_advance(u128 s, u128 inc, uint64_t delta) {
    u128 cur_m = pcg_mult(), cur_p = inc, acc_m = 1, acc_p = 0;
    while (delta) {
        if (delta & 1) {
            acc_m *= cur_m;
            acc_p = acc_p * cur_m + cur_p;
        }
        cur_p = (cur_m + 1) * cur_p;
        cur_m *= cur_m;
        delta >>= 1;
    }
    return acc_m * s + acc_p;
}
MF_DEV uint64_t pcg_out(u128 s) {
    uint64_t hi = (uint64_t)(s >> 64), lo = (uint64_t)s;
    uint64_t x = hi ^ lo;
    unsigned rot = (unsigned)(hi >> 58);
    return (x >> rot) | (x << ((64 - rot) & 63));
}

// One thread per run of kSeedRun consecutive edges: jump once, then step.
constexpr int kSeedRun = 16;
__global__ void k_seed_keys(const int* __restrict__ abort_flag, const int* __restrict__ dE, const double* __restrict__ cost, const int* __restrict__ e0,
                            const int* __restrict__ vmesh, const int* __restrict__ eoff, const int* __restrict__ voff,
                            const unsigned long long* __restrict__ mlo, const unsigned long long* __restrict__ mhi,
                            uint64_t s_hi, uint64_t s_lo, uint64_t i_hi,
                            uint64_t i_lo, uint64_t* __restrict__ key_hi, uint64_t* __restrict__ key_lo) {
    MF_PDL_ENTRY;
    if (*abort_flag) return;
    const int E = *dE;
    const u128 s0 = ((u128)s_hi << 64) | s_lo, inc = ((u128)i_hi << 64) | i_lo;
    const u128 M = pcg_mult();
    for (long long r = blockIdx.x * (long long)blockDim.x + threadIdx.x; r * kSeedRun < E;
         r += (long long)gridDim.x * blockDim.x) {
        int e = (int)(r * kSeedRun);
        int eend = min(E, e + kSeedRun);
        int cur_b = -1;
        u128 st = 0;
        double lo = 0.0, width = 0.0;
        for (; e < eend; e++) {
            int b = mesh_of(vmesh, e0[e]);
            if (b != cur_b) {
                cur_b = b;
                int local = e - (vmesh ? eoff[voff[b]] : 0);
                st = pcg_advance(s0, inc, (uint64_t)local + 1ull);
                lo = f64_unkey(mlo[b]);
                double hi = f64_unkey(mhi[b]);
                width = 1e-12 * (hi - lo);
            } else {
                st = st * M + inc;
            }
            double c = cost[e];
            long long bucket = (width > 0.0) ? (long long)floor((c - lo) / width) : 0ll;
            uint64_t k53 = pcg_out(st) >> 11;
            key_hi[e] = ((uint64_t)bucket << 24) | (k53 >> 29);
            key_lo[e] = ((k53 & ((1ull << 29) - 1ull)) << 35) | (uint64_t)e;
        }
    }
}

// ------------------------------------------------------------------------
// K5: greedy matching by proposals (Suitor algorithm, Manne & Halappanavar).
// Every vertex proposes to the neighbour whose incident edge ranks best among
// those it can win (the neighbour's current suitor edge ranks worse); a
// successful 32-bit CAS on suitor[v] may displace an earlier suitor, which
// then proposes again.  Keys are unique, so the fixed point is the unique
// greedy matching of the rank order -- exactly the sequential scan of
// decimate.py:256-263 run to exhaustion -- with no grid-wide barrier.
struct MatchArgs {
    int N;
    const int* aoff;      // compact adjacency offsets
    const int* ucnt;
    const int* nbr;
    const int* adj_eid;
    const unsigned* adj_k32;  // top 32 bits of each adjacency slot's rank key
    const int* e0;
    const int* e1;
    const uint64_t* key_hi;
    const uint64_t* key_lo;  // nullptr -> secondary key is the edge id
    unsigned long long* suitor;  // per vertex: (k32 << 32) | edge of the best proposal received, ~0 = none
    const int* abort_flag;
    const int* mate;       // nullable: vertices matched by the LD rounds are not eligible
    const int* front0;     // nullable: proposers = residual LD frontier, else all vertices
    const int* front1;
    const int* counters;
    int* acur;             // rank-ordered adjacency cursors (k_adj_sort), -1 = unsorted vertex
};

MF_DEV void edge_key(const MatchArgs& a, int e, uint64_t& h, uint64_t& l) {
    h = a.key_hi[e];
    l = a.key_lo ? a.key_lo[e] : (uint64_t)(unsigned)e;
}
// strict rank order of edge e (prefix ke) against edge f (prefix kf); the full
// 128-bit keys are only gathered when the 32-bit prefixes tie
MF_DEV bool edge_lt(const MatchArgs& a, unsigned ke, int e, unsigned kf, int f) {
    if (ke != kf) return ke < kf;
    uint64_t h1, l1, h2, l2;
    edge_key(a, e, h1, l1);
    edge_key(a, f, h2, l2);
    return key_lt(h1, l1, h2, l2);
}

template <int L>
__global__ void __launch_bounds__(256) k_suitor(MatchArgs a) {
    MF_PDL_ENTRY;
    if (*a.abort_flag) return;
    // 8 lanes per proposer: the adjacency of `cur` is scanned in parallel
    // (one neighbour per lane), the best winnable edge is an argmin over the
    // group, and lane 0 issues a 64-bit CAS of (key prefix | edge id) on the
    // neighbour's suitor word.  Control flow is uniform per group.
    constexpr int LB = L == 8 ? 3 : (L == 4 ? 2 : 1);
    const int g = threadIdx.x >> LB;
    const int l = threadIdx.x & (L - 1);
    const unsigned gmask = (1u << L) - 1u;
    const unsigned mask = gmask << (threadIdx.x & (32 - L));
    const int groups = gridDim.x * (blockDim.x >> LB);
    const int* list = nullptr;
    int nprop = a.N;
    if (a.front0) {
        const int which = __ldcg(a.counters + 3);
        list = which ? a.front1 : a.front0;
        nprop = __ldcg(a.counters + which);
    }
    for (int ui = blockIdx.x * (blockDim.x >> LB) + g; ui < nprop; ui += groups) {
        int cur = list ? __ldcg(list + ui) : ui;
        if (a.mate && __ldcg(a.mate + cur) >= 0) continue;
        while (cur >= 0) {
            const size_t s = (size_t)a.aoff[cur];
            const int nu = a.ucnt[cur];
            int be = -1, bv = -1;
            unsigned bk = 0xffffffffu;
            unsigned long long bsw = ~0ull;  // the suitor word seen when the slot was judged winnable
            const int c0 = a.acur[cur];
            if (c0 >= 0) {
                // rank-ordered adjacency: the best winnable edge is the first winnable slot.
                // A slot is dead for good once its neighbour is LD-matched or holds a better
                // proposal (suitor words only improve), so the cursor moves past dead slots.
                int c = c0;
                for (; c < nu; c += L) {
                    const int j = c + l;
                    bool ok = false;
                    unsigned ke = 0;
                    int e = -1, v = -1;
                    unsigned long long sw = ~0ull;
                    if (j < nu) {
                        e = a.adj_eid[s + j];
                        ke = a.adj_k32[s + j];
                        v = a.nbr[s + j];
                        ok = !(a.mate && __ldcg(a.mate + v) >= 0);
                        if (ok) {
                            sw = ld_volatile(a.suitor + v);
                            ok = sw == ~0ull || edge_lt(a, ke, e, (unsigned)(sw >> 32), (int)(unsigned)sw);
                        }
                    }
                    const unsigned bal = (__ballot_sync(mask, ok) >> (threadIdx.x & (32 - L))) & gmask;
                    if (bal) {
                        const int f = __ffs(bal) - 1;
                        bk = __shfl_sync(mask, ke, f, L);
                        be = __shfl_sync(mask, e, f, L);
                        bv = __shfl_sync(mask, v, f, L);
                        bsw = __shfl_sync(mask, sw, f, L);
                        c += f;
                        break;
                    }
                }
                if (l == 0) a.acur[cur] = c < nu ? c : nu;
            } else {
                for (int j = l; j < nu; j += L) {
                    const int e = a.adj_eid[s + j];
                    const unsigned ke = a.adj_k32[s + j];
                    if (be >= 0 && !edge_lt(a, ke, e, bk, be)) continue;
                    const int v = a.nbr[s + j];
                    if (a.mate && __ldcg(a.mate + v) >= 0) continue;
                    const unsigned long long sw = ld_volatile(a.suitor + v);
                    if (sw != ~0ull && !edge_lt(a, ke, e, (unsigned)(sw >> 32), (int)(unsigned)sw)) continue;
                    bk = ke; be = e; bv = v; bsw = sw;
                }
#pragma unroll
                for (int o = L / 2; o > 0; o >>= 1) {
                    unsigned ok = __shfl_xor_sync(mask, bk, o, L);
                    int oe = __shfl_xor_sync(mask, be, o, L), ov = __shfl_xor_sync(mask, bv, o, L);
                    unsigned long long osw = __shfl_xor_sync(mask, bsw, o, L);
                    if (oe >= 0 && (be < 0 || edge_lt(a, ok, oe, bk, be))) { bk = ok; be = oe; bv = ov; bsw = osw; }
                }
            }
            if (be < 0) break;  // nothing winnable: cur stays unmatched unless proposed to
            int next = -2;      // -2: lost a race, re-scan cur
            if (l == 0) {
                const unsigned long long mine = ((unsigned long long)bk << 32) | (unsigned)be;
                unsigned long long sw = bsw;  // a stale expected value only costs one failed CAS
                while (true) {
                    if (sw != ~0ull && !edge_lt(a, bk, be, (unsigned)(sw >> 32), (int)(unsigned)sw)) break;
                    unsigned long long old = atomicCAS(a.suitor + bv, sw, mine);
                    if (old == sw) {
                        if (sw == ~0ull) next = -1;
                        else {
                            int se = (int)(unsigned)sw;
                            next = (a.e0[se] == bv) ? a.e1[se] : a.e0[se];
                        }
                        break;
                    }
                    sw = old;
                }
            }
            next = __shfl_sync(mask, next, 0, L);
            if (next != -2) cur = next;
        }
    }
}

// Thread-per-proposer Suitor over the rank-ordered adjacency: a proposer walks
// its slots from the cursor and proposes at the first winnable one (the best,
// by the slot order); every proposer is in flight at once (one wave), which
// is what bounds the displacement chains at latency-bound sizes.  Unsorted
// (high-degree) vertices take the full argmin scan.
__global__ void __maxnreg__(48) k_suitor1(MatchArgs a) {
    MF_PDL_ENTRY;
    if (*a.abort_flag) return;
    const int* list = nullptr;
    int nprop = a.N;
    if (a.front0) {
        const int which = __ldcg(a.counters + 3);
        list = which ? a.front1 : a.front0;
        nprop = __ldcg(a.counters + which);
    }
    for (int ui = blockIdx.x * blockDim.x + threadIdx.x; ui < nprop; ui += gridDim.x * blockDim.x) {
        int cur = list ? __ldcg(list + ui) : ui;
        if (a.mate && __ldcg(a.mate + cur) >= 0) continue;
        while (cur >= 0) {
            const size_t s = (size_t)a.aoff[cur];
            const int nu = a.ucnt[cur];
            int be = -1, bv = -1;
            unsigned bk = 0xffffffffu;
            unsigned long long bsw = ~0ull;
            int c = a.acur[cur];
            if (c >= 0) {
                for (; c < nu; c++) {
                    const int v = a.nbr[s + c];
                    if (a.mate && __ldcg(a.mate + v) >= 0) continue;
                    const int e = a.adj_eid[s + c];
                    const unsigned ke = a.adj_k32[s + c];
                    const unsigned long long sw = ld_volatile(a.suitor + v);
                    if (sw == ~0ull || edge_lt(a, ke, e, (unsigned)(sw >> 32), (int)(unsigned)sw)) {
                        bk = ke; be = e; bv = v; bsw = sw;
                        break;
                    }
                }
                a.acur[cur] = c;
            } else {
                for (int j = 0; j < nu; j++) {
                    const int e = a.adj_eid[s + j];
                    const unsigned ke = a.adj_k32[s + j];
                    if (be >= 0 && !edge_lt(a, ke, e, bk, be)) continue;
                    const int v = a.nbr[s + j];
                    if (a.mate && __ldcg(a.mate + v) >= 0) continue;
                    const unsigned long long sw = ld_volatile(a.suitor + v);
                    if (sw != ~0ull && !edge_lt(a, ke, e, (unsigned)(sw >> 32), (int)(unsigned)sw)) continue;
                    bk = ke; be = e; bv = v; bsw = sw;
                }
            }
            if (be < 0) break;  // nothing winnable: cur stays unmatched unless proposed to
            const unsigned long long mine = ((unsigned long long)bk << 32) | (unsigned)be;
            unsigned long long sw = bsw;  // a stale expected value only costs one failed CAS
            int next = -2;  // -2: lost a race, re-scan cur (the lost slot is dead now)
            while (true) {
                if (sw != ~0ull && !edge_lt(a, bk, be, (unsigned)(sw >> 32), (int)(unsigned)sw)) break;
                const unsigned long long old = atomicCAS(a.suitor + bv, sw, mine);
                if (old == sw) {
                    if (sw == ~0ull) next = -1;
                    else {
                        const int se = (int)(unsigned)sw;
                        next = (a.e0[se] == bv) ? a.e1[se] : a.e0[se];
                    }
                    break;
                }
                sw = old;
            }
            if (next != -2) cur = next;
        }
    }
}

// Locally-dominant rounds (persistent, cooperative launch, grid barrier).
// Each round every frontier vertex (8 lanes) picks its best live incident
// edge (lowest rank among edges to unmatched neighbours); an edge that is the
// pick of both endpoints is matched -- it is then the first of its
// neighbourhood in rank order, so the sequential greedy scan accepts it too.
// Matched / exhausted vertices leave the frontier.  After `max_rounds` the
// remaining frontier is finished by k_suitor on the residual graph.
constexpr int kLDRounds = 12;  // most LD rounds a graph holds (default plan: 4 from 2^21, 2 from 2^17)
constexpr int kLDMinVertices = 1 << 21;  // measured: Suitor alone wins at 640k (cfg4), LD at 10M (cfg5)
struct LDArgs {
    int N;
    const int* aoff;
    const int* ucnt;
    const int* nbr;
    const int* adj_eid;
    const unsigned* adj_k32;
    const uint64_t* key_hi;
    const uint64_t* key_lo;
    int* mate;     // -1 unmatched
    int* best;     // per vertex: picked edge
    int* bestu;    // per vertex: the other endpoint of the pick
    int* front0;
    int* front1;
    int* counters;  // [0],[1] frontier sizes, [2] rounds run, [3] which frontier holds the residual
    unsigned* bar;
    int max_rounds;
    const int* abort_flag;
    int* acur;      // per vertex: first possibly-live slot of its rank-ordered adjacency (-1 = unsorted)
    cudaGraphConditionalHandle cond;  // device-driven round loop (WHILE node), 0 = fixed rounds
};

MF_DEV bool ld_lt(const LDArgs& a, unsigned ke, int e, unsigned kf, int f) {
    if (ke != kf) return ke < kf;
    uint64_t h1 = a.key_hi[e], h2 = a.key_hi[f];
    uint64_t l1 = a.key_lo ? a.key_lo[e] : (uint64_t)(unsigned)e, l2 = a.key_lo ? a.key_lo[f] : (uint64_t)(unsigned)f;
    return key_lt(h1, l1, h2, l2);
}

// Block-ordered append: survivors of one block keep their relative order and
// land in one contiguous chunk (one atomic per block), so the frontier stays
// roughly sorted by vertex id and the next round streams the adjacency.
MF_DEV void block_append(bool keep, int v, int* __restrict__ out, int* __restrict__ counter) {
    __shared__ int s_scan[33];
    __shared__ int s_base;
    int tot;
    int pos = block_excl_scan(keep ? 1 : 0, s_scan, &tot);
    if (threadIdx.x == 0) s_base = tot ? atomicAdd(counter, tot) : 0;
    __syncthreads();
    if (keep) out[s_base + pos] = v;
    __syncthreads();
}

// initial frontier: every vertex with an edge (mate reset)
__global__ void __launch_bounds__(256) k_ld_init(LDArgs a) {
    MF_PDL_ENTRY;
    if (*a.abort_flag) return;
    const int nb = (a.N + blockDim.x - 1) / blockDim.x;
    for (int b = blockIdx.x; b < nb; b += gridDim.x) {
        const int v = b * blockDim.x + threadIdx.x;
        bool keep = false;
        if (v < a.N) {
            a.mate[v] = -1;
            keep = a.ucnt[v] > 0;
        }
        block_append(keep, v, a.front0, a.counters);
    }
}

// phase A of round `round` >= 1 (round 0's picks come from k_adj_rank): each
// frontier vertex whose previous pick died picks its best live edge -- the
// first slot from its cursor whose neighbour is unmatched (rank-ordered
// adjacency); unsorted (high-degree) vertices scan every slot.
// `round` < 0: inside the device-driven loop -- the round comes from counters[4]
__global__ void __maxnreg__(48) k_ld_pick(LDArgs a, int round) {
    MF_PDL_ENTRY;
    if (*a.abort_flag) return;
    if (round < 0) {
        round = ld_volatile(a.counters + 4);
        if (round == 0) return;  // round 0's picks come from k_adj_rank
    }
    const int cur = round & 1;
    const int n = a.counters[cur];
    if (n == 0) return;
    const int* Fc = cur ? a.front1 : a.front0;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        const int v = Fc[i];
        // the previous pick stays the best live edge while its other end is unmatched
        // (edges only die): no adjacency reads for those frontier vertices
        const int pu = a.bestu[v];
        if (pu >= 0 && a.mate[pu] < 0) continue;
        const size_t s = (size_t)a.aoff[v];
        const int nu = a.ucnt[v];
        int be = -1, bu = -1;
        int c = a.acur[v];
        if (c >= 0) {
            for (; c < nu; c++) {
                const int u = a.nbr[s + c];
                if (a.mate[u] < 0) {
                    be = a.adj_eid[s + c];
                    bu = u;
                    break;
                }
            }
            a.acur[v] = c;
        } else {
            unsigned bk = 0xffffffffu;
            for (int j = 0; j < nu; j++) {
                const int u = a.nbr[s + j];
                if (a.mate[u] >= 0) continue;
                const int e = a.adj_eid[s + j];
                const unsigned ke = a.adj_k32[s + j];
                if (be < 0 || ld_lt(a, ke, e, bk, be)) { bk = ke; be = e; bu = u; }
            }
        }
        a.best[v] = be;
        a.bestu[v] = bu;
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) a.counters[cur ^ 1] = 0;
}

// phase B: mutual picks are matched; the rest (with a live edge) survive
__global__ void __launch_bounds__(256) k_ld_match(LDArgs a, int round) {
    MF_PDL_ENTRY;
    const bool loop = round < 0;  // device-driven rounds: this kernel decides whether another follows
    if (*a.abort_flag) {
        if (loop && blockIdx.x == 0 && threadIdx.x == 0) cudaGraphSetConditional(a.cond, 0u);
        return;
    }
    if (loop) round = ld_volatile(a.counters + 4);
    const int cur = round & 1;
    const int n = a.counters[cur];
    if (n && blockIdx.x == 0 && threadIdx.x == 0) {
        a.counters[3] = cur ^ 1;  // the residual frontier lives here after this round
        a.counters[2] = round + 1;
    }
    const int* Fc = cur ? a.front1 : a.front0;
    int* Fn = cur ? a.front0 : a.front1;
    const int nb = (n + blockDim.x - 1) / blockDim.x;
    for (int b = blockIdx.x; b < nb; b += gridDim.x) {
        const int i = b * blockDim.x + threadIdx.x;
        bool keep = false;
        int v = 0;
        if (i < n) {
            v = Fc[i];
            const int e = a.best[v];
            if (e >= 0) {
                if (a.best[a.bestu[v]] == e) a.mate[v] = e;
                else keep = true;
            }
        }
        block_append(keep, v, Fn, a.counters + (cur ^ 1));
    }
    if (!loop) return;
    // the last block to finish sees the complete next frontier and sets the loop condition
    __shared__ int s_last;
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        s_last = atomicAdd(a.counters + 5, 1) == (int)gridDim.x - 1;
    }
    __syncthreads();
    if (s_last && threadIdx.x == 0) {
        __threadfence();
        const int next = ld_volatile(a.counters + (cur ^ 1));
        a.counters[5] = 0;
        a.counters[4] = round + 1;
        cudaGraphSetConditional(a.cond, (next > 0 && round + 1 < a.max_rounds) ? 1u : 0u);
    }
}

// Append slot in the candidate segment of v's mesh.  Must be reached by every
// thread of the block (block-uniform loop): one mesh -> one atomic per block
// (a per-warp atomic on a single counter serialises millions of appends);
// batches -> per-mesh counters.
MF_DEV int block_slot(bool keep, int* __restrict__ counter) {
    __shared__ int s_scan[33];
    __shared__ int s_base;
    int tot;
    const int pos = block_excl_scan(keep ? 1 : 0, s_scan, &tot);
    if (threadIdx.x == 0) s_base = tot ? atomicAdd(counter, tot) : 0;
    __syncthreads();
    const int r = s_base + pos;
    __syncthreads();
    return keep ? r : -1;
}
// Two block-aggregated appends from one block scan (counts packed 16:16; blocks <= 1024 threads).
MF_DEV void block_slot2(bool ka, int* __restrict__ ca, int& ra, bool kb, int* __restrict__ cb, int& rb) {
    __shared__ int s_scan[33];
    __shared__ int s_base[2];
    int tot;
    const int pos = block_excl_scan((ka ? 1 : 0) | (kb ? 0x10000 : 0), s_scan, &tot);
    if (threadIdx.x == 0) {
        const int ta = tot & 0xffff, tb = tot >> 16;
        s_base[0] = ta ? atomicAdd(ca, ta) : 0;
        s_base[1] = tb ? atomicAdd(cb, tb) : 0;
    }
    __syncthreads();
    ra = ka ? s_base[0] + (pos & 0xffff) : -1;
    rb = kb ? s_base[1] + (pos >> 16) : -1;
    __syncthreads();
}
MF_DEV int seg_slot_uniform(bool keep, const int* __restrict__ vmesh, const int* __restrict__ voff,
                            int* __restrict__ seg_cnt, int v) {
    if (!vmesh) return block_slot(keep, seg_cnt);
    // batches: a warp's vertices are consecutive, so they span one or two meshes -- one
    // atomic per (warp, mesh) group instead of one per candidate
    const unsigned full = 0xffffffffu;
    const int b = keep ? vmesh[v] : -1;
    const unsigned peers = __match_any_sync(full, b);
    if (!keep) return -1;
    const int lane = threadIdx.x & 31, leader = __ffs(peers) - 1;
    int base = 0;
    if (lane == leader) base = atomicAdd(seg_cnt + b, __popc(peers));
    base = __shfl_sync(peers, base, leader);
    return voff[b] + base + __popc(peers & ((1u << lane) - 1u));
}

// mate = the suitor edge when the proposal is mutual (or the LD match); every
// matched pair is also appended once (from its e0 end) as a budget-truncation
// candidate keyed by its rank (decimate.py:256-258).
__global__ void k_mates(const int* __restrict__ abort_flag, int N, const unsigned long long* __restrict__ suitor,
                        const int* __restrict__ e0, const int* __restrict__ e1, int* __restrict__ mate,
                        const uint64_t* __restrict__ key_hi, const uint64_t* __restrict__ key_lo,
                        const int* __restrict__ vmesh, const int* __restrict__ voff, int* __restrict__ seg_cnt,
                        uint64_t* __restrict__ chi, uint64_t* __restrict__ clo, int* __restrict__ cpay,
                        int* __restrict__ pairlo, int* __restrict__ loose, int* __restrict__ loose_cnt) {
    MF_PDL_ENTRY;
    if (*abort_flag) return;
    // block-uniform trip count: the single-mesh append is aggregated per block.  Unmatched
    // vertices are listed for the absorb stage (the only loose vertices it can see: pairs
    // dropped by the truncation exist only where the budget is met, and then it does not run)
    for (int base = blockIdx.x * blockDim.x; base < N; base += gridDim.x * blockDim.x) {
        const int v = base + threadIdx.x;
        int m = -1;
        bool cand = false;
        if (v < N) {
            m = mate[v];
            unsigned long long w = m >= 0 ? ~0ull : suitor[v];  // m >= 0: matched by the LD rounds
            if (w != ~0ull) {
                int e = (int)(unsigned)w;
                int u = e0[e] == v ? e1[e] : e0[e];
                if ((int)(unsigned)suitor[u] == e && suitor[u] != ~0ull) m = e;
            }
            mate[v] = m;
            const int lo = m >= 0 ? e0[m] : -1;
            pairlo[v] = lo;
            cand = lo == v;
        }
        const bool lz = v < N && m < 0;
        int slot, lslot;
        if (!vmesh) {
            block_slot2(cand, seg_cnt, slot, lz, loose_cnt, lslot);
        } else {
            slot = seg_slot_uniform(cand, vmesh, voff, seg_cnt, v);
            lslot = block_slot(lz, loose_cnt);
        }
        if (lz) loose[lslot] = v;
        if (cand) {
            chi[slot] = key_hi[m];
            clo[slot] = key_lo ? key_lo[m] : (uint64_t)m;
            cpay[slot] = m;
        }
    }
}

// ------------------------------------------------------------------------
// K6: per-segment selection of the k smallest unique 128-bit keys.
// Candidates are compacted in vertex order (so each mesh's candidates are
// contiguous); one block per segment runs an MSD radix select with 11-bit
// digits and shared-memory histograms, first streaming the segment from
// global memory (L2-resident at these sizes) and switching to a shared-memory
// copy of the surviving prefix bucket as soon as it fits.
// Output per segment: mode 1 = all, 2 = none, 3 = keys <= (thr_hi, thr_lo).
constexpr int kSelBits = 11;
constexpr int kSelBins = 1 << kSelBits;
constexpr int kSelCap = 4096;  // keys held in shared memory (64 KiB; a larger carve-out measured slower)
constexpr int kSelThreads = 1024;
// k_select threads: 1024 for one mesh, 512 per mesh of a batch (cheaper barriers; measured
// cfg4 selects 27 -> 19 us, while the single cfg2 mesh prefers 1024: 53 vs 57 us)
constexpr int kSelSmem = kSelBins * 4 + 2 * kSelCap * 8;
constexpr int kSelCapMax = 12288;  // largest stage k_select may be launched with (MF_SEL_CAP)
constexpr int kSelChiCap = 27136;  // single-mesh two-phase path: primary keys + tie secondaries (212 KiB)
constexpr int kSelBucket = 512;    // its compacted bucket (4 KiB static)

MF_DEV int sel_digit(uint64_t hi, uint64_t lo, int shift, int width) {
    // bits [shift, shift+width) of the 128-bit key (may straddle the 64-bit boundary)
    unsigned __int128 k = ((unsigned __int128)hi << 64) | lo;
    return (int)((k >> shift) & ((1u << width) - 1u));
}
MF_DEV bool sel_prefix(uint64_t hi, uint64_t lo, uint64_t phi, uint64_t plo, int top) {
    if (top >= 128) return true;
    unsigned __int128 k = ((unsigned __int128)hi << 64) | lo;
    unsigned __int128 p = ((unsigned __int128)phi << 64) | plo;
    return (k >> top) == (p >> top);
}

// Common-prefix skip.  `o` / `n` are the OR / AND of every key of the bucket
// that was just histogrammed; the surviving sub-bucket agrees on every bit
// below `top` on which the whole bucket agreed, so those bits are copied into
// the prefix and the next digit starts at the highest bit that still differs.
// (Keys built from float64 costs share their sign / exponent bits, and the
// secondary halves share their high zero bits: without the skip each such run
// costs a full pass over the candidates.)
MF_DEV void sel_skip(unsigned __int128& p, int& top, uint64_t oh, uint64_t ol, uint64_t ah, uint64_t al) {
    unsigned __int128 diff = (((unsigned __int128)(oh ^ ah)) << 64) | (ol ^ al);
    if (top < 128) diff &= ((((unsigned __int128)1) << top) - 1);
    if (diff == 0) return;
    const uint64_t dh = (uint64_t)(diff >> 64), dl = (uint64_t)diff;
    const int D = dh ? 127 - __clzll((long long)dh) : 63 - __clzll((long long)dl);
    if (D + 1 >= top) return;
    unsigned __int128 m = ((top < 128) ? ((((unsigned __int128)1) << top) - 1) : ~(unsigned __int128)0) &
                          ~((((unsigned __int128)1) << (D + 1)) - 1);
    unsigned __int128 andv = (((unsigned __int128)ah) << 64) | al;
    p = (p & ~m) | (andv & m);
    top = D + 1;
}

// warp OR / AND reduction of a 128-bit key range summary
MF_DEV void warp_orand(uint64_t& oh, uint64_t& ol, uint64_t& ah, uint64_t& al) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        oh |= __shfl_xor_sync(0xffffffffu, oh, o);
        ol |= __shfl_xor_sync(0xffffffffu, ol, o);
        ah &= __shfl_xor_sync(0xffffffffu, ah, o);
        al &= __shfl_xor_sync(0xffffffffu, al, o);
    }
}

// Histogram increment (plain shared-memory atomic: warp-aggregating the
// contended leading digits measured slower than the conflicts it saves).
MF_DEV void hist_add(int* hist, int d) { atomicAdd(hist + d, 1); }

struct SelectArgs {
    const uint64_t* chi;
    const uint64_t* clo;
    const int* seg_cnt;   // candidates of segment b: [voff[b], voff[b] + seg_cnt[b])
    const int* voff;      // (a mesh never has more candidates than vertices)
    int B;
    const int* act;
    const int* budget;
    const int* removed;  // nullable
    int* ksel;
    int* mode;
    uint64_t* thr_hi;   // prefix while selecting, threshold once decided
    uint64_t* thr_lo;
    const int* abort_flag;
    int* krem;          // resumable state (after the multi-block passes)
    int* top;
    int resume;
    int* gscr;          // multi-block scratch (resume: bucket buffer)
    int cap;            // k_select: keys its shared-memory stage holds (>= kSelCap)
    cudaGraphConditionalHandle cond;  // device-driven multi-block passes (WHILE node), 0 = fixed passes
    int chicap;         // k_select: primary keys the stage holds for the two-phase path (0 = off)
    int bulk;           // k_select: two-phase keys staged by the bulk-copy engine
    int first_all;      // k_select: its first radix pass skips the prefix test (all keys in the bucket)
};

// Multi-block pass scratch (ints): histogram | OR (2 u64), AND (2 u64) | stop |
// compact | count | bucket buffer (kSelCap (hi, lo) pairs).  Once a decide
// leaves a bucket that fits the shared-memory stage, the next histogram pass
// also copies that bucket into the buffer, and k_select resumes from it
// instead of streaming the whole segment again.
constexpr int kSelScrHdr = kSelBins + 16;
constexpr int kSelScratch = kSelScrHdr + 4 * kSelCap;  // ints
constexpr int kSelPasses = 3;  // multi-block passes before the single-CTA stage resumes (5: cfg5 +0.08 ms)
MF_DEV unsigned long long* sel_orand(int* g) { return reinterpret_cast<unsigned long long*>(g + kSelBins); }
MF_DEV int* sel_stop(int* g) { return g + kSelBins + 8; }
MF_DEV int* sel_compact(int* g) { return g + kSelBins + 9; }
MF_DEV int* sel_count(int* g) { return g + kSelBins + 10; }
MF_DEV uint64_t* sel_buf(int* g) { return reinterpret_cast<uint64_t*>(g + kSelScrHdr); }
MF_DEV int* sel_pass(int* g) { return g + kSelBins + 11; }  // pass of the device-driven loop
constexpr int kSelPassesMax = 12;                          // loop cap (128-bit keys, 11-bit digits)

// Block-wide k-th smallest (1-based kr) of vals[0..n) (u64, duplicates allowed) below
// the prefix (p, top): MSD radix with 11-bit digits and the common-prefix skip.
// Returns true when the kr-th is the last element of a digit bucket -- every value in
// [p, p | ones(top)) is then selected -- and false when all 64 bits are fixed (p is the
// exact value, kr its rank among the equal values).  Uniform across the block.
// `scratch` (cap values): once a bucket fits, it is copied there and later passes walk
// only the bucket instead of every value.
MF_DEV bool radix_kth_u64(const uint64_t* vals, int n, int& kr, uint64_t& p, int& top, int* hist, int* s_scan,
                          int* s_sel, unsigned long long* s_oa, uint64_t* scratch, int cap,
                          bool all_in = false) {
    // all_in: every value already shares the prefix above `top` (the caller skipped the bits
    // the whole input shares) -- the first pass then needs neither the prefix test nor the
    // OR / AND of its bucket (which is the whole input, already reflected in `top`)
    bool compacted = false;
    if (n <= 32 && top >= 64) {  // tiny input (typically the ties of phase two): one warp sorts it
        if (threadIdx.x < 32) {
            const int l = threadIdx.x;
            uint64_t x = l < n ? vals[l] : ~0ull;
#pragma unroll
            for (int k = 2; k <= 32; k <<= 1)
#pragma unroll
                for (int j = k >> 1; j > 0; j >>= 1) {
                    const uint64_t y = __shfl_xor_sync(0xffffffffu, x, j);
                    const bool up = ((l & k) == 0), lower = ((l & j) == 0);
                    x = (lower == up) ? (x < y ? x : y) : (x > y ? x : y);
                }
            const uint64_t v = __shfl_sync(0xffffffffu, x, kr - 1);
            const int below = __popc(__ballot_sync(0xffffffffu, l < n && x < v));
            if (l == 0) {
                s_oa[2] = v;
                s_sel[3] = kr - below;
            }
        }
        __syncthreads();
        p = s_oa[2];
        kr = s_sel[3];
        top = 0;
        __syncthreads();
        return false;
    }
    while (top > 0) {
        const int width = top >= kSelBits ? kSelBits : top;
        const int shift = top - width;
        for (int i = threadIdx.x; i < kSelBins; i += blockDim.x) hist[i] = 0;
        if (threadIdx.x < 2) s_oa[threadIdx.x] = threadIdx.x ? ~0ull : 0ull;
        __syncthreads();
        uint64_t o = 0, an = ~0ull;
        if (all_in) {
            const unsigned dmask = (1u << width) - 1u;
#pragma unroll 4
            for (int i = threadIdx.x; i < n; i += blockDim.x) hist_add(hist, (int)((vals[i] >> shift) & dmask));
            all_in = false;
        } else {
            for (int i = threadIdx.x; i < n; i += blockDim.x) {
                const uint64_t x = vals[i];
                if (top >= 64 || (x >> top) == (p >> top)) {
                    hist_add(hist, (int)((x >> shift) & ((1u << width) - 1u)));
                    o |= x;
                    an &= x;
                }
            }
        }
#pragma unroll
        for (int q = 16; q > 0; q >>= 1) {
            o |= __shfl_xor_sync(0xffffffffu, o, q);
            an &= __shfl_xor_sync(0xffffffffu, an, q);
        }
        if ((threadIdx.x & 31) == 0) {
            atomicOr(s_oa, o);
            atomicAnd(s_oa + 1, an);
        }
        __syncthreads();
        const int per = kSelBins / blockDim.x;
        int loc = 0;
        for (int j = 0; j < per; j++) loc += hist[threadIdx.x * per + j];
        int tot;
        const int ex = block_excl_scan(loc, s_scan, &tot);
        if (ex < kr && kr <= ex + loc) {
            int cum = ex;
            for (int j = 0; j < per; j++) {
                const int h = hist[threadIdx.x * per + j];
                if (cum + h >= kr) {
                    s_sel[0] = threadIdx.x * per + j;
                    s_sel[1] = cum;
                    s_sel[2] = h;
                    break;
                }
                cum += h;
            }
        }
        __syncthreads();
        const int d = s_sel[0], h = s_sel[2];
        kr -= s_sel[1];
        p |= (uint64_t)d << shift;
        top = shift;
        const uint64_t diff = (s_oa[0] ^ s_oa[1]) & (shift >= 64 ? ~0ull : ((1ull << shift) - 1ull));
        const uint64_t common = s_oa[1];
        __syncthreads();
        if (h == kr) return true;
        if (!compacted && h <= cap && h > 32 && h < n) {  // walk only the bucket from now on
            if (threadIdx.x == 0) s_sel[3] = 0;
            __syncthreads();
            for (int i = threadIdx.x; i < n; i += blockDim.x) {
                const uint64_t x = vals[i];
                if ((x >> top) == (p >> top)) scratch[atomicAdd(&s_sel[3], 1)] = x;
            }
            __syncthreads();
            vals = scratch;
            n = h;
            compacted = true;
        }
        if (h <= 32 && top > 0) {
            // a small bucket: one warp sorts it and reads the kr-th directly (no more passes)
            uint64_t* small = reinterpret_cast<uint64_t*>(hist);  // the histogram is free now
            if (threadIdx.x == 0) s_sel[3] = 0;
            __syncthreads();
            for (int i = threadIdx.x; i < n; i += blockDim.x) {
                const uint64_t x = vals[i];
                if ((x >> top) == (p >> top)) small[atomicAdd(&s_sel[3], 1)] = x;
            }
            __syncthreads();
            if (threadIdx.x < 32) {
                const int l = threadIdx.x;
                uint64_t x = l < h ? small[l] : ~0ull;
#pragma unroll
                for (int k = 2; k <= 32; k <<= 1)
#pragma unroll
                    for (int j = k >> 1; j > 0; j >>= 1) {
                        const uint64_t y = __shfl_xor_sync(0xffffffffu, x, j);
                        const bool up = ((l & k) == 0), lower = ((l & j) == 0);
                        x = (lower == up) ? (x < y ? x : y) : (x > y ? x : y);
                    }
                const uint64_t v = __shfl_sync(0xffffffffu, x, kr - 1);
                const int below = __popc(__ballot_sync(0xffffffffu, l < h && x < v));
                if (l == 0) {
                    small[32] = v;
                    s_sel[3] = kr - below;
                }
            }
            __syncthreads();
            p = small[32];
            kr = s_sel[3];
            top = 0;
            __syncthreads();
            return false;
        }
        if (diff) {  // skip the bits every value of the bucket shares
            const int D = 63 - __clzll((long long)diff);
            if (D + 1 < top) {
                const uint64_t m = ((top >= 64) ? ~0ull : ((1ull << top) - 1ull)) & ~((1ull << (D + 1)) - 1ull);
                p = (p & ~m) | (common & m);
                top = D + 1;
            }
        }
    }
    return false;
}

template <int NT>
__global__ void __launch_bounds__(NT) k_select(SelectArgs a) {
    MF_PDL_ENTRY;
    if (*a.abort_flag) return;
    extern __shared__ __align__(16) unsigned char s_raw[];
    int* hist = reinterpret_cast<int*>(s_raw);                          // kSelBins
    uint64_t* sh = reinterpret_cast<uint64_t*>(s_raw + kSelBins * 4);   // kSelCap
    uint64_t* sl = sh + a.cap;                                          // a.cap
    __shared__ int s_scan[33];
    __shared__ int s_sel[4];
    __shared__ int s_ncomp;
    __shared__ unsigned long long s_oa[4];
    __shared__ uint64_t s_bucket[kSelBucket];  // the two-phase path's compacted digit bucket
    __shared__ __align__(8) uint64_t s_mbar;    // its bulk key stage
    for (int b = blockIdx.x; b < a.B; b += gridDim.x) {
        const int c0 = a.voff[b], c1 = c0 + a.seg_cnt[b];
        const int cnt = c1 - c0;
        uint64_t phi = 0, plo = 0;
        int kr, top = 128, k;
        if (a.resume) {
            if (a.mode[b] != 0) continue;  // decided by the multi-block passes
            phi = a.thr_hi[b];
            plo = a.thr_lo[b];
            kr = a.krem[b];
            top = a.top[b];
            k = a.ksel[b];
        } else {
            int want = a.act[b] ? a.budget[b] - (a.removed ? a.removed[b] : 0) : 0;
            k = want < cnt ? want : cnt;
            if (k < 0) k = 0;
            if (k == 0 || k >= cnt) {
                if (threadIdx.x == 0) {
                    a.ksel[b] = k;
                    a.mode[b] = (k == 0) ? 2 : 1;
                }
                continue;
            }
            kr = k;
        }
        if (!a.resume && cnt + 1 <= a.chicap) {
            // mid-size segment: the 64-bit primary keys fit the stage -- select on them in
            // shared memory (one coalesced load), then, only among the keys equal to the
            // k-th primary key, on the secondary half gathered from global memory
            const uint64_t* src = a.chi + c0;
            // key i sits at sv[i]; the stage is shifted by one key when the segment starts
            // 8 bytes off a 16-byte boundary, so global and shared addresses agree mod 16
            const int lead = min(cnt, (int)(((uintptr_t)src >> 3) & 1));
            uint64_t* sv = sh + lead;  // a.chicap - 1 keys
            uint64_t o = 0, an = ~0ull;
            if (threadIdx.x < 2) s_oa[threadIdx.x] = threadIdx.x ? ~0ull : 0ull;
            if (a.bulk) {
                // the bulk-copy engine streams the aligned body (one thread issues, the mbarrier
                // counts the bytes); the <= 2 unaligned end keys are plain loads
                const int body = ((cnt - lead) >> 1) << 1;
                if (threadIdx.x == 0) {
                    mbar_init(&s_mbar, 1);
                    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
                }
                __syncthreads();
                if (threadIdx.x == 0) {
                    mbar_expect_tx(&s_mbar, (unsigned)body * 8u);
                    constexpr int kChunk = 4096;  // keys per bulk copy (32 KiB)
                    for (int off = 0; off < body; off += kChunk)
                        bulk_g2s(sv + lead + off, src + lead + off, (unsigned)min(kChunk, body - off) * 8u, &s_mbar);
                }
                if (threadIdx.x == 32 && lead) sv[0] = __ldcg(src);
                if (threadIdx.x == 64 && lead + body < cnt) sv[cnt - 1] = __ldcg(src + cnt - 1);
                mbar_wait(&s_mbar, 0);
                __syncthreads();
                for (int i = threadIdx.x; i < cnt; i += blockDim.x) {
                    o |= sv[i];
                    an &= sv[i];
                }
            } else {
                for (int i0 = threadIdx.x; i0 < cnt; i0 += 8 * blockDim.x) {  // 8 loads in flight per thread
                    uint64_t v8[8];
#pragma unroll
                    for (int q = 0; q < 8; q++) {
                        const int i = i0 + q * blockDim.x;
                        v8[q] = i < cnt ? __ldcg(src + i) : 0;
                    }
#pragma unroll
                    for (int q = 0; q < 8; q++) {
                        const int i = i0 + q * blockDim.x;
                        if (i < cnt) {
                            sv[i] = v8[q];
                            o |= v8[q];
                            an &= v8[q];
                        }
                    }
                }
            }
#pragma unroll
            for (int q = 16; q > 0; q >>= 1) {
                o |= __shfl_xor_sync(0xffffffffu, o, q);
                an &= __shfl_xor_sync(0xffffffffu, an, q);
            }
            __syncthreads();
            if ((threadIdx.x & 31) == 0) {
                atomicOr(s_oa, o);
                atomicAnd(s_oa + 1, an);
            }
            __syncthreads();
            // the bits every primary key shares (sign / exponent of the float64 costs) are fixed
            // before the first pass: histogramming them would pile every key into one or two
            // bins, and those shared-memory atomics serialise
            uint64_t t = 0, q = 0;
            int topc = 64;
            {
                const uint64_t diff = s_oa[0] ^ s_oa[1];
                if (diff) {
                    const int D = 63 - __clzll((long long)diff);
                    if (D < 63) {
                        t = s_oa[1] & ~((1ull << (D + 1)) - 1ull);
                        topc = D + 1;
                    }
                } else {
                    t = s_oa[1];
                    topc = 0;
                }
            }
            __syncthreads();
            const bool whole =
                radix_kth_u64(sv, cnt, kr, t, topc, hist, s_scan, s_sel, s_oa, s_bucket, kSelBucket, a.first_all);
            if (whole) {
                t |= (topc >= 64) ? ~0ull : ((1ull << topc) - 1ull);
                q = ~0ull;
            } else {
                if (threadIdx.x == 0) s_ncomp = 0;
                __syncthreads();
                uint64_t* sq = sv + cnt;  // secondary halves of the primary-key ties
                const int room = a.chicap - cnt - lead;
                for (int i = threadIdx.x; i < cnt; i += blockDim.x)
                    if (sv[i] == t) {
                        const int slot = atomicAdd(&s_ncomp, 1);
                        if (slot < room) sq[slot] = a.clo[c0 + i];
                    }
                __syncthreads();
                const int ne = s_ncomp;
                if (ne > room) {  // more ties than room (pathological): the general path below
                    kr = k;
                    __syncthreads();
                    goto general;
                }
                int topq = 64;
                if (radix_kth_u64(sq, ne, kr, q, topq, hist, s_scan, s_sel, s_oa, s_bucket, kSelBucket))
                    q |= (topq >= 64) ? ~0ull : ((1ull << topq) - 1ull);
            }
            if (threadIdx.x == 0) {
                a.thr_hi[b] = t;
                a.thr_lo[b] = q;
                a.mode[b] = 3;
                a.ksel[b] = k;
            }
            __syncthreads();
            continue;
        }
    general:
        bool in_smem = false;
        int n_s = 0;
        bool done = false;
        if (!a.resume && cnt <= a.cap) {
            // the whole segment fits: one coalesced load, and the bits every key shares are
            // skipped before the first pass
            uint64_t oh = 0, ol = 0, ah = ~0ull, al = ~0ull;
            if (threadIdx.x < 4) s_oa[threadIdx.x] = (threadIdx.x < 2) ? 0ull : ~0ull;
            for (int i = threadIdx.x; i < cnt; i += blockDim.x) {
                const uint64_t h = a.chi[c0 + i], l = a.clo[c0 + i];
                sh[i] = h;
                sl[i] = l;
                oh |= h; ol |= l; ah &= h; al &= l;
            }
            __syncthreads();
            warp_orand(oh, ol, ah, al);
            if ((threadIdx.x & 31) == 0) {
                atomicOr(s_oa, oh); atomicOr(s_oa + 1, ol);
                atomicAnd(s_oa + 2, ah); atomicAnd(s_oa + 3, al);
            }
            __syncthreads();
            unsigned __int128 p0 = 0;
            sel_skip(p0, top, s_oa[0], s_oa[1], s_oa[2], s_oa[3]);
            phi = (uint64_t)(p0 >> 64);
            plo = (uint64_t)p0;
            n_s = cnt;
            in_smem = true;
            __syncthreads();
        }
        if (a.resume && *sel_stop(a.gscr)) {  // the multi-block passes left the bucket in the buffer
            n_s = *sel_count(a.gscr);
            const uint64_t* buf = sel_buf(a.gscr);
            for (int i = threadIdx.x; i < n_s; i += blockDim.x) {
                sh[i] = buf[2 * i];
                sl[i] = buf[2 * i + 1];
            }
            in_smem = true;
            __syncthreads();
        }
        while (!done) {
            int width = top >= kSelBits ? kSelBits : top;
            int shift = top - width;
            for (int i = threadIdx.x; i < kSelBins; i += blockDim.x) hist[i] = 0;
            if (threadIdx.x < 4) s_oa[threadIdx.x] = (threadIdx.x < 2) ? 0ull : ~0ull;
            __syncthreads();
            uint64_t oh = 0, ol = 0, ah = ~0ull, al = ~0ull;
            if (in_smem) {
                for (int i = threadIdx.x; i < n_s; i += blockDim.x)
                    if (sel_prefix(sh[i], sl[i], phi, plo, top)) {
                        hist_add(hist, sel_digit(sh[i], sl[i], shift, width));
                        oh |= sh[i]; ol |= sl[i]; ah &= sh[i]; al &= sl[i];
                    }
            } else {
#pragma unroll 4
                for (int i = c0 + threadIdx.x; i < c1; i += blockDim.x) {
                    uint64_t h = a.chi[i], l = a.clo[i];
                    if (sel_prefix(h, l, phi, plo, top)) {
                        hist_add(hist, sel_digit(h, l, shift, width));
                        oh |= h; ol |= l; ah &= h; al &= l;
                    }
                }
            }
            warp_orand(oh, ol, ah, al);
            if ((threadIdx.x & 31) == 0) {
                atomicOr(s_oa, oh); atomicOr(s_oa + 1, ol);
                atomicAnd(s_oa + 2, ah); atomicAnd(s_oa + 3, al);
            }
            __syncthreads();
            // block scan over the bins: find digit d with cum(d) < kr <= cum(d) + hist[d]
            const int per = kSelBins / NT;  // bins per thread
            int loc = 0;
            for (int j = 0; j < per; j++) loc += hist[threadIdx.x * per + j];
            int tot;
            int ex = block_excl_scan(loc, s_scan, &tot);
            if (ex < kr && kr <= ex + loc) {
                int cum = ex;
                for (int j = 0; j < per; j++) {
                    int h = hist[threadIdx.x * per + j];
                    if (cum + h >= kr) {
                        s_sel[0] = threadIdx.x * per + j;
                        s_sel[1] = cum;
                        s_sel[2] = h;
                        break;
                    }
                    cum += h;
                }
            }
            __syncthreads();
            const int d = s_sel[0];
            kr -= s_sel[1];
            const int hd = s_sel[2];
            unsigned __int128 p = ((unsigned __int128)phi << 64) | plo;
            p |= ((unsigned __int128)d) << shift;
            top = shift;
            if (hd == kr) {
                unsigned __int128 ones = (shift == 0) ? 0 : ((((unsigned __int128)1) << shift) - 1);
                p |= ones;
                if (threadIdx.x == 0) {
                    a.thr_hi[b] = (uint64_t)(p >> 64);
                    a.thr_lo[b] = (uint64_t)p;
                    a.mode[b] = 3;
                    a.ksel[b] = k;
                }
                done = true;
            } else {
                sel_skip(p, top, s_oa[0], s_oa[1], s_oa[2], s_oa[3]);
                phi = (uint64_t)(p >> 64);
                plo = (uint64_t)p;
                if (!in_smem && hd <= a.cap) {
                    // compact the surviving bucket into shared memory
                    if (threadIdx.x == 0) s_ncomp = 0;
                    __syncthreads();
                    for (int i = c0 + threadIdx.x; i < c1; i += blockDim.x) {
                        uint64_t h = a.chi[i], l = a.clo[i];
                        if (sel_prefix(h, l, phi, plo, top)) {
                            int slot = atomicAdd(&s_ncomp, 1);
                            sh[slot] = h;
                            sl[slot] = l;
                        }
                    }
                    __syncthreads();
                    n_s = s_ncomp;
                    in_smem = true;
                }
            }
            __syncthreads();
        }
    }
}

// Cluster selection for one mid-size segment (a single mesh below the
// multi-block threshold): kClCTAs CTAs of one thread-block cluster split the
// candidates; each pass every CTA histograms its slice in its own shared
// memory, rank 0 pulls the slices' histograms (and the bucket's OR / AND)
// through distributed shared memory with plain loads, picks the digit and
// writes the decision into every rank's shared memory, and all ranks carry
// the same selection state (two cluster barriers per pass).  Once the bucket fits, every rank keeps its share
// of it in shared memory, so later passes touch no global memory.
constexpr int kClCTAs = 8;
constexpr int kClThreads = 512;
constexpr int kClSmem = kSelBins * 4 + 2 * kSelCap * 8;
__global__ void __cluster_dims__(kClCTAs, 1, 1) __launch_bounds__(kClThreads) k_select_cl(SelectArgs a) {
    MF_PDL_ENTRY;
    namespace cg = cooperative_groups;
    cg::cluster_group cl = cg::this_cluster();
    const unsigned rank = cl.block_rank();
    extern __shared__ unsigned char s_raw[];
    int* hist = reinterpret_cast<int*>(s_raw);
    uint64_t* sh = reinterpret_cast<uint64_t*>(s_raw + kSelBins * 4);
    uint64_t* sl = sh + kSelCap;
    __shared__ unsigned long long s_oa[4];
    __shared__ int s_scan[33];
    __shared__ int s_sel[3];
    __shared__ int s_dec[3];                 // decision broadcast by rank 0: digit, count below, bucket size
    __shared__ unsigned long long s_moa[4];  // merged OR / AND broadcast by rank 0
    __shared__ int s_ncomp;
    if (*a.abort_flag) return;  // the same word for every rank: the whole cluster leaves together
    const int c0 = a.voff[0], c1 = c0 + a.seg_cnt[0];
    const int cnt = c1 - c0;
    const int want = a.act[0] ? a.budget[0] - (a.removed ? a.removed[0] : 0) : 0;
    int k = want < cnt ? want : cnt;
    if (k < 0) k = 0;
    if (k == 0 || k >= cnt) {
        if (rank == 0 && threadIdx.x == 0) {
            a.ksel[0] = k;
            a.mode[0] = (k == 0) ? 2 : 1;
        }
        return;
    }
    const int per = (cnt + kClCTAs - 1) / kClCTAs;
    const int lo = c0 + min(cnt, (int)rank * per), hi = c0 + min(cnt, ((int)rank + 1) * per);
    uint64_t phi = 0, plo = 0;
    int top = 128, kr = k, n_s = 0;
    bool in_smem = false;
    while (true) {
        const int width = top >= kSelBits ? kSelBits : top;
        const int shift = top - width;
        for (int i = threadIdx.x; i < kSelBins; i += blockDim.x) hist[i] = 0;
        if (threadIdx.x < 4) s_oa[threadIdx.x] = (threadIdx.x < 2) ? 0ull : ~0ull;
        __syncthreads();
        uint64_t oh = 0, ol = 0, ah = ~0ull, al = ~0ull;
        if (in_smem) {
            for (int i = threadIdx.x; i < n_s; i += blockDim.x)
                if (sel_prefix(sh[i], sl[i], phi, plo, top)) {
                    hist_add(hist, sel_digit(sh[i], sl[i], shift, width));
                    oh |= sh[i]; ol |= sl[i]; ah &= sh[i]; al &= sl[i];
                }
        } else {
            for (int i = lo + threadIdx.x; i < hi; i += blockDim.x) {
                const uint64_t h = a.chi[i], l = a.clo[i];
                if (sel_prefix(h, l, phi, plo, top)) {
                    hist_add(hist, sel_digit(h, l, shift, width));
                    oh |= h; ol |= l; ah &= h; al &= l;
                }
            }
        }
        warp_orand(oh, ol, ah, al);
        if ((threadIdx.x & 31) == 0) {
            atomicOr(s_oa, oh); atomicOr(s_oa + 1, ol);
            atomicAnd(s_oa + 2, ah); atomicAnd(s_oa + 3, al);
        }
        cl.sync();  // every slice histogrammed
        if (rank == 0) {
            // pull the slices' histograms and OR / AND words through DSMEM (plain loads)
            const int pb = kSelBins / kClThreads;
            int hb[kSelBins / kClThreads];
            int loc = 0;
#pragma unroll
            for (int j = 0; j < pb; j++) hb[j] = hist[threadIdx.x * pb + j];
            for (int r = 1; r < kClCTAs; r++) {
                const int* hr = cl.map_shared_rank(hist, r);
#pragma unroll
                for (int j = 0; j < pb; j++) hb[j] += hr[threadIdx.x * pb + j];
            }
#pragma unroll
            for (int j = 0; j < pb; j++) loc += hb[j];
            if (threadIdx.x < 4) {
                unsigned long long w = s_oa[threadIdx.x];
                for (int r = 1; r < kClCTAs; r++) {
                    const unsigned long long x = cl.map_shared_rank(s_oa, r)[threadIdx.x];
                    w = (threadIdx.x < 2) ? (w | x) : (w & x);
                }
                s_moa[threadIdx.x] = w;
            }
            int tot;
            const int ex = block_excl_scan(loc, s_scan, &tot);
            if (ex < kr && kr <= ex + loc) {
                int cum = ex;
#pragma unroll
                for (int j = 0; j < pb; j++) {
                    if (cum < kr && cum + hb[j] >= kr) {
                        s_sel[0] = threadIdx.x * pb + j;
                        s_sel[1] = cum;
                        s_sel[2] = hb[j];
                    }
                    cum += hb[j];
                }
            }
            __syncthreads();
            if (threadIdx.x < kClCTAs) {
                int* dec = cl.map_shared_rank(s_dec, threadIdx.x);
                unsigned long long* moa = cl.map_shared_rank(s_moa, threadIdx.x);
                dec[0] = s_sel[0];
                dec[1] = s_sel[1];
                dec[2] = s_sel[2];
                if (threadIdx.x) {
                    moa[0] = s_moa[0]; moa[1] = s_moa[1]; moa[2] = s_moa[2]; moa[3] = s_moa[3];
                }
            }
        }
        cl.sync();  // the decision is in every rank
        const int d = s_dec[0];
        kr -= s_dec[1];
        const int hd = s_dec[2];
        unsigned __int128 p = ((unsigned __int128)phi << 64) | plo;
        p |= ((unsigned __int128)d) << shift;
        top = shift;
        if (hd == kr) {
            const unsigned __int128 ones = (shift == 0) ? 0 : ((((unsigned __int128)1) << shift) - 1);
            p |= ones;
            if (rank == 0 && threadIdx.x == 0) {
                a.thr_hi[0] = (uint64_t)(p >> 64);
                a.thr_lo[0] = (uint64_t)p;
                a.mode[0] = 3;
                a.ksel[0] = k;
            }
            break;
        }
        sel_skip(p, top, s_moa[0], s_moa[1], s_moa[2], s_moa[3]);
        phi = (uint64_t)(p >> 64);
        plo = (uint64_t)p;
        if (!in_smem && hd <= kSelCap) {  // this rank's share of the bucket -> shared memory
            if (threadIdx.x == 0) s_ncomp = 0;
            __syncthreads();
            for (int i = lo + threadIdx.x; i < hi; i += blockDim.x) {
                const uint64_t h = a.chi[i], l = a.clo[i];
                if (sel_prefix(h, l, phi, plo, top)) {
                    const int slot = atomicAdd(&s_ncomp, 1);
                    sh[slot] = h;
                    sl[slot] = l;
                }
            }
            __syncthreads();
            n_s = s_ncomp;
            in_smem = true;
        }
        __syncthreads();
    }
    cl.sync();  // no rank leaves while another may still read its shared memory
}

// Multi-block MSD passes for one large segment (a single big mesh): every
// block histograms its slice of the candidates under the current prefix in
// shared memory and flushes non-zero bins (plus the bucket's OR / AND); one
// block then picks the digit and skips the bits the bucket shares.  Passes
// stop once the surviving bucket fits the shared-memory stage of k_select,
// which resumes from the resulting state.
__global__ void __launch_bounds__(512) k_sel_hist(SelectArgs a, int* __restrict__ ghist, int pass) {
    MF_PDL_ENTRY;
    if (*a.abort_flag) return;
    if (pass < 0) pass = ld_volatile(sel_pass(ghist));
    __shared__ int h[kSelBins];
    __shared__ unsigned long long s_oa[4];
    if (pass > 0 && (a.mode[0] != 0 || *sel_stop(ghist))) return;
    const int top = pass ? a.top[0] : 128;
    const int width = top >= kSelBits ? kSelBits : top;
    const int shift = top - width;
    const uint64_t phi = pass ? a.thr_hi[0] : 0, plo = pass ? a.thr_lo[0] : 0;
    for (int i = threadIdx.x; i < kSelBins; i += blockDim.x) h[i] = 0;
    if (threadIdx.x < 4) s_oa[threadIdx.x] = (threadIdx.x < 2) ? 0ull : ~0ull;
    __syncthreads();
    uint64_t oh = 0, ol = 0, ah = ~0ull, al = ~0ull;
    const int c0 = a.voff[0], c1 = c0 + a.seg_cnt[0];
    const bool compact = pass > 0 && *sel_compact(ghist);  // bucket <= kSelCap: copy it out too
    uint64_t* buf = sel_buf(ghist);
    for (int i = c0 + blockIdx.x * blockDim.x + threadIdx.x; i < c1; i += gridDim.x * blockDim.x) {
        uint64_t hh = a.chi[i], ll = a.clo[i];
        if (sel_prefix(hh, ll, phi, plo, top)) {
            hist_add(h, sel_digit(hh, ll, shift, width));
            oh |= hh; ol |= ll; ah &= hh; al &= ll;
            if (compact) {
                const int slot = atomicAdd(sel_count(ghist), 1);
                buf[2 * slot] = hh;
                buf[2 * slot + 1] = ll;
            }
        }
    }
    warp_orand(oh, ol, ah, al);
    if ((threadIdx.x & 31) == 0) {
        atomicOr(s_oa, oh); atomicOr(s_oa + 1, ol);
        atomicAnd(s_oa + 2, ah); atomicAnd(s_oa + 3, al);
    }
    __syncthreads();
    for (int i = threadIdx.x; i < kSelBins; i += blockDim.x)
        if (h[i]) atomicAdd(ghist + i, h[i]);
    unsigned long long* g = sel_orand(ghist);
    if (threadIdx.x == 0) {
        if (s_oa[0]) atomicOr(g, s_oa[0]);
        if (s_oa[1]) atomicOr(g + 1, s_oa[1]);
        if (~s_oa[2]) atomicAnd(g + 2, s_oa[2]);
        if (~s_oa[3]) atomicAnd(g + 3, s_oa[3]);
    }
}

__global__ void __launch_bounds__(kSelThreads) k_sel_decide(SelectArgs a, int* __restrict__ ghist, int pass) {
    MF_PDL_ENTRY;
    __shared__ int s_scan[33];
    __shared__ int s_sel[3];
    const bool loop = pass < 0;  // device-driven passes: every exit decides whether another follows
    auto stop_loop = [&]() {
        if (loop && threadIdx.x == 0) {
            *sel_pass(ghist) = 0;
            cudaGraphSetConditional(a.cond, 0u);
        }
    };
    if (*a.abort_flag) {
        stop_loop();
        return;
    }
    if (loop) pass = ld_volatile(sel_pass(ghist));
    unsigned long long* g = sel_orand(ghist);
    const int cnt = a.seg_cnt[0];
    int kr;
    uint64_t phi = 0, plo = 0;
    int top = 128;
    auto reset = [&]() {  // scratch back to its neutral state for the next pass / next selection
        for (int i = threadIdx.x; i < kSelBins; i += blockDim.x) ghist[i] = 0;
        if (threadIdx.x < 4) g[threadIdx.x] = (threadIdx.x < 2) ? 0ull : ~0ull;
    };
    if (pass == 0) {
        int want = a.act[0] ? a.budget[0] - (a.removed ? a.removed[0] : 0) : 0;
        int k = want < cnt ? want : cnt;
        if (k < 0) k = 0;
        if (threadIdx.x == 0) {
            a.ksel[0] = k;
            *sel_stop(ghist) = 0;
            *sel_compact(ghist) = 0;
            *sel_count(ghist) = 0;
        }
        if (k == 0 || k >= cnt) {
            if (threadIdx.x == 0) a.mode[0] = (k == 0) ? 2 : 1;
            reset();
            stop_loop();
            return;
        }
        kr = k;
    } else {
        if (a.mode[0] != 0 || *sel_stop(ghist)) {
            stop_loop();
            return;
        }
        kr = a.krem[0];
        phi = a.thr_hi[0];
        plo = a.thr_lo[0];
        top = a.top[0];
    }
    const int width = top >= kSelBits ? kSelBits : top;
    const int shift = top - width;
    const int per = kSelBins / kSelThreads;
    int loc = 0;
    for (int j = 0; j < per; j++) loc += ghist[threadIdx.x * per + j];
    int tot;
    int ex = block_excl_scan(loc, s_scan, &tot);
    if (ex < kr && kr <= ex + loc) {
        int cum = ex;
        for (int j = 0; j < per; j++) {
            int hv = ghist[threadIdx.x * per + j];
            if (cum + hv >= kr) {
                s_sel[0] = threadIdx.x * per + j;
                s_sel[1] = cum;
                s_sel[2] = hv;
                break;
            }
            cum += hv;
        }
    }
    __syncthreads();
    const uint64_t oh = g[0], ol = g[1], ah = g[2], al = g[3];
    __syncthreads();
    reset();
    if (threadIdx.x != 0) return;
    const int d = s_sel[0];
    kr -= s_sel[1];
    unsigned __int128 p = ((unsigned __int128)phi << 64) | plo;
    p |= ((unsigned __int128)d) << shift;
    int ntop = shift;
    if (s_sel[2] == kr) {
        unsigned __int128 ones = (shift == 0) ? 0 : ((((unsigned __int128)1) << shift) - 1);
        p |= ones;
        a.mode[0] = 3;
    } else {
        a.mode[0] = 0;
        sel_skip(p, ntop, oh, ol, ah, al);
        if (*sel_compact(ghist)) *sel_stop(ghist) = 1;       // this pass copied the bucket: hand over
        else if (s_sel[2] <= kSelCap) *sel_compact(ghist) = 1;  // next pass copies it
    }
    a.thr_hi[0] = (uint64_t)(p >> 64);
    a.thr_lo[0] = (uint64_t)p;
    a.krem[0] = kr;
    a.top[0] = ntop;
    if (loop) {
        const bool more = a.mode[0] == 0 && !*sel_stop(ghist) && pass + 1 < kSelPassesMax;
        *sel_pass(ghist) = more ? pass + 1 : 0;
        cudaGraphSetConditional(a.cond, more ? 1u : 0u);
    }
}

// ---- flag producers fused into the decoupled look-back scan (LoadOp functors)
// cluster anchor of v: lower end of its matched pair, the pair it was absorbed into, or itself
// (pairlo[v]: lower end of v's matched pair or -1, written with the final matching)
MF_DEV int cluster_anchor(int v, const int* __restrict__ pairlo, const int* __restrict__ absorbed) {
    const int p = pairlo[v];
    if (p >= 0) return p;
    const int a = absorbed[v];
    return a >= 0 ? a : v;
}
template <int ITEMS>
struct LoadIsRepT {  // v is the lowest member of its cluster
    static constexpr int items = ITEMS;  // two dependent gathers per item: short tiles
    const int* pairlo;
    const int* absorbed;
    const int* minrep;
    MF_DEV int operator()(int v) const { return minrep[cluster_anchor(v, pairlo, absorbed)] == v; }
};
typedef LoadIsRepT<2> LoadIsRep;

struct EpiFacetWrite {  // kept facet f -> output row prefix (order preserving compaction)
    const int* mapped;
    int* Fout;
    MF_DEV void operator()(int f, int pos, int keep) const {
        if (!keep) return;
        Fout[3 * pos] = mapped[3 * f];
        Fout[3 * pos + 1] = mapped[3 * f + 1];
        Fout[3 * pos + 2] = mapped[3 * f + 2];
    }
};
template <int ITEMS>
struct LoadKeepT {  // facet survives: bypassed, or first occurrence of its non-degenerate triple
    static constexpr int items = ITEMS;  // slot -> table gather per item: short tiles
    const int* dM;
    const int* slot;
    const int* table;
    MF_DEV int operator()(int f) const {
        if (f >= *dM) return 0;
        int s = slot[f];
        return s == -2 ? 1 : (s >= 0 && table[s] == f);
    }
};
typedef LoadKeepT<2> LoadKeep;


MF_DEV bool is_selected(int mode, uint64_t h, uint64_t l, uint64_t th, uint64_t tl) {
    return mode == 1 || (mode == 3 && !key_lt(th, tl, h, l));
}

MF_DEV bool seg_valid(const int* __restrict__ vmesh, const int* __restrict__ voff, const int* __restrict__ seg_cnt,
                      int i, int& b) {
    b = vmesh ? vmesh[i] : 0;
    return i - voff[b] < seg_cnt[b];
}

// Unmatch the pairs beyond the budget; removed = number kept.
MF_DEV void trunc_apply_body(const int* __restrict__ abort_flag, int N, const int* __restrict__ vmesh,
                              const int* __restrict__ voff, const int* __restrict__ seg_cnt,
                              const uint64_t* __restrict__ chi, const uint64_t* __restrict__ clo,
                              const int* __restrict__ cpay, const int* __restrict__ mode,
                              const uint64_t* __restrict__ thi, const uint64_t* __restrict__ tlo,
                              const int* __restrict__ e0, const int* __restrict__ e1, int* __restrict__ mate, int B,
                              const int* __restrict__ ksel, int* __restrict__ removed, int* __restrict__ seg_cnt2,
                              int* __restrict__ pairlo, const int* __restrict__ act, const int* __restrict__ budget,
                              cudaGraphConditionalHandle absorb_cond) {
    if (absorb_cond && blockIdx.x == 0 && threadIdx.x == 0) {
        // the absorb stage (an IF node) runs only if some mesh still misses its budget
        bool need = false;
        for (int b = 0; b < B && !need; b++) need = act[b] && ksel[b] < budget[b];
        cudaGraphSetConditional(absorb_cond, need ? 1u : 0u);
    }
    int tid = blockIdx.x * blockDim.x + threadIdx.x, nth = gridDim.x * blockDim.x;
    for (int b = tid; b < B; b += nth) removed[b] = ksel[b];
    (void)seg_cnt2;  // zeroed by k_edges: the absorb phase appends concurrently
    for (int i = tid; i < N; i += nth) {
        int b;
        if (!seg_valid(vmesh, voff, seg_cnt, i, b)) continue;
        if (is_selected(mode[b], chi[i], clo[i], thi[b], tlo[b])) continue;
        const int e = cpay[i], va = e0[e], vb = e1[e];
        mate[va] = -1;
        mate[vb] = -1;
        pairlo[va] = -1;
        pairlo[vb] = -1;
    }
}

// Absorb candidates (decimate.py:207-221): every unmatched vertex with edges
// picks its lowest (cost, rep) incident edge; the matching is maximal here so
// every neighbour is clustered and one pass suffices.
MF_DEV void absorb_cand_body(const int* __restrict__ loose,
                              const int* __restrict__ loose_cnt, const int* __restrict__ aoff,
                              const int* __restrict__ ucnt, const int* __restrict__ nbr,
                              const int* __restrict__ adj_eid, const double* __restrict__ cost,
                              const uint64_t* __restrict__ ckey, const int* __restrict__ pairlo,
                              const int* __restrict__ vmesh,
                              const int* __restrict__ voff, const int* __restrict__ act,
                              const int* __restrict__ budget, const int* __restrict__ removed,
                              int* __restrict__ seg_cnt, uint64_t* __restrict__ chi, uint64_t* __restrict__ clo,
                              int* __restrict__ caux) {
    if (!vmesh && (!act[0] || removed[0] >= budget[0])) return;  // budget met: no absorption this round
    const int L = *loose_cnt;  // the unmatched vertices k_mates listed (a thread each)
    for (int base = blockIdx.x * blockDim.x; base < L; base += gridDim.x * blockDim.x) {
        const int li = base + threadIdx.x;
        const int v = li < L ? loose[li] : -1;
        bool cand = false;
        uint64_t bk = ~0ull;
        int brep = 0x7fffffff;
        int nu = 0;
        if (v >= 0) {
            nu = ucnt[v];
            if (nu > 0 && pairlo[v] < 0) {
                int bm = mesh_of(vmesh, v);
                if (act[bm] && removed[bm] < budget[bm]) {
                    const size_t s = (size_t)aoff[v];
                    // up to 8 slots at a time: neighbour / edge loads, then the anchor gathers,
                    // then the key gathers, each batch in flight together (3 round trips)
                    for (int j0 = 0; j0 < nu; j0 += 8) {
                        int nb[8], ed[8], rp[8];
                        uint64_t ky[8];
#pragma unroll
                        for (int q = 0; q < 8; q++)
                            if (j0 + q < nu) {
                                nb[q] = nbr[s + j0 + q];
                                ed[q] = adj_eid[s + j0 + q];
                            }
#pragma unroll
                        for (int q = 0; q < 8; q++) rp[q] = (j0 + q < nu) ? pairlo[nb[q]] : -1;  // the anchor
#pragma unroll
                        for (int q = 0; q < 8; q++)  // unseeded: ckey == f64_key(cost)
                            ky[q] = rp[q] >= 0 ? (cost ? f64_key(cost[ed[q]]) : ckey[ed[q]]) : ~0ull;
#pragma unroll
                        for (int q = 0; q < 8; q++) {
                            if (rp[q] < 0) continue;  // cannot happen for a maximal matching
                            if (ky[q] < bk || (ky[q] == bk && rp[q] < brep)) { bk = ky[q]; brep = rp[q]; }
                        }
                    }
                    cand = brep != 0x7fffffff;
                }
            }
        }
        const int slot = seg_slot_uniform(cand, vmesh, voff, seg_cnt, v);
        if (cand) {
            chi[slot] = bk;
            clo[slot] = ((uint64_t)(unsigned)brep << 32) | (unsigned)v;
            caux[slot] = brep;
        }
    }
}

// Truncation and absorb candidates in one launch.  They touch disjoint meshes: the
// truncation unmatches pairs only where the budget is met (the selection kept fewer
// than all of them), and absorption runs only where it is not -- so the absorb phase
// needs no barrier behind the truncation (it reads the kept count from `ksel`, which
// is what the truncation stores into `removed`).
struct TruncArgs {
    int N;
    const int *vmesh, *voff, *seg_cnt;
    const uint64_t *chi, *clo;
    const int *cpay, *mode;
    const uint64_t *thi, *tlo;
    const int *e0, *e1;
    int* mate;
    int B;
    const int* ksel;
    int *removed, *seg_cnt2, *pairlo;
    const int *act, *budget;
    cudaGraphConditionalHandle absorb_cond;
};
struct AbsorbArgs {
    const int *loose, *loose_cnt, *aoff, *ucnt, *nbr, *adj_eid;
    const double* cost;
    const uint64_t* ckey;
    const int *pairlo, *vmesh, *voff, *act, *budget, *kept;
    int* seg_cnt;
    uint64_t *chi, *clo;
    int* caux;
};
__global__ void k_trunc_absorb(const int* __restrict__ abort_flag, TruncArgs t, AbsorbArgs a) {
    MF_PDL_ENTRY;
    if (*abort_flag) return;
    trunc_apply_body(abort_flag, t.N, t.vmesh, t.voff, t.seg_cnt, t.chi, t.clo, t.cpay, t.mode, t.thi, t.tlo, t.e0,
                     t.e1, t.mate, t.B, t.ksel, t.removed, t.seg_cnt2, t.pairlo, t.act, t.budget, t.absorb_cond);
    absorb_cand_body(a.loose, a.loose_cnt, a.aoff, a.ucnt, a.nbr, a.adj_eid, a.cost, a.ckey, a.pairlo, a.vmesh, a.voff,
                     a.act, a.budget, a.kept, a.seg_cnt, a.chi, a.clo, a.caux);
}

struct RoundFail {
    int* abort;
    int* fail_ach;     // per mesh: achievable vertices (first failure), -1 = ok
    int* fail_round;   // per mesh
    int* fail_noedge;  // per mesh: the failing round had no edges (decimate.py:239-244)
};

__global__ void k_absorb_apply(int N, const int* __restrict__ vmesh, const int* __restrict__ voff,
                               const int* __restrict__ seg_cnt, const uint64_t* __restrict__ chi,
                               const uint64_t* __restrict__ clo, const int* __restrict__ caux,
                               const int* __restrict__ mode, const uint64_t* __restrict__ thi,
                               const uint64_t* __restrict__ tlo, int* __restrict__ absorbed,
                               int* __restrict__ minrep, int B, const int* __restrict__ act,
                               const int* __restrict__ budget, const int* __restrict__ nin,
                               const int* __restrict__ ksel, int* __restrict__ removed, const int* __restrict__ aoff,
                               RoundFail fail, int round) {
    MF_PDL_ENTRY;
    if (*fail.abort) return;
    int tid = blockIdx.x * blockDim.x + threadIdx.x, nth = gridDim.x * blockDim.x;
    for (int i = tid; i < N; i += nth) {
        int b;
        if (!seg_valid(vmesh, voff, seg_cnt, i, b)) continue;
        if (is_selected(mode[b], chi[i], clo[i], thi[b], tlo[b])) {
            int v = (int)(clo[i] & 0xffffffffull), rep = caux[i];
            absorbed[v] = rep;
            atomicMin(minrep + rep, v);  // cluster's lowest member (decimate.py:224)
        }
    }
    for (int b = tid; b < B; b += nth) {
        if (!act[b]) continue;
        int r = removed[b] + ksel[b];
        removed[b] = r;
        if (r < budget[b]) {
            if (fail.fail_ach[b] < 0) {
                fail.fail_ach[b] = nin[b] - r;
                fail.fail_round[b] = round;
                fail.fail_noedge[b] = (aoff[voff[b + 1]] == aoff[voff[b]]);
            }
            atomicExch(fail.abort, 1);
        }
    }
}

// ------------------------------------------------------------------------
// K7: relabel (decimate.py:130-137, 275-278).  Cluster anchor = lower end of
// the matched pair; output index = rank of the cluster's lowest member.
// rstep = output index; the lowest member of output r is recorded (repv) and
// absorbed vertices are linked into their anchor's list (order fixed later).
__global__ void k_relabel3(int N, const int* __restrict__ abort_flag, const int* __restrict__ pairlo,
                           const int* __restrict__ absorbed,
                           const int* __restrict__ minrep, const int* __restrict__ outidx, int* __restrict__ rstep,
                           int* __restrict__ repv, int* __restrict__ abshead, int* __restrict__ absnext,
                           int* __restrict__ table, unsigned long long* __restrict__ tkey, int tsize, int table_init,
                           unsigned char* __restrict__ has_live, int* __restrict__ deg, int* __restrict__ cursor,
                           int* __restrict__ lowfill, int n1_next) {
    MF_PDL_ENTRY;
    if (*abort_flag) return;
    // the next round's degree / incidence cursor / lower-slot fill words (this round is past
    // the last kernels that use them: k_facet_plane, k_inc_scatter, k_edges)
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n1_next; i += gridDim.x * blockDim.x) {
        deg[i] = 0;
        cursor[i] = 0;
        lowfill[i] = 0;
    }
    // reset the facet dedupe table and the live-facet flags for k_facet_remap
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < tsize; i += gridDim.x * blockDim.x) {
        table[i] = table_init;
        if (tkey) tkey[i] = ~0ull;
    }
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < N; i += gridDim.x * blockDim.x) has_live[i] = 0;
    for (int v = blockIdx.x * blockDim.x + threadIdx.x; v < N; v += gridDim.x * blockDim.x) {
        const int p = pairlo[v];
        const int ab = p >= 0 ? -1 : absorbed[v];
        const int anc = p >= 0 ? p : (ab >= 0 ? ab : v);
        const int rep = minrep[anc];
        const int r = outidx[rep];
        rstep[v] = r;
        if (rep == v) repv[r] = v;
        if (ab >= 0) absnext[v] = atomicExch(abshead + anc, v);
    }
}

// Generic CSR scatter of items by key (order fixed afterwards by the segment sort).
__global__ void k_csr_scatter(int n, const int* __restrict__ abort_flag, const int* __restrict__ key,
                              const int* __restrict__ off, int* __restrict__ cursor, int* __restrict__ members) {
    MF_PDL_ENTRY;
    if (abort_flag && *abort_flag) return;
    for (int v = blockIdx.x * blockDim.x + threadIdx.x; v < n; v += gridDim.x * blockDim.x) {
        int r = key[v];
        members[off[r] + atomicAdd(cursor + r, 1)] = v;
    }
}

// Thread tier of the member sort; longer segments go to the heavy list.
__global__ void k_seg_sort_small(int nseg, const int* __restrict__ abort_flag, const int* __restrict__ off,
                                 int* __restrict__ members, int* __restrict__ heavy, int* __restrict__ heavy_count) {
    MF_PDL_ENTRY;
    if (abort_flag && *abort_flag) return;
    for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < nseg; r += gridDim.x * blockDim.x) {
        int s = off[r], d = off[r + 1] - s;
        if (d <= 1) continue;
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
__global__ void __launch_bounds__(256) k_seg_sort_heavy(const int* __restrict__ abort_flag,
                                                        const int* __restrict__ off, int* __restrict__ members,
                                                        int* __restrict__ tmp, const int* __restrict__ heavy,
                                                        const int* __restrict__ heavy_count) {
    MF_PDL_ENTRY;
    __shared__ int smem[kChunk];
    if (abort_flag && *abort_flag) return;
    const int H = *heavy_count;
    for (int h = blockIdx.x; h < H; h += gridDim.x) {
        int r = heavy[h];
        int s = off[r], d = off[r + 1] - s;
        block_sort_ints(members + s, tmp + s, d, smem);
    }
}

// Member fold of one output cluster: from +0.0 in ascending member order, then / count.
template <int PLACEMENT>
MF_DEV void fold_members(const int* m, int d, const double* __restrict__ P, const double* __restrict__ X, int C,
                         const double* __restrict__ vq, int r, double* __restrict__ Pout, double* __restrict__ Xout) {
    double sx = 0.0, sy = 0.0, sz = 0.0;
    for (int i = 0; i < d; i++) {
        const int v = m[i];
        sx = sx + P[3 * v];
        sy = sy + P[3 * v + 1];
        sz = sz + P[3 * v + 2];
    }
    const double cnt = (double)d;
    double avg[3] = {sx / cnt, sy / cnt, sz / cnt};
    if (PLACEMENT) {  // accumulate_quadrics + optimal_positions(..., 'inverse'), decimate.py:284-286
        double acc[10] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
        for (int i = 0; i < d; i++) {
            const double* q = vq + 10 * (size_t)m[i];
#pragma unroll
            for (int k = 0; k < 10; k++) acc[k] = acc[k] + q[k];
        }
        double t[3];
        mf_optimal_position(acc, acc + 6, avg, t);
        avg[0] = t[0]; avg[1] = t[1]; avg[2] = t[2];
    }
    Pout[3 * r] = avg[0];
    Pout[3 * r + 1] = avg[1];
    Pout[3 * r + 2] = avg[2];
    if (X) {
        for (int k = 0; k < C; k++) {
            double acc = 0.0;
            for (int i = 0; i < d; i++) acc = acc + X[(size_t)m[i] * C + k];
            Xout[(size_t)r * C + k] = acc / cnt;
        }
    }
}


// K8: contraction by member mean (decimate.py:280-283) and feature mean
// (decimate.py:142-145): members = anchor, its matched partner and the
// vertices absorbed into it, folded from +0.0 in ascending order, then / count.
// Inactive (bypassed) meshes copy rows verbatim.  Clusters of <= 4 members (nearly all: a
// pair plus a few absorbed vertices) are sorted and folded in registers; up to kSmallDeg in a
// local array; larger ones are listed and folded by the LAST block of the grid (block sort over
// scratch), so the rare heavy tier costs no extra launch.
template <int PLACEMENT>
MF_DEV void fold_members4(int m0, int m1, int m2, int m3, int d, const double* __restrict__ P,
                          const double* __restrict__ X, int C, const double* __restrict__ vq, int r,
                          double* __restrict__ Pout, double* __restrict__ Xout) {
    const int m[4] = {m0, m1, m2, m3};
    double sx = 0.0, sy = 0.0, sz = 0.0;
#pragma unroll
    for (int i = 0; i < 4; i++)
        if (i < d) {
            sx = sx + P[3 * m[i]];
            sy = sy + P[3 * m[i] + 1];
            sz = sz + P[3 * m[i] + 2];
        }
    const double cnt = (double)d;
    double avg[3] = {sx / cnt, sy / cnt, sz / cnt};
    if (PLACEMENT) {
        double acc[10] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
#pragma unroll
        for (int i = 0; i < 4; i++)
            if (i < d) {
                const double* q = vq + 10 * (size_t)m[i];
#pragma unroll
                for (int k = 0; k < 10; k++) acc[k] = acc[k] + q[k];
            }
        double t[3];
        mf_optimal_position(acc, acc + 6, avg, t);
        avg[0] = t[0]; avg[1] = t[1]; avg[2] = t[2];
    }
    Pout[3 * r] = avg[0];
    Pout[3 * r + 1] = avg[1];
    Pout[3 * r + 2] = avg[2];
    if (X) {
        for (int k = 0; k < C; k++) {
            double acc = 0.0;
#pragma unroll
            for (int i = 0; i < 4; i++)
                if (i < d) acc = acc + X[(size_t)m[i] * C + k];
            Xout[(size_t)r * C + k] = acc / cnt;
        }
    }
}

template <int PLACEMENT>
__global__ void k_contract(int Nout, const int* __restrict__ abort_flag, const int* __restrict__ repv,
                           const int* __restrict__ mate, const int* __restrict__ pairlo, const int* __restrict__ e1,
                           const int* __restrict__ absorbed, const int* __restrict__ abshead,
                           const int* __restrict__ absnext, const int* __restrict__ vmesh,
                           const int* __restrict__ act, const double* __restrict__ P, const double* __restrict__ X,
                           int C, double* __restrict__ Pout, double* __restrict__ Xout,
                           const double* __restrict__ vq, int* __restrict__ heavy, int* __restrict__ heavy_count,
                           int* __restrict__ scratch, int* __restrict__ tmp, int* __restrict__ scratch_used,
                           int* __restrict__ done_blocks) {
    MF_PDL_ENTRY;
    __shared__ int s_last;
    if (*abort_flag) return;
    for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < Nout; r += gridDim.x * blockDim.x) {
        const int v0 = repv[r];
        if (!act[mesh_of(vmesh, v0)]) {
            Pout[3 * r] = P[3 * v0];
            Pout[3 * r + 1] = P[3 * v0 + 1];
            Pout[3 * r + 2] = P[3 * v0 + 2];
            if (X)
                for (int k = 0; k < C; k++) Xout[(size_t)r * C + k] = X[(size_t)v0 * C + k];
            continue;
        }
        const int anc = cluster_anchor(v0, pairlo, absorbed);
        const int me = mate[anc];
        int a = anc, b = INT_MAX, c = INT_MAX, e = INT_MAX;
        int d = 1;
        if (me >= 0) b = e1[me], d = 2;
        int x = abshead[anc];
        if (x >= 0) {
            if (d == 1) b = x; else c = x;
            d++;
            x = absnext[x];
            while (x >= 0 && d < 4) {
                if (d == 2) c = x; else e = x;
                d++;
                x = absnext[x];
            }
        }
        if (x < 0) {  // at most 4 members: sorting network + register fold
            int t;
#define MF_CSWAP(p, q) if (p > q) t = p, p = q, q = t
            MF_CSWAP(a, b);
            MF_CSWAP(c, e);
            MF_CSWAP(a, c);
            MF_CSWAP(b, e);
            MF_CSWAP(b, c);
#undef MF_CSWAP
            fold_members4<PLACEMENT>(a, b, c, e, d, P, X, C, vq, r, Pout, Xout);
            continue;
        }
        int m[kSmallDeg];
        d = 0;
        m[d++] = anc;
        if (me >= 0) m[d++] = e1[me];
        bool big = false;
        for (int y = abshead[anc]; y >= 0; y = absnext[y]) {
            if (d == kSmallDeg) {
                big = true;
                break;
            }
            m[d++] = y;
        }
        if (big) {
            heavy[atomicAdd(heavy_count, 1)] = r;
            continue;
        }
        isort<kSmallDeg>(m, d);
        fold_members<PLACEMENT>(m, d, P, X, C, vq, r, Pout, Xout);
    }
    // the last block to finish folds the listed heavy clusters (block tier)
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        s_last = atomicAdd(done_blocks, 1) == (int)gridDim.x - 1;
    }
    __syncthreads();
    if (!s_last) return;
    __threadfence();
    __shared__ int smem[kChunk];
    __shared__ int s_d, s_base;
    const int H = ld_volatile(heavy_count);
    for (int h = 0; h < H; h++) {
        const int r = heavy[h];
        const int anc = cluster_anchor(repv[r], pairlo, absorbed);
        if (threadIdx.x == 0) {  // clusters are disjoint: their member lists fit in N slots in total
            int d = 1 + (mate[anc] >= 0);
            for (int y = abshead[anc]; y >= 0; y = absnext[y]) d++;
            s_d = d;
            s_base = atomicAdd(scratch_used, d);
            int* m = scratch + s_base;
            int i = 0;
            m[i++] = anc;
            if (mate[anc] >= 0) m[i++] = e1[mate[anc]];
            for (int y = abshead[anc]; y >= 0; y = absnext[y]) m[i++] = y;
        }
        __syncthreads();
        const int d = s_d;
        int* m = scratch + s_base;
        block_sort_ints(m, tmp + s_base, d, smem);
        if (threadIdx.x == 0) fold_members<PLACEMENT>(m, d, P, X, C, vq, r, Pout, Xout);
        __syncthreads();
    }
}

// ------------------------------------------------------------------------
// quality_report (decimate.py:580-602): cluster quadric = sum of the members'
// original vertex quadrics in ascending member order from +0.0
// (accumulate_quadrics, quadrics.py:80-86), evaluated at the output position
// (Quadric.evaluate, quadrics.py:53-58: row-major quadratic form, einsum-order
// linear term).  One thread per output vertex over the cluster CSR.
__global__ void k_quality(int n_out, const int* __restrict__ off, const int* __restrict__ members,
                          const double* __restrict__ vq, const double* __restrict__ Pout, int order,
                          double* __restrict__ err) {
    MF_PDL_ENTRY;
    for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < n_out; r += gridDim.x * blockDim.x) {
        double acc[10] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
        for (int i = off[r]; i < off[r + 1]; i++) {
            const double* q = vq + 10 * (size_t)members[i];
#pragma unroll
            for (int k = 0; k < 10; k++) acc[k] = acc[k] + q[k];
        }
        const double x0 = Pout[3 * (size_t)r], x1 = Pout[3 * (size_t)r + 1], x2 = Pout[3 * (size_t)r + 2];
        const double a00 = acc[0], a01 = acc[1], a02 = acc[2], a11 = acc[3], a12 = acc[4], a22 = acc[5];
        double quad = 0.0;
        quad = quad + (x0 * a00) * x0;
        quad = quad + (x0 * a01) * x1;
        quad = quad + (x0 * a02) * x2;
        quad = quad + (x1 * a01) * x0;
        quad = quad + (x1 * a11) * x1;
        quad = quad + (x1 * a12) * x2;
        quad = quad + (x2 * a02) * x0;
        quad = quad + (x2 * a12) * x1;
        quad = quad + (x2 * a22) * x2;
        const double lin = 2.0 * dot3(acc[6], acc[7], acc[8], x0, x1, x2, order);
        err[r] = (quad + lin) + acc[9];
    }
}

// ------------------------------------------------------------------------
// K9: output facets (decimate.py:147-167).
MF_DEV uint32_t tri_hash(int a, int b, int c) {
    uint32_t h = (uint32_t)a * 0x9E3779B1u;
    h ^= (uint32_t)b * 0x85EBCA77u + (h << 6) + (h >> 2);
    h ^= (uint32_t)c * 0xC2B2AE3Du + (h << 6) + (h >> 2);
    h ^= h >> 16;
    h *= 0x7feb352du;
    h ^= h >> 15;
    h *= 0x846ca68bu;
    h ^= h >> 16;
    return h;
}

// Base slot = min vertex * (slots per output vertex) + a small hash of the
// other two: facets sharing their lowest vertex land in one short run of the
// table, and consecutive facets (spatially coherent) probe neighbouring lines.
// PACKED (output vertex ids < 2^21): the sorted triple is the 64-bit table key
// itself -- CAS on the key, atomicMin on the parallel id word, no fences.
// Otherwise the key is the facet id and the triple lives in `canon` (a fence
// orders its store before the publishing CAS).
constexpr unsigned long long kEmptyKey = ~0ull;
template <bool PACKED>
__global__ void k_facet_remap(const int* __restrict__ dM, const int* __restrict__ abort_flag,
                              const int* __restrict__ F, const int* __restrict__ rstep, const int* __restrict__ vmesh,
                              const int* __restrict__ act, int* __restrict__ mapped, int4* __restrict__ canon,
                              int* __restrict__ slot, unsigned char* __restrict__ has_live, int* __restrict__ table,
                              unsigned long long* __restrict__ tkey, unsigned tmask, unsigned per_vertex) {
    MF_PDL_ENTRY;
    if (*abort_flag) return;
    const int M = *dM;
    for (int f = blockIdx.x * blockDim.x + threadIdx.x; f < M; f += gridDim.x * blockDim.x) {
        int ia = F[3 * f], ib = F[3 * f + 1], ic = F[3 * f + 2];
        int a = rstep[ia], b = rstep[ib], c = rstep[ic];
        mapped[3 * f] = a;
        mapped[3 * f + 1] = b;
        mapped[3 * f + 2] = c;
        if (!act[mesh_of(vmesh, ia)]) {  // bypass: kept verbatim (identity round keeps duplicates)
            slot[f] = -2;
            continue;
        }
        if (a == b || b == c || a == c) {
            slot[f] = -1;
            continue;
        }
        has_live[ia] = 1;
        has_live[ib] = 1;
        has_live[ic] = 1;
        int lo = min(a, min(b, c)), hi = max(a, max(b, c)), mid = a + b + c - lo - hi;
        unsigned h = ((unsigned)lo * per_vertex + (tri_hash(lo, mid, hi) & 7u)) & tmask;
        if (PACKED) {
            const unsigned long long key = ((unsigned long long)lo << 42) | ((unsigned long long)mid << 21) | hi;
            // CAS first: it returns the occupant, so a probe costs one round trip (a load before
            // the CAS made the common empty-slot case two)
            while (true) {
                unsigned long long cur = atomicCAS(tkey + h, kEmptyKey, key);
                if (cur == kEmptyKey || cur == key) {
                    atomicMin(table + h, f);
                    break;
                }
                h = (h + 1) & tmask;
            }
        } else {
            canon[f] = make_int4(lo, mid, hi, 0);
            __threadfence();
            while (true) {
                int cur = __ldcg(table + h);
                if (cur < 0) {
                    int prev = atomicCAS(table + h, -1, f);
                    if (prev < 0) break;
                    cur = prev;
                }
                int4 oc = __ldcg(canon + cur);
                if (oc.x == lo && oc.y == mid && oc.z == hi) {
                    atomicMin(table + h, f);
                    break;
                }
                h = (h + 1) & tmask;
            }
        }
        slot[f] = (int)h;
    }
}


__global__ void k_identity_index(int n, int* __restrict__ a, int* __restrict__ b) {
    MF_PDL_ENTRY;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) a[i] = b[i] = i;
}


// K10: chain replace / mapping across rounds (decimate.py:380-381); the
// round's mapping (decimate.py:159-167) is formed on the fly.
// Round epilogue: per-mesh output facet offsets, per-round counts, the next round's counter
// words cleared, and replace / mapping composed over the original vertices
// (decimate.py:380-381; mapping -1 where a vertex had facets but none survived, :159-167).
MF_DEV void compose_body(int N0, const int* __restrict__ rstep, const int* __restrict__ inc_off,
                         const unsigned char* __restrict__ has_live, const int* __restrict__ vmesh,
                         const int* __restrict__ act, int* __restrict__ rt, int* __restrict__ mt, int first_round, int B,
                         const int* __restrict__ kout, const int* __restrict__ foff_in, int* __restrict__ foff_out,
                         int* __restrict__ foff_fin, int* __restrict__ stats, const int* __restrict__ n_edges,
                         const int* __restrict__ ld_rounds, int* __restrict__ counters, int tid, int nth) {
    // per-mesh output facet offsets = keep-scan prefix at each mesh's first input facet
    for (int b = tid; b <= B; b += nth) {
        foff_out[b] = kout[foff_in[b]];
        if (foff_fin) foff_fin[b] = kout[foff_in[b]];
    }
    if (tid == 0) {  // per-round counts for the host (one readback at the end)
        stats[0] = foff_in[B];
        stats[1] = *n_edges >> 1;  // adjacency slots = 2 per edge
        stats[2] = kout[foff_in[B]];
        stats[3] = *ld_rounds;
    }
    for (int i = tid; i < 64; i += nth) counters[i] = 0;
    for (int i = tid; i < N0; i += nth) {
        int r = first_round ? i : rt[i];
        rt[i] = rstep[r];
        int m = first_round ? i : mt[i];
        if (m < 0) {
            mt[i] = -1;
            continue;
        }
        int ms = rstep[m];
        if (act[mesh_of(vmesh, m)] && inc_off[m + 1] > inc_off[m] && !has_live[m]) ms = -1;
        mt[i] = ms;
    }
}
__global__ void k_compose(int N0, const int* __restrict__ abort_flag, const int* __restrict__ rstep,
                          const int* __restrict__ inc_off, const unsigned char* __restrict__ has_live,
                          const int* __restrict__ vmesh, const int* __restrict__ act, int* __restrict__ rt,
                          int* __restrict__ mt, int first_round, int B, const int* __restrict__ kout,
                          const int* __restrict__ foff_in, int* __restrict__ foff_out, int* __restrict__ foff_fin,
                          int* __restrict__ stats, const int* __restrict__ n_edges, const int* __restrict__ ld_rounds,
                          int* __restrict__ counters) {
    MF_PDL_ENTRY;
    if (*abort_flag) return;
    compose_body(N0, rstep, inc_off, has_live, vmesh, act, rt, mt, first_round, B, kout, foff_in, foff_out, foff_fin,
                 stats, n_edges, ld_rounds, counters, blockIdx.x * blockDim.x + threadIdx.x, gridDim.x * blockDim.x);
}
// One mesh, not its last round: the round epilogue fused with the NEXT round's facet planes
// (independent work -- the planes read this round's output facets / positions; the facet
// count is this round's keep-scan total).  Saves a kernel boundary per round.
__global__ void k_compose_plane(int N0, const int* __restrict__ abort_flag, const int* __restrict__ rstep,
                                const int* __restrict__ inc_off, const unsigned char* __restrict__ has_live,
                                const int* __restrict__ act, int* __restrict__ rt, int* __restrict__ mt,
                                int first_round, const int* __restrict__ kout, const int* __restrict__ foff_in,
                                int* __restrict__ foff_out, int* __restrict__ stats, const int* __restrict__ n_edges,
                                const int* __restrict__ ld_rounds, int* __restrict__ counters,
                                const int* __restrict__ Fn, const double* __restrict__ Pn,
                                const int* __restrict__ act_next, Plane* __restrict__ plane, int* __restrict__ deg,
                                int order) {
    MF_PDL_ENTRY;
    if (*abort_flag) return;
    const int tid = blockIdx.x * blockDim.x + threadIdx.x, nth = gridDim.x * blockDim.x;
    facet_plane_body(kout[foff_in[1]], Fn, Pn, nullptr, act_next, plane, deg, order, tid, nth);
    compose_body(N0, rstep, inc_off, has_live, nullptr, act, rt, mt, first_round, 1, kout, foff_in, foff_out, nullptr,
                 stats, n_edges, ld_rounds, counters, tid, nth);
}

// ------------------------------------------------------------------------
// One kernel instead of a run of memset / memcpy nodes at the start of the
// graph (keeps the whole round chain a sequence of kernel nodes, so every
// edge can be a programmatic-dependent-launch edge).
__global__ void k_graph_init(int* __restrict__ status, int status_words, int fail_lo, int fail_hi,
                             int* __restrict__ foff_a, const int* __restrict__ foff0, int B, int* __restrict__ deg,
                             int* __restrict__ cursor, int* __restrict__ lowfill, int n1, int* __restrict__ counters,
                             unsigned long long* __restrict__ scan_a, unsigned long long* __restrict__ scan_b,
                             int scan_words, int* __restrict__ ghist, int nghist) {
    MF_PDL_ENTRY;
    const int tid = blockIdx.x * blockDim.x + threadIdx.x, nth = gridDim.x * blockDim.x;
    for (int i = tid; i < status_words; i += nth)
        status[i] = (i == 1) ? 0x7f7f7f7f : ((i >= fail_lo && i < fail_hi) ? -1 : 0);
    for (int b = tid; b <= B; b += nth) foff_a[b] = foff0[b];
    for (int i = tid; i < n1; i += nth) {
        deg[i] = 0;
        cursor[i] = 0;
        lowfill[i] = 0;
    }
    for (int i = tid; i < 64; i += nth) counters[i] = 0;
    for (int i = tid; i < scan_words; i += nth) {
        scan_a[i] = 0ull;
        scan_b[i] = 0ull;
    }
    // selection scratch: histogram + OR words zero, AND words all-ones (see kSelScratch)
    for (int i = tid; i < nghist; i += nth) ghist[i] = (i >= kSelBins + 4 && i < kSelBins + 8) ? -1 : 0;
}

// Start of every round chain, one launch: the workspace clears k_graph_init did (the status
// words now arrive pre-initialised with the params upload) fused with the input conversion of
// k_inputs_in -- facets int64 -> int32 with range / repeat validation, positions checked for
// NaN / inf and copied into the workspace.  The input pointers are per call: the captured graph
// node's arguments are updated on replay (device inputs are read in place, no staging copy).
struct InitArgs {
    int* foff_a;
    const int* foff0;
    int B;
    int* deg;
    int* cursor;
    int* lowfill;
    int n1;
    int* counters;
    unsigned long long* scan_a;
    unsigned long long* scan_b;
    int scan_words;
    int* ghist;
    int nghist;
    int64_t M;
    const void* F64;  // int64 [M,3], or int32 when f_is32 (a previous result's device facets)
    int f_is32;
    int* F32;
    const int64_t* voff;
    const int64_t* foff;
    int* badf;
    int64_t n3;
    const double* Psrc;
    double* P0;
    int* badp;
    unsigned long long* vs;  // both look-back buffers of k_vertex_scan
    int vs_words;
};
__global__ void k_init_inputs(InitArgs a) {
    MF_PDL_ENTRY;
    const int tid = blockIdx.x * blockDim.x + threadIdx.x, nth = gridDim.x * blockDim.x;
    for (int b = tid; b <= a.B; b += nth) a.foff_a[b] = a.foff0[b];
    for (int i = tid; i < a.n1; i += nth) {
        a.deg[i] = 0;
        a.cursor[i] = 0;
        a.lowfill[i] = 0;
    }
    for (int i = tid; i < 64; i += nth) a.counters[i] = 0;
    for (int i = tid; i < a.scan_words; i += nth) {
        a.scan_a[i] = 0ull;
        a.scan_b[i] = 0ull;
    }
    // selection scratch: histogram + OR words zero, AND words all-ones (see kSelScratch)
    for (int i = tid; i < a.nghist; i += nth) a.ghist[i] = (i >= kSelBins + 4 && i < kSelBins + 8) ? -1 : 0;
    for (int i = tid; i < a.vs_words; i += nth) a.vs[i] = 0ull;
    const bool copy_p = a.Psrc != a.P0;
    const int64_t T = a.M > a.n3 ? a.M : a.n3;
    for (int64_t f = tid; f < T; f += nth) {
        if (f < a.n3) {
            const double x = a.Psrc[f];
            if (!isfinite(x)) atomicExch(a.badp, 1);
            if (copy_p) a.P0[f] = x;
        }
        if (f >= a.M) continue;
        int lo = 0, hi = a.B;
        while (hi - lo > 1) {
            int mid = (lo + hi) >> 1;
            if (a.foff[mid] <= f) lo = mid; else hi = mid;
        }
        const int64_t vlo = a.voff[lo], vhi = a.voff[lo + 1];
        int64_t x, y, z;
        if (a.f_is32) {
            const int* F = (const int*)a.F64;
            x = F[3 * f], y = F[3 * f + 1], z = F[3 * f + 2];
        } else {
            const int64_t* F = (const int64_t*)a.F64;
            x = F[3 * f], y = F[3 * f + 1], z = F[3 * f + 2];
        }
        const bool ok = x >= vlo && x < vhi && y >= vlo && y < vhi && z >= vlo && z < vhi && x != y && y != z && x != z;
        if (!ok) atomicMin(a.badf, (int)min(f, (int64_t)0x7ffffffe));
        a.F32[3 * f] = (int)x;
        a.F32[3 * f + 1] = (int)y;
        a.F32[3 * f + 2] = (int)z;
    }
}

// ------------------------------------------------------------------------
// boundary conversion / validation
__global__ void k_facets_in(int64_t M, const int64_t* __restrict__ F64, int* __restrict__ F32, int B,
                            const int64_t* __restrict__ voff, const int64_t* __restrict__ foff,
                            int* __restrict__ bad) {
    MF_PDL_ENTRY;
    for (int64_t f = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; f < M; f += (int64_t)gridDim.x * blockDim.x) {
        int lo = 0, hi = B;
        while (hi - lo > 1) {
            int mid = (lo + hi) >> 1;
            if (foff[mid] <= f) lo = mid; else hi = mid;
        }
        int64_t vlo = voff[lo], vhi = voff[lo + 1];
        int64_t a = F64[3 * f], b = F64[3 * f + 1], c = F64[3 * f + 2];
        bool ok = a >= vlo && a < vhi && b >= vlo && b < vhi && c >= vlo && c < vhi && a != b && b != c && a != c;
        if (!ok) atomicMin(bad, (int)min(f, (int64_t)0x7ffffffe));
        F32[3 * f] = (int)a;
        F32[3 * f + 1] = (int)b;
        F32[3 * f + 2] = (int)c;
    }
}
// Both input checks in one launch: facets converted / validated (as k_facets_in) and
// positions checked for NaN / inf.
__global__ void k_inputs_in(int64_t M, const int64_t* __restrict__ F64, int* __restrict__ F32, int B,
                            const int64_t* __restrict__ voff, const int64_t* __restrict__ foff, int* __restrict__ badf,
                            int64_t n3, const double* __restrict__ P, int* __restrict__ badp) {
    MF_PDL_ENTRY;
    const int64_t T = M > n3 ? M : n3;
    for (int64_t f = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; f < T; f += (int64_t)gridDim.x * blockDim.x) {
        if (f < n3 && !isfinite(P[f])) atomicExch(badp, 1);
        if (f >= M) continue;
        int lo = 0, hi = B;
        while (hi - lo > 1) {
            int mid = (lo + hi) >> 1;
            if (foff[mid] <= f) lo = mid; else hi = mid;
        }
        int64_t vlo = voff[lo], vhi = voff[lo + 1];
        int64_t a = F64[3 * f], b = F64[3 * f + 1], c = F64[3 * f + 2];
        bool ok = a >= vlo && a < vhi && b >= vlo && b < vhi && c >= vlo && c < vhi && a != b && b != c && a != c;
        if (!ok) atomicMin(badf, (int)min(f, (int64_t)0x7ffffffe));
        F32[3 * f] = (int)a;
        F32[3 * f + 1] = (int)b;
        F32[3 * f + 2] = (int)c;
    }
}
__global__ void k_f32_to_f64(int64_t n, const float* __restrict__ a, double* __restrict__ b) {
    MF_PDL_ENTRY;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        b[i] = (double)a[i];
}
__global__ void k_i32_to_i64(int64_t n, const int* __restrict__ a, int64_t* __restrict__ b, int64_t add) {
    MF_PDL_ENTRY;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        b[i] = (int64_t)a[i] + add;
}
// any differing 64-bit word -> *diff = 1 (features-are-positions check, mesh.py:28-29)
__global__ void k_words_differ(int64_t n, const unsigned long long* __restrict__ a,
                               const unsigned long long* __restrict__ b, int* __restrict__ diff) {
    MF_PDL_ENTRY;
    bool d = false;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        d |= a[i] != b[i];
    if (__any_sync(0xffffffffu, d) && (threadIdx.x & 31) == 0) *diff = 1;
}
// Fused result emission (mf_decimation_copy): up to 8 jobs, each widening int32 -> int64,
// copying float64, or narrowing float64 -> float32 into a device-writable destination.
constexpr int kEmitI32 = 0, kEmitF64 = 1, kEmitF32 = 2, kEmitW32 = 3;  // W32: int32 copied as is
constexpr int kEmitMax = 12;
struct EmitJobs {
    const void* src[kEmitMax];
    void* dst[kEmitMax];
    int64_t n[kEmitMax];
    int kind[kEmitMax];
    const int* ndev[kEmitMax];  // when set, the job moves min(n, *ndev * 3) elements (a device-side count)
    int count = 0;
    void add(int k, const void* s, void* d, int64_t cnt, const int* rows3 = nullptr) {
        src[count] = s;
        dst[count] = d;
        n[count] = cnt;
        kind[count] = k;
        ndev[count] = rows3;
        count++;
    }
    int64_t total() const {
        int64_t t = 0;
        for (int i = 0; i < count; i++) t += n[i];
        return t;
    }
};
__global__ void k_emit(EmitJobs j) {
    MF_PDL_ENTRY;
    const int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x, nth = (int64_t)gridDim.x * blockDim.x;
    for (int q = 0; q < j.count; q++) {
        const int64_t n = j.ndev[q] ? min(j.n[q], 3 * (int64_t)*j.ndev[q]) : j.n[q];
        const int k = j.kind[q];
        if (k == kEmitW32) {
            const int* sp = (const int*)j.src[q];
            int* dp = (int*)j.dst[q];
            int64_t done = 0;
            if ((((uintptr_t)dp | (uintptr_t)sp) & 15) == 0) {  // four words per thread, 16-byte moves
                const int64_t h = n >> 2;
                for (int64_t i = tid; i < h; i += nth) ((int4*)dp)[i] = ((const int4*)sp)[i];
                done = h << 2;
            }
            for (int64_t i = done + tid; i < n; i += nth) dp[i] = sp[i];
            continue;
        }
        // two elements per thread as one 16-byte store when both ends are 16-byte aligned
        if (k != kEmitF32 && (((uintptr_t)j.dst[q] | (uintptr_t)j.src[q]) & 15) == 0) {
            const int64_t h = n >> 1;
            if (k == kEmitI32) {
                const int2* sp = (const int2*)j.src[q];
                longlong2* dp = (longlong2*)j.dst[q];
                for (int64_t i = tid; i < h; i += nth) {
                    const int2 x = sp[i];
                    dp[i] = make_longlong2(x.x, x.y);
                }
            } else {
                const double2* sp = (const double2*)j.src[q];
                double2* dp = (double2*)j.dst[q];
                for (int64_t i = tid; i < h; i += nth) dp[i] = sp[i];
            }
            if ((n & 1) && tid == 0) {
                if (k == kEmitI32) ((int64_t*)j.dst[q])[n - 1] = ((const int*)j.src[q])[n - 1];
                else ((double*)j.dst[q])[n - 1] = ((const double*)j.src[q])[n - 1];
            }
            continue;
        }
        for (int64_t i = tid; i < n; i += nth) {
            if (j.kind[q] == kEmitI32) ((int64_t*)j.dst[q])[i] = ((const int*)j.src[q])[i];
            else if (j.kind[q] == kEmitF64) ((double*)j.dst[q])[i] = ((const double*)j.src[q])[i];
            else ((float*)j.dst[q])[i] = (float)((const double*)j.src[q])[i];
        }
    }
}
__global__ void k_f64_to_f32(int64_t n, const double* __restrict__ a, float* __restrict__ b) {
    MF_PDL_ENTRY;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        b[i] = (float)a[i];
}

}  // namespace mf
