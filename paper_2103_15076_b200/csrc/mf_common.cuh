// mf_common.cuh -- device helpers shared by the decimation / pooling kernels.
//
// Everything here is integer/byte plumbing sized for B200 (148 SMs, 32-wide
// warps, 126 MB L2): order-preserving keys, warp-aggregated list appends,
// a single-pass decoupled look-back scan, and a software grid barrier for
// the persistent (cooperatively launched) kernels.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#define MF_DEV __device__ __forceinline__

// Programmatic dependent launch: every kernel first waits for its
// predecessor grid (griddepcontrol.wait is a no-op without a programmatic
// edge) and then lets its own dependents start launching, so a graph node's
// launch and prologue overlap the previous node's tail.
#ifdef MF_PDL_EARLY_TRIGGER
#define MF_PDL_ENTRY                                              \
    do {                                                          \
        asm volatile("griddepcontrol.wait;" ::: "memory");        \
        asm volatile("griddepcontrol.launch_dependents;" :::);    \
    } while (0)
#else
// no explicit trigger: a block triggers its dependents when it exits, so a
// dependent grid's CTAs never compete with the primary's unlaunched CTAs
#define MF_PDL_ENTRY                                              \
    do {                                                          \
        asm volatile("griddepcontrol.wait;" ::: "memory");        \
    } while (0)
#endif

namespace mf {

constexpr int kWarp = 32;

// ------------------------------------------------------------------------
// float64 -> order-preserving uint64.  -0.0 is canonicalised to +0.0 and any
// NaN to the largest key, mirroring numpy's comparison semantics inside
// lexsort (equal zeros tie; NaN sorts last) -- decimate.py:183, 217-220.
MF_DEV uint64_t f64_key(double c) {
    uint64_t u = (uint64_t)__double_as_longlong(c);
    if (c == 0.0) u = 0ull;
    if (c != c) u = 0x7FF8000000000000ull;
    return (u >> 63) ? ~u : (u | 0x8000000000000000ull);
}
MF_DEV double f64_unkey(uint64_t k) {
    uint64_t u = (k >> 63) ? (k & 0x7FFFFFFFFFFFFFFFull) : ~k;
    return __longlong_as_double((long long)u);
}

MF_DEV bool key_lt(uint64_t ah, uint64_t al, uint64_t bh, uint64_t bl) {
    return ah < bh || (ah == bh && al < bl);
}

// Lane-aggregated append: one atomic per warp-converged group.
MF_DEV int append_slot(int* counter) {
    unsigned mask = __activemask();
    int lane = threadIdx.x & 31;
    int leader = __ffs(mask) - 1;
    int base = 0;
    if (lane == leader) base = atomicAdd(counter, __popc(mask));
    base = __shfl_sync(mask, base, leader);
    return base + __popc(mask & ((1u << lane) - 1u));
}

MF_DEV int warp_sum(int v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}
MF_DEV int warp_incl_scan(int v) {
    int lane = threadIdx.x & 31;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        int t = __shfl_up_sync(0xffffffffu, v, o);
        if (lane >= o) v += t;
    }
    return v;
}

MF_DEV int ld_volatile(const int* p) { return *(const volatile int*)p; }
MF_DEV unsigned long long ld_volatile(const unsigned long long* p) {
    return *(const volatile unsigned long long*)p;
}

// ------------------------------------------------------------------------
// Bulk-copy engine (TMA, non-tensor form): an mbarrier with a transaction count tracks the bytes
// of cp.async.bulk global->shared copies (k_unpool_tma, k_select's key stage).
MF_DEV unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
MF_DEV void mbar_init(uint64_t* bar, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
MF_DEV void mbar_expect_tx(uint64_t* bar, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}
MF_DEV void mbar_wait(uint64_t* bar, unsigned parity) {
    asm volatile(
        "{\n .reg .pred p;\n LAB_WAIT:\n"
        " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        " @!p bra LAB_WAIT;\n}\n" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}
MF_DEV void bulk_g2s(void* dst, const void* src, unsigned bytes, uint64_t* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_u32(dst)),
                 "l"(src), "r"(bytes), "r"(smem_u32(bar))
                 : "memory");
}

// ------------------------------------------------------------------------
// Software grid barrier for persistent kernels.  The launch must guarantee
// co-residency (cudaLaunchCooperativeKernel with an occupancy-bounded grid).
// `bar` = {arrive counter, generation}; zeroed once per launch.
MF_DEV void grid_sync(unsigned* bar) {
    __syncthreads();
    if (threadIdx.x == 0) {
        volatile unsigned* gen = bar + 1;
        unsigned g = *gen;
        __threadfence();
        unsigned arrived = atomicAdd(bar, 1u) + 1u;
        if (arrived == gridDim.x) {
            bar[0] = 0u;
            __threadfence();
            atomicAdd(bar + 1, 1u);
        } else {
            while (*gen == g) { __nanosleep(32); }
        }
        __threadfence();
    }
    __syncthreads();
}

// ------------------------------------------------------------------------
// Single-pass exclusive scan of int32 with decoupled look-back.
// out[i] = sum(in[0..i)), out[n] = total.  `status` must hold ceil(n/TILE)
// zeroed words and `ticket` one zeroed int (both reset with one memset).
constexpr int kScanBlock = 256;
constexpr int kScanItems = 8;                      // items per thread for plain array loads
constexpr int kScanTile = kScanBlock * kScanItems;
constexpr int kScanTileMin = kScanBlock * 2;       // smallest tile (gathering load functors): sizes the state
// items per thread of a load functor: LoadOp::items when it declares one (functors whose
// load is a chain of dependent gathers use short tiles -- more CTAs in flight), else 8
template <typename T, typename = void>
struct ScanItems {
    static constexpr int value = kScanItems;
};
template <typename T>
struct ScanItems<T, decltype((void)T::items, void())> {
    static constexpr int value = T::items;
};

// plain-array loads (LoadOp::vec4): each thread's 8 items are read and written as two
// 16-byte vectors (the scalar pattern touches 8x the L1 sectors per instruction)
template <typename T, typename = void>
struct ScanVec4 {
    static constexpr bool value = false;
};
template <typename T>
struct ScanVec4<T, decltype((void)T::vec4, void())> {
    static constexpr bool value = T::vec4;
};

constexpr unsigned long long kFlagAgg = 1ull << 32;
constexpr unsigned long long kFlagPre = 2ull << 32;

struct EpiNone {
    MF_DEV void operator()(int, int, int) const {}
};

// `epi(i, exclusive_prefix, value)` runs for every element after its prefix is known
// (lets a compaction write its payload in the same pass).
template <typename LoadOp, typename Epi = EpiNone>
__global__ void __launch_bounds__(kScanBlock) k_scan_excl(LoadOp load, int n, int* __restrict__ out,
                                                          unsigned long long* status, int* ticket,
                                                          const int* __restrict__ abort_flag, Epi epi = Epi(),
                                                          unsigned long long* __restrict__ clear = nullptr,
                                                          int clear_words = 0) {
    MF_PDL_ENTRY;
    // double-buffered look-back state: clear the buffer the NEXT scan will use
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < clear_words; i += gridDim.x * blockDim.x) clear[i] = 0ull;
    if (abort_flag && *abort_flag) return;  // a failed round: every later stage is skipped
    __shared__ int s_tile;
    __shared__ int s_warp[kScanBlock / 32];
    __shared__ int s_prefix;
    // tiles in launch order by ticket -- needed for forward progress only when the grid can be
    // larger than what is resident at once (ticket == nullptr: the host knows every tile is
    // co-resident, blockIdx.x is the tile and one L2 atomic round trip is saved)
    int tile = blockIdx.x;
    if (ticket) {
        if (threadIdx.x == 0) s_tile = atomicAdd(ticket, 1);
        __syncthreads();
        tile = s_tile;
    }
    constexpr int kItems = ScanItems<LoadOp>::value;
    const long long base = (long long)tile * (kScanBlock * kItems) + (long long)threadIdx.x * kItems;
    int v[kItems];
    int tsum = 0;
    constexpr bool kVec = ScanVec4<LoadOp>::value && kItems == 8;
    const bool full = kVec && base + kItems <= n;
    if constexpr (kVec) {
        if (full) {
            const int4* src = reinterpret_cast<const int4*>(load.p + base);
            const int4 a = src[0], b = src[1];
            v[0] = a.x; v[1] = a.y; v[2] = a.z; v[3] = a.w;
            v[4] = b.x; v[5] = b.y; v[6] = b.z; v[7] = b.w;
#pragma unroll
            for (int i = 0; i < kItems; i++) tsum += v[i];
        }
    }
    if (!full) {
#pragma unroll
        for (int i = 0; i < kItems; i++) {
            long long idx = base + i;
            v[i] = (idx < n) ? load((int)idx) : 0;
            tsum += v[i];
        }
    }
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    int incl = warp_incl_scan(tsum);
    if (lane == 31) s_warp[warp] = incl;
    __syncthreads();
    if (warp == 0) {
        int w = (lane < kScanBlock / 32) ? s_warp[lane] : 0;
        int wi = warp_incl_scan(w);
        if (lane < kScanBlock / 32) s_warp[lane] = wi - w;  // exclusive per warp
        int agg = __shfl_sync(0xffffffffu, wi, kScanBlock / 32 - 1);
        // publish + look back
        // the flag and the value share one 64-bit word, so publishing needs no fence: nothing
        // else the consumer reads is ordered by it (the clears above belong to the NEXT scan)
        if (lane == 0) {
            unsigned long long word = (tile == 0 ? kFlagPre : kFlagAgg) | (unsigned)agg;
            atomicExch(status + tile, word);
        }
        int excl = 0;
        if (tile > 0) {
            int pred = tile - 1;
            while (true) {
                int idx = pred - lane;
                unsigned long long s = (idx >= 0) ? ld_volatile(status + idx) : (kFlagPre);
                while (__any_sync(0xffffffffu, (s >> 32) == 0ull)) {
                    if ((s >> 32) == 0ull) s = ld_volatile(status + idx);
                }
                unsigned pmask = __ballot_sync(0xffffffffu, (s >> 32) == 2ull);
                int first = pmask ? (__ffs(pmask) - 1) : 32;
                int val = (lane <= first) ? (int)(unsigned)(s & 0xffffffffull) : 0;
                excl += warp_sum(val);
                if (pmask) break;
                pred -= 32;
            }
            if (lane == 0) atomicExch(status + tile, kFlagPre | (unsigned)(excl + agg));
        }
        if (lane == 0) s_prefix = excl;
    }
    __syncthreads();
    int run = s_prefix + s_warp[warp] + (incl - tsum);
    if constexpr (kVec) {
      if (full) {
        int o[kItems];
#pragma unroll
        for (int i = 0; i < kItems; i++) {
            o[i] = run;
            epi((int)(base + i), run, v[i]);
            run += v[i];
        }
        int4* dst = reinterpret_cast<int4*>(out + base);
        dst[0] = make_int4(o[0], o[1], o[2], o[3]);
        dst[1] = make_int4(o[4], o[5], o[6], o[7]);
        if (base + kItems == n) out[n] = run;
        return;
      }
    }
#pragma unroll
    for (int i = 0; i < kItems; i++) {
        long long idx = base + i;
        if (idx < n) {
            out[idx] = run;
            epi((int)idx, run, v[i]);
        }
        run += v[i];
        if (idx == n - 1) out[n] = run;
    }
    if (n == 0 && tile == 0 && threadIdx.x == 0) out[0] = 0;
}

struct LoadArr {
    static constexpr bool vec4 = true;  // p and out 16-byte aligned (arena allocations)
    const int* p;
    MF_DEV int operator()(int i) const { return p[i]; }
};

// In-register insertion sort of a short int array (segment tiers use this
// for lengths <= the small-tier bound).
template <int CAP>
MF_DEV void isort(int* a, int n) {
    for (int i = 1; i < n; i++) {
        int x = a[i], j = i - 1;
        while (j >= 0 && a[j] > x) { a[j + 1] = a[j]; j--; }
        a[j + 1] = x;
    }
}

// Block-wide bitonic sort of `n` ints in shared memory (padded to pow2 with INT_MAX).
MF_DEV void block_bitonic(int* s, int n_pow2) {
    for (int k = 2; k <= n_pow2; k <<= 1) {
        for (int j = k >> 1; j > 0; j >>= 1) {
            for (int i = threadIdx.x; i < n_pow2; i += blockDim.x) {
                int ixj = i ^ j;
                if (ixj > i) {
                    int a = s[i], b = s[ixj];
                    bool up = ((i & k) == 0);
                    if ((a > b) == up) { s[i] = b; s[ixj] = a; }
                }
            }
            __syncthreads();
        }
    }
}

}  // namespace mf
