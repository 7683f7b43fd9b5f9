// Persistent, warp-specialised, TMA-pipelined tile engine for the sparse passes (sm_100a).
//
// A pass walks the nonzeros of one compressed layout (CSR panels for the row
// pass, CSC for the column pass) tile by tile. A tile is a run of segments
// (rows or columns) whose nonzeros are contiguous and, unless a single
// segment is longer, fit one stage (kPCap). Tiles are cut on the host
// (cf_setup.cu: greedy by nonzeros and segment count, cone-aligned for
// columns). Each persistent CTA owns tiles blockIdx.x, +gridDim.x, ...
//
// Warp roles (one CTA per SM, kStages-deep shared-memory ring):
//   producer warp : cp.async.bulk (TMA 1D) of a tile's index/value slices,
//                   segment pointers and epilogue vectors -> stage, completing
//                   on full[s]; every streamed byte carries an L2 evict-first
//                   hint so the gathered vector stays L2-resident.
//   gather warps  : g[idx] for every staged nonzero (8 independent loads per
//                   lane in flight, evict-last), product written in place over
//                   the staged value; arrive on prod[s]. They never wait for
//                   the reduction, so the L1TEX pipe — whose ~1 random sector
//                   per SM-cycle is the hard limit of this kernel — stays busy.
//   reducer warps : one thread per segment sums its products SEQUENTIALLY in
//                   storage order (np.bincount order, uv.py:10-12), starting
//                   from the carried partial of the previous panel, then runs
//                   the pass epilogue; arrive on empty[s] to free the stage.
// A segment longer than kPCap is handled by the reducer warps alone, streaming
// it through the stage in chunks (rare: only for pathological row lengths).
#pragma once

#include <cstdint>

#include "cf_common.h"

namespace cf {
namespace pass {

constexpr int kPCap = 2048;       // nonzeros per staged tile
constexpr int kPSeg = 256;        // segments per tile (== reducer threads)
constexpr int kStages = 5;        // ring depth
constexpr int kGatherWarps = 8;
constexpr int kReduceWarps = kPSeg / 32;
constexpr int kGatherThreads = kGatherWarps * 32;
constexpr int kReduceThreads = kReduceWarps * 32;
constexpr int kPThreads = kGatherThreads + kReduceThreads + 32;   // + producer warp
constexpr int kPVecs = 5;         // epilogue vectors staged per tile (incl. the panel carry)
constexpr int kReduceBarrier = 1; // named barrier id of the reducer group

struct alignas(16) Stage {
    int32_t meta[4];                   // s0, s1, k0, k1 (written by the producer)
    int32_t idx[kPCap + 8];
    double val[kPCap + 4];
    int32_t ptr[kPSeg + 12];
    double vec[kPVecs][kPSeg + 4];
};

struct Smem {
    Stage st[kStages];
    alignas(8) uint64_t full[kStages];
    alignas(8) uint64_t prod[kStages];
    alignas(8) uint64_t empty[kStages];
    double acc[kPSeg];
    double red[32];
};

constexpr size_t kSmemBytes = sizeof(Smem);

// ---------------------------------------------------------------- PTX helpers
__device__ __forceinline__ uint32_t smem_addr(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ uint64_t pol_first() {
    uint64_t p;
    asm("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ uint64_t pol_last() {
    uint64_t p;
    asm("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_addr(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n"
        ".reg .pred P1;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
        "@!P1 bra WAIT_%=;\n"
        "}\n" ::"r"(smem_addr(bar)),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar, uint64_t pol) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], "
        "%4;" ::"r"(smem_addr(dst)),
        "l"(src), "r"(bytes), "r"(smem_addr(bar)), "l"(pol)
        : "memory");
}
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
__device__ __forceinline__ void fence_mbar_init() { asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
__device__ __forceinline__ void reducer_sync() {
    asm volatile("bar.sync %0, %1;" ::"n"(kReduceBarrier), "n"(kReduceThreads) : "memory");
}

__device__ __forceinline__ int rtid() { return (int)threadIdx.x - kGatherThreads; }

// deterministic reduction over the reducer group; result valid in reducer thread 0
template <class Op>
__device__ double reducer_reduce(double v, double* red, Op op) {
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) v = op(v, __shfl_xor_sync(0xffffffffu, v, off));
    const int w = rtid() >> 5, l = rtid() & 31;
    reducer_sync();
    if (l == 0) red[w] = v;
    reducer_sync();
    if (w == 0) {
        v = (l < kReduceWarps) ? red[l] : 0.0;
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) v = op(v, __shfl_xor_sync(0xffffffffu, v, off));
    }
    return v;
}

__device__ __forceinline__ double ld_gather(const double* p, uint64_t pol) {
    double v;
    asm("ld.global.nc.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(v) : "l"(p), "l"(pol));
    return v;
}
__device__ __forceinline__ double ld_first(const double* p, uint64_t pol) {
    double v;
    asm("ld.global.nc.L1::no_allocate.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(v) : "l"(p), "l"(pol));
    return v;
}
__device__ __forceinline__ int32_t ld_first(const int32_t* p, uint64_t pol) {
    int32_t v;
    asm("ld.global.nc.L1::no_allocate.L2::cache_hint.s32 %0, [%1], %2;" : "=r"(v) : "l"(p), "l"(pol));
    return v;
}
__device__ __forceinline__ void st_hint(double* p, double v, uint64_t pol) {
    asm volatile("st.global.L2::cache_hint.f64 [%0], %1, %2;" ::"l"(p), "d"(v), "l"(pol) : "memory");
}

// Aligned superset copy of `count` elements starting at `first`: the copy
// starts at the 16-byte boundary below `first`; the consumer finds element 0
// at lead_of(first).
template <class T>
__device__ __forceinline__ int lead_of(const T* first) {
    return (int)(((uintptr_t)first & 15u) / sizeof(T));
}
template <class T>
__device__ __forceinline__ uint32_t span_bytes(const T* first, int64_t count) {
    if (count <= 0) return 0u;
    const uintptr_t a = (uintptr_t)first & ~(uintptr_t)15u;
    const uintptr_t e = (uintptr_t)(first + count);
    return (uint32_t)(((e - a) + 15u) & ~(uintptr_t)15u);
}
template <class T>
__device__ __forceinline__ void copy_span(void* dst, const T* first, int64_t count, uint64_t* bar, uint64_t pol) {
    const uint32_t bytes = span_bytes(first, count);
    if (count > 0 && bytes) bulk_g2s(dst, (const void*)((uintptr_t)first & ~(uintptr_t)15u), bytes, bar, pol);
}

// Tile boundaries: tb[t] = {first segment, first nonzero}; tile t = [tb[t], tb[t+1]).
struct Tiles {
    const int2* tb;
    int32_t n_tiles;
};

// ---------------------------------------------------------------- the engine
// P (the pass policy) provides, all __device__ unless noted:
//   int nvec() const; const double* vec(int v) const   staged epilogue vectors, indexed by segment
//   const int32_t* ptr() / idx(); const double* val() / gvec()
//   bool carry_in() const                               acc starts from staged vec[nvec()-1]
//   void check(double a, int j, double g)               per-nonzero hook (report finiteness)
//   void epilogue(Smem&, Stage&, int tile, int s0, int nseg, const int32_t* ptrb, const double* const* vecb)
//                                                       reducer threads only (reducer_sync() allowed)
//   void finish(Smem&)                                  reducer threads only, after the last tile
template <class P>
__device__ __forceinline__ void issue_tile(const P& p, const Tiles& T, int t, Stage& st, uint64_t* bar,
                                           uint64_t pol) {
    const int2 lo = T.tb[t], hi = T.tb[t + 1];
    const int s0 = lo.x, s1 = hi.x, k0 = lo.y, k1 = hi.y;
    st.meta[0] = s0;
    st.meta[1] = s1;
    st.meta[2] = k0;
    st.meta[3] = k1;
    const bool fits = (k1 - k0) <= kPCap;
    const int nv = p.nvec();
    uint32_t total = span_bytes(p.ptr() + s0, s1 - s0 + 1);
    if (fits && k1 > k0) total += span_bytes(p.idx() + k0, k1 - k0) + span_bytes(p.val() + k0, k1 - k0);
    for (int v = 0; v < nv; ++v) total += span_bytes(p.vec(v) + s0, s1 - s0);
    mbar_expect_tx(bar, total);
    copy_span(st.ptr, p.ptr() + s0, s1 - s0 + 1, bar, pol);
    if (fits && k1 > k0) {
        copy_span(st.idx, p.idx() + k0, k1 - k0, bar, pol);
        copy_span(st.val, p.val() + k0, k1 - k0, bar, pol);
    }
    for (int v = 0; v < nv; ++v) copy_span(st.vec[v], p.vec(v) + s0, s1 - s0, bar, pol);
}

template <class P>
__global__ void __launch_bounds__(kPThreads, 1) k_pass(const P p0, const Tiles T, const int32_t* done) {
    if (done && *done) return;
    P p = p0;  // per-thread mutable copy (report accumulators live in registers)
    extern __shared__ __align__(128) unsigned char smem_raw[];
    Smem& sm = *reinterpret_cast<Smem*>(smem_raw);
    const int G = gridDim.x;
    const int my = (T.n_tiles > (int)blockIdx.x) ? (T.n_tiles - (int)blockIdx.x + G - 1) / G : 0;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        for (int s = 0; s < kStages; ++s) {
            mbar_init(&sm.full[s], 1);
            mbar_init(&sm.prod[s], kGatherWarps);
            mbar_init(&sm.empty[s], kReduceWarps);
        }
        fence_mbar_init();
    }
    __syncthreads();

    if (warp == kGatherWarps + kReduceWarps) {
        // ------------------------------------------------ producer
        if (lane == 0) {
            const uint64_t pf = pol_first();
            for (int i = 0; i < my; ++i) {
                const int s = i % kStages;
                if (i >= kStages) {
                    mbar_wait(&sm.empty[s], (uint32_t)(((i / kStages) - 1) & 1));
                    fence_proxy_async();
                }
                issue_tile(p, T, blockIdx.x + i * G, sm.st[s], &sm.full[s], pf);
            }
        }
        return;
    }

    if (warp < kGatherWarps) {
        // ------------------------------------------------ gatherers
        const uint64_t pl = pol_last();
        const double* __restrict__ g = p.gvec();
        const int gt = threadIdx.x;
        for (int i = 0; i < my; ++i) {
            const int s = i % kStages;
            Stage& st = sm.st[s];
            mbar_wait(&sm.full[s], (uint32_t)((i / kStages) & 1));
            const int k0 = st.meta[2], len = st.meta[3] - k0;
            if (len <= kPCap) {
                const int32_t* ib = st.idx + lead_of(p.idx() + k0);
                double* vb = st.val + lead_of(p.val() + k0);
                int e = gt;
                for (; e + 7 * kGatherThreads < len; e += 8 * kGatherThreads) {
                    int j[8];
                    double gv[8];
#pragma unroll
                    for (int u = 0; u < 8; ++u) j[u] = ib[e + u * kGatherThreads];
#pragma unroll
                    for (int u = 0; u < 8; ++u) gv[u] = ld_gather(g + j[u], pl);
#pragma unroll
                    for (int u = 0; u < 8; ++u) {
                        const double a = vb[e + u * kGatherThreads];
                        p.check(a, j[u], gv[u]);
                        vb[e + u * kGatherThreads] = __dmul_rn(a, gv[u]);
                    }
                }
                int j[8];
                double gv[8];
                int cnt = 0;
#pragma unroll
                for (int u = 0; u < 8; ++u) {
                    const int ee = e + u * kGatherThreads;
                    j[u] = ee < len ? ib[ee] : 0;
                }
#pragma unroll
                for (int u = 0; u < 8; ++u)
                    if (e + u * kGatherThreads < len) gv[u] = ld_gather(g + j[u], pl);
#pragma unroll
                for (int u = 0; u < 8; ++u) {
                    const int ee = e + u * kGatherThreads;
                    if (ee < len) {
                        const double a = vb[ee];
                        p.check(a, j[u], gv[u]);
                        vb[ee] = __dmul_rn(a, gv[u]);
                        ++cnt;
                    }
                }
                (void)cnt;
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(&sm.prod[s]);
        }
        return;
    }

    // ---------------------------------------------------- reducers
    const int rt = threadIdx.x - kGatherThreads;   // 0 .. kReduceThreads-1
    const uint64_t pf = pol_first(), pl = pol_last();
    for (int i = 0; i < my; ++i) {
        const int s = i % kStages;
        Stage& st = sm.st[s];
        mbar_wait(&sm.prod[s], (uint32_t)((i / kStages) & 1));
        const int s0 = st.meta[0], s1 = st.meta[1], k0 = st.meta[2], k1 = st.meta[3];
        const int nseg = s1 - s0, len = k1 - k0;
        const int32_t* ptrb = st.ptr + lead_of(p.ptr() + s0);
        const double* vecb[kPVecs];
        const int nv = p.nvec();
#pragma unroll
        for (int v = 0; v < kPVecs; ++v) vecb[v] = v < nv ? st.vec[v] + lead_of(p.vec(v) + s0) : nullptr;
        const double* carry = p.carry_in() ? vecb[nv - 1] : nullptr;
        if (len <= kPCap) {
            const double* vb = st.val + lead_of(p.val() + k0);
            for (int q = rt; q < nseg; q += kReduceThreads) {
                const int a = ptrb[q] - k0, b = ptrb[q + 1] - k0;
                double acc = carry ? carry[q] : 0.0;
                int k = a;
                for (; k + 3 < b; k += 4) {
                    const double v0 = vb[k], v1 = vb[k + 1], v2 = vb[k + 2], v3 = vb[k + 3];
                    acc = __dadd_rn(__dadd_rn(__dadd_rn(__dadd_rn(acc, v0), v1), v2), v3);
                }
                for (; k < b; ++k) acc = __dadd_rn(acc, vb[k]);
                sm.acc[q] = acc;
            }
        } else {
            // one long segment: stream it through the stage's value buffer
            for (int q = rt; q < nseg; q += kReduceThreads) sm.acc[q] = carry ? carry[q] : 0.0;
            double* buf = st.val;
            const double* __restrict__ g = p.gvec();
            for (int c0 = k0; c0 < k1; c0 += kPCap) {
                const int cl = min(kPCap, k1 - c0);
                for (int e = rt; e < cl; e += kReduceThreads) {
                    const int jj = ld_first(p.idx() + c0 + e, pf);
                    const double a = ld_first(p.val() + c0 + e, pf);
                    const double gj = ld_gather(g + jj, pl);
                    p.check(a, jj, gj);
                    buf[e] = __dmul_rn(a, gj);
                }
                reducer_sync();
                for (int q = rt; q < nseg; q += kReduceThreads) {
                    const int a = max(ptrb[q], c0) - c0, b = min(ptrb[q + 1], c0 + cl) - c0;
                    if (a < b) {
                        double acc = sm.acc[q];
                        for (int k = a; k < b; ++k) acc = __dadd_rn(acc, buf[k]);
                        sm.acc[q] = acc;
                    }
                }
                reducer_sync();
            }
        }
        p.epilogue(sm, st, (int)blockIdx.x + i * G, s0, nseg, ptrb, vecb);
        reducer_sync();
        if ((rt & 31) == 0) mbar_arrive(&sm.empty[s]);
    }
    p.finish(sm);
}

}  // namespace pass
}  // namespace cf
