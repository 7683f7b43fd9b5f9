// Persistent, TMA-pipelined, warp-local jagged-diagonal tile engine for the sparse passes (sm_100a).
//
// A pass walks one compressed layout (CSR panels for the row pass, CSC for the
// column pass) tile by tile. A tile is a run of <= kPSeg segments (rows or
// columns) with <= kPCap nonzeros, cut on the host (cf_setup.cu), or one
// segment longer than kMaxDiag ("long tile", streamed in chunks).
//
// Inside a normal tile every WARP BLOCK of 32 consecutive segments is stored
// in jagged-diagonal order (k_build_jds): the block's segments are ranked by
// length (descending, stable), rank r holds local segment perm[r], and the
// k-th nonzero of rank r sits at joff_w[k] + r. So
//   * lane r owns one segment: it gathers g[idx] for its nonzeros (kUnroll
//     independent loads in flight) and sums the products SEQUENTIALLY in
//     canonical order — np.bincount's order (uv.py:10-12), bit-identical;
//   * a warp reads idx/val of 32 segments at consecutive shared-memory
//     addresses (conflict-free); lanes drop out in length order;
//   * the rank -> natural-order transpose of the sums stays inside the warp, so
//     the epilogue runs in natural segment order with no CTA barrier: its
//     vectors are loaded straight from global memory (coalesced, issued at
//     tile start so they arrive during the gathers) and its stores coalesce.
// The L1TEX pipe's ~1 random sector per SM-cycle (the gathers) is then the
// dominant consumer of the only hot on-chip resource.
//
// Warp roles: per compute group (kPSeg threads) one producer warp issues
// cp.async.bulk (TMA 1D) copies of a future tile's idx/val/perm/joff into the
// group's slots of a kStages ring (full[s] mbarrier, L2 evict-first hint on
// every streamed byte); the group's warps consume (empty[s] when done).
// Groups alternate tiles; a group needs a barrier only for cone epilogues and
// long tiles. The ring is kept small on purpose: shared memory beyond ~150 KB
// per SM starves the L1 that the outstanding gathers need (profiles/r01_probes.md).
#pragma once

#include <cmath>
#include <cstdint>

#include "cf_common.h"

namespace cf {
namespace pass {

#ifndef CF_STAGES
#define CF_STAGES 4
#endif
#ifndef CF_GROUPS
#define CF_GROUPS 2
#endif
#ifndef CF_UNROLL
#define CF_UNROLL 20
#endif
#ifndef CF_GATHER_NOALLOC
#define CF_GATHER_NOALLOC 1        // gathers bypass L1 allocation (measured: +3%)
#endif
#ifndef CF_PCAP
#define CF_PCAP 3072
#endif
#ifndef CF_PSEG
#define CF_PSEG 256
#endif
constexpr int kPCap = CF_PCAP;     // nonzeros per staged tile
constexpr int kPSeg = CF_PSEG;     // segments per tile (== threads of a compute group)
constexpr int kMaxDiag = 256;      // longest segment inside a normal tile (longer ones get their own tile)
constexpr int kStages = CF_STAGES; // ring depth (all groups)
constexpr int kGroups = CF_GROUPS; // compute groups; group g consumes the CTA's tiles i = g, g+kGroups, ...
constexpr int kUnroll = CF_UNROLL; // independent gathers in flight per thread
constexpr int kComputeWarps = kPSeg / 32;      // per group
constexpr int kComputeThreads = kPSeg;         // per group
constexpr int kPThreads = kGroups * (kComputeThreads + 32);   // + one producer warp per group
constexpr int kJoffHdr = 2 * kComputeWarps;    // per-warp {start, maxlen} header of a tile's joff
constexpr int kJoffMax = kJoffHdr + kComputeWarps * (kMaxDiag + 1);
constexpr int kFvTab = 256;
static_assert(kStages % kGroups == 0, "a ring slot must be reused by the same compute group (mbarrier parity)");

struct alignas(16) Stage {
    int32_t meta[4];                    // s0, nseg, k0, len (written by the producer)
    int32_t meta2[4];                   // joff length (0 = long tile), first joff entry
    int32_t idx[kPCap + 8];
    double val[kPCap + 4];
    uint8_t perm[kPSeg + 16];
    uint16_t joff[kJoffMax + 16];
};

struct Smem {
    Stage st[kStages];
    alignas(8) uint64_t full[kStages];
    alignas(8) uint64_t empty[kStages];
    double fvtab[kFvTab];               // 1/(1+cnt) for small column counts (uv.py:82)
    double wacc[kGroups][kPSeg];        // rank -> natural transpose of the sums (warp-private slices)
    int32_t wcnt[kGroups][kPSeg];
    double cscr[kGroups][4][kPSeg];     // cone epilogue: x+, w, delta, delta+
    double red[kGroups][32];
};

constexpr size_t kSmemBytes = sizeof(Smem);

// x / mu; exact multiply when mu is a power of two (then x * (1/mu) == x / mu bit for bit)
struct MuDiv {
    double mu, inv;
    bool pow2;
    __device__ __forceinline__ double operator()(double x) const { return pow2 ? x * inv : x / mu; }
};
__host__ inline MuDiv make_mudiv(double mu) {
    int e = 0;
    const double fr = frexp(mu, &e);
    MuDiv d{mu, 1.0 / mu, fr == 0.5 && e > -1000 && e < 1000};
    return d;
}

// Epilogue vectors of one segment, loaded by the policy (natural order, coalesced).
struct Vals {
    double v[5];
};

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

// compute group of the calling thread and its thread index inside the group
__device__ __forceinline__ int group_id() { return (int)threadIdx.x / kComputeThreads; }
__device__ __forceinline__ int group_tid() { return (int)threadIdx.x % kComputeThreads; }
// named barrier of the caller's compute group (ids 1..kGroups; 0 is __syncthreads)
__device__ __forceinline__ void group_sync() {
    asm volatile("bar.sync %0, %1;" ::"r"(1 + group_id()), "n"(kComputeThreads) : "memory");
}

// deterministic reduction over the caller's compute group; result valid in its thread 0
template <class Op>
__device__ double group_reduce(double v, double* red, Op op) {
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) v = op(v, __shfl_xor_sync(0xffffffffu, v, off));
    const int w = group_tid() >> 5, l = group_tid() & 31;
    group_sync();
    if (l == 0) red[w] = v;
    group_sync();
    if (w == 0) {
        v = (l < kComputeWarps) ? red[l] : 0.0;
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) v = op(v, __shfl_xor_sync(0xffffffffu, v, off));
    }
    return v;
}

__device__ __forceinline__ double ld_gather(const double* p, uint64_t pol) {
    double v;
#if CF_GATHER_NOALLOC
    asm("ld.global.nc.L1::no_allocate.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(v) : "l"(p), "l"(pol));
#else
    asm("ld.global.nc.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(v) : "l"(p), "l"(pol));
#endif
    return v;
}
// streamed once: no L1 allocation, L2 evict-first
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
// starts at the 16-byte boundary below `first`; element 0 lands at lead_of(first).
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
    if (bytes) bulk_g2s(dst, (const void*)((uintptr_t)first & ~(uintptr_t)15u), bytes, bar, pol);
}

// Tile table: tb[t] = {first segment, first nonzero, first joff entry, joff length (0 = long tile)};
// tile t spans [tb[t].x, tb[t+1].x) segments and [tb[t].y, tb[t+1].y) nonzeros.
struct Tiles {
    const int4* tb;
    int32_t n_tiles;
};

// The JDS layout of a pass: idx/val in warp-local jagged-diagonal order inside
// every normal tile (canonical order inside long tiles); perm (rank -> local
// segment of the warp block, one byte per segment position); joff per tile =
// {start, maxlen} per warp block, then every block's diagonal starts
// (tile-relative nonzero offsets).
struct Jds {
    const int32_t* idx;
    const double* val;
    const uint8_t* perm;
    const uint16_t* joff;
};

// ---------------------------------------------------------------- the engine
// P (the pass policy) provides (device):
//   const double* gvec() const                 gathered operand
//   Vals load(int s) const                     epilogue vectors of segment s (global index, natural order)
//   bool carry_in() const; double carry(const Vals&) const   starting value of a segment's sum
//   static constexpr int kUnroll               gathers in flight per thread
//   static constexpr bool kGroupEpilogue       epilogue needs all segments of the tile at once (cones)
//   void check(double a, int j, double g)      per-nonzero hook (report finiteness)
//   void segment(Smem&, int tile, int s0, int q, int cnt, double acc, const Vals&)
//                                              epilogue of local segment q (natural order)
//   void group(Smem&, int tile, int s0, int nseg)   (kGroupEpilogue) after a group barrier
//   void finish(Smem&)                         compute threads, after the last tile
__device__ __forceinline__ void issue_tile(const Jds& L, int4 lo, int4 hi, Stage& st, uint64_t* bar, uint64_t pol) {
    const int s0 = lo.x, nseg = hi.x - lo.x, k0 = lo.y, len = hi.y - lo.y, j0 = lo.z, jn = lo.w;
    st.meta[0] = s0;
    st.meta[1] = nseg;
    st.meta[2] = k0;
    st.meta[3] = len;
    st.meta2[0] = jn;
    st.meta2[1] = j0;
    if (jn == 0) {  // long tile: nothing staged (streamed by the consumers)
        mbar_expect_tx(bar, 0);
        return;
    }
    const uint32_t total = span_bytes(L.idx + k0, len) + span_bytes(L.val + k0, len) +
                           span_bytes(L.perm + s0, nseg) + span_bytes(L.joff + j0, jn);
    mbar_expect_tx(bar, total);
    copy_span(st.idx, L.idx + k0, len, bar, pol);
    copy_span(st.val, L.val + k0, len, bar, pol);
    copy_span(st.perm, L.perm + s0, nseg, bar, pol);
    copy_span(st.joff, L.joff + j0, jn, bar, pol);
}

template <class P>
__global__ void __launch_bounds__(kPThreads, 1) k_pass(const P p0, const Jds L, const Tiles T, const int32_t* done) {
    if (done && *done) return;
    P p = p0;  // per-thread mutable copy (report accumulators live in registers)
    extern __shared__ __align__(128) unsigned char smem_raw[];
    Smem& sm = *reinterpret_cast<Smem*>(smem_raw);
    const int G = gridDim.x;
    const int my = (T.n_tiles > (int)blockIdx.x) ? (T.n_tiles - (int)blockIdx.x + G - 1) / G : 0;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int c = threadIdx.x; c < kFvTab; c += blockDim.x) sm.fvtab[c] = 1.0 / (1.0 + (double)c);
    if (threadIdx.x == 0) {
        for (int s = 0; s < kStages; ++s) {
            mbar_init(&sm.full[s], 1);
            mbar_init(&sm.empty[s], kComputeWarps);
        }
        fence_mbar_init();
    }
    __syncthreads();

    if (warp >= kGroups * kComputeWarps) {
        // ------------------------------------------------ producers: warp kGroups*kComputeWarps + g feeds group g
        const int pg = warp - kGroups * kComputeWarps;
        if (lane == 0) {
            const uint64_t pf = pol_first();
            // the next tile's table entries are loaded before waiting for its slot
            int4 lo = make_int4(0, 0, 0, 0), hi = lo;
            if (pg < my) {
                lo = T.tb[blockIdx.x + pg * G];
                hi = T.tb[blockIdx.x + pg * G + 1];
            }
            for (int i = pg; i < my; i += kGroups) {
                const int s = i % kStages;
                int4 nlo = lo, nhi = hi;
                if (i + kGroups < my) {
                    nlo = T.tb[blockIdx.x + (i + kGroups) * G];
                    nhi = T.tb[blockIdx.x + (i + kGroups) * G + 1];
                }
                if (i >= kStages) {
                    mbar_wait(&sm.empty[s], (uint32_t)(((i / kStages) - 1) & 1));
                    fence_proxy_async();
                }
                issue_tile(L, lo, hi, sm.st[s], &sm.full[s], pf);
                lo = nlo;
                hi = nhi;
            }
        }
        return;
    }

    // ---------------------------------------------------- compute warps
    const uint64_t pl = pol_last(), pf = pol_first();
    const double* __restrict__ g = p.gvec();
    const int grp = group_id();
    const int gt = group_tid();
    const int gw = gt >> 5;      // warp within the group = warp block of the tile
    double* wacc = sm.wacc[grp] + gw * 32;
    int32_t* wcnt = sm.wcnt[grp] + gw * 32;
    for (int i = grp; i < my; i += kGroups) {
        const int s = i % kStages;
        Stage& st = sm.st[s];
        mbar_wait(&sm.full[s], (uint32_t)((i / kStages) & 1));
        const int s0 = st.meta[0], nseg = st.meta[1], k0 = st.meta[2], len = st.meta[3];
        const int jn = st.meta2[0];
        const int tile = (int)blockIdx.x + i * G;
        if (jn > 0) {
            const int nb = min(32, nseg - gw * 32);   // segments of this warp block
            if (nb > 0) {
                const int32_t* ib = st.idx + lead_of(L.idx + k0);
                const double* vb = st.val + lead_of(L.val + k0);
                const uint8_t* pb = st.perm + lead_of(L.perm + s0) + gw * 32;
                const uint16_t* jh = st.joff + lead_of(L.joff + st.meta2[1]);
                const uint16_t* jb = jh + jh[2 * gw];   // this block's diagonal starts
                const int mlen = jh[2 * gw + 1];
                const bool nat = lane < nb;             // natural segment gw*32 + lane exists
                const Vals vv = nat ? p.load(s0 + gw * 32 + lane) : Vals{};
                const int r = lane;                     // rank within the block
                const int q = nat ? (int)pb[r] : 0;     // local segment (within the block) of rank r
                const double c0 = p.carry_in() ? p.carry(vv) : 0.0;
                double acc = __shfl_sync(0xffffffffu, c0, q);
                int cnt = 0;
                constexpr int U = P::kUnroll;
                for (int k = 0; k < mlen; k += U) {
                    int e[U];
                    bool ok[U];
                    bool any = false;
#pragma unroll
                    for (int u = 0; u < U; ++u) {
                        const int kk = k + u;
                        const int a = kk < mlen ? (int)jb[kk] : 0;
                        const int b = kk < mlen ? (int)jb[kk + 1] : 0;
                        ok[u] = nat && (b - a) > r;
                        e[u] = a + r;
                        any |= ok[u];
                    }
                    if (!__any_sync(0xffffffffu, any)) break;
                    int jj[U];
                    double av[U], gv[U];
#pragma unroll
                    for (int u = 0; u < U; ++u) {
                        jj[u] = ok[u] ? ib[e[u]] : 0;
                        av[u] = ok[u] ? vb[e[u]] : 0.0;
                    }
#pragma unroll
#ifdef CF_EXP_LOCALGATHER
                    for (int u = 0; u < U; ++u) gv[u] = ok[u] ? ld_gather(g + (jj[u] & 4095), pl) : 0.0;
#else
                    for (int u = 0; u < U; ++u) gv[u] = ok[u] ? ld_gather(g + jj[u], pl) : 0.0;
#endif
#pragma unroll
                    for (int u = 0; u < U; ++u)
                        if (ok[u]) {
                            p.check(av[u], jj[u], gv[u]);
                            acc = __dadd_rn(acc, __dmul_rn(av[u], gv[u]));
                            ++cnt;
                        }
                }
                // rank -> natural order inside the warp
                if (nat) {
                    wacc[q] = acc;
                    wcnt[q] = cnt;
                }
                __syncwarp();
                if (nat) p.segment(sm, tile, s0, gw * 32 + lane, wcnt[lane], wacc[lane], vv);
                __syncwarp();
            }
        } else {
            // long tile: one segment [k0, k0+len), canonical order, chunked through the stage
            double* buf = st.val;
            double* lacc = sm.wacc[grp];
            Vals vv{};
            if (gt == 0) {
                vv = p.load(s0);
                lacc[0] = p.carry_in() ? p.carry(vv) : 0.0;
            }
            group_sync();
            for (int c0 = 0; c0 < len; c0 += kPCap) {
                const int cl = min(kPCap, len - c0);
                for (int e = gt; e < cl; e += kComputeThreads) {
                    const int jj = ld_first(L.idx + k0 + c0 + e, pf);
                    const double a = ld_first(L.val + k0 + c0 + e, pf);
                    const double gj = ld_gather(g + jj, pl);
                    p.check(a, jj, gj);
                    buf[e] = __dmul_rn(a, gj);
                }
                group_sync();
                if (gt == 0) {
                    double acc = lacc[0];
                    for (int e = 0; e < cl; ++e) acc = __dadd_rn(acc, buf[e]);
                    lacc[0] = acc;
                }
                group_sync();
            }
            if (gt == 0) p.segment(sm, tile, s0, 0, len, lacc[0], vv);
            group_sync();
        }
        if (P::kGroupEpilogue) {
            group_sync();
            p.group(sm, tile, s0, nseg);
            group_sync();   // cone scratch of this group is rewritten by its next tile
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&sm.empty[s]);
    }
    p.finish(sm);
}

}  // namespace pass
}  // namespace cf
