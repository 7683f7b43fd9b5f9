// Persistent warp-local jagged-diagonal tile engine for the sparse passes (sm_100a).
//
// A pass walks one compressed layout (CSR panels for the row pass, CSC for the
// column pass) tile by tile. A tile is a run of <= kPSeg segments (rows or
// columns) with <= kPCap nonzeros, cut on the host (cf_setup.cu), or one
// segment longer than kMaxDiag ("long tile").
//
// Inside a normal tile every WARP BLOCK of 32 consecutive segments is stored
// in jagged-diagonal order (k_build_jds): the block's segments are ranked by
// length (descending, stable), rank r holds local segment perm[r], and the
// k-th nonzero of rank r sits at k0 + start_w + sum_{j<k} width_j + r
// (width_j = ranks longer than j). pl[rank] = perm | len << 5 | start_w << 14,
// so each lane knows its own length and the offsets come from warp ballots.
//   * lane r owns one segment: it loads idx/val of its nonzeros straight from
//     global memory (a diagonal is contiguous, so the warp's loads coalesce;
//     L1 no-allocate, L2 evict-first), gathers g[idx] (kUnroll independent
//     loads in flight, L2 evict-last) and sums the products SEQUENTIALLY in
//     canonical order — np.bincount's order (uv.py:10-12), bit-identical;
//   * the rank -> natural-order transpose of the sums stays inside the warp, so
//     the epilogue runs in natural segment order with no CTA barrier: its
//     vectors are loaded straight from global memory (coalesced, issued at
//     block start so they arrive during the gathers) and its stores coalesce.
// Nothing is staged in shared memory. Measured (profiles/r01_probes.md): a
// random fp64 gather costs one L1TEX->L2 request, ~1 per SM-cycle, and that
// request port is the bound; TMA bulk staging of idx/val added ~40 % to a
// pass and shared memory above ~128 KB per SM starves the L1 the gathers need.
// So each CTA is one group of kPSeg threads (one warp per warp block), several
// CTAs per SM, a few KB of shared memory for the transposes and cone epilogues.
#pragma once

#include <cmath>
#include <cstdint>

#include "cf_common.h"

namespace cf {
namespace pass {

#ifndef CF_TMA
#define CF_TMA 0                   // 1: producer-warp TMA ring; 0: direct coalesced loads (measured faster)
#endif
#ifndef CF_UNROLL
#define CF_UNROLL 3
#endif
#ifndef CF_MINB
#define CF_MINB 6                  // (direct engine) resident CTAs per SM the registers are sized for
#endif
#ifndef CF_STAGES
#define CF_STAGES 4                // (TMA engine) ring depth, all groups
#endif
#ifndef CF_GROUPS
#define CF_GROUPS 2                // (TMA engine) compute groups per CTA
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
constexpr int kPCap = CF_PCAP;     // nonzeros per tile
constexpr int kPSeg = CF_PSEG;     // segments per tile (== threads of a compute group)
constexpr int kMaxDiag = 256;      // longest segment inside a normal tile (longer ones get their own tile)
constexpr int kUnroll = CF_UNROLL; // independent gathers in flight per thread
constexpr int kComputeWarps = kPSeg / 32;      // per group
constexpr int kComputeThreads = kPSeg;         // per group
#if CF_TMA
constexpr int kGroups = CF_GROUPS; // group g consumes the CTA's tiles i = g, g+kGroups, ...
constexpr int kStages = CF_STAGES;
constexpr int kPThreads = kGroups * (kComputeThreads + 32);   // + one producer warp per group
constexpr int kMinBlocks = 1;
static_assert(kStages % kGroups == 0, "a ring slot must be reused by the same compute group (mbarrier parity)");
#else
constexpr int kGroups = 1;
constexpr int kPThreads = kComputeThreads;
constexpr int kMinBlocks = CF_MINB;
#endif
constexpr int kLongChunk = kComputeWarps * 128;   // long tiles: products buffered per chunk (in the vals buffer)
constexpr int kFvTab = 256;
constexpr int kPlPermBits = 5, kPlLenBits = 9;
static_assert(kMaxDiag < (1 << kPlLenBits), "segment length must fit pl");

#if CF_TMA
struct alignas(16) Stage {
    int32_t meta[4];                    // s0, nseg, k0, len (written by the producer)
    int32_t meta2[4];                   // normal (1) / long (0) tile
    int32_t idx[kPCap + 8];
    double val[kPCap + 4];
    uint32_t pl[kPSeg + 4];
};
#endif

struct Smem {
#if CF_TMA
    Stage st[kStages];
    alignas(8) uint64_t full[kStages];
    alignas(8) uint64_t empty[kStages];
#endif
    double fvtab[kFvTab];               // 1/(1+cnt) for small column counts (uv.py:82)
    double wacc[kGroups][kPSeg];        // rank -> natural transpose of the sums (warp-private slices)
    int32_t wcnt[kGroups][kPSeg];
    double red[kGroups][32];
    double vals[kGroups * kComputeWarps][4][32];  // epilogue vectors of a warp block (cp.async); long tiles: products
    double cscr[kGroups][4][kPSeg];     // cone epilogue only: x+, w, delta, delta+ (last member)
};
static_assert(sizeof(((Smem*)0)->vals) / kGroups >= kLongChunk * sizeof(double), "long-tile buffer");

constexpr size_t kSmemBytes = sizeof(Smem);
// policies without a cone epilogue do not allocate the cone scratch
constexpr size_t kSmemBytesNoCones = offsetof(Smem, cscr);

// Staged tiles (the latency-bound Wide/Medium dispatch of the direct engine):
// the whole tile's idx/val are copied to shared memory with 16-byte cp.async at
// tile start, so a lane pays one DRAM round trip per tile instead of one per
// batch of diagonals. Placed after the full Smem.
struct alignas(16) TileStage {
    int32_t idx[kPCap + 8];
    double val[kPCap + 4];
};
template <class P>
constexpr size_t smem_bytes() {
    return (P::kStaged && !CF_TMA) ? kSmemBytes + sizeof(TileStage)
                                   : (P::kGroupEpilogue ? kSmemBytes : kSmemBytesNoCones);
}

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

// Epilogue vectors of one segment (natural order), copied global -> shared by
// cp.async at block start (no registers held while the gathers are in flight).
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
// Programmatic dependent launch (sm_90+): a kernel launched with
// cudaLaunchAttributeProgrammaticStreamSerialization may start while its
// predecessor drains; pdl_wait() blocks until the predecessor has completed and
// its writes are visible (a no-op without the attribute). pdl_trigger() lets
// the successor launch once every CTA of this grid has triggered or exited.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

// compute group of the calling thread and its thread index inside the group
#if CF_TMA
__device__ __forceinline__ int group_id() { return (int)threadIdx.x / kComputeThreads; }
__device__ __forceinline__ int group_tid() { return (int)threadIdx.x % kComputeThreads; }
// named barrier of the caller's compute group (ids 1..kGroups; 0 is __syncthreads)
__device__ __forceinline__ void group_sync() {
    asm volatile("bar.sync %0, %1;" ::"r"(1 + group_id()), "n"(kComputeThreads) : "memory");
}
#else
__device__ __forceinline__ int group_id() { return 0; }
__device__ __forceinline__ int group_tid() { return (int)threadIdx.x; }
__device__ __forceinline__ void group_sync() { __syncthreads(); }
#endif

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

__device__ __forceinline__ void cp_async8(double* dst, const double* src, uint64_t pol) {
    asm volatile("cp.async.ca.shared.global.L2::cache_hint [%0], [%1], 8, %2;" ::"r"(smem_addr(dst)), "l"(src),
                 "l"(pol)
                 : "memory");
}
__device__ __forceinline__ void cp_async16(void* dst, const void* src, uint64_t pol) {
    asm volatile("cp.async.cg.shared.global.L2::cache_hint [%0], [%1], 16, %2;" ::"r"(smem_addr(dst)), "l"(src),
                 "l"(pol)
                 : "memory");
}
// 16-byte-aligned superset copy of [first, first + count) into dst by the calling CTA's
// threads; element 0 lands at dst + ((uintptr_t)first & 15) bytes
template <class T>
__device__ __forceinline__ void stage_span(void* dst, const T* first, int count, uint64_t pol) {
    if (count <= 0) return;
    const uintptr_t a = (uintptr_t)first & ~(uintptr_t)15u;
    const uintptr_t e = ((uintptr_t)(first + count) + 15u) & ~(uintptr_t)15u;
    const int chunks = (int)((e - a) >> 4);
    for (int c = threadIdx.x; c < chunks; c += blockDim.x)
        cp_async16(static_cast<char*>(dst) + 16 * c, reinterpret_cast<const char*>(a) + 16 * c, pol);
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_group 0;" ::: "memory"); }

// Tile table: tb[t] = {first segment, first nonzero, normal (1) / long (0), 0};
// tile t spans [tb[t].x, tb[t+1].x) segments and [tb[t].y, tb[t+1].y) nonzeros.
struct Tiles {
    const int4* tb;
    int32_t n_tiles;
    int32_t stageable = 1;   // every tile fits a TileStage (cut at kPCap nonzeros)
};

// The JDS layout of a pass: idx/val in warp-local jagged-diagonal order inside
// every normal tile (canonical order inside long tiles); pl per segment
// position = local segment of rank r in the warp block | its length << 5 |
// the block's first nonzero (tile-relative) << 14.
struct Jds {
    const int32_t* idx;
    const double* val;
    const uint32_t* pl;
    int64_t n_idx = 0;     // entries of idx/val (bounds of the checked build)
    int64_t g_len = 0;     // length of the gathered vector (bounds of the checked build)
};

// ---------------------------------------------------------------- the engine
// P (the pass policy) provides (device):
//   const double* gvec() const                 gathered operand
//   static constexpr int kVals                 epilogue vectors per segment (<= 4)
//   void load_async(int s, double* slot) const cp.async vector f of segment s (global index) to slot[32 f]
//   bool carry_in() const; double carry(int s) const   starting value of a segment's sum
//   static constexpr int kUnroll               gathers in flight per thread
//   static constexpr int kMinBlocks            resident CTAs per SM the registers are sized for
//   static constexpr bool kStaged              (direct engine) stage each tile's idx/val in shared memory
//   static constexpr bool kGroupEpilogue       epilogue needs all segments of the tile at once (cones)
//   void check(double a, int j, double g)      per-nonzero hook (report finiteness)
//   void segment(Smem&, int tile, int s0, int q, int cnt, double acc, const Vals&)
//                                              epilogue of local segment q (natural order)
//   void group(Smem&, int tile, int s0, int nseg)   (kGroupEpilogue) after a group barrier
//   void finish(Smem&)                         compute threads, after the last tile

// rank r's pl entry -> its length, and the block's first nonzero (from rank 0)
__device__ __forceinline__ int pl_len(uint32_t pr) { return (int)((pr >> kPlPermBits) & ((1u << kPlLenBits) - 1u)); }
__device__ __forceinline__ int pl_start(uint32_t pr) { return (int)(pr >> (kPlPermBits + kPlLenBits)); }

// idx/val of diagonals [k, k+U) of the caller's warp block; pos advances past them
template <int U>
__device__ __forceinline__ void load_batch(const Jds& L, int (&nj)[U], double (&nv)[U], int& pos, int mylen, int k,
                                           uint64_t pf) {
#pragma unroll
    for (int u = 0; u < U; ++u) {
        const bool ok = mylen > k + u;
        if (ok) CF_DASSERT(pos >= 0 && pos < L.n_idx);
        nj[u] = ok ? ld_first(L.idx + pos, pf) : 0;
        nv[u] = ok ? ld_first(L.val + pos, pf) : 0.0;
        if (ok) CF_DASSERT(nj[u] >= 0 && nj[u] < L.g_len);
        pos += __popc(__ballot_sync(0xffffffffu, ok));   // width of diagonal k+u
    }
}

// long tile: one segment [k0, k0+len) in canonical order; the products of a
// chunk are buffered and summed in order by thread 0
template <class P>
__device__ __forceinline__ void long_tile(P& p, Smem& sm, const Jds& L, int tile, int s0, int k0, int len) {
    const int gt = group_tid(), grp = group_id();
    const uint64_t pf = pol_first(), pl_ = pol_last();
    const double* __restrict__ g = p.gvec();
    double* lacc = sm.wacc[grp];
    double* lbuf = &sm.vals[grp * kComputeWarps][0][0];
    Vals vv{};
    group_sync();   // the previous tile's epilogue vectors (same buffer) are consumed
    if (gt == 0) {
        if (P::kVals > 0) {
            p.load_async(s0, &lacc[1]);
            cp_async_commit();
            cp_async_wait_all();
            for (int f = 0; f < P::kVals; ++f) vv.v[f] = lacc[1 + 32 * f];
        }
        lacc[0] = p.carry_in() ? p.carry(s0) : 0.0;
    }
    group_sync();
    for (int c0 = 0; c0 < len; c0 += kLongChunk) {
        const int cl = min(kLongChunk, len - c0);
        for (int e = gt; e < cl; e += kComputeThreads) {
            CF_DASSERT(k0 + c0 + e < L.n_idx);
            const int jj = ld_first(L.idx + k0 + c0 + e, pf);
            CF_DASSERT(jj >= 0 && jj < L.g_len);
            const double a = ld_first(L.val + k0 + c0 + e, pf);
            const double gj = ld_gather(g + jj, pl_);
            p.check(a, jj, gj);
            lbuf[e] = __dmul_rn(a, gj);
        }
        group_sync();
        if (gt == 0) {
            double acc = lacc[0];
            for (int e = 0; e < cl; ++e) acc = __dadd_rn(acc, lbuf[e]);
            lacc[0] = acc;
        }
        group_sync();
    }
    if (gt == 0) p.segment(sm, tile, s0, 0, len, lacc[0], vv);
    group_sync();
}

#if CF_TMA
// PTX: mbarriers and TMA bulk copies (producer-warp ring)
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

__device__ __forceinline__ void issue_tile(const Jds& L, int4 lo, int4 hi, Stage& st, uint64_t* bar, uint64_t pol) {
    const int s0 = lo.x, nseg = hi.x - lo.x, k0 = lo.y, len = hi.y - lo.y, normal = lo.z;
    st.meta[0] = s0;
    st.meta[1] = nseg;
    st.meta[2] = k0;
    st.meta[3] = len;
    st.meta2[0] = normal;
    if (!normal) {  // long tile: nothing staged (streamed by the consumers)
        mbar_expect_tx(bar, 0);
        return;
    }
    const uint32_t total =
        span_bytes(L.idx + k0, len) + span_bytes(L.val + k0, len) + span_bytes(L.pl + s0, nseg);
    mbar_expect_tx(bar, total);
    copy_span(st.idx, L.idx + k0, len, bar, pol);
    copy_span(st.val, L.val + k0, len, bar, pol);
    copy_span(st.pl, L.pl + s0, nseg, bar, pol);
}

// Per compute group (kPSeg threads) one producer warp copies a future tile's
// idx/val/pl into the group's slots of a kStages ring with cp.async.bulk (TMA
// 1D; full[s] mbarrier, L2 evict-first); the group's warps consume (empty[s]).
// Groups alternate tiles. Inside a tile, warp w takes warp block w.
template <class P>
__global__ void __launch_bounds__(kPThreads, 1) k_pass(const P p0, const Jds L, const Tiles T, const int32_t* done) {
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
    pdl_wait();
    pdl_trigger();
    if (done && *done) return;

    if (warp >= kGroups * kComputeWarps) {
        // ------------------------------------------------ producers: warp kGroups*kComputeWarps + g feeds group g
        const int pg = warp - kGroups * kComputeWarps;
        if (lane == 0) {
            const uint64_t pf = pol_first();
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
    const double* __restrict__ g = p.gvec();
    const int grp = group_id();
    const int gt = group_tid();
    const int gw = gt >> 5;      // warp within the group = warp block of the tile
    double* wacc = sm.wacc[grp] + gw * 32;
    int32_t* wcnt = sm.wcnt[grp] + gw * 32;
    double* slot = &sm.vals[grp * kComputeWarps + gw][0][lane];
    constexpr int U = P::kUnroll;
    for (int i = grp; i < my; i += kGroups) {
        const int s = i % kStages;
        Stage& st = sm.st[s];
        mbar_wait(&sm.full[s], (uint32_t)((i / kStages) & 1));
        const int s0 = st.meta[0], nseg = st.meta[1], k0 = st.meta[2], len = st.meta[3];
        const int tile = (int)blockIdx.x + i * G;
        if (st.meta2[0]) {
            const int nb = min(32, nseg - gw * 32);   // segments of this warp block
            if (nb > 0) {
                const bool nat = lane < nb;             // natural segment gw*32 + lane exists
                const int seg = s0 + gw * 32 + lane;
                if (P::kVals > 0) {
                    if (nat) p.load_async(seg, slot);
                    cp_async_commit();
                }
                const int32_t* ib = st.idx + lead_of(L.idx + k0);
                const double* vb = st.val + lead_of(L.val + k0);
                const uint32_t pr = nat ? st.pl[lead_of(L.pl + s0) + gw * 32 + lane] : 0u;
                const int q = (int)(pr & 31u);          // local segment (within the block) of rank r
                const int mylen = pl_len(pr);
                const int mlen = __shfl_sync(0xffffffffu, mylen, 0);   // rank 0 is the longest
                int pos = __shfl_sync(0xffffffffu, pl_start(pr), 0) + lane;
                // rank r's own carry (no shuffle: the load's latency hides behind the gathers)
                double acc = (p.carry_in() && nat) ? p.carry(s0 + gw * 32 + q) : 0.0;
                for (int k = 0; k < mlen; k += U) {
                    // indices first; the values are read from shared memory only
                    // when the gathers land (keeps U fewer doubles live)
                    const int p0 = pos;
                    int jj[U];
                    double gv[U];
#pragma unroll
                    for (int u = 0; u < U; ++u) {
                        const bool ok = mylen > k + u;
                        jj[u] = ok ? ib[pos] : 0;
                        pos += __popc(__ballot_sync(0xffffffffu, ok));   // width of diagonal k+u
                    }
#pragma unroll
                    for (int u = 0; u < U; ++u)
                        gv[u] = (mylen > k + u) ? ld_gather(g + jj[u], pol_last()) : 0.0;
                    int p1 = p0;
#pragma unroll
                    for (int u = 0; u < U; ++u) {
                        const bool ok = mylen > k + u;
                        if (ok) {
                            const double a = vb[p1];
                            p.check(a, jj[u], gv[u]);
                            acc = __dadd_rn(acc, __dmul_rn(a, gv[u]));
                        }
                        p1 += __popc(__ballot_sync(0xffffffffu, ok));
                    }
                }
                // rank -> natural order inside the warp (a segment's count is its length)
                if (nat) {
                    wacc[q] = acc;
                    wcnt[q] = mylen;
                }
                Vals vv{};
                if (P::kVals > 0) {
                    cp_async_wait_all();
#pragma unroll
                    for (int f = 0; f < P::kVals; ++f) vv.v[f] = slot[32 * f];
                }
                __syncwarp();
                if (nat) p.segment(sm, tile, s0, gw * 32 + lane, wcnt[lane], wacc[lane], vv);
                __syncwarp();
            }
        } else {
            long_tile(p, sm, L, tile, s0, k0, len);
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

#else
// load_batch from a staged tile (positions relative to the staged arrays)
template <int U>
__device__ __forceinline__ void load_batch_smem(const int32_t* ib, const double* vb, int (&nj)[U], double (&nv)[U],
                                                int& pos, int mylen, int k) {
#pragma unroll
    for (int u = 0; u < U; ++u) {
        const bool ok = mylen > k + u;
        if (ok) CF_DASSERT(pos >= 0 && pos < kPCap + 8);
        nj[u] = ok ? ib[pos] : 0;
        nv[u] = ok ? vb[pos] : 0.0;
        pos += __popc(__ballot_sync(0xffffffffu, ok));   // width of diagonal k+u
    }
}

// Each warp walks its warp blocks (block gw of tiles blockIdx.x, +G, ...):
// pl -> idx/val of U diagonals -> U gathers -> sequential sums, then the
// natural-order epilogue. Many resident warps hide the dependent chain.
template <class P>
__global__ void __launch_bounds__(kPThreads, P::kMinBlocks) k_pass(const P p0, const Jds L, const Tiles T,
                                                               const int32_t* done) {
    P p = p0;  // per-thread mutable copy (report accumulators live in registers)
    extern __shared__ __align__(128) unsigned char smem_raw[];
    Smem& sm = *reinterpret_cast<Smem*>(smem_raw);
    const int G = gridDim.x;
    const int lane = threadIdx.x & 31;
    const int gt = threadIdx.x;
    const int gw = gt >> 5;      // warp = warp block of the tile
    for (int c = gt; c < kFvTab; c += kPThreads) sm.fvtab[c] = 1.0 / (1.0 + (double)c);
    __syncthreads();
    pdl_wait();   // everything above is independent of the previous kernel
    pdl_trigger();
    if (done && *done) return;
    constexpr int U = P::kUnroll;
    for (int tile = blockIdx.x; tile < T.n_tiles; tile += G) {
        const int4 lo = __ldg(T.tb + tile), hi = __ldg(T.tb + tile + 1);
        const int s0 = lo.x, nseg = hi.x - lo.x, k0 = lo.y, len = hi.y - lo.y;
        CF_DASSERT(nseg >= 0 && len >= 0 && k0 >= 0 && (int64_t)k0 + len <= L.n_idx);
        CF_DASSERT(!lo.z || (nseg <= kPSeg && (!P::kStaged || len <= kPCap)));
        if (lo.z) {
            const int32_t* ib = nullptr;
            const double* vb = nullptr;
            if constexpr (P::kStaged) {
                TileStage& ts = *reinterpret_cast<TileStage*>(smem_raw + kSmemBytes);
                __syncthreads();   // the previous tile's readers are done with the stage
                stage_span(ts.idx, L.idx + k0, len, pol_first());
                stage_span(ts.val, L.val + k0, len, pol_first());
                cp_async_commit();
                ib = ts.idx + (((uintptr_t)(L.idx + k0) & 15u) >> 2);
                vb = ts.val + (((uintptr_t)(L.val + k0) & 15u) >> 3);
            }
            const int nb = min(32, nseg - gw * 32);   // segments of this warp block
            const bool nat = lane < nb;                 // natural segment gw*32 + lane exists
            const int seg = s0 + gw * 32 + lane;
            const uint32_t pr =
                (nb > 0 && nat) ? (uint32_t)ld_first(reinterpret_cast<const int32_t*>(L.pl) + seg, pol_first()) : 0u;
            if constexpr (P::kStaged) {
                cp_async_wait_all();
                __syncthreads();
            }
            if (nb > 0) {
                double* slot = &sm.vals[gw][0][lane];
                if (P::kVals > 0) {
                    if (nat) p.load_async(seg, slot);
                    cp_async_commit();
                }
                const int q = (int)(pr & 31u);          // local segment (within the block) of rank r
                const int mylen = pl_len(pr);
                const int mlen = __shfl_sync(0xffffffffu, mylen, 0);   // rank 0 is the longest
                int pos = (P::kStaged ? 0 : k0) + __shfl_sync(0xffffffffu, pl_start(pr), 0) + lane;
                // rank r's own carry (no shuffle: the load's latency hides behind the gathers)
                double acc = (p.carry_in() && nat) ? p.carry(s0 + gw * 32 + q) : 0.0;
                const double* __restrict__ g = p.gvec();
                for (int k = 0; k < mlen; k += U) {
                    int nj[U];
                    double nv[U], gv[U];
                    if constexpr (P::kStaged)
                        load_batch_smem<U>(ib, vb, nj, nv, pos, mylen, k);
                    else
                        load_batch<U>(L, nj, nv, pos, mylen, k, pol_first());
#pragma unroll
                    for (int u = 0; u < U; ++u) {
                        if (mylen > k + u) CF_DASSERT(nj[u] >= 0 && nj[u] < L.g_len);
                        gv[u] = (mylen > k + u) ? ld_gather(g + (uint32_t)nj[u], pol_last()) : 0.0;
                    }
#pragma unroll
                    for (int u = 0; u < U; ++u) {
                        if (mylen > k + u) p.check(nv[u], nj[u], gv[u]);
                        // no predicate: a lane past its segment adds 0.0*0.0 = +0.0, which leaves acc
                        // unchanged (a sum that starts at +0.0 is never -0.0 in round-to-nearest)
                        acc = __dadd_rn(acc, __dmul_rn(nv[u], gv[u]));
                    }
                }
                // rank -> natural order inside the warp (a segment's count is its length)
                double* wacc = sm.wacc[0] + gw * 32;
                int32_t* wcnt = sm.wcnt[0] + gw * 32;
                if (nat) {
                    wacc[q] = acc;
                    wcnt[q] = mylen;
                }
                Vals vv{};
                if (P::kVals > 0) {
                    cp_async_wait_all();
#pragma unroll
                    for (int f = 0; f < P::kVals; ++f) vv.v[f] = slot[32 * f];
                }
                __syncwarp();
                if (nat) p.segment(sm, tile, s0, gw * 32 + lane, wcnt[lane], wacc[lane], vv);
                __syncwarp();
            }
        } else {
            long_tile(p, sm, L, tile, s0, k0, len);
        }
        if (P::kGroupEpilogue) {
            __syncthreads();
            p.group(sm, tile, s0, nseg);
            __syncthreads();   // cone scratch is rewritten by the next tile
        }
    }
    p.finish(sm);
}
#endif

}  // namespace pass
}  // namespace cf
