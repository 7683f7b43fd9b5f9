// Persistent jagged-diagonal tile engine for the sparse passes (sm_100a).
//
// A pass walks one compressed layout (CSR panels for the row pass, CSC for the
// column pass) tile by tile. A tile is a run of <= kPSeg segments (rows or
// columns) with <= kPCap nonzeros, cut on the host (cf_setup.cu), or one
// segment longer than kMaxDiag ("long tile").
//
// Inside a normal tile the segments are RANKED BY LENGTH over the whole tile
// (descending, stable) and every WARP BLOCK of 32 consecutive ranks is stored in
// jagged-diagonal order (k_build_jds): the k-th nonzero of rank r sits at
//   base + start_w + sum_{j<k} width_j + (r mod 32),
// width_j = ranks of the block longer than j, start_w = the block's offset, a
// multiple of 32 elements, so a full diagonal is one aligned 128-byte line of idx
// and two of val. Ranking over the tile makes the 32 lengths of a block nearly
// equal, so nearly every diagonal is full: 0.10 L1TEX requests per nonzero for
// idx/val instead of 0.20 with per-block ranking (profiles/r02_probes.md).
// pl[rank] = local segment | length << 8 | start_w << 17, so each lane knows its
// segment, its length and its block's offset. While k is below the block's
// shortest length every diagonal is 32 wide (constant offsets); the narrower
// diagonals after it take their offsets from warp ballots.
//   * lane r owns one segment: it loads idx/val of its nonzeros straight from
//     global memory (L1 no-allocate, L2 evict-first), gathers g[idx] (kUnroll
//     independent loads in flight, L2 evict-last) and sums the products
//     SEQUENTIALLY in canonical order — np.bincount's order (uv.py:10-12),
//     bit-identical;
//   * the sums go through shared memory back to natural segment order, so the
//     epilogue runs in natural order with coalesced vector loads and stores. The
//     large passes hand the sums over through mbarriers without a CTA barrier
//     (the deferred flow, see k_pass) and load the epilogue vectors straight into
//     registers; the staged small passes and the cone group epilogue use one CTA
//     barrier per tile and cp.async the vectors at tile start.
// Measured (profiles/r01_probes.md, r02_probes.md): a random fp64 gather costs one
// L1TEX->L2 request, ~1 per SM-cycle, and that request port is the bound; TMA
// staging and TMA gathers were slower; shared memory above ~128 KB per SM starves
// the L1 the gathers need. So each CTA is one group of kPSeg threads (one warp per
// warp block), several CTAs per SM, a few KB of shared memory.
#pragma once

#include <cmath>
#include <cstdint>

#include "cf_common.h"

namespace cf {
namespace pass {

#ifndef CF_UNROLL
#define CF_UNROLL 4
#endif
#ifndef CF_MINB
#define CF_MINB 5                  // resident CTAs per SM the registers are sized for (6 spills with the deferred pipeline)
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
#ifndef CF_DEFERRED
#define CF_DEFERRED 1              // deferred-epilogue pipeline (mbarriers) instead of one CTA barrier per tile
#endif
#ifndef CF_FULL_DIAG
#define CF_FULL_DIAG 1             // full-width diagonals without predicates (block_sums)
#endif
#ifndef CF_FULL_UNROLL
#define CF_FULL_UNROLL 0           // diagonals per batch on the full-width part (0: the policy's kUnroll)
#endif
#ifndef CF_PRED_TAIL
#define CF_PRED_TAIL 1             // predicated loads/gathers/adds on the narrow diagonals (block_sums)
#endif
#ifndef CF_TAIL_UNROLL
#define CF_TAIL_UNROLL 0           // diagonals per batch on the narrow part (0: the policy's kUnroll)
#endif
#ifndef CF_EPI_DIRECT
#define CF_EPI_DIRECT 1            // deferred flow: epilogue vectors loaded straight into registers at the epilogue (+1 %; 0: cp.async at hand-in)
#endif
#ifndef CF_BULK_PREFETCH
#define CF_BULK_PREFETCH 0         // L2-prefetch the idx/val/pl of the tile this many rounds ahead (measured slower)
#endif
constexpr int kPCap = CF_PCAP;     // nonzeros per tile
constexpr int kPSeg = CF_PSEG;     // segments per tile (== threads of a CTA)
constexpr int kMaxDiag = 256;      // longest segment inside a normal tile (longer ones get their own tile)
constexpr int kUnroll = CF_UNROLL; // independent gathers in flight per thread
constexpr int kComputeWarps = kPSeg / 32;
constexpr int kComputeThreads = kPSeg;
constexpr int kGroups = 1;
constexpr int kPThreads = kComputeThreads;
constexpr int kMinBlocks = CF_MINB;
// JDS slack per tile (cf_common.h kTilePad): every warp block starts at a multiple of 32
// elements, and so does every tile (host: base_t = align32(k0_t + kTilePad * t))
static_assert(kTilePad >= kComputeWarps * 31 + 31, "tile padding must cover the block alignment");
constexpr int kLongChunk = kComputeWarps * 128;   // long tiles: products buffered per chunk (in the vals buffer)
constexpr int kFvTab = 256;
constexpr int kPlLenBits = 9;   // pl = local segment | length << kPlPermBits | block start << (kPlPermBits + 9)
static_assert(kPSeg <= (1 << kPlPermBits), "tile-local segment must fit pl");
static_assert(kMaxDiag < (1 << kPlLenBits), "segment length must fit pl");

// Laid out so each flow allocates only a prefix: staged tiles without cones stop after vals,
// the deferred flow after the third sum buffer and its mbarriers, the cone group epilogue
// takes everything. Less shared memory leaves more L1 for the gathers in flight.
struct alignas(16) Smem {   // 16-byte multiple: a TileStage follows the allocated prefix
    double fvtab[kFvTab];               // 1/(1+cnt) for small column counts (uv.py:82)
    double wacc[2][kPSeg];              // rank -> natural transpose of the sums (buffers 0, 1)
    int32_t wcnt[2][kPSeg];
    double red[kGroups][32];
    double vals[kComputeWarps][4][32];  // epilogue vectors of a warp block (cp.async); long tiles: products
    double wacc2[kPSeg];                // deferred flow only: the third sum buffer
    int32_t wcnt2[kPSeg];
    alignas(8) uint64_t full[3];        // deferred flow only: tile sums of a buffer handed in by every warp
    alignas(16) double cscr[kGroups][4][kPSeg];   // cone group epilogue only: x+, w, delta, delta+
};
static_assert(offsetof(Smem, wacc2) % 16 == 0 && offsetof(Smem, cscr) % 16 == 0, "TileStage alignment");
static_assert(sizeof(((Smem*)0)->vals) >= kLongChunk * sizeof(double), "long-tile buffer");
__device__ __forceinline__ double* wacc_buf(Smem& sm, int b) { return b < 2 ? sm.wacc[b] : sm.wacc2; }
__device__ __forceinline__ int32_t* wcnt_buf(Smem& sm, int b) { return b < 2 ? sm.wcnt[b] : sm.wcnt2; }

constexpr size_t kSmemBytes = sizeof(Smem);
// prefixes: staged tiles without cones stop after vals; the deferred flow after the mbarriers;
// the cone group epilogue takes the whole struct
constexpr size_t kSmemBytesStaged = offsetof(Smem, wacc2);
constexpr size_t kSmemBytesDeferred = (offsetof(Smem, full) + sizeof(((Smem*)0)->full) + 15) / 16 * 16;

// Staged tiles (the latency-bound Wide/Medium dispatch): the whole tile's idx/val
// span (with its alignment slack) is copied to shared memory with 16-byte cp.async
// at tile start, so a lane pays one DRAM round trip per tile instead of one per batch
// of diagonals. Placed after the barrier flow's prefix of Smem.
struct alignas(16) TileStage {   // staged tiles are block-ranked and packed: no alignment slack
    int32_t idx[kPCap + 40];
    double val[kPCap + 40];
};
// offset of the TileStage (staged policies): after the prefix the flow uses
template <class P>
__host__ __device__ constexpr size_t stage_offset() {
    return P::kGroupEpilogue ? kSmemBytes : kSmemBytesStaged;
}
template <class P>
constexpr size_t smem_bytes() {
    return P::kStaged ? stage_offset<P>() + sizeof(TileStage)
                      : (P::kGroupEpilogue ? kSmemBytes : kSmemBytesDeferred);
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

// compute group of the calling thread (one group per CTA) and its index inside the group
__device__ __forceinline__ int group_id() { return 0; }
__device__ __forceinline__ int group_tid() { return (int)threadIdx.x; }
__device__ __forceinline__ void group_sync() { __syncthreads(); }

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
// predicated forms returning 0 where !ok: one zeroing move plus a predicated load into
// the same register (a C++ `ok ? ld : 0` becomes a load into a temporary and a select)
__device__ __forceinline__ int32_t ld_first_if(const int32_t* p, uint64_t pol, bool ok) {
    int32_t v;
    asm volatile("{\n .reg .pred q;\n setp.ne.u32 q, %3, 0;\n mov.b32 %0, 0;\n"
                 " @q ld.global.nc.L1::no_allocate.L2::cache_hint.s32 %0, [%1], %2;\n}"
                 : "=&r"(v) : "l"(p), "l"(pol), "r"((unsigned)ok));
    return v;
}
__device__ __forceinline__ double ld_first_if(const double* p, uint64_t pol, bool ok) {
    double v;
    asm volatile("{\n .reg .pred q;\n setp.ne.u32 q, %3, 0;\n mov.b64 %0, 0;\n"
                 " @q ld.global.nc.L1::no_allocate.L2::cache_hint.f64 %0, [%1], %2;\n}"
                 : "=&d"(v) : "l"(p), "l"(pol), "r"((unsigned)ok));
    return v;
}
__device__ __forceinline__ double ld_gather_if(const double* p, uint64_t pol, bool ok) {
    double v;
    asm volatile("{\n .reg .pred q;\n setp.ne.u32 q, %3, 0;\n mov.b64 %0, 0;\n"
#if CF_GATHER_NOALLOC
                 " @q ld.global.nc.L1::no_allocate.L2::cache_hint.f64 %0, [%1], %2;\n}"
#else
                 " @q ld.global.nc.L2::cache_hint.f64 %0, [%1], %2;\n}"
#endif
                 : "=&d"(v) : "l"(p), "l"(pol), "r"((unsigned)ok));
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
// L2 prefetch of a byte span by the TMA unit (one instruction, no L1TEX requests); the span
// is widened to 16-byte boundaries (the buffers carry 64 bytes of slack)
__device__ __forceinline__ void bulk_prefetch_l2(const void* first, int64_t bytes) {
    if (bytes <= 0) return;
    const uintptr_t a = (uintptr_t)first & ~(uintptr_t)15u;
    const uintptr_t e = ((uintptr_t)first + (uintptr_t)bytes + 15u) & ~(uintptr_t)15u;
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(a), "r"((uint32_t)(e - a)) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_group 0;" ::: "memory"); }

// mbarriers: the deferred-epilogue pipeline of k_pass (warps hand a tile's sums to the
// warps that run its epilogue without a CTA-wide barrier)
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];" ::"r"(smem_addr(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n"
        ".reg .pred P1;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.acquire.cta.shared::cta.b64 P1, [%0], %1;\n"
        "@!P1 bra WAIT_%=;\n"
        "}\n" ::"r"(smem_addr(bar)),
        "r"(parity)
        : "memory");
}

// Tile table: tb[t] = {first segment, first canonical nonzero, normal (1) / long (0),
// JDS base}; tile t spans [tb[t].x, tb[t+1].x) segments, [tb[t].y, tb[t+1].y) canonical
// nonzeros, and its jagged-diagonal copy starts at tb[t].w (a multiple of 32 elements;
// long tiles: the canonical order there).
struct Tiles {
    const int4* tb;
    int32_t n_tiles;
    int32_t stageable = 1;   // every tile fits a TileStage (cut at kPCap nonzeros)
};

// The JDS layout of a pass: idx/val in jagged-diagonal order per warp block of
// tile-ranked segments (canonical order inside long tiles); pl per rank position =
// tile-local segment of the rank | its length << 8 | the block's first element
// (tile-relative, a multiple of 32) << 17.
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

// The sums of warp block gw of a normal tile (ranks [32 gw, 32 gw + 32)): pl -> idx/val
// of U diagonals -> U gathers -> sequential sums; each rank's sum and count go to
// wacc/wcnt at its tile-local segment (natural order).
template <class P>
__device__ __forceinline__ void block_sums(P& p, const Jds& L, const int32_t* ib, const double* vb, int s0, int kj,
                                           int gw, int lane, int nb, uint32_t pr, double* wacc, int32_t* wcnt) {
    constexpr int U = P::kUnroll;
    const bool has = lane < nb;
    const int q = (int)(pr & ((1u << kPlPermBits) - 1u));   // tile-local segment of my rank
    const int mylen = pl_len(pr);
    const int mlen = __shfl_sync(0xffffffffu, mylen, 0);   // rank 32 gw is the block's longest
    int pos = (P::kStaged ? 0 : kj) + __shfl_sync(0xffffffffu, pl_start(pr), 0) + lane;
    // my segment's carry (no shuffle: the load's latency hides behind the gathers)
    double acc = (p.carry_in() && has) ? p.carry(s0 + q) : 0.0;
    const double* __restrict__ g = p.gvec();
    int k = 0;
#if CF_FULL_DIAG
    // Full diagonals: the ranks are sorted by length, so while k is below the block's
    // shortest length (rank 31; 0 for a partial block) every diagonal is 32 wide and
    // lane l's element k sits at pos + 32 k: constant offsets, no predicates, no ballots.
    constexpr int UF = CF_FULL_UNROLL > 0 ? CF_FULL_UNROLL : U;
    const int mmin = __shfl_sync(0xffffffffu, mylen, 31);
    if (mmin >= UF) {
        const uint64_t pf = pol_first(), plast = pol_last();
        for (; k + UF <= mmin; k += UF) {
            int nj[UF];
            double nv[UF], gv[UF];
#pragma unroll
            for (int u = 0; u < UF; ++u) {
                if constexpr (P::kStaged) {
                    CF_DASSERT(pos + 32 * u < kPCap + 8);
                    nj[u] = ib[pos + 32 * u];
                    nv[u] = vb[pos + 32 * u];
                } else {
                    CF_DASSERT(pos + 32 * u < L.n_idx);
                    nj[u] = ld_first(L.idx + (pos + 32 * u), pf);
                    nv[u] = ld_first(L.val + (pos + 32 * u), pf);
                }
            }
#pragma unroll
            for (int u = 0; u < UF; ++u) {
                CF_DASSERT(nj[u] >= 0 && nj[u] < L.g_len);
                gv[u] = ld_gather(g + (uint32_t)nj[u], plast);
            }
#pragma unroll
            for (int u = 0; u < UF; ++u) {
                p.check(nv[u], nj[u], gv[u]);
                acc = __dadd_rn(acc, __dmul_rn(nv[u], gv[u]));
            }
            pos += 32 * UF;
        }
    }
#endif
#if CF_PRED_TAIL
    // the rest (diagonals narrower than 32, or all of a partial block): per-lane
    // predicated loads, gathers and adds; the ranks are sorted, so the lanes of
    // diagonal k+u are a prefix and its width is the ballot's popcount
    constexpr int UT = CF_TAIL_UNROLL > 0 ? CF_TAIL_UNROLL : U;
    for (; k < mlen; k += UT) {
        int nj[UT];
        double nv[UT], gv[UT];
#pragma unroll
        for (int u = 0; u < UT; ++u) {
            const bool ok = mylen > k + u;
            if constexpr (P::kStaged) {
                if (ok) CF_DASSERT(pos >= 0 && pos < kPCap + 8);
                nj[u] = ok ? ib[pos] : 0;
                nv[u] = ok ? vb[pos] : 0.0;
            } else {
                if (ok) CF_DASSERT(pos >= 0 && pos < L.n_idx);
                const uint32_t upos = (uint32_t)pos;   // one IMAD.WIDE.U32 per address
                nj[u] = ld_first_if(L.idx + upos, pol_first(), ok);
                nv[u] = ld_first_if(L.val + upos, pol_first(), ok);
            }
            pos += __popc(__ballot_sync(0xffffffffu, ok));   // width of diagonal k+u
        }
#pragma unroll
        for (int u = 0; u < UT; ++u) {
            const bool ok = mylen > k + u;
            if (ok) CF_DASSERT(nj[u] >= 0 && nj[u] < L.g_len);
            gv[u] = ld_gather_if(g + (uint32_t)nj[u], pol_last(), ok);
        }
#pragma unroll
        for (int u = 0; u < UT; ++u) {
            if (mylen > k + u) p.check(nv[u], nj[u], gv[u]);
            acc = __dadd_rn(acc, __dmul_rn(nv[u], gv[u]));   // +0.0 * +0.0 past my segment: acc unchanged
        }
    }
#else
    for (; k < mlen; k += U) {
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
#endif
    if (has) {
        wacc[q] = acc;
        wcnt[q] = mylen;
    }
}

// Each CTA walks its tiles (blockIdx.x, +G, ...); warp gw takes the tile's warp block
// gw. The sums go to natural order through shared memory and lane l of warp gw runs
// the epilogue of natural segment 32 gw + l.
//   * deferred flow (direct loads, per-segment epilogue): no CTA barrier. A warp
//     writes tile i's sums (of rank block (gw + i) mod 8: the blocks rotate, so every
//     warp gets as many long blocks as short ones), then runs the epilogue of tile i-1 once every warp has
//     handed in tile i-1 (mbarrier full[(i-1) % 3]), cp.asyncs tile i's epilogue
//     vectors, and arrives on full[i % 3]. Three sum buffers: a warp writes tile i+2's
//     sums only after waiting on tile i+1, whose arrivals all follow the epilogues of
//     tile i. A slow warp therefore delays the others by up to two tiles, not every tile.
//   * barrier flow (staged tiles, cone group epilogue): one CTA barrier per tile.
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
    constexpr bool kDeferred = CF_DEFERRED && !P::kStaged && !P::kGroupEpilogue;
    for (int c = gt; c < kFvTab; c += kPThreads) sm.fvtab[c] = 1.0 / (1.0 + (double)c);
    if (kDeferred && gt == 0) {
        for (int b = 0; b < 3; ++b) mbar_init(&sm.full[b], kComputeWarps);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    pdl_wait();   // everything above is independent of the previous kernel
    pdl_trigger();
    if (done && *done) return;
    double* slot = &sm.vals[gw][0][lane];
    // deferred flow: the tile whose epilogue is pending (this warp's view)
    int seq = 0;                              // normal tiles handed in so far
    int pv_tile = -1, pv_s0 = 0, pv_nb = 0;
    auto drain = [&]() {                      // run the pending epilogue (deferred flow)
        if (pv_tile < 0) return;
        const int b = (seq - 1) % 3;
        mbar_wait(&sm.full[b], (uint32_t)(((seq - 1) / 3) & 1));
        if (pv_nb > 0) {
            Vals vv{};
#if CF_EPI_DIRECT
            if (P::kVals > 0 && lane < pv_nb) p.load_direct(pv_s0 + gw * 32 + lane, vv);
#else
            if (P::kVals > 0) {
                cp_async_wait_all();
#pragma unroll
                for (int f = 0; f < P::kVals; ++f) vv.v[f] = slot[32 * f];
            }
#endif
            __syncwarp();
            if (lane < pv_nb)
                p.segment(sm, pv_tile, pv_s0, gw * 32 + lane, wcnt_buf(sm, b)[gw * 32 + lane],
                          wacc_buf(sm, b)[gw * 32 + lane], vv);
            __syncwarp();
        }
        pv_tile = -1;
    };
    int buf = 0;   // barrier flow
    for (int tile = blockIdx.x; tile < T.n_tiles; tile += G) {
        const int4 lo = __ldg(T.tb + tile), hi = __ldg(T.tb + tile + 1);
        // x: first segment, y: first canonical nonzero, z: normal/long, w: JDS base (multiple of 32)
        const int s0 = lo.x, nseg = hi.x - lo.x, len = hi.y - lo.y, kj = lo.w;
        CF_DASSERT(nseg >= 0 && len >= 0 && kj >= 0 && (int64_t)kj + len <= L.n_idx && (kj & 31) == 0);
        CF_DASSERT(!lo.z || (nseg <= kPSeg && (!P::kStaged || len <= kPCap)));
        if (CF_BULK_PREFETCH > 0 && !P::kStaged && threadIdx.x == 0) {
            const int nt = tile + CF_BULK_PREFETCH * G;
            if (nt < T.n_tiles) {
                const int4 a = __ldg(T.tb + nt), b = __ldg(T.tb + nt + 1);
                bulk_prefetch_l2(L.idx + a.w, (int64_t)(b.w - a.w) * 4);
                bulk_prefetch_l2(L.val + a.w, (int64_t)(b.w - a.w) * 8);
                bulk_prefetch_l2(L.pl + a.x, (int64_t)(b.x - a.x) * 4);
            }
        }
        const int nb = min(32, nseg - gw * 32);     // ranks (and natural segments) of this warp block
        if (!lo.z) {
            if constexpr (kDeferred) drain();
            long_tile(p, sm, L, tile, s0, kj, len);
        } else if constexpr (kDeferred) {
            // the sums of rank block bw, rotating with the tile sequence: ranking over the tile
            // makes block 0 the longest, so a fixed block per warp would keep one warp behind
            const int bw = (gw + seq) % kComputeWarps;
            const int nbw = min(32, nseg - bw * 32);
            const uint32_t pr =
                lane < nbw ? (uint32_t)ld_first(reinterpret_cast<const int32_t*>(L.pl) + s0 + bw * 32 + lane, pol_first())
                           : 0u;
            const int b = seq % 3;
            if (nbw > 0) block_sums(p, L, nullptr, nullptr, s0, kj, bw, lane, nbw, pr, wacc_buf(sm, b), wcnt_buf(sm, b));
            drain();                                  // the previous tile's epilogue
            if (!CF_EPI_DIRECT && P::kVals > 0 && nb > 0) {
                if (lane < nb) p.load_async(s0 + gw * 32 + lane, slot);   // this tile's epilogue vectors
                cp_async_commit();
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(&sm.full[b]);
            pv_tile = tile;
            pv_s0 = s0;
            pv_nb = nb;
            ++seq;
        } else {
            const int32_t* ib = nullptr;
            const double* vb = nullptr;
            if constexpr (P::kStaged) {
                TileStage& ts = *reinterpret_cast<TileStage*>(smem_raw + stage_offset<P>());
                __syncthreads();   // the previous tile's readers are done with the stage
                // a staged tile is block-ranked and packed: its len elements start at kj
                CF_DASSERT(lo.z == 2 && len <= kPCap);
                stage_span(ts.idx, L.idx + kj, len, pol_first());
                stage_span(ts.val, L.val + kj, len, pol_first());
                cp_async_commit();
                ib = ts.idx + (((uintptr_t)(L.idx + kj) & 15u) >> 2);
                vb = ts.val + (((uintptr_t)(L.val + kj) & 15u) >> 3);
            }
            const uint32_t pr =
                lane < nb ? (uint32_t)ld_first(reinterpret_cast<const int32_t*>(L.pl) + s0 + gw * 32 + lane, pol_first())
                          : 0u;
            if constexpr (P::kStaged) {
                cp_async_wait_all();
                __syncthreads();
            }
            if (nb > 0 && P::kVals > 0) {
                if (lane < nb) p.load_async(s0 + gw * 32 + lane, slot);   // natural segment 32 gw + lane
                cp_async_commit();
            }
            if (nb > 0) block_sums(p, L, ib, vb, s0, kj, gw, lane, nb, pr, sm.wacc[buf], sm.wcnt[buf]);
            Vals vv{};
            if (nb > 0 && P::kVals > 0) {
                cp_async_wait_all();
#pragma unroll
                for (int f = 0; f < P::kVals; ++f) vv.v[f] = slot[32 * f];
            }
            // every rank's sum of this tile is in wacc[buf] (wacc[buf ^ 1] is next); a tile ranked
            // inside its warp blocks (normal flag 2) hands its sums only to its own warp
            if (lo.z == 2)
                __syncwarp();
            else
                __syncthreads();
            if (nb > 0) {
                __syncwarp();
                if (lane < nb)
                    p.segment(sm, tile, s0, gw * 32 + lane, sm.wcnt[buf][gw * 32 + lane], sm.wacc[buf][gw * 32 + lane],
                              vv);
                __syncwarp();
            }
            buf ^= 1;
        }
        if (P::kGroupEpilogue) {
            __syncthreads();
            p.group(sm, tile, s0, nseg);
            __syncthreads();   // cone scratch is rewritten by the next tile
        }
    }
    if constexpr (kDeferred) drain();
    p.finish(sm);
}

}  // namespace pass
}  // namespace cf
