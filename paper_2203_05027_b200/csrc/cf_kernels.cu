// Iteration, report, projection and export kernels of libcfb200 (sm_100a, fp64).
//
// The reference iteration (solver.py:312-317) is x_update -> y_update ->
// z_update -> dual_update over o-length per-nonzero vectors y, gamma. Because
// U U^T = diag(d) the reference's gamma equals -U^T lam after every iteration
// (DESIGN.md §2), so one iteration is exactly two sparse
// passes with closed-form epilogues:
//
//   col pass (CSC, canonical order)  x+ = fv*(cnt*x + A^T h + z + delta/mu - c/mu)
//                                     z+ = Proj_K(x+ - delta/mu);  delta+ = delta + mu*(z+ - x+)
//   row pass (CSR)                    r = fu*(d*b + A x+);  lam+ = lam + mu*(r - b);
//                                     h+ = (b - r) - lam+/mu
//
// Both passes (and the report's A^T lam pass, and the plain operators) run on
// the persistent TMA-pipelined tile engine of cf_pass.cuh with a per-pass
// policy struct (RowIter, ColIter, ColReport, RowSpmv, ColSpmv) supplying the
// staged epilogue vectors and the epilogue. Segment sums are sequential in
// storage order, so A x and A^T lam are bit-identical to the reference's
// apply_U(apply_Vt(x)) and apply_V(apply_Ut(lam)). Everything is compiled with
// -fmad=false so every fp64 operation rounds like its numpy counterpart.
#include <algorithm>
#include <cmath>

#include "cf_common.h"
#include <utility>

#include <nvtx3/nvToolsExt.h>

#include "cf_pass.cuh"
#include "cf_report.cuh"

namespace cf {
namespace {

// np.max semantics: NaN propagates
__device__ __forceinline__ double nanmax(double a, double b) { return (a > b || a != a) ? a : b; }
__device__ __forceinline__ bool finite(double v) { return isfinite(v); }

struct SumOp {
    __device__ double operator()(double a, double b) const { return a + b; }
};
struct MaxOp {
    __device__ double operator()(double a, double b) const { return nanmax(a, b); }
};

// Deterministic block reduction (fixed xor-shuffle tree + fixed warp order).
// Result valid in thread 0. `sh` needs blockDim/32 doubles.
template <class Op>
__device__ double block_reduce(double v, double* sh, Op op) {
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) v = op(v, __shfl_xor_sync(0xffffffffu, v, off));
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31, nw = blockDim.x >> 5;
    __syncthreads();
    if (l == 0) sh[w] = v;
    __syncthreads();
    if (w == 0) {
        v = (l < nw) ? sh[l] : 0.0;
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) v = op(v, __shfl_xor_sync(0xffffffffu, v, off));
    }
    return v;
}

// Lorentz-cone projection of one block (cones.py:76-92; branch order :78-80),
// tail sum of squares sequential like np.bincount (cones.py:69-72).
__device__ __forceinline__ void project_block_dev(const double* w, int q, double* out) {
    const double w0 = w[0];
    double ssq = 0.0;
    for (int t = 1; t < q; ++t) ssq = __dadd_rn(ssq, __dmul_rn(w[t], w[t]));
    const double alpha = sqrt(ssq);
    if (alpha <= -w0) {
        for (int t = 0; t < q; ++t) out[t] = 0.0;
    } else if (alpha <= w0) {
        for (int t = 0; t < q; ++t) out[t] = w[t];
    } else {
        const double factor = w0 / (2.0 * alpha);
        for (int t = 1; t < q; ++t) out[t] = __dadd_rn(__dmul_rn(0.5, w[t]), __dmul_rn(factor, w[t]));
        out[0] = __dadd_rn(__dmul_rn(0.5, w0), __dmul_rn(0.5, alpha));
    }
}

static_assert(kTileSeg == pass::kPSeg && kTileNnz == pass::kPCap, "host tile cutter and pass engine disagree");
using pass::kComputeThreads;
using pass::kPSeg;
using pass::Smem;

// ---------------------------------------------------------------- pass policies
// A policy supplies the gathered operand, the per-segment epilogue vectors
// (loaded in natural order straight from global memory) and the epilogue.
using pass::Vals;

struct Layout {
    const double* g_;
    static constexpr bool kGroupEpilogue = false;
    static constexpr int kUnroll = pass::kUnroll;   // gathers in flight per thread
    static constexpr int kMinBlocks = pass::kMinBlocks;
    static constexpr int kWideUnroll = 16;          // ... when the tiles cannot fill the GPU (Wide<P>)
    static constexpr int kMediumUnroll = 6;         // ... when they fill it in one wave of 4 CTAs/SM
    static constexpr bool kStaged = false;          // tile idx/val staged in shared memory
    __device__ __forceinline__ const double* gvec() const { return g_; }
    static constexpr int kVals = 0;
    __device__ __forceinline__ void load_async(int, double*) const {}
    __device__ __forceinline__ void load_direct(int, Vals&) const {}
    __device__ __forceinline__ bool carry_in() const { return false; }
    __device__ __forceinline__ double carry(int) const { return 0.0; }
    __device__ __forceinline__ void check(double, int, double) {}
    __device__ __forceinline__ void group(Smem&, int, int, int) {}
    __device__ __forceinline__ void finish(Smem&) {}
};

// Row pass of the iteration: y_update + lam/gamma of dual_update (solver.py:179-183,
// 194-195) in the reduced form r = fu*(d*b + A x+), lam+ = lam + mu(r - b),
// h = b - r - lam+/mu. With column panels, every panel but the last only
// carries the partial row sums (in `carry`), continuing the sequential order.
#ifndef CF_CARRY_L1
#define CF_CARRY_L1 1   // panel carries read through L1 (row pass -0.6 %, profiles/r02_carry_l1.log)
#endif
struct RowIter : Layout {
    int64_t seg_off;       // p * m
    bool last;             // last panel: ADMM update
    bool has_carry;        // panel > 0: the sum continues from carry[i]
    double* carry_buf;     // partial A x between panels (= the plan's ax buffer)
    const double* b;
    const double* dn;      // d_i = sum_k a_ik^2: fu = 1/(1+d) and d b are recomputed (the same
                           // IEEE operations as k_row_diag's, so the same bits; one vector
                           // streamed instead of two)
    double* lam;
    double* h;
    double* br;            // optional: b - r
    double* ax;            // optional: A x (report iterations)
    const double* rcorr;   // optional: warm-start U eps / mu
    double mu;
    pass::MuDiv div;
    static constexpr int kVals = 3;   // b, lam, d (last panel only)
    __device__ __forceinline__ bool carry_in() const { return has_carry; }
    __device__ __forceinline__ double carry(int s) const {
#if CF_CARRY_L1
        // the lanes of a rank block read rows scattered over the tile's 2 KB of carries:
        // through L1 the tile's lines go to L2 once instead of once per warp
        double v;
        asm("ld.global.nc.L1::evict_first.L2::cache_hint.f64 %0, [%1], %2;"
            : "=d"(v) : "l"(carry_buf + (s - seg_off)), "l"(pass::pol_first()));
        return v;
#else
        return pass::ld_first(carry_buf + (s - seg_off), pass::pol_first());
#endif
    }
    __device__ __forceinline__ void load_async(int s, double* slot) const {
        if (!last) return;
        const uint64_t pf = pass::pol_first();
        const int64_t i = s - seg_off;
        pass::cp_async8(slot, b + i, pf);
        pass::cp_async8(slot + 32, lam + i, pf);
        pass::cp_async8(slot + 64, dn + i, pf);
    }
    __device__ __forceinline__ void load_direct(int s, Vals& v) const {
        if (!last) return;
        const uint64_t pf = pass::pol_first();
        const uint32_t i = (uint32_t)(s - seg_off);   // local row (< m): one IMAD.WIDE.U32 per address
        v.v[0] = pass::ld_first(b + i, pf);
        v.v[1] = pass::ld_first(lam + i, pf);
        v.v[2] = pass::ld_first(dn + i, pf);
    }
    __device__ __forceinline__ void segment(Smem&, int, int s0, int q, int, double axi, const Vals& v) {
        const uint32_t i = (uint32_t)(s0 + q - seg_off);   // local row (< m)
        if (!last) {
            carry_buf[i] = axi;
            return;
        }
        const double bi = v.v[0], li = v.v[1], di = v.v[2];
        const double fui = 1.0 / (1.0 + di), dbi = di * bi;   // k_row_diag (uv.py:81)
        double si = dbi + axi;                  // (U t)_i with t = a b + x
        if (rcorr) si = si - rcorr[i];
        const double r = fui * si;              // r = U y+ = fu (U t)
        const double ln = li + mu * (r - bi);   // solver.py:194
        const double bmr = bi - r;
        const double hi = bmr - div(ln);        // h = b - r - lam+/mu
        // on report iterations (ax != null) lam is gathered next by the report's A^T lam pass
        pass::st_hint(lam + i, ln, ax ? pass::pol_last() : pass::pol_first());
        pass::st_hint(h + i, hi, pass::pol_last());   // gathered by the next column pass
        if (br) br[i] = bmr;
        if (ax) ax[i] = axi;
    }
};

// y = A x (apply_U . apply_Vt, uv.py:106-131), panel by panel with y as the carry.
struct RowSpmv : Layout {
    int64_t seg_off;
    bool has_carry;
    double* y;
    __device__ __forceinline__ bool carry_in() const { return has_carry; }
    __device__ __forceinline__ double carry(int s) const { return y[s - seg_off]; }
    __device__ __forceinline__ void segment(Smem&, int, int s0, int q, int, double acc, const Vals&) {
        y[s0 + q - seg_off] = acc;
    }
};

// x = A^T y (apply_V . apply_Ut), band by band with y as the carry.
struct ColSpmv : Layout {
    int64_t seg_off;       // band * n
    bool last;             // (unused: every band writes y)
    bool has_carry;        // band > 0: the sum continues from y[j]
    double* y;
    __device__ __forceinline__ bool carry_in() const { return has_carry; }
    __device__ __forceinline__ double carry(int s) const { return y[s - seg_off]; }
    __device__ __forceinline__ void segment(Smem&, int, int s0, int q, int, double acc, const Vals&) {
        y[s0 + q - seg_off] = acc;
    }
};

// Column-pass state shared by the column policies: the band (segment = band*n + col),
// the carry of the partial column sums between bands, and the epilogue vectors
// x, z, delta, c of column j (read by the last band only).
struct ColVecs : Layout {
    const double* x_in;
    const double* z_in;
    const double* d_in;
    const double* c;
    int64_t seg_off;       // band * n
    bool last;             // last band: run the epilogue
    bool has_carry;        // band > 0: the sum continues from carry_buf[j]
    double* carry_buf;     // partial sums between bands (the plan's atcarry)
    const int32_t* colptr; // bands > 1: canonical column pointers (the full column count)
    static constexpr int kVals = 4;
    __device__ __forceinline__ bool carry_in() const { return has_carry; }
    __device__ __forceinline__ double carry(int s) const { return carry_buf[s - seg_off]; }
    __device__ __forceinline__ void load_async(int s, double* slot) const {
        if (!last) return;
        const uint64_t pf = pass::pol_first();
        const int64_t j = s - seg_off;
        pass::cp_async8(slot, x_in + j, pf);
        pass::cp_async8(slot + 32, z_in + j, pf);
        pass::cp_async8(slot + 64, d_in + j, pf);
        pass::cp_async8(slot + 96, c + j, pf);
    }
    __device__ __forceinline__ void load_direct(int s, Vals& v) const {
        if (!last) return;
        const uint64_t pf = pass::pol_first();
        const int64_t j = s - seg_off;
        v.v[0] = pass::ld_first(x_in + j, pf);
        v.v[1] = pass::ld_first(z_in + j, pf);
        v.v[2] = pass::ld_first(d_in + j, pf);
        v.v[3] = pass::ld_first(c + j, pf);
    }
    // a band before the last only hands its partial sum on
    __device__ __forceinline__ bool carry_out(int64_t j, double acc) const {
        if (last) return false;
        pass::st_hint(carry_buf + j, acc, pass::pol_last());
        return true;
    }
};

// Column pass of the iteration: x_update (solver.py:168-176) in the reduced form
// V(y + gamma/mu) = cnt*x + A^T h, then z = Proj_K(x+ - delta/mu), delta update.
// CONES=false: all blocks of size 1 (cones.py:108-109 shortcut), fused per column.
// CONES=true : x+, w, delta per column to shared memory, then (group epilogue) one thread per cone.
// MODE kLP: all blocks of size 1 (cones.py:108-109 shortcut), fused per column.
// MODE kGroupCones: x+, w, delta to shared memory, group barrier, one thread per cone.
// MODE kWarpCones: every cone has the same size cs in {2,4,...,32} and starts at a
//   multiple of cs, so a cone is cs adjacent lanes of one warp (natural order):
//   the tail norm is summed in order through shuffles, no barrier.
constexpr int kLP = 0, kGroupCones = 1, kWarpCones = 2;

template <int MODE>
struct ColIter : ColVecs {
    static constexpr bool kGroupEpilogue = MODE == kGroupCones;
    double* x;
    double* z;
    double* delta;
    const double* vterm;   // optional: V(y0 + gamma0/mu) (first warm iteration)
    const double* ccorr;   // optional: V eps / mu (second warm iteration)
    const int32_t* tile_cone;
    const int32_t* tile_big;
    const int32_t* cone_ptr;
    double* wbuf;
    double mu;
    pass::MuDiv div;
    int32_t cs;            // kWarpCones: the uniform cone size
    __device__ __forceinline__ void segment(Smem& sm, int, int s0, int q, int cnt, double ath, const Vals& vv) {
        const int j = (int)(s0 + q - seg_off);
        if (carry_out(j, ath)) return;
        if (colptr) cnt = colptr[j + 1] - colptr[j];   // banded: the band holds part of the column
        const double fv = cnt < pass::kFvTab ? sm.fvtab[cnt] : 1.0 / (1.0 + (double)cnt);   // uv.py:82
        const double xj = vv.v[0], zj = vv.v[1], dj = vv.v[2], cj = vv.v[3];
        const double dm = div(dj);
        double v = vterm ? vterm[j] : __dadd_rn(__dmul_rn((double)cnt, xj), ath);
        if (ccorr) v = v - ccorr[j];
        const double xp = fv * (((v + zj) + dm) - div(cj));   // solver.py:171-176 operand order
        const double w = xp - dm;                            // solver.py:188
        if (MODE == kLP) {
            const double zp = w > 0.0 ? w : 0.0;             // NaN -> 0, -0 -> +0
            const double dp = dj + mu * (zp - xp);           // solver.py:196
            pass::st_hint(x + j, xp, pass::pol_last());      // gathered by the next row pass
            pass::st_hint(z + j, zp, pass::pol_first());
            pass::st_hint(delta + j, dp, pass::pol_first());
        } else if (MODE == kWarpCones) {
            // project_block (cones.py:76-92) on cs adjacent lanes; the callers of segment()
            // are the tile's lanes < nb, converged, and nb is a multiple of cs
            const unsigned mask = __activemask();
            const int lane = threadIdx.x & 31;
            const int head = lane & ~(cs - 1);
            double ssq = 0.0;
            for (int t = 1; t < cs; ++t) {
                const double wt = __shfl_sync(mask, w, head + t);
                ssq = __dadd_rn(ssq, __dmul_rn(wt, wt));
            }
            const double w0 = __shfl_sync(mask, w, head);
            const double alpha = sqrt(ssq);
            double zp;
            if (alpha <= -w0) {
                zp = 0.0;
            } else if (alpha <= w0) {
                zp = w;
            } else if (lane == head) {
                zp = __dadd_rn(__dmul_rn(0.5, w0), __dmul_rn(0.5, alpha));
            } else {
                const double factor = w0 / (2.0 * alpha);
                zp = __dadd_rn(__dmul_rn(0.5, w), __dmul_rn(factor, w));
            }
            const double dp = dj + mu * (zp - xp);
            pass::st_hint(x + j, xp, pass::pol_last());
            pass::st_hint(z + j, zp, pass::pol_first());
            pass::st_hint(delta + j, dp, pass::pol_first());
        } else {
            const int gi = pass::group_id();
            sm.cscr[gi][0][q] = xp;
            sm.cscr[gi][1][q] = w;
            sm.cscr[gi][2][q] = dj;
        }
    }
    __device__ __forceinline__ void group(Smem& sm, int tile, int sseg0, int nseg) {
        if (!last) return;
        const int s0 = (int)(sseg0 - seg_off);   // first column of the tile
        const int gi = pass::group_id();
        const double* sxp = sm.cscr[gi][0];
        const double* sw = sm.cscr[gi][1];
        const double* sd = sm.cscr[gi][2];
        double* sdn = sm.cscr[gi][3];
        double* szp = sm.wacc[gi];   // the warp transposes of this tile are done
        const int t = pass::group_tid();
        const int big = tile_big[tile];
        if (big >= 0) {  // piece of a cone wider than a tile: k_big_cone projects it
            for (int q = t; q < nseg; q += kComputeThreads) {
                pass::st_hint(x + s0 + q, sxp[q], pass::pol_last());
                wbuf[s0 + q] = sw[q];
            }
            return;
        }
        const int q0 = tile_cone[tile], q1 = tile_cone[tile + 1];
        for (int c = q0 + t; c < q1; c += kComputeThreads) {
            const int off = cone_ptr[c] - s0, size = cone_ptr[c + 1] - cone_ptr[c];
            project_block_dev(sw + off, size, szp + off);
            for (int u = 0; u < size; ++u) sdn[off + u] = sd[off + u] + mu * (szp[off + u] - sxp[off + u]);
        }
        pass::group_sync();
        for (int q = t; q < nseg; q += kComputeThreads) {
            pass::st_hint(x + s0 + q, sxp[q], pass::pol_last());
            pass::st_hint(z + s0 + q, szp[q], pass::pol_first());
            pass::st_hint(delta + s0 + q, sdn[q], pass::pol_first());
        }
    }
};

// Column part of compute_report (solver.py:208-225): atl = A^T lam (bincount order),
// dual = atl + c, stat = dual - delta, pobj = c.x, cone_gap = max|x - z| and the
// finiteness of x, z, delta (the implicit y and gamma are checked per row by
// k_row_report). Per-thread partials are reduced once per CTA (finish).
struct ColReport : ColVecs {
    static constexpr int kUnroll = 8;      // 8 report accumulators per thread
    static constexpr int kWideUnroll = 8;
    static constexpr int kMediumUnroll = 4;
    static constexpr int kMinBlocks = 2;   // (more registers; runs once per check_every iterations)
    double* part;          // [kReportFieldsCol][kGroups][gridDim.x]
    double d2, dmx, s2, smx, amx, cx, cg, nf;
    __device__ __forceinline__ void segment(Smem&, int, int s0, int q, int, double atl, const Vals& vv) {
        if (carry_out(s0 + q - seg_off, atl)) return;
        const double xj = vv.v[0], zj = vv.v[1], dj = vv.v[2], cj = vv.v[3];
        const double dual = atl + cj;
        const double stat = dual - dj;
        d2 = d2 + dual * dual;
        dmx = nanmax(dmx, fabs(dual));
        s2 = s2 + stat * stat;
        smx = nanmax(smx, fabs(stat));
        amx = nanmax(amx, fabs(atl));
        cx = cx + cj * xj;
        cg = nanmax(cg, fabs(xj - zj));
        if (!isfinite(xj) || !isfinite(zj) || !isfinite(dj)) nf = 1.0;
    }
    __device__ __forceinline__ void finish(Smem& sm) {
        if (!last) return;   // (uniform over the grid)
        const int G = gridDim.x;
        const double vals[8] = {d2, dmx, s2, smx, amx, cx, cg, nf};
        const bool is_sum[8] = {true, false, true, false, false, true, false, false};
#pragma unroll
        for (int f = 0; f < 8; ++f) {
            const double v = is_sum[f] ? pass::group_reduce(vals[f], sm.red[pass::group_id()], SumOp())
                                       : pass::group_reduce(vals[f], sm.red[pass::group_id()], MaxOp());
            if (pass::group_tid() == 0) part[(f * pass::kGroups + pass::group_id()) * G + blockIdx.x] = v;
        }
    }
};

// Cones larger than kSmallCone: one CTA per cone. Tail norm by a fixed
// per-thread sequential split + deterministic tree (not the reference's
// sequential order: agrees to rounding).
struct BigConeArgs {
    const int32_t* big_cone;
    const int32_t* cone_ptr;
    const double* wbuf;
    const double* x;   // x+
    double* z;
    double* delta;
    double* out;       // projection-only mode: write here instead of z/delta
    double mu;
    const int32_t* done;
};
__global__ void __launch_bounds__(1024) k_big_cone(const BigConeArgs a) {
    pass::pdl_wait();
    pass::pdl_trigger();
    if (a.done && *a.done) return;
    __shared__ double sh[32];
    __shared__ double s_alpha;
    const int q = a.big_cone[blockIdx.x];
    const int off = a.cone_ptr[q], size = a.cone_ptr[q + 1] - off;
    const double* w = a.wbuf + off;
    double ssq = 0.0;
    for (int t = 1 + threadIdx.x; t < size; t += blockDim.x) ssq = __dadd_rn(ssq, __dmul_rn(w[t], w[t]));
    ssq = block_reduce(ssq, sh, SumOp());
    if (threadIdx.x == 0) s_alpha = sqrt(ssq);
    __syncthreads();
    const double alpha = s_alpha, w0 = w[0];
    const int branch = (alpha <= -w0) ? 0 : ((alpha <= w0) ? 1 : 2);
    const double factor = branch == 2 ? w0 / (2.0 * alpha) : 0.0;
    for (int t = threadIdx.x; t < size; t += blockDim.x) {
        double zt;
        if (branch == 0) zt = 0.0;
        else if (branch == 1) zt = w[t];
        else if (t == 0) zt = __dadd_rn(__dmul_rn(0.5, w0), __dmul_rn(0.5, alpha));
        else zt = __dadd_rn(__dmul_rn(0.5, w[t]), __dmul_rn(factor, w[t]));
        if (a.out) {
            a.out[off + t] = zt;
        } else {
            a.z[off + t] = zt;
            a.delta[off + t] = a.delta[off + t] + a.mu * (zt - a.x[off + t]);
        }
    }
}

// ---------------------------------------------------------------- report
// Row part of compute_report (solver.py:213-214,219,224): prim = ax - b.
struct RowReportArgs {
    const double* ax;
    const double* b;
    const double* lam;
    const double* br;     // b - r of the report iteration (y_k = x_j + a_k br_i), may be null
    const double* amax;   // max |a_k| of each row
    double* part;    // [kReportFieldsRow][gridDim.x]
    int32_t m;
    const int32_t* done;
};
__global__ void __launch_bounds__(kThreads) k_row_report(const RowReportArgs a) {
    pass::pdl_wait();
    pass::pdl_trigger();
    if (a.done && *a.done) return;
    __shared__ double sh[32];
    double s2 = 0.0, mx = 0.0, axm = 0.0, bl = 0.0, nf = 0.0;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < a.m; i += gridDim.x * blockDim.x) {
        const double axi = a.ax[i], bi = a.b[i], li = a.lam[i];
        const double pr = axi - bi;
        // implicit gamma_k = -a_k lam_i and the a_k (b_i - r_i) part of y_k: all finite iff
        // their largest magnitude is
        const double am = a.amax[i];
        if (!finite(am * li) || (a.br && !finite(am * a.br[i]))) nf = 1.0;
        s2 = s2 + pr * pr;
        mx = nanmax(mx, fabs(pr));
        axm = nanmax(axm, fabs(axi));
        bl = bl + bi * li;
        if (!finite(li)) nf = 1.0;
    }
    const int G = gridDim.x;
    double v;
    v = block_reduce(s2, sh, SumOp());
    if (threadIdx.x == 0) a.part[0 * G + blockIdx.x] = v;
    v = block_reduce(mx, sh, MaxOp());
    if (threadIdx.x == 0) a.part[1 * G + blockIdx.x] = v;
    v = block_reduce(axm, sh, MaxOp());
    if (threadIdx.x == 0) a.part[2 * G + blockIdx.x] = v;
    v = block_reduce(bl, sh, SumOp());
    if (threadIdx.x == 0) a.part[3 * G + blockIdx.x] = v;
    v = block_reduce(nf, sh, MaxOp());
    if (threadIdx.x == 0) a.part[4 * G + blockIdx.x] = v;
}

struct FinalizeArgs {
    const double* part_row;
    const double* part_col;
    const int32_t* nf_flag;  // non-finite implicit y / gamma seen by the report's gather warps
    int32_t g_row;
    int32_t g_col;
    int64_t k;
    int32_t check;      // apply check_termination
    cf_config cfg;
    cf_report* slot;
    int32_t* done;      // may be null
};
template <class Op>
__device__ double reduce_partials(const double* p, int G, double* sh, Op op) {
    double v = 0.0;
    for (int t = threadIdx.x; t < G; t += blockDim.x) v = op(v, p[t]);
    return block_reduce(v, sh, op);
}
// Final stage of compute_report (solver.py:219-242) + check_termination
// (solver.py:245-272) + the max_iters rule (:322-323).
__global__ void __launch_bounds__(1024) k_finalize(const FinalizeArgs a) {
    pass::pdl_wait();
    pass::pdl_trigger();
    if (a.done && *a.done) return;
    __shared__ double sh[32];
    double f[kReportFieldsRow + kReportFieldsCol];
    const SumOp sum;
    const MaxOp mx;
    f[0] = reduce_partials(a.part_row + 0 * a.g_row, a.g_row, sh, sum);
    f[1] = reduce_partials(a.part_row + 1 * a.g_row, a.g_row, sh, mx);
    f[2] = reduce_partials(a.part_row + 2 * a.g_row, a.g_row, sh, mx);
    f[3] = reduce_partials(a.part_row + 3 * a.g_row, a.g_row, sh, sum);
    f[4] = reduce_partials(a.part_row + 4 * a.g_row, a.g_row, sh, mx);
    f[5] = reduce_partials(a.part_col + 0 * a.g_col, a.g_col, sh, sum);
    f[6] = reduce_partials(a.part_col + 1 * a.g_col, a.g_col, sh, mx);
    f[7] = reduce_partials(a.part_col + 2 * a.g_col, a.g_col, sh, sum);
    f[8] = reduce_partials(a.part_col + 3 * a.g_col, a.g_col, sh, mx);
    f[9] = reduce_partials(a.part_col + 4 * a.g_col, a.g_col, sh, mx);
    f[10] = reduce_partials(a.part_col + 5 * a.g_col, a.g_col, sh, sum);
    f[11] = reduce_partials(a.part_col + 6 * a.g_col, a.g_col, sh, mx);
    f[12] = reduce_partials(a.part_col + 7 * a.g_col, a.g_col, sh, mx);
    if (threadIdx.x != 0) return;
    const ReportFields rf{f[0], f[1], f[2], f[3], f[4], f[5], f[6], f[7], f[8], f[9], f[10], f[11], f[12]};
    cf_report r = assemble_report(rf, a.k, a.nf_flag && *a.nf_flag);
    int status = a.check ? decide_status(r, a.cfg, a.k) : r.status;
    r.status = status;
    *a.slot = r;
    if (a.done && status != CF_STATUS_RUNNING) *a.done = 1;
}

// ---------------------------------------------------------------- projection utility
// project_product (cones.py:103-110) of an arbitrary vector.
__global__ void k_project_lp(const double* w, double* out, int64_t n) {
    for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < n; j += (int64_t)gridDim.x * blockDim.x) {
        const double v = w[j];
        out[j] = v > 0.0 ? v : 0.0;
    }
}
__global__ void k_project_small(const double* w, double* out, const int32_t* cone_ptr, int64_t n_blocks) {
    for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < n_blocks;
         q += (int64_t)gridDim.x * blockDim.x) {
        const int off = cone_ptr[q], size = cone_ptr[q + 1] - off;
        if (size > kSmallCone) continue;  // big cones: k_big_cone
        project_block_dev(w + off, size, out + off);
    }
}

// ---------------------------------------------------------------- state export (K5)
// y_k = x_j + a_k (b_i - r_i) [- eps_k/mu right after a warm start]; gamma_k = -a_k lam_i,
// written in canonical (CSC) order.
__global__ void k_export(const int32_t* colptr, const int32_t* rowidx, const double* val, const double* x,
                         const double* br, const double* lam, const double* eps, double mu, double* y,
                         double* gamma, int64_t n) {
    for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < n; j += (int64_t)gridDim.x * blockDim.x) {
        const double xj = x[j];
        for (int k = colptr[j]; k < colptr[j + 1]; ++k) {
            const int i = rowidx[k];
            const double av = val[k];
            if (y) {
                double yk = xj + av * br[i];
                if (eps) yk = yk - eps[k] / mu;
                y[k] = yk;
            }
            if (gamma) gamma[k] = -(av * lam[i]);
        }
    }
}

// ---------------------------------------------------------------- warm start (App. A.3)
// vterm[j] = sum_{k in col j} (y0_k + gamma0_k/mu)   (apply_V, bincount order)
// eps_k    = gamma0_k + a_k lam0_i
// ccorr[j] = (sum_{k in col j} eps_k) / mu
__global__ void k_warm_cols(const int32_t* colptr, const int32_t* rowidx, const double* val, const double* y0,
                            const double* g0, const double* lam0, double mu, double* vterm, double* eps,
                            double* ccorr, int64_t n) {
    for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < n; j += (int64_t)gridDim.x * blockDim.x) {
        double v = 0.0, e = 0.0;
        for (int k = colptr[j]; k < colptr[j + 1]; ++k) {
            v = v + (y0[k] + g0[k] / mu);
            const double ek = g0[k] + val[k] * lam0[rowidx[k]];
            eps[k] = ek;
            e = e + ek;
        }
        vterm[j] = v;
        ccorr[j] = e / mu;
    }
}
// rcorr[i] = (sum_{p in row i} a_p eps_{csc(p)}) / mu
__global__ void k_warm_rows(const int32_t* rowptr, const double* valr, const int32_t* csr2csc, const double* eps,
                            double mu, double* rcorr, int64_t m, int32_t panels) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m; i += (int64_t)gridDim.x * blockDim.x) {
        double s = 0.0;
        for (int32_t pn = 0; pn < panels; ++pn) {
            const int64_t seg = pn * m + i;
            for (int p = rowptr[seg]; p < rowptr[seg + 1]; ++p) s = s + valr[p] * eps[csr2csc[p]];
        }
        rcorr[i] = s / mu;
    }
}

// fu_i = 1/(1 + sum a^2) (uv.py:81, bincount order = CSR order), db_i = d_i b_i
// also amax_i = max_k |a_k| of row i: a_k*v is finite for every k of row i iff amax_i*v is
// (the report's exact row-level test of the implicit y and gamma, solver.py:208-211)
__global__ void k_row_diag(const int32_t* rowptr, const double* valr, const double* b, double* fu, double* db,
                           double* amax, double* dn, int64_t m, int32_t panels) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m; i += (int64_t)gridDim.x * blockDim.x) {
        double d = 0.0, am = 0.0;
        for (int32_t pn = 0; pn < panels; ++pn) {
            const int64_t seg = pn * m + i;
            for (int p = rowptr[seg]; p < rowptr[seg + 1]; ++p) {
                d = d + valr[p] * valr[p];
                am = fmax(am, fabs(valr[p]));
            }
        }
        fu[i] = 1.0 / (1.0 + d);
        db[i] = d * b[i];
        amax[i] = am;
        dn[i] = d;
    }
}

// the row sums d_i = sum_k a_ik^2 (canonical order) and max |a_ik| of the plan's entries
__global__ void k_row_norms(const int32_t* rowptr, const double* valr, double* dout, double* amax, int64_t m,
                            int32_t panels) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m; i += (int64_t)gridDim.x * blockDim.x) {
        double d = 0.0, am = 0.0;
        for (int32_t pn = 0; pn < panels; ++pn) {
            const int64_t seg = pn * m + i;
            for (int p = rowptr[seg]; p < rowptr[seg + 1]; ++p) {
                d = d + valr[p] * valr[p];
                am = fmax(am, fabs(valr[p]));
            }
        }
        dout[i] = d;
        amax[i] = am;
    }
}
// fu = 1/(1+d) (uv.py:81), d*b and amax from given (e.g. all-reduced) row norms
__global__ void k_set_row_diag(const double* din, const double* amax_in, const double* b, double* fu, double* db,
                               double* amax, double* dn, int64_t m) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m; i += (int64_t)gridDim.x * blockDim.x) {
        const double d = din[i];
        fu[i] = 1.0 / (1.0 + d);
        db[i] = d * b[i];
        amax[i] = amax_in[i];
        dn[i] = d;
    }
}

inline int grid_for(int64_t work, int threads) {
    int64_t g = (work + threads - 1) / threads;
    if (g < 1) g = 1;
    if (g > 148 * 16) g = 148 * 16;
    return (int)g;
}

// every tile of [t0, t1) is block-ranked and packed, so it fits a TileStage
// (unpacked[t] = tile-ranked tiles among the first t; size = tiles + 1)
int32_t stageable(const std::vector<int32_t>& unpacked, int64_t t0, int64_t t1) {
    if (t0 < 0 || t1 <= t0 || t1 >= (int64_t)unpacked.size() + 1) return 0;
    return unpacked[t1] - unpacked[t0] == 0 ? 1 : 0;
}

pass::Tiles row_panel_tiles(const cf_plan* p, int panel) {
    const int64_t t0 = p->row_panel_tile[panel], t1 = p->row_panel_tile[panel + 1];
    return pass::Tiles{p->row_tb.p + t0, (int32_t)(t1 - t0), stageable(p->row_unpacked, t0, t1)};
}
pass::Tiles col_band_tiles(const cf_plan* p, int band) {
    const int64_t t0 = p->col_band_tile[band], t1 = p->col_band_tile[band + 1];
    return pass::Tiles{p->col_tb.p + t0, (int32_t)(t1 - t0), stageable(p->col_unpacked, t0, t1)};
}
pass::Jds row_jds(const cf_plan* p) {
    return pass::Jds{p->rj_idx.p, p->rj_val.p, p->rj_pl.p, (int64_t)p->rj_idx.n, p->n};
}
pass::Jds col_jds(const cf_plan* p) {
    return pass::Jds{p->cj_idx.p, p->cj_val.p, p->cj_pl.p, (int64_t)p->cj_idx.n, p->m};
}

// L2 persisting window for the gathered vector of the next pass launches
// (CF_L2_PERSIST_MB=<set-aside MB>; off by default). Set by the pass launchers.
struct L2Window {
    const void* ptr = nullptr;
    size_t bytes = 0;
};
thread_local L2Window g_l2win;
size_t l2_persist_bytes() {
    static const size_t v = [] {
        const char* e = getenv("CF_L2_PERSIST_MB");
        if (!e || atoi(e) <= 0) return (size_t)0;
        int dev = 0, maxp = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&maxp, cudaDevAttrMaxPersistingL2CacheSize, dev);
        const size_t want = std::min<size_t>((size_t)atoi(e) << 20, (size_t)maxp);
        if (cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, want) != cudaSuccess) {
            cudaGetLastError();
            return (size_t)0;
        }
        return want;
    }();
    return v;
}
struct L2WindowScope {
    L2Window saved;
    L2WindowScope(const void* p, size_t b) : saved(g_l2win) { g_l2win = L2Window{p, b}; }
    ~L2WindowScope() { g_l2win = saved; }
};

// Launch with programmatic stream serialization (the kernel calls pdl_wait()
// before touching its predecessor's results): the launch overlaps the
// predecessor's tail instead of waiting for it to drain.
template <class... KArgs, class... Args>
cudaError_t launch_pdl(void (*kernel)(KArgs...), unsigned grid, unsigned block, size_t smem, cudaStream_t st,
                       Args&&... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(block);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute at[2];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    const size_t persist = g_l2win.ptr ? l2_persist_bytes() : 0;
    if (persist) {
        static const size_t max_win = [] {
            int dev = 0, v = 0;
            cudaGetDevice(&dev);
            cudaDeviceGetAttribute(&v, cudaDevAttrMaxAccessPolicyWindowSize, dev);
            return (size_t)v;
        }();
        const size_t nb = std::min(g_l2win.bytes, max_win);
        at[1].id = cudaLaunchAttributeAccessPolicyWindow;
        at[1].val.accessPolicyWindow.base_ptr = const_cast<void*>(g_l2win.ptr);
        at[1].val.accessPolicyWindow.num_bytes = nb;
        at[1].val.accessPolicyWindow.hitRatio = nb ? (float)std::min(1.0, (double)persist / (double)nb) : 0.f;
        at[1].val.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
        at[1].val.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
        cfg.numAttrs = 2;
    }
    return cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
}

#ifndef CF_MEDIUM_MINB
#define CF_MEDIUM_MINB 4
#endif
#ifndef CF_CARVEOUT
#define CF_CARVEOUT 1      // size the carve-out of the unstaged variants for kMinBlocks CTAs too
#endif
#ifndef CF_STAGED_CTAS
#define CF_STAGED_CTAS 3   // staged CTAs per SM the shared-memory carve-out is sized for (0: driver default)
#endif
#ifndef CF_STAGED_CAP
#define CF_STAGED_CAP 0   // >0: at most this many staged CTAs per SM (their shared memory starves the gathers' L1)
#endif
// resident CTAs of k_pass<P> on the device (computed once, thread-safe: plans are
// created and run from several host threads by solve_batch / run_bench)
template <class P>
int pass_capacity() {
    static const int cap = [] {
        int per_sm = 0, sms = 0, dev = 0;
        bool ok = cudaFuncSetAttribute(pass::k_pass<P>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)pass::smem_bytes<P>()) == cudaSuccess;
        // The L1 left beside the shared-memory carve-out is what keeps the gathers in flight, so
        // size the carve-out for the CTAs per SM the variant is meant to run (staged tiles hold
        // ~54 KB each: 3 per SM, 1e6 nonzeros 25 -> 20 us per iteration; the others kMinBlocks)
        const int ctas = P::kStaged ? CF_STAGED_CTAS : (CF_CARVEOUT ? P::kMinBlocks : 0);
        if (ok && ctas > 0) {
            const double need = (double)ctas * (double)(pass::smem_bytes<P>() + 1024);
            const int pct = std::min(100, (int)std::ceil(100.0 * need / (228.0 * 1024.0)));
            ok = cudaFuncSetAttribute(pass::k_pass<P>, cudaFuncAttributePreferredSharedMemoryCarveout, pct) ==
                 cudaSuccess;
        }
        ok = ok && cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, pass::k_pass<P>, pass::kPThreads,
                                                                 pass::smem_bytes<P>()) == cudaSuccess;
        ok = ok && cudaGetDevice(&dev) == cudaSuccess;
        ok = ok && cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) == cudaSuccess;
        return ok ? std::max(per_sm, 1) * sms : 0;
    }();
    return cap;
}

template <class P>
int persistent_grid(int n_tiles) {
    const int g = pass_capacity<P>();
    if (g <= 0) {
        set_error("k_pass occupancy query failed");
        return 0;
    }
    return n_tiles < g ? (n_tiles > 0 ? n_tiles : 1) : g;
}

#ifndef CF_STAGED_SMALL
#define CF_STAGED_SMALL 1   // Wide/Medium stage each tile's idx/val in shared memory (direct engine)
#endif
// Small and mid-size problems are latency-bound: every tile should get its own
// CTA in ONE wave, and each lane then keeps more gathers in flight instead.
//   n_tiles <=  2 x 148: Wide   (16 in flight, 2 CTAs / SM, staged tiles)
//   n_tiles <= 12 x 148: Medium ( 6 in flight, 4 CTAs / SM, staged tiles)
//   otherwise          : the persistent default (3 in flight, 6 CTAs / SM, direct loads)
// (tools/prof_sizes.py: 1e6 nnz 25.5 -> 19.8 us/iteration, 3e6 55.6 -> 51.8; 1e7 is
// faster unstaged)
template <class P>
struct Wide : P {
    static constexpr int kUnroll = P::kWideUnroll;
    static constexpr int kMinBlocks = 2;
    static constexpr bool kStaged = CF_STAGED_SMALL;
};
template <class P>
struct Medium : P {
    static constexpr int kUnroll = P::kMediumUnroll;
    static constexpr int kMinBlocks = CF_MEDIUM_MINB;
    static constexpr bool kStaged = CF_STAGED_SMALL;
};
// large passes over long segments (>= 16 nonzeros on average): 4 diagonals in flight,
// 5 CTAs/SM (C3's row pass 0.258 -> 0.237 ms; C2's 10-long segments keep the default)
template <class P>
struct Long : P {
    static constexpr int kUnroll = 4;
    static constexpr int kMinBlocks = 5;
};
constexpr double kLongSegments = 16.0;
constexpr int kWideTiles = 148 * 2;
constexpr int kMediumTiles = kStagedMaxTiles;

template <class Q>
int launch_variant(const Q& pol, const pass::Jds& L, const pass::Tiles& T, const int32_t* done, cudaStream_t st,
                   int* grid_out) {
    int grid = persistent_grid<Q>(T.n_tiles);
    if (grid <= 0) return CF_ECUDA;
    if (CF_STAGED_CAP > 0 && Q::kStaged) grid = std::min(grid, CF_STAGED_CAP * 148);
    if (grid_out) *grid_out = grid;
    CF_CUDA(launch_pdl(pass::k_pass<Q>, (unsigned)grid, (unsigned)pass::kPThreads, pass::smem_bytes<Q>(), st, pol, L,
                       T, done));
    return CF_OK;
}

template <class P>
int launch_pass(const P& pol, const pass::Jds& L, const pass::Tiles& T, const int32_t* done, cudaStream_t st,
                int* grid_out = nullptr, double avg_len = 0.0) {
    if (T.n_tiles == 0) return CF_OK;
    if (T.stageable && T.n_tiles <= kWideTiles) return launch_variant(Wide<P>{pol}, L, T, done, st, grid_out);
    if (T.stageable && T.n_tiles <= kMediumTiles) return launch_variant(Medium<P>{pol}, L, T, done, st, grid_out);
    if constexpr (P::kUnroll < 4) {
        if (avg_len >= kLongSegments) return launch_variant(Long<P>{pol}, L, T, done, st, grid_out);
    }
    return launch_variant(pol, L, T, done, st, grid_out);
}

// average segment length of a pass: nonzeros / segments (rows per panel, columns per band)
double row_avg_len(const cf_plan* p) { return p->m ? (double)p->o / ((double)p->n_panels * (double)p->m) : 0.0; }
double col_avg_len(const cf_plan* p) { return p->n ? (double)p->o / ((double)p->n_bands * (double)p->n) : 0.0; }

// the band fields of a column policy (seg_off/last/has_carry are set per launch)
template <class P>
void col_vecs_bands(const cf_plan* p, P& c) {
    c.carry_buf = p->atcarry.p;
    c.colptr = p->n_bands > 1 ? p->colptr.p : nullptr;
}

// run a column policy band by band (segment = band*n + col); the last band runs the
// epilogue, earlier bands carry their partial sums (grid_out: the last band's grid)
template <class P>
int launch_col_bands(cf_plan* p, P pol, const int32_t* done, int64_t* nl, int* grid_out = nullptr) {
    const int B = p->n_bands;
    for (int b = 0; b < B; ++b) {
        pol.seg_off = (int64_t)b * p->n;
        pol.last = (b == B - 1);
        pol.has_carry = b > 0;
        CF_TRY(launch_pass(pol, col_jds(p), col_band_tiles(p, b), done, p->stream, pol.last ? grid_out : nullptr,
                           col_avg_len(p)));
        if (nl) ++*nl;
    }
    return CF_OK;
}

template <int MODE>
ColIter<MODE> col_iter(cf_plan* p, const IterOpts& opt) {
    ColIter<MODE> c{};
    c.g_ = p->h.p;
    c.x_in = p->x.p;
    c.z_in = p->z.p;
    c.d_in = p->delta.p;
    c.c = p->c.p;
    c.x = p->x.p;
    c.z = p->z.p;
    c.delta = p->delta.p;
    c.tile_cone = p->tile_cone.p;
    c.tile_big = p->tile_big.p;
    c.cone_ptr = p->cone_ptr.p;
    c.wbuf = p->wbuf.p;
    c.vterm = opt.vterm;
    c.ccorr = opt.ccorr;
    c.mu = opt.mu;
    c.div = pass::make_mudiv(opt.mu);
    c.cs = p->warp_cone;
    col_vecs_bands(p, c);
    return c;
}

}  // namespace

// ---------------------------------------------------------------- launch wrappers
int launch_row_only(cf_plan* p, const IterOpts& opt, const int32_t* done, int64_t* launches) {
    int64_t nl = 0;
    const int64_t m = p->m;
    for (int pn = 0; pn < p->n_panels && m > 0; ++pn) {
        RowIter r{};
        r.g_ = p->x.p;
        r.seg_off = (int64_t)pn * m;
        r.last = (pn == p->n_panels - 1);
        r.has_carry = pn > 0;
        r.carry_buf = p->ax.p;
        r.b = p->b.p;
        r.dn = p->dn.p;
        r.lam = p->lam.p;
        r.h = p->h.p;
        r.mu = opt.mu;
        r.div = pass::make_mudiv(opt.mu);
        r.rcorr = opt.rcorr;
        r.br = (opt.report || p->keep_br) ? p->br.p : nullptr;
        r.ax = opt.report ? p->ax.p : nullptr;
        const int64_t c0 = std::min<int64_t>(p->n, (int64_t)pn * p->panel_cols);
        const int64_t c1 = std::min<int64_t>(p->n, c0 + p->panel_cols);
        L2WindowScope w(g_l2win.ptr ? (const void*)(p->x.p + c0) : nullptr, (size_t)(c1 - c0) * 8);
        CF_TRY(launch_pass(r, row_jds(p), row_panel_tiles(p, pn), done, p->stream, nullptr, row_avg_len(p)));
        ++nl;
    }
    if (launches) *launches += nl;
    return CF_OK;
}

int launch_iteration(cf_plan* p, const IterOpts& opt, const int32_t* done, int64_t* launches) {
    int64_t nl = 0;
    cudaEvent_t e_a = nullptr, e_b = nullptr, e_c = nullptr;
    // per-pass events break the programmatic-launch overlap of the passes they bracket
    // (~11 us per iteration at C2), so a loop can sample every prof_stride-th iteration
    // (the last iteration of each stride: the loop's first iteration, with its launch
    // latency exposed, is sampled only when every iteration is)
    const bool prof = p->profiling && (p->prof_iter++ % p->prof_stride) == p->prof_stride - 1;
    if (prof) {
        while (p->prof_events.size() < p->prof_used + 3) {
            cudaEvent_t e;
            CF_CUDA(cudaEventCreate(&e));
            p->prof_events.push_back(e);
        }
        e_a = p->prof_events[p->prof_used];
        e_b = p->prof_events[p->prof_used + 1];
        e_c = p->prof_events[p->prof_used + 2];
        p->prof_used += 3;
        CF_CUDA(cudaEventRecord(e_a, p->stream));
    }
    {
        // NVTX ranges (host enqueue of each pass; free without a profiler attached)
        nvtxRangePushA("cf col pass");
        L2WindowScope w(p->h.p, (size_t)p->m * 8);
        const int rc = launch_col_only(p, opt, done, &nl);
        nvtxRangePop();
        CF_TRY(rc);
    }
    if (prof) CF_CUDA(cudaEventRecord(e_b, p->stream));
    {
        nvtxRangePushA("cf row pass");
        L2WindowScope w(p->x.p, (size_t)p->n * 8);
        const int rc = launch_row_only(p, opt, done, &nl);
        nvtxRangePop();
        CF_TRY(rc);
    }
    if (prof) CF_CUDA(cudaEventRecord(e_c, p->stream));
    if (launches) *launches += nl;
    return CF_OK;
}

// one launch per run of tiles with one cone size (cf_plan::col_runs; a single band)
int launch_col_runs(cf_plan* p, const IterOpts& opt, const int32_t* done, int64_t* nl) {
    for (const auto& r : p->col_runs) {
        const pass::Tiles T{p->col_tb.p + r.t0, (int32_t)(r.t1 - r.t0), stageable(p->col_unpacked, r.t0, r.t1)};
        auto run = [&](auto c) {
            c.seg_off = 0;
            c.last = true;
            c.has_carry = false;
            return launch_pass(c, col_jds(p), T, done, p->stream, nullptr, col_avg_len(p));
        };
        if (r.cls == 1) {
            CF_TRY(run(col_iter<kLP>(p, opt)));
        } else if (r.cls > 1) {
            auto c = col_iter<kWarpCones>(p, opt);
            c.cs = r.cls;
            CF_TRY(run(c));
        } else {
            auto c = col_iter<kGroupCones>(p, opt);
            c.tile_cone += r.t0;   // the kernel indexes them by tile within the launch
            c.tile_big += r.t0;
            CF_TRY(run(c));
        }
        ++*nl;
    }
    return CF_OK;
}

int launch_col_only(cf_plan* p, const IterOpts& opt, const int32_t* done, int64_t* launches) {
    int64_t nl = 0;
    if (p->n > 0) {
        if (!p->col_runs.empty()) {
            CF_TRY(launch_col_runs(p, opt, done, &nl));
        } else if (p->all_unit) {
            CF_TRY(launch_col_bands(p, col_iter<kLP>(p, opt), done, &nl));
        } else if (p->warp_cone) {
            CF_TRY(launch_col_bands(p, col_iter<kWarpCones>(p, opt), done, &nl));
        } else {
            CF_TRY(launch_col_bands(p, col_iter<kGroupCones>(p, opt), done, &nl));
        }
        if (!p->all_unit && p->n_big > 0) {
            BigConeArgs g{};
            g.big_cone = p->big_cone.p;
            g.cone_ptr = p->cone_ptr.p;
            g.wbuf = p->wbuf.p;
            g.x = p->x.p;
            g.z = p->z.p;
            g.delta = p->delta.p;
            g.mu = opt.mu;
            g.done = done;
            CF_CUDA(launch_pdl(k_big_cone, (unsigned)p->n_big, 1024u, 0, p->stream, g));
            ++nl;
        }
    }
    if (launches) *launches += nl;
    return CF_OK;
}

void prof_reset(cf_plan* p) {
    p->prof_used = 0;
    p->prof_iter = 0;
    p->prof_samples = 0;
    p->prof_row_ms = p->prof_col_ms = 0.0;
}

void prof_collect(cf_plan* p) {
    for (size_t i = 0; i + 3 <= p->prof_used; i += 3) {
        float t1 = 0.f, t2 = 0.f;
        cudaEventElapsedTime(&t1, p->prof_events[i], p->prof_events[i + 1]);
        cudaEventElapsedTime(&t2, p->prof_events[i + 1], p->prof_events[i + 2]);
        p->prof_col_ms += t1;
        p->prof_row_ms += t2;
        ++p->prof_samples;
    }
    p->prof_used = 0;
}

int launch_spmv_rows(cf_plan* p, const double* x, double* y) {
    const int64_t m = p->m;
    for (int pn = 0; pn < p->n_panels && m > 0; ++pn) {
        RowSpmv r{};
        r.g_ = x;
        r.seg_off = (int64_t)pn * m;
        r.has_carry = pn > 0;
        r.y = y;
        CF_TRY(launch_pass(r, row_jds(p), row_panel_tiles(p, pn), nullptr, p->stream, nullptr, row_avg_len(p)));
    }
    return CF_OK;
}

int launch_spmv_cols(cf_plan* p, const double* y, double* x) {
    if (p->n == 0) return CF_OK;
    ColSpmv c{};
    c.g_ = y;
    c.y = x;
    return launch_col_bands(p, c, nullptr, nullptr);
}

int launch_spmv_cols_range(cf_plan* p, const double* y, double* x, int64_t col_lo, int64_t col_hi) {
    if (p->n == 0 || p->col_tile_start.size() < 2 || col_hi <= col_lo) return CF_OK;
    if (p->n_bands > 1) {
        // the bands' tile boundaries differ, so a column's bands could not be kept in order
        // across ranges: the first range runs the whole banded pass, the others are no-ops
        return col_lo == 0 ? launch_spmv_cols(p, y, x) : CF_OK;
    }
    // the tiles that start in [col_lo, col_hi)
    const auto& ts = p->col_tile_start;   // first column of each tile, + the end (n)
    const int64_t t0 = std::lower_bound(ts.begin(), ts.end() - 1, (int32_t)col_lo) - ts.begin();
    const int64_t t1 =
        std::lower_bound(ts.begin(), ts.end() - 1, (int32_t)std::min<int64_t>(col_hi, p->n)) - ts.begin();
    if (t1 <= t0) return CF_OK;
    ColSpmv c{};
    c.g_ = y;
    c.y = x;
    return launch_pass(c, col_jds(p), pass::Tiles{p->col_tb.p + t0, (int32_t)(t1 - t0), stageable(p->col_unpacked, t0, t1)}, nullptr,
                       p->stream);
}

int launch_report(cf_plan* p, double mu, bool ax_ready, const cf_config* cfg, int64_t k, int64_t slot,
                  const int32_t* done, int64_t* launches) {
    (void)mu;
    int64_t nl = 0;
    if (!ax_ready) {
        CF_TRY(launch_spmv_rows(p, p->x.p, p->ax.p));
        nl += p->n_panels;
    }
    if (p->m > 0) {
        RowReportArgs a{};
        a.ax = p->ax.p;
        a.b = p->b.p;
        a.lam = p->lam.p;
        a.br = p->br_valid ? p->br.p : nullptr;
        a.amax = p->amax.p;
        a.part = p->part_row.p;
        a.m = (int32_t)p->m;
        a.done = done;
        CF_CUDA(launch_pdl(k_row_report, (unsigned)p->row_report_ctas, (unsigned)kThreads, 0, p->stream, a));
        ++nl;
    }
    int g_col = 0;
    if (p->n > 0) {
        ColReport c{};
        c.d2 = c.dmx = c.s2 = c.smx = c.amx = c.cx = c.cg = c.nf = 0.0;
        c.g_ = p->lam.p;
        c.x_in = p->x.p;
        c.z_in = p->z.p;
        c.d_in = p->delta.p;
        c.c = p->c.p;
        c.part = p->part_col.p;
        col_vecs_bands(p, c);
        CF_TRY(launch_col_bands(p, c, done, &nl, &g_col));
        g_col *= pass::kGroups;  // one partial per (field, group, CTA)
    }
    FinalizeArgs f{};
    f.part_row = p->part_row.p;
    f.part_col = p->part_col.p;
    f.nf_flag = nullptr;
    f.g_row = p->m > 0 ? p->row_report_ctas : 0;
    f.g_col = g_col;
    f.k = k;
    f.check = cfg ? 1 : 0;
    if (cfg) f.cfg = *cfg;
    f.slot = p->report_slot.p + slot;
    f.done = const_cast<int32_t*>(done);
    CF_CUDA(launch_pdl(k_finalize, 1u, 1024u, 0, p->stream, f));
    ++nl;
    if (launches) *launches += nl;
    return CF_OK;
}

int launch_project(cf_plan* p, const double* w, double* out) {
    if (p->n == 0) return CF_OK;
    if (p->all_unit) {
        k_project_lp<<<grid_for(p->n, 256), 256, 0, p->stream>>>(w, out, p->n);
        CF_LAUNCHED();
        return CF_OK;
    }
    k_project_small<<<grid_for(p->n_blocks, 128), 128, 0, p->stream>>>(w, out, p->cone_ptr.p, p->n_blocks);
    CF_LAUNCHED();
    if (p->n_big > 0) {
        BigConeArgs g{};
        g.big_cone = p->big_cone.p;
        g.cone_ptr = p->cone_ptr.p;
        g.wbuf = w;
        g.out = out;
        k_big_cone<<<(unsigned)p->n_big, 1024, 0, p->stream>>>(g);
        CF_LAUNCHED();
    }
    return CF_OK;
}

int launch_export(cf_plan* p, double mu, double* y, double* gamma) {
    if (p->n == 0 || p->o == 0) return CF_OK;
    const double* eps = (p->since_warm == 1) ? p->eps.p : nullptr;
    k_export<<<grid_for(p->n, 128), 128, 0, p->stream>>>(p->colptr.p, p->rowidx.p, p->valc.p, p->x.p, p->br.p,
                                                         p->lam.p, eps, mu, y, gamma, p->n);
    CF_LAUNCHED();
    return CF_OK;
}

int launch_warm_start(cf_plan* p, double mu) {
    if (p->n > 0) {
        k_warm_cols<<<grid_for(p->n, 128), 128, 0, p->stream>>>(p->colptr.p, p->rowidx.p, p->valc.p, p->y0.p,
                                                                p->gamma0.p, p->lam.p, mu, p->vterm1.p, p->eps.p,
                                                                p->ccorr.p, p->n);
        CF_LAUNCHED();
    }
    if (p->m > 0) {
        k_warm_rows<<<grid_for(p->m, 128), 128, 0, p->stream>>>(p->rowptr.p, p->valr.p, p->csr2csc.p, p->eps.p, mu,
                                                                p->rcorr.p, p->m, p->n_panels);
        CF_LAUNCHED();
    }
    return CF_OK;
}

int launch_row_diag(cf_plan* p) {
    if (p->m == 0) return CF_OK;
    k_row_diag<<<grid_for(p->m, 128), 128, 0, p->stream>>>(p->rowptr.p, p->valr.p, p->b.p, p->fu.p, p->db.p,
                                                          p->amax.p, p->dn.p, p->m, p->n_panels);
    CF_LAUNCHED();
    return CF_OK;
}

int launch_row_norms(cf_plan* p, double* dout, double* amax) {
    if (p->m == 0) return CF_OK;
    k_row_norms<<<grid_for(p->m, 128), 128, 0, p->stream>>>(p->rowptr.p, p->valr.p, dout, amax, p->m, p->n_panels);
    CF_LAUNCHED();
    return CF_OK;
}

int launch_set_row_diag(cf_plan* p, const double* din, const double* amax_in) {
    if (p->m == 0) return CF_OK;
    k_set_row_diag<<<grid_for(p->m, 128), 128, 0, p->stream>>>(din, amax_in, p->b.p, p->fu.p, p->db.p, p->amax.p,
                                                                p->dn.p, p->m);
    CF_LAUNCHED();
    return CF_OK;
}

int max_col_report_ctas() { return std::max(persistent_grid<ColReport>(1 << 30), kMediumTiles); }

// ---------------------------------------------------------------- row-sharded building blocks
namespace {
__global__ void k_col_update(int64_t n, const double* ath, const double* cnt, const double* c, double* x, double* z,
                             double* delta, double mu, int64_t n_blocks, const int32_t* cone_ptr, double* wbuf) {
    for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < n; j += (int64_t)gridDim.x * blockDim.x) {
        const double cj = cnt[j];
        const double fv = 1.0 / (1.0 + cj);
        const double xj = x[j], zj = z[j], dj = delta[j];
        const double dm = dj / mu;
        const double v = __dadd_rn(__dmul_rn(cj, xj), ath[j]);
        const double xp = fv * (((v + zj) + dm) - c[j] / mu);
        const double w = xp - dm;
        x[j] = xp;
        if (!cone_ptr) {
            const double zp = w > 0.0 ? w : 0.0;
            z[j] = zp;
            delta[j] = dj + mu * (zp - xp);
        } else {
            wbuf[j] = w;
        }
    }
}
// k_col_update with the reduce and the broadcast fused in: A^T h of the slice is the sum of
// the `world` ranks' partials read over P2P in rank order (deterministic), and x+ goes to
// every rank's x replica. Only x crosses the link on the way out; z and delta stay local.
__global__ void k_col_update_p2p(int64_t n, const double* const* parts, int world, const double* cnt,
                                 const double* c, double* x, double* z, double* delta, double mu,
                                 const int32_t* cone_ptr, double* wbuf, double* const* x_dst, int n_dst) {
    for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < n; j += (int64_t)gridDim.x * blockDim.x) {
        double ath = parts[0][j];
        for (int s = 1; s < world; ++s) ath = __dadd_rn(ath, parts[s][j]);
        const double cj = cnt[j];
        const double fv = 1.0 / (1.0 + cj);
        const double xj = x[j], zj = z[j], dj = delta[j];
        const double dm = dj / mu;
        const double v = __dadd_rn(__dmul_rn(cj, xj), ath);
        const double xp = fv * (((v + zj) + dm) - c[j] / mu);
        const double w = xp - dm;
        x[j] = xp;
        for (int s = 0; s < n_dst; ++s) x_dst[s][j] = xp;
        if (!cone_ptr) {
            const double zp = w > 0.0 ? w : 0.0;
            z[j] = zp;
            delta[j] = dj + mu * (zp - xp);
        } else {
            wbuf[j] = w;
        }
    }
    __threadfence_system();   // peer stores performed before the kernel retires
}
__global__ void k_cone_update(int64_t n_blocks, const int32_t* cone_ptr, const double* wbuf, const double* x,
                              double* z, double* delta, double mu) {
    for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < n_blocks;
         q += (int64_t)gridDim.x * blockDim.x) {
        const int off = cone_ptr[q], size = cone_ptr[q + 1] - off;
        project_block_dev(wbuf + off, size, z + off);
        for (int u = 0; u < size; ++u) delta[off + u] = delta[off + u] + mu * (z[off + u] - x[off + u]);
    }
}
// column parts of compute_report over a column slice: per-CTA partials (part[f * G + cta]),
// then k_col_parts_final reduces them in CTA order (deterministic)
__global__ void k_col_parts(int64_t n, const double* atl, const double* c, const double* x, const double* z,
                            const double* delta, double* part) {
    __shared__ double sh[32];
    const int G = gridDim.x;
    double d2 = 0.0, dmx = 0.0, s2 = 0.0, smx = 0.0, amx = 0.0, cx = 0.0, cg = 0.0, nf = 0.0;
    for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < n; j += (int64_t)G * blockDim.x) {
        const double dual = atl[j] + c[j];
        const double stat = dual - delta[j];
        d2 = d2 + dual * dual;
        dmx = nanmax(dmx, fabs(dual));
        s2 = s2 + stat * stat;
        smx = nanmax(smx, fabs(stat));
        amx = nanmax(amx, fabs(atl[j]));
        cx = cx + c[j] * x[j];
        cg = nanmax(cg, fabs(x[j] - z[j]));
        if (!isfinite(x[j]) || !isfinite(z[j]) || !isfinite(delta[j]) || !isfinite(atl[j])) nf = 1.0;
    }
    const double vals[8] = {d2, dmx, s2, smx, amx, cx, cg, nf};
    const bool is_sum[8] = {true, false, true, false, false, true, false, false};
    for (int f = 0; f < 8; ++f) {
        const double v = is_sum[f] ? block_reduce(vals[f], sh, SumOp()) : block_reduce(vals[f], sh, MaxOp());
        if (threadIdx.x == 0) part[f * G + blockIdx.x] = v;
    }
}
__global__ void k_col_parts_final(const double* part, int G, double* out) {
    __shared__ double sh[32];
    const bool is_sum[8] = {true, false, true, false, false, true, false, false};
    for (int f = 0; f < 8; ++f) {
        const double v = is_sum[f] ? reduce_partials(part + f * G, G, sh, SumOp()) : reduce_partials(part + f * G, G, sh, MaxOp());
        if (threadIdx.x == 0) out[f] = v;
    }
}
__global__ void k_row_parts_final(const double* part_row, int G, double* out) {
    __shared__ double sh[32];
    const SumOp sum;
    const MaxOp mx;
    const double f0 = reduce_partials(part_row + 0 * G, G, sh, sum);
    const double f1 = reduce_partials(part_row + 1 * G, G, sh, mx);
    const double f2 = reduce_partials(part_row + 2 * G, G, sh, mx);
    const double f3 = reduce_partials(part_row + 3 * G, G, sh, sum);
    const double f4 = reduce_partials(part_row + 4 * G, G, sh, mx);
    if (threadIdx.x == 0) {
        out[0] = f0;
        out[1] = f1;
        out[2] = f2;
        out[3] = f3;
        out[4] = f4;
    }
}
// the row epilogue of RowIter (y_update + lam/gamma, solver.py:179-183,194-195) from a
// full A x: the column-sharded driver's row step
__global__ void k_row_update(int64_t m, const double* ax, const double* b, const double* fu, const double* db,
                             double* lam, double* h, double* br, double mu, pass::MuDiv div) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m; i += (int64_t)gridDim.x * blockDim.x) {
        const double bi = b[i];
        const double r = fu[i] * (db[i] + ax[i]);
        const double ln = lam[i] + mu * (r - bi);
        const double bmr = bi - r;
        lam[i] = ln;
        h[i] = bmr - div(ln);
        if (br) br[i] = bmr;
    }
}
__global__ void k_counts(const int32_t* colptr, int64_t n, double* cnt) {
    for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < n; j += (int64_t)gridDim.x * blockDim.x)
        cnt[j] = (double)(colptr[j + 1] - colptr[j]);
}
}  // namespace

int launch_row_update(int64_t m, const double* ax, const double* b, const double* fu, const double* db, double* lam,
                      double* h, double* br, double mu, cudaStream_t st) {
    if (m == 0) return CF_OK;
    k_row_update<<<grid_for(m, 256), 256, 0, st>>>(m, ax, b, fu, db, lam, h, br, mu, pass::make_mudiv(mu));
    CF_LAUNCHED();
    return CF_OK;
}

int launch_col_update(int64_t n, const double* ath, const double* cnt, const double* c, double* x, double* z,
                      double* delta, double mu, int64_t n_blocks, const int32_t* cone_ptr, cudaStream_t st) {
    if (n == 0) return CF_OK;
    DevBuf<double> w;
    if (cone_ptr) CF_TRY(w.alloc(n));
    k_col_update<<<grid_for(n, 256), 256, 0, st>>>(n, ath, cnt, c, x, z, delta, mu, n_blocks, cone_ptr, w.p);
    CF_LAUNCHED();
    if (cone_ptr) {
        k_cone_update<<<grid_for(n_blocks, 128), 128, 0, st>>>(n_blocks, cone_ptr, w.p, x, z, delta, mu);
        CF_LAUNCHED();
        CF_CUDA(cudaStreamSynchronize(st));  // w is released at return
    }
    return CF_OK;
}

int launch_col_update_p2p(int64_t n, const double* const* parts, int world, const double* cnt, const double* c,
                          double* x, double* z, double* delta, double mu, int64_t n_blocks, const int32_t* cone_ptr,
                          double* const* x_dst, int n_dst, cudaStream_t st) {
    if (n == 0) return CF_OK;
    DevBuf<double> w;
    if (cone_ptr) CF_TRY(w.alloc(n));
    k_col_update_p2p<<<grid_for(n, 256), 256, 0, st>>>(n, parts, world, cnt, c, x, z, delta, mu, cone_ptr, w.p,
                                                       x_dst, n_dst);
    CF_LAUNCHED();
    if (cone_ptr) {
        k_cone_update<<<grid_for(n_blocks, 128), 128, 0, st>>>(n_blocks, cone_ptr, w.p, x, z, delta, mu);
        CF_LAUNCHED();
        CF_CUDA(cudaStreamSynchronize(st));  // w is released at return
    }
    return CF_OK;
}

int col_parts_ctas(int64_t n) { return (int)std::min<int64_t>(148 * 8, std::max<int64_t>(1, (n + 2047) / 2048)); }

int launch_col_parts(int64_t n, const double* atl, const double* c, const double* x, const double* z,
                     const double* delta, double* out8_dev, double* work, cudaStream_t st) {
    const int G = col_parts_ctas(n);
    k_col_parts<<<G, 256, 0, st>>>(n, atl, c, x, z, delta, work);
    CF_LAUNCHED();
    k_col_parts_final<<<1, 1024, 0, st>>>(work, G, out8_dev);
    CF_LAUNCHED();
    return CF_OK;
}

int launch_row_parts(cf_plan* p, double* out5_dev) {
    if (p->m == 0) {
        CF_CUDA(cudaMemsetAsync(out5_dev, 0, 5 * sizeof(double), p->stream));
        return CF_OK;
    }
    RowReportArgs a{};
    a.ax = p->ax.p;
    a.b = p->b.p;
    a.lam = p->lam.p;
    a.br = p->br_valid ? p->br.p : nullptr;
    a.amax = p->amax.p;
    a.part = p->part_row.p;
    a.m = (int32_t)p->m;
    k_row_report<<<p->row_report_ctas, kThreads, 0, p->stream>>>(a);
    CF_LAUNCHED();
    k_row_parts_final<<<1, 1024, 0, p->stream>>>(p->part_row.p, p->row_report_ctas, out5_dev);
    CF_LAUNCHED();
    return CF_OK;
}

int launch_row_parts_range(cf_plan* p, int64_t r0, int64_t r1, const double* ax, double* out5_dev) {
    if (r1 <= r0) {
        CF_CUDA(cudaMemsetAsync(out5_dev, 0, 5 * sizeof(double), p->stream));
        return CF_OK;
    }
    RowReportArgs a{};
    a.ax = ax;
    a.b = p->b.p + r0;
    a.lam = p->lam.p + r0;
    a.br = p->br_valid ? p->br.p + r0 : nullptr;
    a.amax = p->amax.p + r0;
    a.part = p->part_row.p;
    a.m = (int32_t)(r1 - r0);
    k_row_report<<<p->row_report_ctas, kThreads, 0, p->stream>>>(a);
    CF_LAUNCHED();
    k_row_parts_final<<<1, 1024, 0, p->stream>>>(p->part_row.p, p->row_report_ctas, out5_dev);
    CF_LAUNCHED();
    return CF_OK;
}

int launch_counts(cf_plan* p, double* cnt) {
    if (p->n == 0) return CF_OK;
    k_counts<<<grid_for(p->n, 256), 256, 0, p->stream>>>(p->colptr.p, p->n, cnt);
    CF_LAUNCHED();
    return CF_OK;
}

}  // namespace cf
