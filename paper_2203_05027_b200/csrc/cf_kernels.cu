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
// Both passes run the same tile engine: a CTA owns a tile of up to kMaxSeg
// segments (rows or columns) whose nonzeros are contiguous; it streams the
// tile's (index, value) pairs with coalesced evict-first loads, gathers the
// dense operand (x or h, kept L2-resident with evict-last), stages the
// products in shared memory and then reduces each segment SEQUENTIALLY in
// storage order - the order np.bincount uses (uv.py:10-12) - so A x and
// A^T lam are bit-identical to the reference's apply_U(apply_Vt(x)) and
// apply_V(apply_Ut(lam)). Everything is compiled with -fmad=false so every
// fp64 operation rounds like its numpy counterpart.
#include <cmath>

#include "cf_common.h"

namespace cf {
namespace {

// ---------------------------------------------------------------- memory helpers
__device__ __forceinline__ uint64_t policy_evict_first() {
    uint64_t p;
    asm("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ uint64_t policy_evict_last() {
    uint64_t p;
    asm("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
    return p;
}
// streamed once per pass: do not pollute L1, leave L2 first
__device__ __forceinline__ double ld_stream(const double* ptr, uint64_t pol) {
    double v;
    asm("ld.global.nc.L1::no_allocate.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(v) : "l"(ptr), "l"(pol));
    return v;
}
__device__ __forceinline__ int32_t ld_stream(const int32_t* ptr, uint64_t pol) {
    int32_t v;
    asm("ld.global.nc.L1::no_allocate.L2::cache_hint.s32 %0, [%1], %2;" : "=r"(v) : "l"(ptr), "l"(pol));
    return v;
}
// random gather of the dense operand: keep it resident in L2
__device__ __forceinline__ double ld_gather(const double* ptr, uint64_t pol) {
    double v;
    asm("ld.global.nc.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(v) : "l"(ptr), "l"(pol));
    return v;
}
__device__ __forceinline__ void st_keep(double* ptr, double v, uint64_t pol) {
    asm volatile("st.global.L2::cache_hint.f64 [%0], %1, %2;" ::"l"(ptr), "d"(v), "l"(pol) : "memory");
}

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

// ---------------------------------------------------------------- tile engine
// sacc[s] = sum_{k in [sptr[s], sptr[s+1])} val[k] * g[idx[k]], sequential in k.
// Chunks of kCap products go through shared memory, so segments of any
// length are handled (a segment spanning chunks keeps its partial in sacc).
// Thread t owns segments t, t+kThreads, ... in both the init and the reduce
// phase, so no barrier is needed between them.
__device__ __forceinline__ void tile_gather_reduce(const int32_t* __restrict__ idx,
                                                   const double* __restrict__ val,
                                                   const double* __restrict__ g, const int32_t* sptr,
                                                   int nseg, double* sacc, double* sprod) {
    const uint64_t pol_s = policy_evict_first();
    const uint64_t pol_g = policy_evict_last();
    const int k0 = sptr[0], k1 = sptr[nseg];
    for (int s = threadIdx.x; s < nseg; s += kThreads) sacc[s] = 0.0;
    for (int c0 = k0; c0 < k1; c0 += kCap) {
        const int len = min(kCap, k1 - c0);
        const int32_t* ip = idx + c0;
        const double* vp = val + c0;
        int t = threadIdx.x;
        for (; t + 3 * kThreads < len; t += 4 * kThreads) {
            const int j0 = ld_stream(ip + t, pol_s);
            const int j1 = ld_stream(ip + t + kThreads, pol_s);
            const int j2 = ld_stream(ip + t + 2 * kThreads, pol_s);
            const int j3 = ld_stream(ip + t + 3 * kThreads, pol_s);
            const double a0 = ld_stream(vp + t, pol_s);
            const double a1 = ld_stream(vp + t + kThreads, pol_s);
            const double a2 = ld_stream(vp + t + 2 * kThreads, pol_s);
            const double a3 = ld_stream(vp + t + 3 * kThreads, pol_s);
            const double g0 = ld_gather(g + j0, pol_g);
            const double g1 = ld_gather(g + j1, pol_g);
            const double g2 = ld_gather(g + j2, pol_g);
            const double g3 = ld_gather(g + j3, pol_g);
            sprod[t] = __dmul_rn(a0, g0);
            sprod[t + kThreads] = __dmul_rn(a1, g1);
            sprod[t + 2 * kThreads] = __dmul_rn(a2, g2);
            sprod[t + 3 * kThreads] = __dmul_rn(a3, g3);
        }
        for (; t < len; t += kThreads)
            sprod[t] = __dmul_rn(ld_stream(vp + t, pol_s), ld_gather(g + ld_stream(ip + t, pol_s), pol_g));
        __syncthreads();
        for (int s = threadIdx.x; s < nseg; s += kThreads) {
            const int a = max(sptr[s], c0) - c0;
            const int e = min(sptr[s + 1], c0 + len) - c0;
            if (a < e) {
                double acc = sacc[s];
                for (int k = a; k < e; ++k) acc = __dadd_rn(acc, sprod[k]);
                sacc[s] = acc;
            }
        }
        __syncthreads();
    }
}

// ---------------------------------------------------------------- row pass
struct RowArgs {
    const int32_t* rowptr;
    const int32_t* colidx;
    const double* val;
    const double* x;      // gathered operand
    const double* b;
    const double* fu;
    const double* db;     // d * b
    double* lam;
    double* h;
    double* br;           // optional: b - r (SolverState.y export, report finiteness)
    double* ax;           // optional: A x (report)
    const double* rcorr;  // optional warm-start correction U eps / mu
    int32_t m;
    int32_t rows_per_tile;
    double mu;
    const int32_t* done;
};

// MODE 0: ADMM row update (y_update + lam/gamma parts of dual_update,
//         solver.py:179-183,194-195). MODE 1: ax = A x only (apply_U . apply_Vt).
template <int MODE>
__global__ void __launch_bounds__(kThreads) k_row_pass(const RowArgs a) {
    if (a.done && *a.done) return;
    __shared__ double sprod[kCap];
    __shared__ double sacc[kMaxSeg];
    __shared__ int32_t sptr[kMaxSeg + 1];
    const int r0 = blockIdx.x * a.rows_per_tile;
    const int nseg = min(a.rows_per_tile, a.m - r0);
    for (int s = threadIdx.x; s <= nseg; s += kThreads) sptr[s] = a.rowptr[r0 + s];
    __syncthreads();
    tile_gather_reduce(a.colidx, a.val, a.x, sptr, nseg, sacc, sprod);
    const uint64_t pol_keep = policy_evict_last();
    for (int s = threadIdx.x; s < nseg; s += kThreads) {
        const int i = r0 + s;
        const double axi = sacc[s];
        if (MODE == 1) {
            a.ax[i] = axi;
            continue;
        }
        const double bi = a.b[i], li = a.lam[i];
        double si = a.db[i] + axi;                 // (U t)_i with t = a b + x (App. A)
        if (a.rcorr) si = si - a.rcorr[i];
        const double r = a.fu[i] * si;              // r = U y+ = fu * U t
        const double ln = li + a.mu * (r - bi);    // solver.py:194
        const double bmr = bi - r;
        const double hi = bmr - ln / a.mu;          // h = b - r - lam+/mu
        a.lam[i] = ln;
        st_keep(a.h + i, hi, pol_keep);
        if (a.br) a.br[i] = bmr;
        if (a.ax) a.ax[i] = axi;
    }
}

// ---------------------------------------------------------------- column pass
struct ColArgs {
    const int32_t* colptr;
    const int32_t* rowidx;
    const double* val;
    const double* h;        // gathered operand
    const double* c;
    double* x;
    double* z;
    double* delta;
    const double* vterm;    // optional: V(y0 + gamma0/mu) replaces cnt*x + A^T h (first warm iteration)
    const double* ccorr;    // optional: V eps / mu subtracted (second warm iteration)
    const int32_t* tile_start;
    const int32_t* tile_cone;
    const int32_t* tile_big;
    const int32_t* cone_ptr;
    double* wbuf;
    int32_t n;
    int32_t cols_per_tile;
    double mu;
    const int32_t* done;
};

// Lorentz-cone projection of one block (cones.py:76-92; branch order :78-80).
// w, out, xp, dold, dnew are shared-memory (or global) arrays indexed by
// position inside the block.
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

// MODE 0: LP (all blocks of size 1, cones.py:108-109 shortcut), fused.
// MODE 1: general cones; small cones projected in the tile, big cones deferred.
// MODE 2: x = A^T y only (apply_V . apply_Ut).
template <int MODE>
__global__ void __launch_bounds__(kThreads) k_col_pass(const ColArgs a) {
    if (a.done && *a.done) return;
    __shared__ double sprod[kCap];
    __shared__ double sacc[kMaxSeg];
    __shared__ int32_t sptr[kMaxSeg + 1];
    int c0, nseg;
    if (a.tile_start) {
        c0 = a.tile_start[blockIdx.x];
        nseg = a.tile_start[blockIdx.x + 1] - c0;
    } else {
        c0 = blockIdx.x * a.cols_per_tile;
        nseg = min(a.cols_per_tile, a.n - c0);
    }
    for (int s = threadIdx.x; s <= nseg; s += kThreads) sptr[s] = a.colptr[c0 + s];
    __syncthreads();
    tile_gather_reduce(a.rowidx, a.val, a.h, sptr, nseg, sacc, sprod);
    if (MODE == 2) {
        for (int s = threadIdx.x; s < nseg; s += kThreads) a.x[c0 + s] = sacc[s];
        return;
    }
    const uint64_t pol_keep = policy_evict_last();
    const double mu = a.mu;
    // x-update (solver.py:168-176) in the reference's operand order:
    // fv * (((V(..) + z) + delta/mu) - c/mu)
    double* sxp = sprod;                 // x+      (reuses the product buffer)
    double* sw = sprod + kMaxSeg;        // x+ - delta/mu
    double* sd = sprod + 2 * kMaxSeg;    // delta (old)
    double* sdn = sprod + 3 * kMaxSeg;   // delta+
    for (int s = threadIdx.x; s < nseg; s += kThreads) {
        const int j = c0 + s;
        const int cnt = sptr[s + 1] - sptr[s];
        const double fv = 1.0 / (1.0 + (double)cnt);   // uv.py:82
        const double xj = a.x[j], zj = a.z[j], dj = a.delta[j], cj = a.c[j];
        const double dm = dj / mu;
        double v = a.vterm ? a.vterm[j] : __dadd_rn(__dmul_rn((double)cnt, xj), sacc[s]);
        if (a.ccorr) v = v - a.ccorr[j];
        const double xp = fv * (((v + zj) + dm) - cj / mu);
        const double w = xp - dm;                        // z_update argument, solver.py:188
        if (MODE == 0) {
            const double zp = w > 0.0 ? w : 0.0;         // np.where(w > 0, w, 0): NaN -> 0, -0 -> +0
            const double dp = dj + mu * (zp - xp);       // solver.py:196
            st_keep(a.x + j, xp, pol_keep);
            a.z[j] = zp;
            a.delta[j] = dp;
        } else {
            sxp[s] = xp;
            sw[s] = w;
            sd[s] = dj;
        }
    }
    if (MODE == 0) return;
    __syncthreads();
    const int big = a.tile_big[blockIdx.x];
    if (big >= 0) {  // part of a cone larger than kSmallCone: projected by k_big_cone
        for (int s = threadIdx.x; s < nseg; s += kThreads) {
            st_keep(a.x + c0 + s, sxp[s], pol_keep);
            a.wbuf[c0 + s] = sw[s];
        }
        return;
    }
    double* sz = sacc;  // A^T h no longer needed
    const int q0 = a.tile_cone[blockIdx.x], q1 = a.tile_cone[blockIdx.x + 1];
    for (int q = q0 + threadIdx.x; q < q1; q += kThreads) {
        const int off = a.cone_ptr[q] - c0;
        const int sz_q = a.cone_ptr[q + 1] - a.cone_ptr[q];
        project_block_dev(sw + off, sz_q, sz + off);
        for (int t = 0; t < sz_q; ++t) sdn[off + t] = sd[off + t] + mu * (sz[off + t] - sxp[off + t]);
    }
    __syncthreads();
    for (int s = threadIdx.x; s < nseg; s += kThreads) {
        st_keep(a.x + c0 + s, sxp[s], pol_keep);
        a.z[c0 + s] = sz[s];
        a.delta[c0 + s] = sdn[s];
    }
}

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
    double* part;    // [kReportFieldsRow][gridDim.x]
    int32_t m;
    const int32_t* done;
};
__global__ void __launch_bounds__(kThreads) k_row_report(const RowReportArgs a) {
    if (a.done && *a.done) return;
    __shared__ double sh[32];
    double s2 = 0.0, mx = 0.0, axm = 0.0, bl = 0.0, nf = 0.0;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < a.m; i += gridDim.x * blockDim.x) {
        const double axi = a.ax[i], bi = a.b[i], li = a.lam[i];
        const double pr = axi - bi;
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

// Column part (solver.py:215-218,223,225): atl = A^T lam (sequential,
// bincount order), dual = atl + c, stat = dual - delta; plus the finiteness
// of x, z, delta and of the implicit y_k = x_j + a_k (b_i - r_i) and
// gamma_k = -a_k lam_i (solver.py:208-211).
struct ColReportArgs {
    const int32_t* colptr;
    const int32_t* rowidx;
    const double* val;
    const double* lam;
    const double* br;    // may be null (then the y check reduces to x)
    const double* c;
    const double* x;
    const double* z;
    const double* delta;
    const int32_t* tile_start;
    int32_t n;
    int32_t cols_per_tile;
    double* part;        // [kReportFieldsCol][gridDim.x]
    const int32_t* done;
};
__global__ void __launch_bounds__(kThreads) k_col_report(const ColReportArgs a) {
    if (a.done && *a.done) return;
    __shared__ double sprod[kCap];
    __shared__ double sacc[kMaxSeg];
    __shared__ int32_t sptr[kMaxSeg + 1];
    __shared__ double sh[32];
    int c0, nseg;
    if (a.tile_start) {
        c0 = a.tile_start[blockIdx.x];
        nseg = a.tile_start[blockIdx.x + 1] - c0;
    } else {
        c0 = blockIdx.x * a.cols_per_tile;
        nseg = min(a.cols_per_tile, a.n - c0);
    }
    for (int s = threadIdx.x; s <= nseg; s += kThreads) sptr[s] = a.colptr[c0 + s];
    __syncthreads();
    double nf = 0.0;
    // same engine as the column pass, with the y/gamma checks in the gather loop
    {
        const uint64_t pol_s = policy_evict_first();
        const int k0 = sptr[0], k1 = sptr[nseg];
        for (int s = threadIdx.x; s < nseg; s += kThreads) sacc[s] = 0.0;
        for (int cc = k0; cc < k1; cc += kCap) {
            const int len = min(kCap, k1 - cc);
            for (int t = threadIdx.x; t < len; t += kThreads) {
                const int i = ld_stream(a.rowidx + cc + t, pol_s);
                const double av = ld_stream(a.val + cc + t, pol_s);
                const double p = __dmul_rn(av, a.lam[i]);
                if (!finite(p)) nf = 1.0;
                if (a.br && !finite(av * a.br[i])) nf = 1.0;
                sprod[t] = p;
            }
            __syncthreads();
            for (int s = threadIdx.x; s < nseg; s += kThreads) {
                const int lo = max(sptr[s], cc) - cc;
                const int hi = min(sptr[s + 1], cc + len) - cc;
                if (lo < hi) {
                    double acc = sacc[s];
                    for (int k = lo; k < hi; ++k) acc = __dadd_rn(acc, sprod[k]);
                    sacc[s] = acc;
                }
            }
            __syncthreads();
        }
    }
    double d2 = 0.0, dmx = 0.0, s2 = 0.0, smx = 0.0, amx = 0.0, cx = 0.0, cg = 0.0;
    for (int s = threadIdx.x; s < nseg; s += kThreads) {
        const int j = c0 + s;
        const double atl = sacc[s];
        const double xj = a.x[j], zj = a.z[j], dj = a.delta[j], cj = a.c[j];
        const double dual = atl + cj;
        const double stat = dual - dj;
        d2 = d2 + dual * dual;
        dmx = nanmax(dmx, fabs(dual));
        s2 = s2 + stat * stat;
        smx = nanmax(smx, fabs(stat));
        amx = nanmax(amx, fabs(atl));
        cx = cx + cj * xj;
        cg = nanmax(cg, fabs(xj - zj));
        if (!finite(xj) || !finite(zj) || !finite(dj)) nf = 1.0;
    }
    const int G = gridDim.x;
    double v;
    v = block_reduce(d2, sh, SumOp());
    if (threadIdx.x == 0) a.part[0 * G + blockIdx.x] = v;
    v = block_reduce(dmx, sh, MaxOp());
    if (threadIdx.x == 0) a.part[1 * G + blockIdx.x] = v;
    v = block_reduce(s2, sh, SumOp());
    if (threadIdx.x == 0) a.part[2 * G + blockIdx.x] = v;
    v = block_reduce(smx, sh, MaxOp());
    if (threadIdx.x == 0) a.part[3 * G + blockIdx.x] = v;
    v = block_reduce(amx, sh, MaxOp());
    if (threadIdx.x == 0) a.part[4 * G + blockIdx.x] = v;
    v = block_reduce(cx, sh, SumOp());
    if (threadIdx.x == 0) a.part[5 * G + blockIdx.x] = v;
    v = block_reduce(cg, sh, MaxOp());
    if (threadIdx.x == 0) a.part[6 * G + blockIdx.x] = v;
    v = block_reduce(nf, sh, MaxOp());
    if (threadIdx.x == 0) a.part[7 * G + blockIdx.x] = v;
}

struct FinalizeArgs {
    const double* part_row;
    const double* part_col;
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
    cf_report r;
    r.iter = a.k;
    r.prim_res_inf = f[1];
    r.prim_res_2 = sqrt(f[0]);
    r.dual_res_inf = f[6];
    r.dual_res_2 = sqrt(f[5]);
    r.stat_res_inf = f[8];
    r.stat_res_2 = sqrt(f[7]);
    r.ax_inf = f[2];
    r.atl_inf = f[9];
    r.cone_gap = f[11];
    r.pobj = f[10];
    const double blam = f[3];
    r.dobj = -blam;
    r.gap = r.pobj + blam;
    r.nonfinite = (f[4] > 0.0 || f[12] > 0.0) ? 1 : 0;
    int status = r.nonfinite ? CF_STATUS_DIVERGED : CF_STATUS_RUNNING;
    if (a.check && status == CF_STATUS_RUNNING) {
        const cf_config& c = a.cfg;
        bool ok;
        if (c.term_mode == CF_TERM_OSQP) {
            // Python max(a, b) returns a unless b > a
            const double mp = (c.b_inf > r.ax_inf) ? c.b_inf : r.ax_inf;
            const double md = (c.c_inf > r.atl_inf) ? c.c_inf : r.atl_inf;
            const double ep = c.eps_abs + c.eps_rel * mp;
            const double ed = c.eps_abs + c.eps_rel * md;
            ok = (r.prim_res_inf < ep) && (r.stat_res_inf < ed);
        } else if (c.term_mode == CF_TERM_SCS) {
            ok = (r.prim_res_2 <= c.scs_prim_bound) && (r.stat_res_2 <= c.scs_dual_bound) &&
                 (fabs(r.gap) <= c.eps_gap * ((1.0 + fabs(r.pobj)) + fabs(r.dobj)));
        } else {
            ok = (r.prim_res_2 < c.target_prim_res) && (fabs(r.gap) < c.target_gap);
        }
        status = ok ? CF_STATUS_SOLVED : CF_STATUS_RUNNING;
        if (status == CF_STATUS_RUNNING && a.k == c.max_iters) status = CF_STATUS_MAX_ITERS;
    }
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
                            double mu, double* rcorr, int64_t m) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m; i += (int64_t)gridDim.x * blockDim.x) {
        double s = 0.0;
        for (int p = rowptr[i]; p < rowptr[i + 1]; ++p) s = s + valr[p] * eps[csr2csc[p]];
        rcorr[i] = s / mu;
    }
}

// fu_i = 1/(1 + sum a^2) (uv.py:81, bincount order = CSR order), db_i = d_i b_i
__global__ void k_row_diag(const int32_t* rowptr, const double* valr, const double* b, double* fu, double* db,
                           int64_t m) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m; i += (int64_t)gridDim.x * blockDim.x) {
        double d = 0.0;
        for (int p = rowptr[i]; p < rowptr[i + 1]; ++p) d = d + valr[p] * valr[p];
        fu[i] = 1.0 / (1.0 + d);
        db[i] = d * b[i];
    }
}

inline int grid_for(int64_t work, int threads) {
    int64_t g = (work + threads - 1) / threads;
    if (g < 1) g = 1;
    if (g > 148 * 16) g = 148 * 16;
    return (int)g;
}

RowArgs row_args(cf_plan* p) {
    RowArgs a{};
    a.rowptr = p->rowptr.p;
    a.colidx = p->colidx.p;
    a.val = p->valr.p;
    a.x = p->x.p;
    a.b = p->b.p;
    a.fu = p->fu.p;
    a.db = p->db.p;
    a.lam = p->lam.p;
    a.h = p->h.p;
    a.m = (int32_t)p->m;
    a.rows_per_tile = p->rows_per_tile;
    return a;
}
ColArgs col_args(cf_plan* p) {
    ColArgs a{};
    a.colptr = p->colptr.p;
    a.rowidx = p->rowidx.p;
    a.val = p->valc.p;
    a.h = p->h.p;
    a.c = p->c.p;
    a.x = p->x.p;
    a.z = p->z.p;
    a.delta = p->delta.p;
    a.tile_start = p->all_unit ? nullptr : p->tile_start.p;
    a.tile_cone = p->tile_cone.p;
    a.tile_big = p->tile_big.p;
    a.cone_ptr = p->cone_ptr.p;
    a.wbuf = p->wbuf.p;
    a.n = (int32_t)p->n;
    a.cols_per_tile = p->cols_per_tile;
    return a;
}

}  // namespace

// ---------------------------------------------------------------- launch wrappers
int launch_iteration(cf_plan* p, const IterOpts& opt, const int32_t* done, int64_t* launches) {
    int64_t nl = 0;
    cudaEvent_t e_a = nullptr, e_b = nullptr, e_c = nullptr;
    if (p->profiling) {
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
    if (p->n > 0) {
        ColArgs a = col_args(p);
        a.vterm = opt.vterm;
        a.ccorr = opt.ccorr;
        a.mu = opt.mu;
        a.done = done;
        if (p->all_unit) {
            k_col_pass<0><<<(unsigned)p->col_tiles, kThreads, 0, p->stream>>>(a);
        } else {
            k_col_pass<1><<<(unsigned)p->col_tiles, kThreads, 0, p->stream>>>(a);
            if (p->n_big > 0) {
                BigConeArgs g{};
                g.big_cone = p->big_cone.p;
                g.cone_ptr = p->cone_ptr.p;
                g.wbuf = p->wbuf.p;
                g.x = p->x.p;
                g.z = p->z.p;
                g.delta = p->delta.p;
                g.mu = opt.mu;
                g.done = done;
                k_big_cone<<<(unsigned)p->n_big, 1024, 0, p->stream>>>(g);
                ++nl;
            }
        }
        ++nl;
        CF_LAUNCHED();
    }
    if (p->profiling) CF_CUDA(cudaEventRecord(e_b, p->stream));
    if (p->m > 0) {
        RowArgs a = row_args(p);
        a.mu = opt.mu;
        a.done = done;
        a.rcorr = opt.rcorr;
        a.br = (opt.report || p->keep_br) ? p->br.p : nullptr;
        a.ax = opt.report ? p->ax.p : nullptr;
        k_row_pass<0><<<(unsigned)p->row_tiles, kThreads, 0, p->stream>>>(a);
        ++nl;
        CF_LAUNCHED();
    }
    if (p->profiling) CF_CUDA(cudaEventRecord(e_c, p->stream));
    if (launches) *launches += nl;
    return CF_OK;
}

void prof_reset(cf_plan* p) {
    p->prof_used = 0;
    p->prof_row_ms = p->prof_col_ms = 0.0;
}

void prof_collect(cf_plan* p) {
    for (size_t i = 0; i + 3 <= p->prof_used; i += 3) {
        float t1 = 0.f, t2 = 0.f;
        cudaEventElapsedTime(&t1, p->prof_events[i], p->prof_events[i + 1]);
        cudaEventElapsedTime(&t2, p->prof_events[i + 1], p->prof_events[i + 2]);
        p->prof_col_ms += t1;
        p->prof_row_ms += t2;
    }
    p->prof_used = 0;
}

int launch_spmv_rows(cf_plan* p, const double* x, double* y) {
    if (p->m == 0) return CF_OK;
    RowArgs a = row_args(p);
    a.x = x;
    a.ax = y;
    k_row_pass<1><<<(unsigned)p->row_tiles, kThreads, 0, p->stream>>>(a);
    CF_LAUNCHED();
    return CF_OK;
}

int launch_spmv_cols(cf_plan* p, const double* y, double* x) {
    if (p->n == 0) return CF_OK;
    ColArgs a = col_args(p);
    a.h = y;
    a.x = x;
    k_col_pass<2><<<(unsigned)p->col_tiles, kThreads, 0, p->stream>>>(a);
    CF_LAUNCHED();
    return CF_OK;
}

int launch_report(cf_plan* p, double mu, bool ax_ready, const cf_config* cfg, int64_t k, int64_t slot,
                  const int32_t* done, int64_t* launches) {
    (void)mu;
    int64_t nl = 0;
    if (!ax_ready) {
        CF_TRY(launch_spmv_rows(p, p->x.p, p->ax.p));
        ++nl;
    }
    if (p->m > 0) {
        RowReportArgs a{};
        a.ax = p->ax.p;
        a.b = p->b.p;
        a.lam = p->lam.p;
        a.part = p->part_row.p;
        a.m = (int32_t)p->m;
        a.done = done;
        k_row_report<<<p->row_report_ctas, kThreads, 0, p->stream>>>(a);
        ++nl;
        CF_LAUNCHED();
    }
    if (p->n > 0) {
        ColReportArgs a{};
        a.colptr = p->colptr.p;
        a.rowidx = p->rowidx.p;
        a.val = p->valc.p;
        a.lam = p->lam.p;
        a.br = p->br_valid ? p->br.p : nullptr;
        a.c = p->c.p;
        a.x = p->x.p;
        a.z = p->z.p;
        a.delta = p->delta.p;
        a.tile_start = p->all_unit ? nullptr : p->tile_start.p;
        a.n = (int32_t)p->n;
        a.cols_per_tile = p->cols_per_tile;
        a.part = p->part_col.p;
        a.done = done;
        k_col_report<<<(unsigned)p->col_tiles, kThreads, 0, p->stream>>>(a);
        ++nl;
        CF_LAUNCHED();
    }
    FinalizeArgs f{};
    f.part_row = p->part_row.p;
    f.part_col = p->part_col.p;
    f.g_row = p->m > 0 ? p->row_report_ctas : 0;
    f.g_col = p->n > 0 ? (int32_t)p->col_tiles : 0;
    f.k = k;
    f.check = cfg ? 1 : 0;
    if (cfg) f.cfg = *cfg;
    f.slot = p->report_slot.p + slot;
    f.done = const_cast<int32_t*>(done);
    k_finalize<<<1, 1024, 0, p->stream>>>(f);
    ++nl;
    CF_LAUNCHED();
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
                                                                p->rcorr.p, p->m);
        CF_LAUNCHED();
    }
    return CF_OK;
}

int launch_row_diag(cf_plan* p) {
    if (p->m == 0) return CF_OK;
    k_row_diag<<<grid_for(p->m, 128), 128, 0, p->stream>>>(p->rowptr.p, p->valr.p, p->b.p, p->fu.p, p->db.p, p->m);
    CF_LAUNCHED();
    return CF_OK;
}

}  // namespace cf
