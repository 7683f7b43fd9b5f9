// Batched solver (SURVEY §2 "Batched solver", config C4): many independent small
// problems, each solved by ONE CTA that keeps the problem's CSR + CSC copy and all
// iterates in shared memory and runs the whole loop of solve() (solver.py:309-334)
// with per-problem termination. Persistent CTAs pull problems from an atomic queue,
// so a problem that needs 100k iterations does not hold up the others.
//
// The batch is set up as ONE block-diagonal problem through the plan's device
// setup (validate + canonical sort + CSR), so problem p owns rows
// [row_off[p], row_off[p+1]) and columns [col_off[p], col_off[p+1]) and its CSR
// and CSC slices are contiguous. Arithmetic is that of the plan's passes:
// sequential canonical-order sums (bit-identical to np.bincount), the same
// epilogue expressions, the same report assembly and termination test
// (cf_report.cuh). The reference's batch mechanism is a process pool over
// solve() (bench.py:96-106); solve_batch() returns what [solve(p) for p in ps]
// returns.
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <mutex>

#include "cf_common.h"
#include "cf_report.cuh"

namespace cf {
namespace {

#ifndef CF_CLUSTER_SEG
#define CF_CLUSTER_SEG 8   // loads in flight per batch in the cluster kernel's segment sums
#endif
#ifndef CF_BATCH_THREADS
#define CF_BATCH_THREADS 256
#endif
#ifndef CF_BATCH_MINB
#define CF_BATCH_MINB 4   // 4 problems per SM (C4: 114M -> 120M problem-iterations/s; the spills sit in the report)
#endif
constexpr int kBT = CF_BATCH_THREADS;   // threads per problem CTA

struct BatchArgs {
    int32_t P;
    const int64_t* row_off;   // P+1
    const int64_t* col_off;   // P+1
    const int64_t* cone_off;  // P+1 first cone of each problem (cones mode)
    const int32_t* rowptr;
    const int32_t* colidx;
    const double* valr;
    const int32_t* colptr;
    const int32_t* rowidx;
    const double* valc;
    const double* b;
    const double* c;
    const double* fu;
    const double* db;
    const int32_t* cone_ptr;
    int32_t cones;            // 0: all blocks of size 1
    const cf_config* cfg;     // per problem
    double* x_out;
    double* lam_out;
    cf_report* trace;         // [P][trace_cap]
    int64_t trace_cap;
    int32_t* n_reports;       // [P]
    cf_report* final_report;  // [P]
    int32_t* queue;
    int32_t cap_m, cap_n, cap_o, cap_k;   // smem capacities (rows, cols, nonzeros, cones)
};

__device__ __forceinline__ double nanmax_b(double a, double b) { return (a > b || a != a) ? a : b; }

template <bool MAX, int NT = kBT>
__device__ double block_reduce_b(double v, double* sh) {
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
        const double o = __shfl_xor_sync(0xffffffffu, v, off);
        v = MAX ? nanmax_b(v, o) : v + o;
    }
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    __syncthreads();
    if (l == 0) sh[w] = v;
    __syncthreads();
    if (w == 0) {
        v = (l < NT / 32) ? sh[l] : 0.0;
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) {
            const double o = __shfl_xor_sync(0xffffffffu, v, off);
            v = MAX ? nanmax_b(v, o) : v + o;
        }
    }
    return v;   // valid in thread 0
}

// x / mu; an exact multiply when mu is a power of two (x * (1/mu) == x / mu bit for bit)
struct MuDivB {
    double mu, inv;
    bool pow2;
    __device__ __forceinline__ double operator()(double x) const { return pow2 ? x * inv : x / mu; }
};
__device__ __forceinline__ MuDivB make_mudiv_b(double mu) {
    int e = 0;
    const double fr = frexp(mu, &e);
    return MuDivB{mu, 1.0 / mu, fr == 0.5 && e > -1000 && e < 1000};
}

// seg_dot with every load of a batch of kB issued before the batch's adds, the tail
// predicated instead of a one-by-one remainder loop: the dependent chain of a short
// segment is ceil(len/kB) x (idx -> gather) + len adds. Same sequential order of the same
// __dadd_rn/__dmul_rn, so bit-identical to seg_dot (the cluster kernel's passes are
// latency chains, not issue-bound like the batched kernel's).
template <int kB>
__device__ __forceinline__ double seg_dot_pf(const double* __restrict__ val, const int32_t* __restrict__ idx,
                                             const double* __restrict__ g, int p0, int p1) {
    double acc = 0.0;
    for (int q = p0; q < p1; q += kB) {
        int ii[kB];
        double vv[kB], gg[kB];
#pragma unroll
        for (int e = 0; e < kB; ++e) {
            ii[e] = q + e < p1 ? idx[q + e] : 0;
            vv[e] = q + e < p1 ? val[q + e] : 0.0;
        }
#pragma unroll
        for (int e = 0; e < kB; ++e) gg[e] = q + e < p1 ? g[ii[e]] : 0.0;
#pragma unroll
        for (int e = 0; e < kB; ++e)
            if (q + e < p1) acc = __dadd_rn(acc, __dmul_rn(vv[e], gg[e]));
    }
    return acc;
}

// sequential sum of val[q] * g[idx[q]] over [p0, p1) in order, four independent
// shared-memory loads in flight (the adds stay in canonical order)
__device__ __forceinline__ double seg_dot(const double* __restrict__ val, const int32_t* __restrict__ idx,
                                          const double* __restrict__ g, int p0, int p1) {
    double acc = 0.0;
    int q = p0;
    for (; q + 4 <= p1; q += 4) {
        const int i0 = idx[q], i1 = idx[q + 1], i2 = idx[q + 2], i3 = idx[q + 3];
        const double v0 = val[q], v1 = val[q + 1], v2 = val[q + 2], v3 = val[q + 3];
        const double g0 = g[i0], g1 = g[i1], g2 = g[i2], g3 = g[i3];
        acc = __dadd_rn(acc, __dmul_rn(v0, g0));
        acc = __dadd_rn(acc, __dmul_rn(v1, g1));
        acc = __dadd_rn(acc, __dmul_rn(v2, g2));
        acc = __dadd_rn(acc, __dmul_rn(v3, g3));
    }
    for (; q < p1; ++q) acc = __dadd_rn(acc, __dmul_rn(val[q], g[idx[q]]));
    return acc;
}

__device__ __forceinline__ void project_block_b(const double* w, int q, double* out) {
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

#ifndef CF_BATCH_RANK
#define CF_BATCH_RANK 1  // LP problems relabelled by row/column length (less divergence in the dot loops)
#endif
#ifndef CF_BATCH_SEG
#define CF_BATCH_SEG 0   // 0: seg_dot (unrolled by 4); N: seg_dot_pf<N>
#endif
__device__ __forceinline__ double batch_seg_dot(const double* __restrict__ val, const int32_t* __restrict__ idx,
                                                const double* __restrict__ g, int p0, int p1) {
#if CF_BATCH_SEG
    return seg_dot_pf<CF_BATCH_SEG>(val, idx, g, p0, p1);
#else
    return seg_dot(val, idx, g, p0, p1);
#endif
}

__global__ void __launch_bounds__(kBT, CF_BATCH_MINB) k_batch(const BatchArgs a) {
    extern __shared__ __align__(16) unsigned char smem[];
    const int CM = a.cap_m, CN = a.cap_n, CO = a.cap_o;
    // shared-memory carve-up (doubles first)
    double* valr = reinterpret_cast<double*>(smem);
    double* valc = valr + CO;
    double* b = valc + CO;
    double* fu = b + CM;
    double* db = fu + CM;
    double* lam = db + CM;
    double* h = lam + CM;
    double* br = h + CM;
    double* ax = br + CM;
    double* c = ax + CM;
    double* x = c + CN;
    double* z = x + CN;
    double* dl = z + CN;
    double* wv = dl + CN;     // cones: x+ - delta/mu, then z+
    double* fvs = wv + CN;    // 1/(1+cnt_j) (uv.py:82), constant per problem
    double* cmu = fvs + CN;   // c_j / mu, constant per problem
    double* red = cmu + CN;   // 32
    int32_t* colidx = reinterpret_cast<int32_t*>(red + 32);
    int32_t* rowidx = colidx + CO;
    int32_t* rowptr = rowidx + CO;
    int32_t* colptr = rowptr + CM + 1;
    int32_t* cptr = colptr + CN + 1;   // cone offsets (local), cap_k + 1
#if CF_BATCH_RANK
    int32_t* cperm = cptr + a.cap_k + 1;   // columns by length, longest first (cap_n)
    int32_t* rperm = cperm + CN;           // rows by length, longest first (cap_m)
#endif
    __shared__ int32_t s_prob, s_status;
    const int t = threadIdx.x;

    for (;;) {
        if (t == 0) s_prob = atomicAdd(a.queue, 1);
        __syncthreads();
        const int pid = s_prob;
        if (pid >= a.P) break;
        const int64_t r0 = a.row_off[pid], c0 = a.col_off[pid];
        const int m = (int)(a.row_off[pid + 1] - r0), n = (int)(a.col_off[pid + 1] - c0);
        const int64_t kr0 = a.rowptr[r0], kc0 = a.colptr[c0];
        const int o = (int)(a.colptr[c0 + n] - kc0);
        const cf_config cfg = a.cfg[pid];
        const double mu = cfg.mu;
        const MuDivB div = make_mudiv_b(mu);
        // ---- load the problem (canonical CSC, CSR, vectors) and a cold start (solver.py:309)
        CF_DASSERT(m >= 0 && n >= 0 && o >= 0 && m <= a.cap_m && n <= a.cap_n && o <= a.cap_o);
#if CF_BATCH_RANK
        // LP problems are relabelled: rows and columns in order of decreasing length (ties by
        // index), so the lanes of a warp run dot loops of similar lengths (a warp costs its
        // longest lane) and the epilogues stay contiguous in shared memory. Only labels
        // change: every row and column keeps its entries in canonical order, so each sum is
        // the same sequence of operations and the iterates are unchanged (the report's
        // cross-thread sums associate differently: rounding only). Cone problems keep
        // their natural order (a cone is a contiguous column range).
        const bool ranked = !a.cones;
        if (ranked) {
            int32_t* crank = reinterpret_cast<int32_t*>(wv);   // scratch during the load (cap_n)
            int32_t* rrank = reinterpret_cast<int32_t*>(ax);   // (cap_m)
            for (int j = t; j < n; j += kBT) {
                const int64_t lj = a.colptr[c0 + j + 1] - a.colptr[c0 + j];
                int r = 0;
                for (int q = 0; q < n; ++q) {
                    const int64_t lq = a.colptr[c0 + q + 1] - a.colptr[c0 + q];
                    r += (lq > lj) || (lq == lj && q < j);
                }
                crank[j] = r;
                cperm[r] = j;
            }
            for (int i = t; i < m; i += kBT) {
                const int64_t li = a.rowptr[r0 + i + 1] - a.rowptr[r0 + i];
                int r = 0;
                for (int q = 0; q < m; ++q) {
                    const int64_t lq = a.rowptr[r0 + q + 1] - a.rowptr[r0 + q];
                    r += (lq > li) || (lq == li && q < i);
                }
                rrank[i] = r;
                rperm[r] = i;
            }
            __syncthreads();
            if (t == 0) {   // pointers in rank order
                colptr[0] = 0;
                for (int r = 0; r < n; ++r)
                    colptr[r + 1] = colptr[r] + (int32_t)(a.colptr[c0 + cperm[r] + 1] - a.colptr[c0 + cperm[r]]);
            } else if (t == 32) {
                rowptr[0] = 0;
                for (int r = 0; r < m; ++r)
                    rowptr[r + 1] = rowptr[r] + (int32_t)(a.rowptr[r0 + rperm[r] + 1] - a.rowptr[r0 + rperm[r]]);
            }
            __syncthreads();
            for (int r = t; r < n; r += kBT) {   // column r = natural column cperm[r], entries in order
                const int64_t g0 = a.colptr[c0 + cperm[r]];
                const int d0 = colptr[r], len = colptr[r + 1] - d0;
                for (int e = 0; e < len; ++e) {
                    rowidx[d0 + e] = rrank[a.rowidx[g0 + e] - r0];
                    valc[d0 + e] = a.valc[g0 + e];
                }
            }
            for (int r = t; r < m; r += kBT) {   // row r = natural row rperm[r]
                const int64_t g0 = a.rowptr[r0 + rperm[r]];
                const int d0 = rowptr[r], len = rowptr[r + 1] - d0;
                for (int e = 0; e < len; ++e) {
                    colidx[d0 + e] = crank[a.colidx[g0 + e] - c0];
                    valr[d0 + e] = a.valr[g0 + e];
                }
            }
            for (int r = t; r < m; r += kBT) {
                const int i = rperm[r];
                b[r] = a.b[r0 + i];
                fu[r] = a.fu[r0 + i];
                db[r] = a.db[r0 + i];
            }
            for (int r = t; r < n; r += kBT) {
                const int j = cperm[r];
                const double cj = a.c[c0 + j];
                c[r] = cj;
                cmu[r] = div(cj);
                fvs[r] = 1.0 / (1.0 + (double)(a.colptr[c0 + j + 1] - a.colptr[c0 + j]));
            }
            __syncthreads();   // crank / rrank (in wv / ax) are read above
        } else
#endif
        {
            for (int i = t; i <= m; i += kBT) rowptr[i] = (int32_t)(a.rowptr[r0 + i] - kr0);
            for (int j = t; j <= n; j += kBT) colptr[j] = (int32_t)(a.colptr[c0 + j] - kc0);
            for (int k = t; k < o; k += kBT) {
                colidx[k] = (int32_t)(a.colidx[kr0 + k] - c0);
                valr[k] = a.valr[kr0 + k];
                rowidx[k] = (int32_t)(a.rowidx[kc0 + k] - r0);
                valc[k] = a.valc[kc0 + k];
            }
            for (int i = t; i < m; i += kBT) {
                b[i] = a.b[r0 + i];
                fu[i] = a.fu[r0 + i];
                db[i] = a.db[r0 + i];
            }
            for (int j = t; j < n; j += kBT) {
                const double cj = a.c[c0 + j];
                c[j] = cj;
                cmu[j] = div(cj);
                fvs[j] = 1.0 / (1.0 + (double)(a.colptr[c0 + j + 1] - a.colptr[c0 + j]));
            }
        }
        for (int k = t; k < o; k += kBT) CF_DASSERT(colidx[k] >= 0 && colidx[k] < n && rowidx[k] >= 0 && rowidx[k] < m);
        for (int i = t; i < m; i += kBT) {
            lam[i] = 0.0;
            h[i] = 0.0;
            br[i] = 0.0;
        }
        for (int j = t; j < n; j += kBT) {
            x[j] = 0.0;
            z[j] = 0.0;
            dl[j] = 0.0;
        }
        int nk = 0;
        if (a.cones) {
            const int64_t q0 = a.cone_off[pid];
            nk = (int)(a.cone_off[pid + 1] - q0);
            for (int q = t; q <= nk; q += kBT) cptr[q] = (int32_t)(a.cone_ptr[q0 + q] - c0);
        }
        if (t == 0) s_status = CF_STATUS_RUNNING;
        __syncthreads();
        int nrep = 0;
        cf_report last{};
        // reports at k % check_every == 0 or k == max_iters (solver.py:319), tracked by a
        // countdown instead of a 64-bit modulo (a software division) per iteration
        int64_t next_report = cfg.check_every < cfg.max_iters ? cfg.check_every : cfg.max_iters;
        for (int64_t k = 1; k <= cfg.max_iters; ++k) {
            const bool report = k == next_report;
            if (report) next_report = (k + cfg.check_every < cfg.max_iters) ? k + cfg.check_every : cfg.max_iters;
            // ---- column pass: x_update, z_update, delta update (solver.py:168-176,186-188,196)
            for (int j = t; j < n; j += kBT) {
                const int p0 = colptr[j], p1 = colptr[j + 1];
                const double ath = batch_seg_dot(valc, rowidx, h, p0, p1);
                const int cnt = p1 - p0;
                const double fv = fvs[j];
                const double xj = x[j], zj = z[j], dj = dl[j];
                const double dm = div(dj);
                const double v = __dadd_rn(__dmul_rn((double)cnt, xj), ath);
                const double xp = fv * (((v + zj) + dm) - cmu[j]);
                const double w = xp - dm;
                x[j] = xp;
                if (!a.cones) {
                    const double zp = w > 0.0 ? w : 0.0;
                    z[j] = zp;
                    dl[j] = dj + mu * (zp - xp);
                } else {
                    wv[j] = w;
                }
            }
            if (a.cones) {
                __syncthreads();
                for (int q = t; q < nk; q += kBT) {
                    const int off = cptr[q], size = cptr[q + 1] - off;
                    project_block_b(wv + off, size, z + off);
                    for (int u = 0; u < size; ++u) dl[off + u] = dl[off + u] + mu * (z[off + u] - x[off + u]);
                }
            }
            __syncthreads();
            // ---- row pass: y_update + lam/gamma of dual_update (solver.py:179-183,194-195)
            for (int i = t; i < m; i += kBT) {
                const int p0 = rowptr[i], p1 = rowptr[i + 1];
                const double axi = batch_seg_dot(valr, colidx, x, p0, p1);
                const double bi = b[i];
                const double r = fu[i] * (db[i] + axi);
                const double ln = lam[i] + mu * (r - bi);
                const double bmr = bi - r;
                lam[i] = ln;
                h[i] = bmr - div(ln);
                if (report) {
                    br[i] = bmr;
                    ax[i] = axi;
                }
            }
            __syncthreads();
            if (!report) continue;
            // ---- compute_report (solver.py:206-242)
            double prim2 = 0.0, primi = 0.0, axm = 0.0, blam = 0.0, nfr = 0.0;
            for (int i = t; i < m; i += kBT) {
                const double pr = ax[i] - b[i];
                prim2 = prim2 + pr * pr;
                primi = nanmax_b(primi, fabs(pr));
                axm = nanmax_b(axm, fabs(ax[i]));
                blam = blam + b[i] * lam[i];
                if (!isfinite(lam[i])) nfr = 1.0;
            }
            double d2 = 0.0, dmx = 0.0, s2 = 0.0, smx = 0.0, amx = 0.0, cx = 0.0, cg = 0.0, nfc = 0.0;
            for (int j = t; j < n; j += kBT) {
                double atl = 0.0;
                for (int q = colptr[j]; q < colptr[j + 1]; ++q) {
                    const int i = rowidx[q];
                    const double pa = __dmul_rn(valc[q], lam[i]);
                    if (!isfinite(pa) || !isfinite(valc[q] * br[i])) nfc = 1.0;
                    atl = __dadd_rn(atl, pa);
                }
                const double dual = atl + c[j];
                const double stat = dual - dl[j];
                d2 = d2 + dual * dual;
                dmx = nanmax_b(dmx, fabs(dual));
                s2 = s2 + stat * stat;
                smx = nanmax_b(smx, fabs(stat));
                amx = nanmax_b(amx, fabs(atl));
                cx = cx + c[j] * x[j];
                cg = nanmax_b(cg, fabs(x[j] - z[j]));
                if (!isfinite(x[j]) || !isfinite(z[j]) || !isfinite(dl[j])) nfc = 1.0;
            }
            ReportFields f;
            f.prim2 = block_reduce_b<false>(prim2, red);
            f.prim_inf = block_reduce_b<true>(primi, red);
            f.ax_inf = block_reduce_b<true>(axm, red);
            f.blam = block_reduce_b<false>(blam, red);
            f.nf_row = block_reduce_b<true>(nfr, red);
            f.dual2 = block_reduce_b<false>(d2, red);
            f.dual_inf = block_reduce_b<true>(dmx, red);
            f.stat2 = block_reduce_b<false>(s2, red);
            f.stat_inf = block_reduce_b<true>(smx, red);
            f.atl_inf = block_reduce_b<true>(amx, red);
            f.pobj = block_reduce_b<false>(cx, red);
            f.cone_gap = block_reduce_b<true>(cg, red);
            f.nf_col = block_reduce_b<true>(nfc, red);
            if (t == 0) {
                cf_report r = assemble_report(f, k, false);
                r.status = decide_status(r, cfg, k);
                if (nrep < a.trace_cap) a.trace[(int64_t)pid * a.trace_cap + nrep] = r;
                ++nrep;
                last = r;
                s_status = r.status;
            }
            __syncthreads();
            if (s_status != CF_STATUS_RUNNING) break;
        }
        // ---- SolveResult (solver.py:329-334)
#if CF_BATCH_RANK
        if (ranked) {
            for (int r = t; r < n; r += kBT) a.x_out[c0 + cperm[r]] = x[r];
            for (int r = t; r < m; r += kBT) a.lam_out[r0 + rperm[r]] = lam[r];
        } else
#endif
        {
            for (int j = t; j < n; j += kBT) a.x_out[c0 + j] = x[j];
            for (int i = t; i < m; i += kBT) a.lam_out[r0 + i] = lam[i];
        }
        if (t == 0) {
            a.final_report[pid] = last;
            a.n_reports[pid] = nrep;
        }
        __syncthreads();
    }
}

size_t batch_smem(int cm, int cn, int co, int ck) {
    return sizeof(double) * (size_t)(2 * co + 7 * cm + 7 * cn + 32) +
           sizeof(int32_t) * ((size_t)2 * co + cm + 1 + cn + 1 + ck + 1 + (CF_BATCH_RANK ? (size_t)cn + cm : 0)) + 16;
}

}  // namespace
}  // namespace cf

using namespace cf;

extern "C" int cf_batch_solve(int64_t n_problems, const int64_t* row_off, const int64_t* col_off, int64_t o,
                              const int64_t* rows, const int64_t* cols, const double* vals, const double* b,
                              const double* c, int64_t n_blocks, const int64_t* block_sizes,
                              const cf_config* cfgs, double* x_out, double* lam_out, cf_report* final_reports,
                              int32_t* n_reports, cf_report* trace, int64_t trace_cap, cf_problem_checks* checks,
                              double* elapsed_ms) {
    if (n_problems < 1 || !row_off || !col_off || !cfgs || !x_out || !lam_out || !final_reports || !n_reports ||
        trace_cap < 0 || (trace_cap > 0 && !trace)) {
        set_error("cf_batch_solve: bad arguments");
        return CF_EINVAL;
    }
    const int64_t P = n_problems, M = row_off[P], N = col_off[P];
    if (row_off[0] != 0 || col_off[0] != 0 || P >= INT32_MAX) {
        set_error("cf_batch_solve: offsets must start at 0");
        return CF_EINVAL;
    }
    int cap_m = 0, cap_n = 0;
    for (int64_t p = 0; p < P; ++p) {
        if (row_off[p + 1] < row_off[p] || col_off[p + 1] < col_off[p]) {
            set_error("cf_batch_solve: offsets must be non-decreasing");
            return CF_EINVAL;
        }
        cap_m = std::max<int>(cap_m, (int)(row_off[p + 1] - row_off[p]));
        cap_n = std::max<int>(cap_n, (int)(col_off[p + 1] - col_off[p]));
        if (cfgs[p].max_iters < 1 || cfgs[p].check_every < 1 || !(cfgs[p].mu > 0)) {
            set_error("cf_batch_solve: invalid config of problem " + std::to_string(p));
            return CF_EINVAL;
        }
    }
    // one block-diagonal plan: device validate + canonical CSC + CSR (single panel, no pass tiles)
    cf_plan* plan = nullptr;
    int rc = cf_plan_create_mode(M, N, o, rows, cols, vals, b, c, n_blocks, block_sizes, 0, nullptr, checks,
                                 /*batch_mode=*/1, &plan);
    if (rc != CF_OK) return rc;
    struct Guard {
        cf_plan* p;
        ~Guard() { cf_plan_destroy(p); }
    } guard{plan};
    cudaStream_t st = plan->stream;
    // per-problem nonzeros and cones
    std::vector<int32_t> cp(N + 1);
    CF_CUDA(cudaMemcpyAsync(cp.data(), plan->colptr.p, (N + 1) * 4, cudaMemcpyDeviceToHost, st));
    CF_CUDA(cudaStreamSynchronize(st));
    int cap_o = 0;
    for (int64_t p = 0; p < P; ++p) cap_o = std::max<int>(cap_o, cp[col_off[p + 1]] - cp[col_off[p]]);
    std::vector<int64_t> cone_off(P + 1, 0);
    int cap_k = 0;
    if (!plan->all_unit) {
        std::vector<int64_t> starts(n_blocks + 1, 0);
        for (int64_t q = 0; q < n_blocks; ++q) starts[q + 1] = starts[q] + block_sizes[q];
        for (int64_t p = 0; p <= P; ++p) {
            const auto it = std::lower_bound(starts.begin(), starts.end(), col_off[p]);
            if (it == starts.end() || *it != col_off[p]) {
                set_error("cf_batch_solve: a cone block crosses the boundary of problem " + std::to_string(p));
                return CF_EINVAL;
            }
            cone_off[p] = it - starts.begin();
        }
        for (int64_t p = 0; p < P; ++p) cap_k = std::max<int>(cap_k, (int)(cone_off[p + 1] - cone_off[p]));
    }
    const size_t smem = batch_smem(cap_m, cap_n, cap_o, cap_k);
    int dev = 0, max_smem = 0, sms = 0;
    CF_CUDA(cudaGetDevice(&dev));
    CF_CUDA(cudaDeviceGetAttribute(&max_smem, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev));
    CF_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    if (smem > (size_t)max_smem) {
        set_error("cf_batch_solve: the largest problem needs " + std::to_string(smem) +
                  " bytes of shared memory (> " + std::to_string(max_smem) + "); solve it with cf_plan_solve");
        return CF_EINVAL;
    }
    // process-wide attribute: set once to the limit so concurrent batches never lower each other's
    static std::once_flag attr_once;
    static cudaError_t attr_err = cudaSuccess;
    std::call_once(attr_once, [&] {
        cudaFuncAttributes fa{};
        attr_err = cudaFuncGetAttributes(&fa, k_batch);
        if (attr_err == cudaSuccess)
            attr_err = cudaFuncSetAttribute(k_batch, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                            max_smem - (int)fa.sharedSizeBytes);
    });
    CF_CUDA(attr_err);
    int per_sm = 0;
    CF_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_batch, kBT, smem));
    const int grid = (int)std::min<int64_t>(P, (int64_t)std::max(per_sm, 1) * sms);
    // device-side arguments and outputs
    DevBuf<int64_t> d_roff, d_coff, d_koff;
    DevBuf<cf_config> d_cfg;
    DevBuf<double> d_x, d_lam;
    DevBuf<cf_report> d_final, d_trace;
    DevBuf<int32_t> d_nrep, d_queue;
    CF_TRY(d_roff.alloc(P + 1));
    CF_TRY(d_coff.alloc(P + 1));
    CF_TRY(d_koff.alloc(P + 1));
    CF_TRY(d_cfg.alloc(P));
    CF_TRY(d_x.alloc(N));
    CF_TRY(d_lam.alloc(M));
    CF_TRY(d_final.alloc(P));
    CF_TRY(d_trace.alloc(std::max<int64_t>(1, P * trace_cap)));
    CF_TRY(d_nrep.alloc(P));
    CF_TRY(d_queue.alloc(1));
    CF_CUDA(cudaMemcpyAsync(d_roff.p, row_off, (P + 1) * 8, cudaMemcpyHostToDevice, st));
    CF_CUDA(cudaMemcpyAsync(d_coff.p, col_off, (P + 1) * 8, cudaMemcpyHostToDevice, st));
    CF_CUDA(cudaMemcpyAsync(d_koff.p, cone_off.data(), (P + 1) * 8, cudaMemcpyHostToDevice, st));
    CF_CUDA(cudaMemcpyAsync(d_cfg.p, cfgs, P * sizeof(cf_config), cudaMemcpyHostToDevice, st));
    CF_CUDA(cudaMemsetAsync(d_queue.p, 0, 4, st));
    BatchArgs a{};
    a.P = (int32_t)P;
    a.row_off = d_roff.p;
    a.col_off = d_coff.p;
    a.cone_off = d_koff.p;
    a.rowptr = plan->rowptr.p;
    a.colidx = plan->colidx.p;
    a.valr = plan->valr.p;
    a.colptr = plan->colptr.p;
    a.rowidx = plan->rowidx.p;
    a.valc = plan->valc.p;
    a.b = plan->b.p;
    a.c = plan->c.p;
    a.fu = plan->fu.p;
    a.db = plan->db.p;
    a.cone_ptr = plan->cone_ptr.p;
    a.cones = plan->all_unit ? 0 : 1;
    a.cfg = d_cfg.p;
    a.x_out = d_x.p;
    a.lam_out = d_lam.p;
    a.trace = d_trace.p;
    a.trace_cap = trace_cap;
    a.n_reports = d_nrep.p;
    a.final_report = d_final.p;
    a.queue = d_queue.p;
    a.cap_m = cap_m;
    a.cap_n = cap_n;
    a.cap_o = cap_o;
    a.cap_k = cap_k;
    CF_CUDA(cudaEventRecord(plan->ev0, st));
    k_batch<<<grid, kBT, smem, st>>>(a);
    CF_LAUNCHED();
    CF_CUDA(cudaEventRecord(plan->ev1, st));
    CF_CUDA(cudaEventSynchronize(plan->ev1));
    float ms = 0.f;
    CF_CUDA(cudaEventElapsedTime(&ms, plan->ev0, plan->ev1));
    if (elapsed_ms) *elapsed_ms = ms;
    CF_CUDA(cudaMemcpyAsync(x_out, d_x.p, N * 8, cudaMemcpyDeviceToHost, st));
    CF_CUDA(cudaMemcpyAsync(lam_out, d_lam.p, M * 8, cudaMemcpyDeviceToHost, st));
    CF_CUDA(cudaMemcpyAsync(final_reports, d_final.p, P * sizeof(cf_report), cudaMemcpyDeviceToHost, st));
    CF_CUDA(cudaMemcpyAsync(n_reports, d_nrep.p, P * 4, cudaMemcpyDeviceToHost, st));
    if (trace_cap > 0)
        CF_CUDA(cudaMemcpyAsync(trace, d_trace.p, P * trace_cap * sizeof(cf_report), cudaMemcpyDeviceToHost, st));
    CF_CUDA(cudaStreamSynchronize(st));
    return CF_OK;
}

// ============================================================================
// Cluster-resident solver (mid-size problems, e.g. config C1): ONE problem spread
// over a thread-block cluster of C CTAs (C = 1..16). CTA q owns a contiguous,
// nonzero-balanced block of rows and a cone-aligned block of columns, keeps its
// CSR rows and CSC columns in shared memory, and holds a full REPLICA of the
// gathered vectors (x for the row pass, h for the column pass; lam and b - r on
// report iterations). After updating its slice a CTA stores it into every peer's
// replica through distributed shared memory, and one cluster barrier per pass
// orders the stores before the peers' gathers. The whole loop of solve()
// (solver.py:309-334) runs in one launch with two cluster barriers per iteration,
// in place of the plan's kernel chain (whose per-iteration cost at C1 is launch
// and dependent-latency bound). Arithmetic is k_batch's: the same sequential
// canonical-order sums and epilogue expressions, so x and lam are bit-identical to
// cf_plan_solve; the report's fixed-order reduction differs only in rounding.
// ============================================================================
#include <cooperative_groups.h>

#include <mutex>

namespace cf {
namespace {

namespace cg = cooperative_groups;

constexpr int kCT = 512;              // threads per cluster CTA
constexpr int kMaxCluster = 16;
// reports the cluster kernel keeps on the device (112 B each); larger max_iters/check_every
// ratios go to the plan path, whose host trace grows one report at a time
constexpr int64_t kMaxClusterTrace = 1 << 16;

struct ClusterArgs {
    int32_t C;
    int32_t M, N;                     // problem rows / columns (replica lengths)
    int32_t row_cut[kMaxCluster + 1];
    int32_t col_cut[kMaxCluster + 1];
    int32_t cone_cut[kMaxCluster + 1];
    const int32_t* rowptr;            // canonical CSR / CSC of the plan (global indices)
    const int32_t* colidx;
    const double* valr;
    const int32_t* colptr;
    const int32_t* rowidx;
    const double* valc;
    const double* b;
    const double* c;
    const double* fu;
    const double* db;
    const int32_t* cone_ptr;
    int32_t cones;
    cf_config cfg;
    double* x_out;
    double* lam_out;
    cf_report* trace;
    int64_t trace_cap;
    int32_t* n_reports;
    cf_report* final_report;
    int32_t cap_m, cap_n, cap_or, cap_oc, cap_k;
};

size_t cluster_smem(int M, int N, int cm, int cn, int cor, int coc, int ck) {
    // every term in size_t: m and n may reach INT32_MAX / 4 through the C ABI
    const size_t nd = (size_t)N + 3 * (size_t)M + (size_t)cor + (size_t)coc + 4 * (size_t)cm + 6 * (size_t)cn + 32 +
                      16 * (size_t)kMaxCluster;
    const size_t ni = (size_t)cor + (size_t)coc + (size_t)cm + 1 + (size_t)cn + 1 + (size_t)ck + 1;
    return sizeof(double) * nd + sizeof(int32_t) * ni + 16;
}

__global__ void __launch_bounds__(kCT, 1) k_cluster(const ClusterArgs a) {
    extern __shared__ __align__(16) unsigned char smem[];
    cg::cluster_group cluster = cg::this_cluster();
    const int q = (int)cluster.block_rank();
    const int C = a.C, M = a.M, N = a.N;
    const int CM = a.cap_m, CN = a.cap_n;
    double* xr = reinterpret_cast<double*>(smem);   // replicas (global indices)
    double* hr = xr + N;
    double* lamr = hr + M;
    double* brr = lamr + M;
    double* valr = brr + M;                          // own rows / columns
    double* valc = valr + a.cap_or;
    double* b = valc + a.cap_oc;
    double* fu = b + CM;
    double* db = fu + CM;
    double* ax = db + CM;
    double* c = ax + CM;
    double* z = c + CN;
    double* dl = z + CN;
    double* wv = dl + CN;
    double* fvs = wv + CN;
    double* cmu = fvs + CN;
    double* red = cmu + CN;                          // 32
    double* parts = red + 32;                        // [C][16] report partials (CTA 0)
    int32_t* colidx = reinterpret_cast<int32_t*>(parts + 16 * kMaxCluster);
    int32_t* rowidx = colidx + a.cap_or;
    int32_t* rowptr = rowidx + a.cap_oc;
    int32_t* colptr = rowptr + CM + 1;
    int32_t* cptr = colptr + CN + 1;
    __shared__ int32_t s_status;
    __shared__ double* s_peer_x[kMaxCluster];
    __shared__ double* s_peer_h[kMaxCluster];
    __shared__ double* s_peer_lam[kMaxCluster];
    __shared__ double* s_peer_br[kMaxCluster];
    __shared__ int32_t* s_peer_status[kMaxCluster];
    __shared__ double* s_parts0;
    const int t = threadIdx.x;
    const int r0 = a.row_cut[q], m = a.row_cut[q + 1] - r0;
    const int c0 = a.col_cut[q], n = a.col_cut[q + 1] - c0;
    const int kr0 = a.rowptr[r0], kc0 = a.colptr[c0];
    const int orr = a.rowptr[r0 + m] - kr0, occ = a.colptr[c0 + n] - kc0;
    const cf_config& cfg = a.cfg;
    const double mu = cfg.mu;
    const MuDivB div = make_mudiv_b(mu);
    // ---- load the CTA's rows and columns, cold start (solver.py:309)
    for (int i = t; i <= m; i += kCT) rowptr[i] = a.rowptr[r0 + i] - kr0;
    for (int j = t; j <= n; j += kCT) colptr[j] = a.colptr[c0 + j] - kc0;
    CF_DASSERT(m <= a.cap_m && n <= a.cap_n && orr <= a.cap_or && occ <= a.cap_oc);
    for (int k = t; k < orr; k += kCT) {
        colidx[k] = a.colidx[kr0 + k];
        CF_DASSERT(colidx[k] >= 0 && colidx[k] < N);
        valr[k] = a.valr[kr0 + k];
    }
    for (int k = t; k < occ; k += kCT) {
        rowidx[k] = a.rowidx[kc0 + k];
        CF_DASSERT(rowidx[k] >= 0 && rowidx[k] < M);
        valc[k] = a.valc[kc0 + k];
    }
    for (int i = t; i < M; i += kCT) {
        hr[i] = 0.0;
        lamr[i] = 0.0;
        brr[i] = 0.0;
    }
    for (int j = t; j < N; j += kCT) xr[j] = 0.0;
    for (int i = t; i < m; i += kCT) {
        b[i] = a.b[r0 + i];
        fu[i] = a.fu[r0 + i];
        db[i] = a.db[r0 + i];
        ax[i] = 0.0;
    }
    for (int j = t; j < n; j += kCT) {
        const double cj = a.c[c0 + j];
        c[j] = cj;
        cmu[j] = div(cj);
        fvs[j] = 1.0 / (1.0 + (double)(a.colptr[c0 + j + 1] - a.colptr[c0 + j]));
        z[j] = 0.0;
        dl[j] = 0.0;
    }
    int nk = 0;
    if (a.cones) {
        const int k0 = a.cone_cut[q];
        nk = a.cone_cut[q + 1] - k0;
        for (int u = t; u <= nk; u += kCT) cptr[u] = a.cone_ptr[k0 + u] - c0;
    }
    if (t < C) {
        s_peer_x[t] = cluster.map_shared_rank(xr, t);
        s_peer_h[t] = cluster.map_shared_rank(hr, t);
        s_peer_lam[t] = cluster.map_shared_rank(lamr, t);
        s_peer_br[t] = cluster.map_shared_rank(brr, t);
        s_peer_status[t] = cluster.map_shared_rank(&s_status, t);
    }
    if (t == 0) {
        s_status = CF_STATUS_RUNNING;
        s_parts0 = cluster.map_shared_rank(parts, 0);
    }
    cluster.sync();   // every CTA resident and initialised before any remote store
    int nrep = 0;
    cf_report last{};
    int64_t next_report = cfg.check_every < cfg.max_iters ? cfg.check_every : cfg.max_iters;
    for (int64_t k = 1; k <= cfg.max_iters; ++k) {
        const bool report = k == next_report;
        if (report) next_report = (k + cfg.check_every < cfg.max_iters) ? k + cfg.check_every : cfg.max_iters;
        // ---- column pass on the CTA's columns (solver.py:168-176,186-188,196)
        for (int j = t; j < n; j += kCT) {
            const int p0 = colptr[j], p1 = colptr[j + 1];
            const double ath = seg_dot_pf<CF_CLUSTER_SEG>(valc, rowidx, hr, p0, p1);
            const int cnt = p1 - p0;
            const double fv = fvs[j];
            const double xj = xr[c0 + j], zj = z[j], dj = dl[j];
            const double dm = div(dj);
            const double v = __dadd_rn(__dmul_rn((double)cnt, xj), ath);
            const double xp = fv * (((v + zj) + dm) - cmu[j]);
            const double w = xp - dm;
            xr[c0 + j] = xp;
            for (int u = 0; u < C; ++u)
                if (u != q) s_peer_x[u][c0 + j] = xp;
            if (!a.cones) {
                const double zp = w > 0.0 ? w : 0.0;
                z[j] = zp;
                dl[j] = dj + mu * (zp - xp);
            } else {
                wv[j] = w;
            }
        }
        if (a.cones) {
            __syncthreads();
            for (int u = t; u < nk; u += kCT) {
                const int off = cptr[u], size = cptr[u + 1] - off;
                project_block_b(wv + off, size, z + off);
                for (int e = 0; e < size; ++e) dl[off + e] = dl[off + e] + mu * (z[off + e] - xr[c0 + off + e]);
            }
        }
        cluster.sync();   // x replicas complete
        // ---- row pass on the CTA's rows (solver.py:179-183,194-195)
        for (int i = t; i < m; i += kCT) {
            const int p0 = rowptr[i], p1 = rowptr[i + 1];
            const double axi = seg_dot_pf<CF_CLUSTER_SEG>(valr, colidx, xr, p0, p1);
            const double bi = b[i];
            const double r = fu[i] * (db[i] + axi);
            const double ln = lamr[r0 + i] + mu * (r - bi);
            const double bmr = bi - r;
            const double hn = bmr - div(ln);
            hr[r0 + i] = hn;
            lamr[r0 + i] = ln;
            for (int u = 0; u < C; ++u)
                if (u != q) s_peer_h[u][r0 + i] = hn;
            if (report) {
                brr[r0 + i] = bmr;
                for (int u = 0; u < C; ++u)
                    if (u != q) {
                        s_peer_lam[u][r0 + i] = ln;
                        s_peer_br[u][r0 + i] = bmr;
                    }
                ax[i] = axi;
            }
        }
        cluster.sync();   // h (and on reports lam, b - r) replicas complete
        if (!report) continue;
        // ---- compute_report (solver.py:206-242): per-CTA partials, CTA 0 combines in rank order
        double prim2 = 0.0, primi = 0.0, axm = 0.0, blam = 0.0, nfr = 0.0;
        for (int i = t; i < m; i += kCT) {
            const double pr = ax[i] - b[i];
            prim2 = prim2 + pr * pr;
            primi = nanmax_b(primi, fabs(pr));
            axm = nanmax_b(axm, fabs(ax[i]));
            blam = blam + b[i] * lamr[r0 + i];
            if (!isfinite(lamr[r0 + i])) nfr = 1.0;
        }
        double d2 = 0.0, dmx = 0.0, s2 = 0.0, smx = 0.0, amx = 0.0, cx = 0.0, cgp = 0.0, nfc = 0.0;
        for (int j = t; j < n; j += kCT) {
            double atl = 0.0;
            for (int p = colptr[j]; p < colptr[j + 1]; ++p) {
                const int i = rowidx[p];
                const double pa = __dmul_rn(valc[p], lamr[i]);
                if (!isfinite(pa) || !isfinite(valc[p] * brr[i])) nfc = 1.0;
                atl = __dadd_rn(atl, pa);
            }
            const double xj = xr[c0 + j];
            const double dual = atl + c[j];
            const double stat = dual - dl[j];
            d2 = d2 + dual * dual;
            dmx = nanmax_b(dmx, fabs(dual));
            s2 = s2 + stat * stat;
            smx = nanmax_b(smx, fabs(stat));
            amx = nanmax_b(amx, fabs(atl));
            cx = cx + c[j] * xj;
            cgp = nanmax_b(cgp, fabs(xj - z[j]));
            if (!isfinite(xj) || !isfinite(z[j]) || !isfinite(dl[j])) nfc = 1.0;
        }
        double f[13];
        f[0] = block_reduce_b<false, kCT>(prim2, red);
        f[1] = block_reduce_b<true, kCT>(primi, red);
        f[2] = block_reduce_b<true, kCT>(axm, red);
        f[3] = block_reduce_b<false, kCT>(blam, red);
        f[4] = block_reduce_b<true, kCT>(nfr, red);
        f[5] = block_reduce_b<false, kCT>(d2, red);
        f[6] = block_reduce_b<true, kCT>(dmx, red);
        f[7] = block_reduce_b<false, kCT>(s2, red);
        f[8] = block_reduce_b<true, kCT>(smx, red);
        f[9] = block_reduce_b<true, kCT>(amx, red);
        f[10] = block_reduce_b<false, kCT>(cx, red);
        f[11] = block_reduce_b<true, kCT>(cgp, red);
        f[12] = block_reduce_b<true, kCT>(nfc, red);
        if (t == 0)
            for (int e = 0; e < 13; ++e) s_parts0[q * 16 + e] = f[e];
        cluster.sync();
        if (q == 0 && t == 0) {
            double g[13];
            for (int e = 0; e < 13; ++e) g[e] = parts[e];
            for (int u = 1; u < C; ++u) {
                const double* pu = parts + u * 16;
                g[0] = g[0] + pu[0];
                g[1] = nanmax_b(g[1], pu[1]);
                g[2] = nanmax_b(g[2], pu[2]);
                g[3] = g[3] + pu[3];
                g[4] = nanmax_b(g[4], pu[4]);
                g[5] = g[5] + pu[5];
                g[6] = nanmax_b(g[6], pu[6]);
                g[7] = g[7] + pu[7];
                g[8] = nanmax_b(g[8], pu[8]);
                g[9] = nanmax_b(g[9], pu[9]);
                g[10] = g[10] + pu[10];
                g[11] = nanmax_b(g[11], pu[11]);
                g[12] = nanmax_b(g[12], pu[12]);
            }
            ReportFields rf;
            rf.prim2 = g[0];
            rf.prim_inf = g[1];
            rf.ax_inf = g[2];
            rf.blam = g[3];
            rf.nf_row = g[4];
            rf.dual2 = g[5];
            rf.dual_inf = g[6];
            rf.stat2 = g[7];
            rf.stat_inf = g[8];
            rf.atl_inf = g[9];
            rf.pobj = g[10];
            rf.cone_gap = g[11];
            rf.nf_col = g[12];
            cf_report r = assemble_report(rf, k, false);
            r.status = decide_status(r, cfg, k);
            if (nrep < a.trace_cap) a.trace[nrep] = r;
            last = r;
            s_status = r.status;
            for (int u = 1; u < C; ++u) *s_peer_status[u] = r.status;
        }
        ++nrep;
        cluster.sync();   // status visible everywhere; parts free for the next report
        if (s_status != CF_STATUS_RUNNING) break;
    }
    // ---- SolveResult (solver.py:329-334)
    for (int j = t; j < n; j += kCT) a.x_out[c0 + j] = xr[c0 + j];
    for (int i = t; i < m; i += kCT) a.lam_out[r0 + i] = lamr[r0 + i];
    if (q == 0 && t == 0) {
        *a.final_report = last;
        *a.n_reports = nrep;
    }
    cluster.sync();   // no CTA leaves while a peer may still address its shared memory
}

// positions (indices into allowed) of C+1 cuts balancing ptr's counts over the
// candidate boundaries allowed (increasing, allowed[0] = 0)
void balanced_cuts(const std::vector<int32_t>& ptr, const std::vector<int32_t>& allowed, int C, int32_t* cut) {
    const int64_t total = (int64_t)ptr[allowed.back()] - ptr[0];
    cut[0] = 0;
    size_t pos = 0;
    for (int q = 1; q < C; ++q) {
        const int64_t target = total * q / C;
        while (pos + 1 < allowed.size() && (int64_t)ptr[allowed[pos]] < target) ++pos;
        cut[q] = std::max<int32_t>(cut[q - 1], (int32_t)pos);
    }
    cut[C] = (int32_t)allowed.size() - 1;
}

}  // namespace
}  // namespace cf

namespace {
// cf_cluster_solve declines (cluster_used = 0, CF_OK) and the caller builds a plan;
// CF_VERBOSE=1 says why
int decline(const char* why) {
    if (getenv("CF_VERBOSE")) fprintf(stderr, "cf_cluster_solve: declined: %s\n", why);
    return CF_OK;
}
}  // namespace

extern "C" int cf_cluster_solve(int64_t m, int64_t n, int64_t o, const int64_t* rows, const int64_t* cols,
                                const double* vals, const double* b, const double* c, int64_t n_blocks,
                                const int64_t* block_sizes, const cf_config* cfg, double* x_out, double* lam_out,
                                cf_report* final_report, int32_t* n_reports, cf_report* trace, int64_t trace_cap,
                                cf_problem_checks* checks, int32_t* cluster_used, double* elapsed_ms) {
    if (m < 1 || n < 1 || o < 0 || !cfg || !x_out || !lam_out || !final_report || !n_reports || !cluster_used ||
        trace_cap < 0 || (trace_cap > 0 && !trace)) {
        set_error("cf_cluster_solve: bad arguments");
        return CF_EINVAL;
    }
    *cluster_used = 0;
    if (cfg->max_iters < 1 || cfg->check_every < 1 || !(cfg->mu > 0)) {
        set_error("cf_cluster_solve: invalid config");
        return CF_EINVAL;
    }
    if (m + 1 >= INT32_MAX / 4 || n + 1 >= INT32_MAX / 4) return CF_OK;   // not eligible
    {
        int ndev = 0;
        if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
            (void)cudaGetLastError();
            set_error("cf_cluster_solve: no CUDA device visible (libcfb200 has no CPU path)");
            return CF_ECUDA;
        }
    }
    // Decide the fit from host-side row/column counts BEFORE any device setup, so a problem
    // that does not fit costs one O(o) count here and the caller builds its plan only once.
    // Out-of-range entries are skipped; an invalid problem fails in cf_plan_create_mode below.
    std::vector<int32_t> rp(m + 1, 0), cp(n + 1, 0), kp;
    for (int64_t k = 0; k < o; ++k) {
        if (rows[k] >= 0 && rows[k] < m) ++rp[rows[k] + 1];
        if (cols[k] >= 0 && cols[k] < n) ++cp[cols[k] + 1];
    }
    for (int64_t i = 0; i < m; ++i) rp[i + 1] += rp[i];
    for (int64_t j = 0; j < n; ++j) cp[j + 1] += cp[j];
    int64_t maxsize = 0, ksum = 0;
    for (int64_t q = 0; q < n_blocks; ++q) maxsize = std::max<int64_t>(maxsize, block_sizes[q]);
    const bool all_unit = (n_blocks == 0 || maxsize == 1);
    if (!all_unit) {
        kp.resize(n_blocks + 1);
        kp[0] = 0;
        for (int64_t q = 0; q < n_blocks; ++q) {
            ksum += std::max<int64_t>(0, block_sizes[q]);
            if (ksum > n) return CF_OK;   // invalid cones: the plan path reports it
            kp[q + 1] = (int32_t)ksum;
        }
    }
    int dev = 0, max_smem = 0;
    CF_CUDA(cudaGetDevice(&dev));
    CF_CUDA(cudaDeviceGetAttribute(&max_smem, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev));
    // candidate cut points: every row; column cuts only at cone boundaries
    std::vector<int32_t> row_allowed(m + 1), col_allowed;
    for (int64_t i = 0; i <= m; ++i) row_allowed[i] = (int32_t)i;
    if (all_unit) {
        col_allowed.resize(n + 1);
        for (int64_t j = 0; j <= n; ++j) col_allowed[j] = (int32_t)j;
    } else {
        col_allowed = kp;
    }
    ClusterArgs a{};
    size_t smem = 0;
    int C = 0;
    const char* force = getenv("CF_CLUSTER_SIZE");   // experiments: try only this cluster size
    const int only = force ? atoi(force) : 0;
    for (int cand = 1; cand <= kMaxCluster; cand *= 2) {
        if (only > 0 && cand != only) continue;
        ClusterArgs t{};
        balanced_cuts(rp, row_allowed, cand, t.row_cut);
        std::vector<int32_t> kc(cand + 1);
        balanced_cuts(cp, col_allowed, cand, kc.data());
        for (int q = 0; q <= cand; ++q) {
            t.col_cut[q] = col_allowed[kc[q]];
            t.cone_cut[q] = all_unit ? 0 : kc[q];
        }
        int cm = 0, cn = 0, cor = 0, coc = 0, ck = 0;
        for (int q = 0; q < cand; ++q) {
            cm = std::max(cm, t.row_cut[q + 1] - t.row_cut[q]);
            cn = std::max(cn, t.col_cut[q + 1] - t.col_cut[q]);
            cor = std::max(cor, rp[t.row_cut[q + 1]] - rp[t.row_cut[q]]);
            coc = std::max(coc, cp[t.col_cut[q + 1]] - cp[t.col_cut[q]]);
            ck = std::max(ck, t.cone_cut[q + 1] - t.cone_cut[q]);
        }
        const size_t s = cluster_smem((int)m, (int)n, cm, cn, cor, coc, ck);
        if (s + 1024 > (size_t)max_smem) continue;   // room for the kernel's static shared memory
        t.C = cand;
        t.cap_m = cm;
        t.cap_n = cn;
        t.cap_or = cor;
        t.cap_oc = coc;
        t.cap_k = ck;
        a = t;
        smem = s;
        C = cand;
        // Measured (tools/cluster_sizes.py): a larger cluster shortens each CTA's
        // passes but adds barrier and remote-store cost. Take the smallest size with at most
        // ~2,800 nonzeros and 1,024 rows or columns per CTA, and at least 4 CTAs once o >= 2,000.
        if (cor <= 2800 && coc <= 2800 && cm <= 1024 && cn <= 1024 && (cand >= 4 || o < 2000)) break;
    }
    if (C == 0) return decline("no cluster size fits the shared memory");   // the caller uses cf_plan_solve
    if (trace_cap > kMaxClusterTrace) return decline("trace too long");   // the plan path streams its trace
    cf_plan* plan = nullptr;
    int rc = cf_plan_create_mode(m, n, o, rows, cols, vals, b, c, n_blocks, block_sizes, 0, nullptr, checks,
                                 /*batch_mode=*/1, &plan);
    if (rc != CF_OK) return rc;
    struct Guard {
        cf_plan* p;
        ~Guard() { cf_plan_destroy(p); }
    } guard{plan};
    cudaStream_t st = plan->stream;
    // function attributes are process-wide: set them once, to the limits, so concurrent
    // solves (solve_batch / run_bench threads) never lower each other's
    static std::once_flag attr_once;
    static cudaError_t attr_err = cudaSuccess;
    std::call_once(attr_once, [&] {
        cudaFuncAttributes fa{};
        attr_err = cudaFuncGetAttributes(&fa, k_cluster);
        if (attr_err == cudaSuccess)
            attr_err = cudaFuncSetAttribute(k_cluster, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                            max_smem - (int)fa.sharedSizeBytes);
        if (attr_err == cudaSuccess)
            attr_err = cudaFuncSetAttribute(k_cluster, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    });
    if (attr_err != cudaSuccess) return decline(cudaGetErrorString(attr_err));   // cannot configure the kernel
    DevBuf<double> d_x, d_lam;
    DevBuf<cf_report> d_final, d_trace;
    DevBuf<int32_t> d_nrep;
    // an out-of-memory here means "does not fit": decline, the plan path allocates its own
    if (d_x.alloc(n) != CF_OK || d_lam.alloc(m) != CF_OK || d_final.alloc(1) != CF_OK ||
        d_trace.alloc(std::max<int64_t>(1, trace_cap)) != CF_OK || d_nrep.alloc(1) != CF_OK) {
        (void)cudaGetLastError();
        return decline("out of device memory");
    }
    a.M = (int32_t)m;
    a.N = (int32_t)n;
    a.rowptr = plan->rowptr.p;
    a.colidx = plan->colidx.p;
    a.valr = plan->valr.p;
    a.colptr = plan->colptr.p;
    a.rowidx = plan->rowidx.p;
    a.valc = plan->valc.p;
    a.b = plan->b.p;
    a.c = plan->c.p;
    a.fu = plan->fu.p;
    a.db = plan->db.p;
    a.cone_ptr = plan->cone_ptr.p;
    a.cones = plan->all_unit ? 0 : 1;
    a.cfg = *cfg;
    a.x_out = d_x.p;
    a.lam_out = d_lam.p;
    a.trace = d_trace.p;
    a.trace_cap = trace_cap;
    a.n_reports = d_nrep.p;
    a.final_report = d_final.p;
    cudaLaunchConfig_t lc{};
    lc.gridDim = dim3(C, 1, 1);
    lc.blockDim = dim3(kCT, 1, 1);
    lc.dynamicSmemBytes = smem;
    lc.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = C;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    lc.attrs = attr;
    lc.numAttrs = 1;
    // a cluster of C CTAs with this much shared memory may not be schedulable (MPS, an
    // SM-limited context, a busy GPU): treat that like "does not fit"
    int active = 0;
    {
        const cudaError_t oe = cudaOccupancyMaxActiveClusters(&active, k_cluster, &lc);
        if (oe != cudaSuccess || active < 1) {
            (void)cudaGetLastError();
            return decline(oe != cudaSuccess ? cudaGetErrorString(oe) : "no active cluster of this size fits");
        }
    }
    CF_CUDA(cudaEventRecord(plan->ev0, st));
    {
        const cudaError_t le = cudaLaunchKernelEx(&lc, k_cluster, a);
        if (le == cudaErrorLaunchOutOfResources ||
            le == cudaErrorMemoryAllocation || le == cudaErrorInvalidClusterSize) {
            (void)cudaGetLastError();
            return decline(cudaGetErrorString(le));
        }
        CF_CUDA(le);
    }
    CF_LAUNCHED();
    CF_CUDA(cudaEventRecord(plan->ev1, st));
    CF_CUDA(cudaEventSynchronize(plan->ev1));
    float ms = 0.f;
    CF_CUDA(cudaEventElapsedTime(&ms, plan->ev0, plan->ev1));
    if (elapsed_ms) *elapsed_ms = ms;
    CF_CUDA(cudaMemcpyAsync(x_out, d_x.p, n * 8, cudaMemcpyDeviceToHost, st));
    CF_CUDA(cudaMemcpyAsync(lam_out, d_lam.p, m * 8, cudaMemcpyDeviceToHost, st));
    CF_CUDA(cudaMemcpyAsync(final_report, d_final.p, sizeof(cf_report), cudaMemcpyDeviceToHost, st));
    CF_CUDA(cudaMemcpyAsync(n_reports, d_nrep.p, 4, cudaMemcpyDeviceToHost, st));
    if (trace_cap > 0)
        CF_CUDA(cudaMemcpyAsync(trace, d_trace.p, trace_cap * sizeof(cf_report), cudaMemcpyDeviceToHost, st));
    CF_CUDA(cudaStreamSynchronize(st));
    *cluster_used = C;
    return CF_OK;
}
