// C ABI of libcfb200 (include/cfb200.h): plan lifetime, warm start / state
// export, the iteration loop of solve() (solver.py:309-334) with device-side
// termination, and the matrix-free operators.
#include <nvtx3/nvToolsExt.h>
#include <atomic>
#include <cstdio>
#include <vector>
#include <algorithm>
#include <cstring>
#include <string>
#include <vector>

#include "cf_common.h"

namespace cf {

static thread_local std::string g_last_error;

void set_error(const std::string& msg) { g_last_error = msg; }

cudaError_t pool_alloc(void** p, size_t bytes) {
    static thread_local int configured_dev = -1;
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    if (configured_dev != dev) {
        cudaMemPool_t pool;
        if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
            uint64_t keep = UINT64_MAX;
            cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
        }
        cudaGetLastError();
        configured_dev = dev;
    }
    e = cudaMallocAsync(p, bytes, 0);
    if (e != cudaSuccess) return e;
    return cudaStreamSynchronize(0);
}

void pool_free(void* p) {
    // callers synchronise the plan stream before releasing (plan destroy, scoped setup scratch)
    cudaFreeAsync(p, 0);
    cudaStreamSynchronize(0);
}

// checked build: canary bytes behind every DevBuf (cf_common.h kGuardBytes)
static std::atomic<long long> g_guard_violations{0};
void guard_fill(void* p, size_t used, size_t total) {
    cudaMemset(static_cast<char*>(p) + used, 0xA5, total - used);
    cudaDeviceSynchronize();
}
void guard_check(const void* p, size_t used, size_t total) {
    std::vector<unsigned char> h(total - used);
    cudaDeviceSynchronize();
    if (cudaMemcpy(h.data(), static_cast<const char*>(p) + used, h.size(), cudaMemcpyDeviceToHost) != cudaSuccess) {
        cudaGetLastError();
        return;
    }
    for (size_t i = 0; i < h.size(); ++i) {
        if (h[i] != 0xA5) {
            fprintf(stderr, "CF_CHECKED: device buffer of %zu bytes written at byte %zu past its end\n", used, i);
            ++g_guard_violations;
            return;
        }
    }
}

int cuda_fail(cudaError_t e, const char* what, const char* file, int line) {
    cudaGetLastError();  // clear sticky-free errors
    set_error(std::string(what) + " failed: " + cudaGetErrorString(e) + " (" + file + ":" + std::to_string(line) + ")");
    return e == cudaErrorMemoryAllocation ? CF_ENOMEM : CF_ECUDA;
}

namespace {

int check_plan(const cf_plan* p, const char* fn) {
    if (!p) {
        set_error(std::string(fn) + ": plan is NULL");
        return CF_EINVAL;
    }
    return CF_OK;
}

int check_mu(double mu, const char* fn) {
    if (!(mu > 0)) {
        set_error(std::string(fn) + ": mu must be > 0");
        return CF_EINVAL;
    }
    return CF_OK;
}

// options of the next iteration: warm-start corrections
IterOpts next_opts(const cf_plan* p, double mu, bool report) {
    IterOpts o;
    o.mu = mu;
    o.report = report;
    if (p->since_warm == 0) {
        o.vterm = p->vterm1.p;
        o.rcorr = p->rcorr.p;
    } else if (p->since_warm == 1) {
        o.ccorr = p->ccorr.p;
    }
    return o;
}

void advance(cf_plan* p, int64_t iters, bool br_written) {
    p->iter += iters;
    p->since_warm = (int)std::min<int64_t>(2, p->since_warm + iters);
    if (iters > 0) p->br_valid = br_written;
}

}  // namespace
}  // namespace cf

using namespace cf;

extern "C" {

const char* cf_last_error(void) { return g_last_error.c_str(); }

int cf_abi_version(void) { return CF_ABI_VERSION; }

long long cf_debug_guard_violations(void) { return CF_CHECKED ? cf::g_guard_violations.load() : -1; }

int cf_device_count(int* count) {
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess) {
        cudaGetLastError();
        n = 0;
    }
    if (count) *count = n;
    return CF_OK;
}

int cf_plan_destroy(cf_plan* p) {
    if (!p) return CF_OK;
    if (p->stream) cudaStreamSynchronize(p->stream);
    if (p->host_reports) cudaFreeHost(p->host_reports);
    if (p->ev0) cudaEventDestroy(p->ev0);
    if (p->ev1) cudaEventDestroy(p->ev1);
    for (cudaEvent_t e : p->prof_events) cudaEventDestroy(e);
    cudaStream_t st = p->own_stream ? p->stream : nullptr;
    if (p->x_own) p->x.p = p->x_own;   // an external x (cf_plan_bind_x) belongs to the caller
    if (p->h_own) p->h.p = p->h_own;   // likewise an external h (cf_plan_bind_h)
    delete p;  // DevBuf destructors free device memory
    if (st) cudaStreamDestroy(st);
    return CF_OK;
}

int cf_plan_info(const cf_plan* p, int64_t* m, int64_t* n, int64_t* o, int64_t* row_tiles, int64_t* col_tiles,
                 int64_t* big_cones, int32_t* all_unit) {
    CF_TRY(check_plan(p, "cf_plan_info"));
    if (m) *m = p->m;
    if (n) *n = p->n;
    if (o) *o = p->o;
    if (row_tiles) *row_tiles = p->row_tiles;
    if (col_tiles) *col_tiles = p->col_tiles;
    if (big_cones) *big_cones = p->n_big;
    if (all_unit) *all_unit = p->all_unit ? 1 : 0;
    return CF_OK;
}

int cf_plan_set_rhs(cf_plan* p, const double* b, const double* c, int on_device) {
    CF_TRY(check_plan(p, "cf_plan_set_rhs"));
    const cudaMemcpyKind kind = on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice;
    if (b && p->m) CF_CUDA(cudaMemcpyAsync(p->b.p, b, p->m * 8, kind, p->stream));
    if (c && p->n) CF_CUDA(cudaMemcpyAsync(p->c.p, c, p->n * 8, kind, p->stream));
    if (b) CF_TRY(launch_row_diag(p));
    CF_CUDA(cudaStreamSynchronize(p->stream));
    return CF_OK;
}

int cf_plan_set_state(cf_plan* p, double mu, const double* x, const double* y, const double* z, const double* lam,
                      const double* gamma, const double* delta) {
    CF_TRY(check_plan(p, "cf_plan_set_state"));
    CF_TRY(check_mu(mu, "cf_plan_set_state"));
    const int given = (x != nullptr) + (y != nullptr) + (z != nullptr) + (lam != nullptr) + (gamma != nullptr) +
                      (delta != nullptr);
    if (given != 0 && given != 6) {
        set_error("cf_plan_set_state: give all six vectors (warm start) or none (cold start)");
        return CF_EINVAL;
    }
    cudaStream_t st = p->stream;
    const int64_t m = p->m, n = p->n, o = p->o;
    p->br_valid = false;
    p->iter = 0;
    p->export_mu = mu;
    CF_CUDA(cudaMemsetAsync(p->h.p, 0, std::max<int64_t>(m, 1) * 8, st));
    if (given == 0) {
        CF_CUDA(cudaMemsetAsync(p->x.p, 0, std::max<int64_t>(n, 1) * 8, st));
        CF_CUDA(cudaMemsetAsync(p->z.p, 0, std::max<int64_t>(n, 1) * 8, st));
        CF_CUDA(cudaMemsetAsync(p->delta.p, 0, std::max<int64_t>(n, 1) * 8, st));
        CF_CUDA(cudaMemsetAsync(p->lam.p, 0, std::max<int64_t>(m, 1) * 8, st));
        p->since_warm = 2;
        p->y0.release();
        p->gamma0.release();
        CF_CUDA(cudaStreamSynchronize(st));
        return CF_OK;
    }
    if (n) {
        CF_CUDA(cudaMemcpyAsync(p->x.p, x, n * 8, cudaMemcpyHostToDevice, st));
        CF_CUDA(cudaMemcpyAsync(p->z.p, z, n * 8, cudaMemcpyHostToDevice, st));
        CF_CUDA(cudaMemcpyAsync(p->delta.p, delta, n * 8, cudaMemcpyHostToDevice, st));
    }
    if (m) CF_CUDA(cudaMemcpyAsync(p->lam.p, lam, m * 8, cudaMemcpyHostToDevice, st));
    CF_TRY(p->y0.alloc(o));
    CF_TRY(p->gamma0.alloc(o));
    CF_TRY(p->eps.alloc(o));
    CF_TRY(p->vterm1.alloc(n));
    CF_TRY(p->ccorr.alloc(n));
    CF_TRY(p->rcorr.alloc(m));
    if (o) {
        CF_CUDA(cudaMemcpyAsync(p->y0.p, y, o * 8, cudaMemcpyHostToDevice, st));
        CF_CUDA(cudaMemcpyAsync(p->gamma0.p, gamma, o * 8, cudaMemcpyHostToDevice, st));
    }
    CF_CUDA(cudaMemsetAsync(p->vterm1.p, 0, std::max<int64_t>(n, 1) * 8, st));
    CF_CUDA(cudaMemsetAsync(p->ccorr.p, 0, std::max<int64_t>(n, 1) * 8, st));
    CF_CUDA(cudaMemsetAsync(p->rcorr.p, 0, std::max<int64_t>(m, 1) * 8, st));
    CF_TRY(launch_warm_start(p, mu));
    p->since_warm = 0;
    CF_CUDA(cudaStreamSynchronize(st));  // host inputs may be freed after return
    return CF_OK;
}

int cf_plan_set_export(cf_plan* p, int keep) {
    CF_TRY(check_plan(p, "cf_plan_set_export"));
    p->keep_br = keep != 0;
    return CF_OK;
}

int cf_plan_get_state(cf_plan* p, double* x, double* y, double* z, double* lam, double* gamma, double* delta,
                      int64_t* iter) {
    CF_TRY(check_plan(p, "cf_plan_get_state"));
    cudaStream_t st = p->stream;
    const int64_t m = p->m, n = p->n, o = p->o;
    if (x && n) CF_CUDA(cudaMemcpyAsync(x, p->x.p, n * 8, cudaMemcpyDeviceToHost, st));
    if (z && n) CF_CUDA(cudaMemcpyAsync(z, p->z.p, n * 8, cudaMemcpyDeviceToHost, st));
    if (delta && n) CF_CUDA(cudaMemcpyAsync(delta, p->delta.p, n * 8, cudaMemcpyDeviceToHost, st));
    if (lam && m) CF_CUDA(cudaMemcpyAsync(lam, p->lam.p, m * 8, cudaMemcpyDeviceToHost, st));
    if (iter) *iter = p->iter;
    if ((y || gamma) && o) {
        if (p->iter == 0) {
            if (p->since_warm == 0) {
                if (y) CF_CUDA(cudaMemcpyAsync(y, p->y0.p, o * 8, cudaMemcpyDeviceToHost, st));
                if (gamma) CF_CUDA(cudaMemcpyAsync(gamma, p->gamma0.p, o * 8, cudaMemcpyDeviceToHost, st));
            } else {
                if (y) std::memset(y, 0, o * 8);
                if (gamma) std::memset(gamma, 0, o * 8);
            }
        } else {
            if (y && !p->br_valid) {
                set_error("cf_plan_get_state: y needs b - r of the last iteration; enable cf_plan_set_export "
                          "before iterating");
                return CF_ESTATE;
            }
            DevBuf<double> dy, dg;
            if (y) CF_TRY(dy.alloc(o));
            if (gamma) CF_TRY(dg.alloc(o));
            // mu only enters through eps (first iteration after a warm start)
            CF_TRY(launch_export(p, p->export_mu, y ? dy.p : nullptr, gamma ? dg.p : nullptr));
            if (y) CF_CUDA(cudaMemcpyAsync(y, dy.p, o * 8, cudaMemcpyDeviceToHost, st));
            if (gamma) CF_CUDA(cudaMemcpyAsync(gamma, dg.p, o * 8, cudaMemcpyDeviceToHost, st));
            CF_CUDA(cudaStreamSynchronize(st));
        }
    }
    CF_CUDA(cudaStreamSynchronize(st));
    return CF_OK;
}

int cf_plan_iterate(cf_plan* p, double mu, int64_t n_iters) {
    CF_TRY(check_plan(p, "cf_plan_iterate"));
    CF_TRY(check_mu(mu, "cf_plan_iterate"));
    if (n_iters < 0) {
        set_error("cf_plan_iterate: n_iters < 0");
        return CF_EINVAL;
    }
    int64_t launches = 0;
    p->export_mu = mu;
    prof_reset(p);
    CF_CUDA(cudaEventRecord(p->ev0, p->stream));
    for (int64_t t = 0; t < n_iters; ++t) {
        IterOpts opt = next_opts(p, mu, false);
        CF_TRY(launch_iteration(p, opt, nullptr, &launches));
        advance(p, 1, p->keep_br);
    }
    CF_CUDA(cudaEventRecord(p->ev1, p->stream));
    CF_CUDA(cudaEventSynchronize(p->ev1));
    prof_collect(p);
    float ms = 0;
    CF_CUDA(cudaEventElapsedTime(&ms, p->ev0, p->ev1));
    p->last_loop_ms = ms;
    p->last_launches = launches;
    p->last_timed_iters = n_iters;
    return CF_OK;
}

int cf_plan_report(cf_plan* p, double mu, cf_report* out) {
    CF_TRY(check_plan(p, "cf_plan_report"));
    CF_TRY(check_mu(mu, "cf_plan_report"));
    if (!out) {
        set_error("cf_plan_report: out is NULL");
        return CF_EINVAL;
    }
    CF_TRY(launch_report(p, mu, false, nullptr, p->iter, 0, nullptr, nullptr));
    CF_CUDA(cudaMemcpyAsync(out, p->report_slot.p, sizeof(cf_report), cudaMemcpyDeviceToHost, p->stream));
    CF_CUDA(cudaStreamSynchronize(p->stream));
    return CF_OK;
}

int cf_plan_solve(cf_plan* p, const cf_config* cfg, double* x_out, double* lam_out, cf_report* trace,
                  int64_t trace_cap, int64_t* n_reports) {
    CF_TRY(check_plan(p, "cf_plan_solve"));
    if (!cfg || !trace || !n_reports) {
        set_error("cf_plan_solve: NULL cfg/trace/n_reports");
        return CF_EINVAL;
    }
    CF_TRY(check_mu(cfg->mu, "cf_plan_solve"));
    if (cfg->max_iters < 1 || cfg->check_every < 1) {
        set_error("cf_plan_solve: max_iters and check_every must be >= 1");
        return CF_EINVAL;
    }
    const int64_t n_chunks = (cfg->max_iters + cfg->check_every - 1) / cfg->check_every;
    if (trace_cap < 0) {
        set_error("cf_plan_solve: trace_cap < 0");
        return CF_EINVAL;
    }
    *n_reports = 0;
    p->trace_all.clear();
    cudaStream_t st = p->stream;
    p->export_mu = cfg->mu;
    prof_reset(p);
    CF_CUDA(cudaMemsetAsync(p->done.p, 0, 4, st));
    constexpr int kDepth = 3;  // chunks in flight before the host looks at a report
    cudaEvent_t evs[kDepth];
    for (int i = 0; i < kDepth; ++i) CF_CUDA(cudaEventCreateWithFlags(&evs[i], cudaEventDisableTiming));
    int64_t launches = 0, read = 0, k_final = 0;
    bool finished = false;
    const int since_warm0 = p->since_warm;
    int rc = CF_OK;
    CF_CUDA(cudaEventRecord(p->ev0, st));
    auto consume = [&](int64_t c) -> int {
        CF_CUDA(cudaEventSynchronize(evs[c % kDepth]));
        const cf_report& r = p->host_reports[c % p->host_ring];
        p->trace_all.push_back(r);
        if (read < trace_cap) trace[read] = r;
        ++read;
        if (r.status != CF_STATUS_RUNNING) {
            finished = true;
            k_final = r.iter;
        }
        return CF_OK;
    };
    for (int64_t c = 0; c < n_chunks && !finished; ++c) {
        const int64_t k0 = c * cfg->check_every;
        const int64_t nit = std::min(cfg->check_every, cfg->max_iters - k0);
        nvtxRangePushA("cf chunk");
        struct PopRange {
            ~PopRange() { nvtxRangePop(); }
        } pop_range;
        for (int64_t i = 1; i <= nit; ++i) {
            IterOpts opt = next_opts(p, cfg->mu, i == nit);
            rc = launch_iteration(p, opt, p->done.p, &launches);
            if (rc != CF_OK) break;
            p->since_warm = (int)std::min<int64_t>(2, p->since_warm + 1);
        }
        if (rc != CF_OK) break;
        const int64_t slot = c % p->host_ring;
        rc = launch_report(p, cfg->mu, true, cfg, k0 + nit, slot, p->done.p, &launches);
        if (rc != CF_OK) break;
        CF_CUDA(cudaMemcpyAsync(p->host_reports + slot, p->report_slot.p + slot, sizeof(cf_report),
                                cudaMemcpyDeviceToHost, st));
        CF_CUDA(cudaEventRecord(evs[c % kDepth], st));
        if (c - read + 1 >= kDepth) CF_TRY(consume(read));
    }
    while (rc == CF_OK && !finished && read < n_chunks) {
        // drain the chunks still in flight
        const int64_t enq = std::min<int64_t>(n_chunks, read + kDepth);
        (void)enq;
        CF_TRY(consume(read));
    }
    CF_CUDA(cudaEventRecord(p->ev1, st));
    CF_CUDA(cudaEventSynchronize(p->ev1));
    prof_collect(p);
    for (int i = 0; i < kDepth; ++i) cudaEventDestroy(evs[i]);
    if (rc != CF_OK) return rc;
    float ms = 0;
    CF_CUDA(cudaEventElapsedTime(&ms, p->ev0, p->ev1));
    p->last_loop_ms = ms;
    p->last_launches = launches;
    if (!finished) k_final = cfg->max_iters;  // unreachable: the last report is max_iters
    p->last_timed_iters = k_final;
    // state bookkeeping: the device stopped after iteration k_final
    p->since_warm = since_warm0;
    advance(p, k_final, true);
    *n_reports = read;
    if (x_out && p->n) CF_CUDA(cudaMemcpyAsync(x_out, p->x.p, p->n * 8, cudaMemcpyDeviceToHost, st));
    if (lam_out && p->m) CF_CUDA(cudaMemcpyAsync(lam_out, p->lam.p, p->m * 8, cudaMemcpyDeviceToHost, st));
    CF_CUDA(cudaStreamSynchronize(st));
    return CF_OK;
}

int cf_plan_trace(cf_plan* p, int64_t start, int64_t count, cf_report* out) {
    CF_TRY(check_plan(p, "cf_plan_trace"));
    if (start < 0 || count < 0 || start + count > (int64_t)p->trace_all.size() || (count > 0 && !out)) {
        set_error("cf_plan_trace: range outside the last solve's trace");
        return CF_EINVAL;
    }
    for (int64_t i = 0; i < count; ++i) out[i] = p->trace_all[start + i];
    return CF_OK;
}

int cf_apply_A(cf_plan* p, const double* x_dev, double* y_dev) {
    CF_TRY(check_plan(p, "cf_apply_A"));
    CF_TRY(launch_spmv_rows(p, x_dev, y_dev));
    CF_CUDA(cudaStreamSynchronize(p->stream));
    return CF_OK;
}

int cf_apply_At(cf_plan* p, const double* y_dev, double* x_dev) {
    CF_TRY(check_plan(p, "cf_apply_At"));
    CF_TRY(launch_spmv_cols(p, y_dev, x_dev));
    CF_CUDA(cudaStreamSynchronize(p->stream));
    return CF_OK;
}

int cf_apply_At_async(cf_plan* p, const double* y_dev, double* x_dev) {
    CF_TRY(check_plan(p, "cf_apply_At_async"));
    CF_TRY(launch_spmv_cols(p, y_dev, x_dev));
    return CF_OK;
}

int cf_apply_At_cols(cf_plan* p, const double* y_dev, double* x_dev, int64_t col_lo, int64_t col_hi) {
    CF_TRY(check_plan(p, "cf_apply_At_cols"));
    CF_TRY(launch_spmv_cols_range(p, y_dev, x_dev, col_lo, col_hi));
    return CF_OK;
}

int cf_project(cf_plan* p, const double* w_dev, double* out_dev) {
    CF_TRY(check_plan(p, "cf_project"));
    CF_TRY(launch_project(p, w_dev, out_dev));
    CF_CUDA(cudaStreamSynchronize(p->stream));
    return CF_OK;
}

int cf_plan_vector(cf_plan* p, int which, double** ptr, int64_t* len) {
    CF_TRY(check_plan(p, "cf_plan_vector"));
    if (!ptr || !len) {
        set_error("cf_plan_vector: NULL output");
        return CF_EINVAL;
    }
    switch (which) {
        case CF_VEC_X: *ptr = p->x.p; *len = p->n; break;
        case CF_VEC_Z: *ptr = p->z.p; *len = p->n; break;
        case CF_VEC_DELTA: *ptr = p->delta.p; *len = p->n; break;
        case CF_VEC_LAM: *ptr = p->lam.p; *len = p->m; break;
        case CF_VEC_H: *ptr = p->h.p; *len = p->m; break;
        case CF_VEC_AX: *ptr = p->ax.p; *len = p->m; break;
        case CF_VEC_B: *ptr = p->b.p; *len = p->m; break;
        case CF_VEC_C: *ptr = p->c.p; *len = p->n; break;
        case CF_VEC_FU: *ptr = p->fu.p; *len = p->m; break;
        case CF_VEC_DB: *ptr = p->db.p; *len = p->m; break;
        case CF_VEC_BR: *ptr = p->br.p; *len = p->m; break;
        default: set_error("cf_plan_vector: unknown vector"); return CF_EINVAL;
    }
    return CF_OK;
}

int cf_plan_column_counts(cf_plan* p, double* cnt_dev) {
    CF_TRY(check_plan(p, "cf_plan_column_counts"));
    CF_TRY(launch_counts(p, cnt_dev));
    CF_CUDA(cudaStreamSynchronize(p->stream));
    return CF_OK;
}

int cf_plan_row_step(cf_plan* p, double mu, int report) {
    CF_TRY(check_plan(p, "cf_plan_row_step"));
    CF_TRY(check_mu(mu, "cf_plan_row_step"));
    // the row half of launch_iteration: the column update already happened on the slices
    IterOpts opt;
    opt.mu = mu;
    opt.report = report != 0;
    CF_TRY(launch_row_only(p, opt));
    p->br_valid = opt.report || p->keep_br;
    return CF_OK;
}

int cf_plan_col_step(cf_plan* p, double mu) {
    CF_TRY(check_plan(p, "cf_plan_col_step"));
    CF_TRY(check_mu(mu, "cf_plan_col_step"));
    // the column half of launch_iteration; the row half happens elsewhere (column sharding)
    IterOpts opt;
    opt.mu = mu;
    CF_TRY(launch_col_only(p, opt));
    return CF_OK;
}

int cf_apply_A_async(cf_plan* p, const double* x_dev, double* y_dev) {
    CF_TRY(check_plan(p, "cf_apply_A_async"));
    CF_TRY(launch_spmv_rows(p, x_dev, y_dev));
    return CF_OK;
}

int cf_plan_row_norms(cf_plan* p, double* d_dev, double* amax_dev) {
    CF_TRY(check_plan(p, "cf_plan_row_norms"));
    CF_TRY(launch_row_norms(p, d_dev, amax_dev));
    CF_CUDA(cudaStreamSynchronize(p->stream));
    return CF_OK;
}

int cf_plan_set_row_norms(cf_plan* p, const double* d_dev, const double* amax_dev) {
    CF_TRY(check_plan(p, "cf_plan_set_row_norms"));
    CF_TRY(launch_set_row_diag(p, d_dev, amax_dev));
    CF_CUDA(cudaStreamSynchronize(p->stream));
    return CF_OK;
}

int cf_plan_row_update(cf_plan* p, double mu, int report) {
    CF_TRY(check_plan(p, "cf_plan_row_update"));
    CF_TRY(check_mu(mu, "cf_plan_row_update"));
    // the plan's ax holds the FULL A x (the all-reduced partials of the column slices)
    CF_TRY(launch_row_update(p->m, p->ax.p, p->b.p, p->fu.p, p->db.p, p->lam.p, p->h.p,
                             (report || p->keep_br) ? p->br.p : nullptr, mu, p->stream));
    p->br_valid = report || p->keep_br;
    return CF_OK;
}

int cf_plan_row_update_range(cf_plan* p, double mu, int report, int64_t r0, int64_t r1, const double* ax_dev) {
    CF_TRY(check_plan(p, "cf_plan_row_update_range"));
    CF_TRY(check_mu(mu, "cf_plan_row_update_range"));
    if (r0 < 0 || r1 < r0 || r1 > p->m || (r1 > r0 && !ax_dev)) {
        set_error("cf_plan_row_update_range: rows outside the plan or NULL A x");
        return CF_EINVAL;
    }
    if (r1 == r0) return CF_OK;
    const bool keep = report || p->keep_br;
    CF_TRY(launch_row_update(r1 - r0, ax_dev, p->b.p + r0, p->fu.p + r0, p->db.p + r0, p->lam.p + r0, p->h.p + r0,
                             keep ? p->br.p + r0 : nullptr, mu, p->stream));
    p->br_valid = keep;
    return CF_OK;
}

int cf_plan_row_parts_range(cf_plan* p, int64_t r0, int64_t r1, const double* ax_dev, double* out5) {
    CF_TRY(check_plan(p, "cf_plan_row_parts_range"));
    if (r0 < 0 || r1 < r0 || r1 > p->m || !out5 || (r1 > r0 && !ax_dev)) {
        set_error("cf_plan_row_parts_range: bad arguments");
        return CF_EINVAL;
    }
    DevBuf<double> d;
    CF_TRY(d.alloc(5));
    CF_TRY(launch_row_parts_range(p, r0, r1, ax_dev, d.p));
    CF_CUDA(cudaMemcpyAsync(out5, d.p, 5 * sizeof(double), cudaMemcpyDeviceToHost, p->stream));
    CF_CUDA(cudaStreamSynchronize(p->stream));
    return CF_OK;
}

int cf_plan_bind_h(cf_plan* p, double* h_ext) {
    CF_TRY(check_plan(p, "cf_plan_bind_h"));
    const size_t bytes = (size_t)std::max<int64_t>(p->m, 1) * sizeof(double);
    if (h_ext) {
        if (!p->h_own) p->h_own = p->h.p;
        if (h_ext != p->h.p) CF_CUDA(cudaMemcpyAsync(h_ext, p->h.p, bytes, cudaMemcpyDeviceToDevice, p->stream));
        p->h.p = h_ext;
    } else if (p->h_own) {
        CF_CUDA(cudaMemcpyAsync(p->h_own, p->h.p, bytes, cudaMemcpyDeviceToDevice, p->stream));
        p->h.p = p->h_own;
        p->h_own = nullptr;
    }
    CF_CUDA(cudaStreamSynchronize(p->stream));
    return CF_OK;
}

int cf_plan_row_parts(cf_plan* p, double* out5) {
    CF_TRY(check_plan(p, "cf_plan_row_parts"));
    DevBuf<double> d;
    CF_TRY(d.alloc(5));
    CF_TRY(launch_row_parts(p, d.p));
    CF_CUDA(cudaMemcpyAsync(out5, d.p, 5 * sizeof(double), cudaMemcpyDeviceToHost, p->stream));
    CF_CUDA(cudaStreamSynchronize(p->stream));
    return CF_OK;
}

int cf_column_update(int64_t n, const double* ath, const double* cnt, const double* c, double* x, double* z,
                     double* delta, double mu, int64_t n_blocks, const int32_t* cone_ptr, void* stream) {
    CF_TRY(check_mu(mu, "cf_column_update"));
    CF_TRY(launch_col_update(n, ath, cnt, c, x, z, delta, mu, n_blocks, cone_ptr, (cudaStream_t)stream));
    return CF_OK;
}

int cf_column_update_p2p(int64_t n, const double* const* parts, int32_t world, const double* cnt, const double* c,
                         double* x, double* z, double* delta, double mu, int64_t n_blocks, const int32_t* cone_ptr,
                         double* const* x_dst, int32_t n_dst, void* stream) {
    CF_TRY(check_mu(mu, "cf_column_update_p2p"));
    if (world < 1 || n_dst < 0 || !parts || (n_dst > 0 && !x_dst)) {
        set_error("cf_column_update_p2p: world >= 1 partials and n_dst >= 0 destinations required");
        return CF_EINVAL;
    }
    CF_TRY(launch_col_update_p2p(n, parts, world, cnt, c, x, z, delta, mu, n_blocks, cone_ptr, x_dst, n_dst,
                                 (cudaStream_t)stream));
    return CF_OK;
}

int cf_ipc_alloc(int64_t bytes, void** dev_ptr, void* handle) {
    if (!dev_ptr || !handle || bytes < 0) {
        set_error("cf_ipc_alloc: NULL output or negative size");
        return CF_EINVAL;
    }
    *dev_ptr = nullptr;
    CF_CUDA(cudaMalloc(dev_ptr, (size_t)bytes + 64));   // +64: the pass engine reads 16-byte supersets
    CF_CUDA(cudaMemset(*dev_ptr, 0, (size_t)bytes + 64));
    cudaIpcMemHandle_t h;
    CF_CUDA(cudaIpcGetMemHandle(&h, *dev_ptr));
    memcpy(handle, &h, sizeof(h));
    return CF_OK;
}

int cf_ipc_free(void* dev_ptr) {
    if (dev_ptr) CF_CUDA(cudaFree(dev_ptr));
    return CF_OK;
}

int cf_ipc_open(const void* handle, void** dev_ptr) {
    if (!dev_ptr || !handle) {
        set_error("cf_ipc_open: NULL argument");
        return CF_EINVAL;
    }
    cudaIpcMemHandle_t h;
    memcpy(&h, handle, sizeof(h));
    CF_CUDA(cudaIpcOpenMemHandle(dev_ptr, h, cudaIpcMemLazyEnablePeerAccess));
    return CF_OK;
}

int cf_ipc_close(void* dev_ptr) {
    if (dev_ptr) CF_CUDA(cudaIpcCloseMemHandle(dev_ptr));
    return CF_OK;
}

int cf_plan_bind_x(cf_plan* p, double* x_ext) {
    CF_TRY(check_plan(p, "cf_plan_bind_x"));
    const size_t bytes = (size_t)std::max<int64_t>(p->n, 1) * sizeof(double);
    if (x_ext) {
        if (!p->x_own) p->x_own = p->x.p;
        if (x_ext != p->x.p) CF_CUDA(cudaMemcpyAsync(x_ext, p->x.p, bytes, cudaMemcpyDeviceToDevice, p->stream));
        p->x.p = x_ext;
    } else if (p->x_own) {
        CF_CUDA(cudaMemcpyAsync(p->x_own, p->x.p, bytes, cudaMemcpyDeviceToDevice, p->stream));
        p->x.p = p->x_own;
        p->x_own = nullptr;
    }
    CF_CUDA(cudaStreamSynchronize(p->stream));
    return CF_OK;
}

int cf_column_parts(int64_t n, const double* atl, const double* c, const double* x, const double* z,
                    const double* delta, double* out8, void* stream) {
    DevBuf<double> d;   // the 8 results, then the per-CTA partials
    CF_TRY(d.alloc(8 + 8 * (size_t)col_parts_ctas(n)));
    CF_TRY(launch_col_parts(n, atl, c, x, z, delta, d.p, d.p + 8, (cudaStream_t)stream));
    CF_CUDA(cudaMemcpyAsync(out8, d.p, 8 * sizeof(double), cudaMemcpyDeviceToHost, (cudaStream_t)stream));
    CF_CUDA(cudaStreamSynchronize((cudaStream_t)stream));
    return CF_OK;
}

int cf_plan_last_timing(const cf_plan* p, double* loop_ms, int64_t* launches, double* row_pass_ms,
                        double* col_pass_ms, int64_t* timed_iters) {
    CF_TRY(check_plan(p, "cf_plan_last_timing"));
    if (loop_ms) *loop_ms = p->last_loop_ms;
    if (launches) *launches = p->last_launches;
    // totals over the loop: the sampled iterations' sums scaled to every timed iteration
    const double scale = (p->prof_samples > 0 && p->last_timed_iters > 0)
                             ? (double)p->last_timed_iters / (double)p->prof_samples : 1.0;
    if (row_pass_ms) *row_pass_ms = p->prof_row_ms * scale;
    if (col_pass_ms) *col_pass_ms = p->prof_col_ms * scale;
    if (timed_iters) *timed_iters = p->last_timed_iters;
    return CF_OK;
}

int cf_plan_set_profiling(cf_plan* p, int enable) {
    CF_TRY(check_plan(p, "cf_plan_set_profiling"));
    p->profiling = enable != 0;
    p->prof_stride = enable > 1 ? enable : 1;
    return CF_OK;
}

int cf_plan_sync(cf_plan* p) {
    CF_TRY(check_plan(p, "cf_plan_sync"));
    CF_CUDA(cudaStreamSynchronize(p->stream));
    return CF_OK;
}

}  // extern "C"
