/*
 * cfb200.h — C ABI of the B200-native iteration engine for the UV-decomposition
 * ADMM conic solver (arXiv 2203.05027, reference package `conefree`).
 *
 * The reference is pure Python/numpy and has no FFI; each entry point below
 * replaces one reference function (file:line relative to /root/reference/pkg/src/conefree)
 * and is bound from Python with ctypes by paper_2203_05027_b200/_lib.py
 * (see INTEGRATION.md for the binding a maintainer would add to conefree).
 *
 * Conventions
 *   - plain pointers + sizes only; no torch / numpy types cross this boundary.
 *   - every function returns int: CF_OK (0) or a CF_E* code; cf_last_error()
 *     returns a thread-local message for the last failure on this thread.
 *   - fp64 everywhere (the reference computes in float64, model.py:59-61).
 *   - "canonical order" of nonzeros = column-major (sorted by column, then row),
 *     exactly the order build_uv produces (uv.py:76); y and gamma vectors of
 *     SolverState are exchanged in that order.
 *   - a plan owns all device memory it allocates; one plan is driven from one
 *     host thread at a time; plans are independent of each other.
 */
#ifndef CFB200_H
#define CFB200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define CF_ABI_VERSION 1

/* return codes */
#define CF_OK 0
#define CF_EINVAL 1          /* bad argument (sizes, nulls, unsupported shape) */
#define CF_ECUDA 2           /* CUDA runtime failure (message in cf_last_error) */
#define CF_ENOMEM 3          /* device allocation failed */
#define CF_EPROBLEM 4        /* validate() found violations: see cf_problem_checks */
#define CF_ESTATE 5          /* call not valid in the plan's current state */
#define CF_IO_PARSE 6        /* CONEPROB parse error: line + message as fileio.ParseError */
#define CF_IO_FALLBACK 7     /* input outside the native parser's subset: use the Python parser */

/* report status, mirrors the strings of solver.py:241,272,323 */
#define CF_STATUS_RUNNING 0
#define CF_STATUS_SOLVED 1
#define CF_STATUS_MAX_ITERS 2
#define CF_STATUS_DIVERGED 3

/* termination modes, solver.py:58 TERM_MODES */
#define CF_TERM_OSQP 0
#define CF_TERM_SCS 1
#define CF_TERM_TARGET 2

typedef struct cf_plan cf_plan;

/* Solver settings. Replaces SolverConfig (solver.py:61-103). The norm-dependent
 * bounds are computed by the caller exactly as check_termination does
 * (solver.py:252-271) so host and device take bit-identical decisions. */
typedef struct cf_config {
    double mu;                 /* SolverConfig.mu */
    int64_t max_iters;         /* SolverConfig.max_iters */
    int64_t check_every;       /* SolverConfig.check_every */
    int32_t term_mode;         /* CF_TERM_* */
    int32_t reserved0;
    double eps_abs;            /* osqp: eps_abs */
    double eps_rel;            /* osqp: eps_rel */
    double b_inf;              /* osqp: _norms(p.b)[0] */
    double c_inf;              /* osqp: _norms(p.c)[0] */
    double scs_prim_bound;     /* scs: eps_prim * (1.0 + _norms(p.b)[1]) */
    double scs_dual_bound;     /* scs: eps_dual * (1.0 + _norms(p.c)[1]) */
    double eps_gap;            /* scs: eps_gap */
    double target_prim_res;    /* target mode */
    double target_gap;         /* target mode */
} cf_config;

/* One evaluated report. Replaces IterationReport (solver.py:141-158). */
typedef struct cf_report {
    int64_t iter;
    int32_t status;            /* CF_STATUS_* after check_termination */
    int32_t nonfinite;         /* 1 when any state entry was non-finite (solver.py:208-211) */
    double prim_res_inf, prim_res_2;
    double dual_res_inf, dual_res_2;
    double stat_res_inf, stat_res_2;
    double ax_inf, atl_inf;
    double cone_gap;
    double pobj, dobj, gap;
} cf_report;

/* Problem-check counters filled by cf_plan_create (model.py:152-217). */
typedef struct cf_problem_checks {
    int64_t bad_row;           /* rows outside [0, m)      model.py:155 */
    int64_t bad_col;           /* cols outside [0, n)      model.py:158 */
    int64_t nonfinite_val;     /* non-finite values        model.py:161 */
    int64_t zero_val;          /* exact zero values        model.py:164 */
    int64_t duplicates;        /* duplicate positions      model.py:167-175 */
    int64_t nonfinite_b;       /* model.py:198-201 */
    int64_t nonfinite_c;
} cf_problem_checks;

/* ---------------------------------------------------------------- basics */
const char* cf_last_error(void);
int cf_abi_version(void);
/* Checked build only (libcfb200_checked.so, -DCF_CHECKED=1): device buffers found written
 * past their end when released (guard canaries); -1 in the product build. */
long long cf_debug_guard_violations(void);
/* number of visible CUDA devices (0 on a CPU-only host; never an error) */
int cf_device_count(int* count);

/* ---------------------------------------------------------------- setup
 * cf_plan_create: validate + build_uv + ConeWorkview.from_spec on the device.
 * Replaces validate's triplet/vector checks (model.py:152-201), build_uv
 * (uv.py:64-98) and ConeWorkview.from_spec (cones.py:39-59).
 *   rows/cols/vals: o triplets in ANY order (model.py:47-49); int64/int64/f64.
 *   b (m), c (n): f64.  block_sizes (n_blocks, host): the ConeSpec.
 *   inputs_on_device: 0 = rows/cols/vals/b/c are host pointers (copied with
 *   cudaMemcpyAsync), 1 = device pointers (read, never written or retained).
 *   stream: cudaStream_t the plan issues all work on (NULL = the plan creates one;
 *           (void*)1 = cudaStreamLegacy, the legacy default stream, e.g. torch's default).
 * On CF_EPROBLEM, *checks tells which checks failed and *out is NULL; the
 * caller produces the reference's messages (solver.py:300-302). */
int cf_plan_create(int64_t m, int64_t n, int64_t o,
                   const int64_t* rows, const int64_t* cols, const double* vals,
                   const double* b, const double* c,
                   int64_t n_blocks, const int64_t* block_sizes,
                   int inputs_on_device, void* stream,
                   cf_problem_checks* checks, cf_plan** out);
int cf_plan_destroy(cf_plan* plan);
/* dims and the device tile geometry chosen at setup (for tests/bench). */
int cf_plan_info(const cf_plan* plan, int64_t* m, int64_t* n, int64_t* o,
                 int64_t* row_tiles, int64_t* col_tiles, int64_t* big_cones, int32_t* all_unit);
/* replace b and/or c (device or host per inputs_on_device; NULL = keep). */
int cf_plan_set_rhs(cf_plan* plan, const double* b, const double* c, int inputs_on_device);

/* ---------------------------------------------------------------- state
 * cf_plan_set_state: warm start (solver.py:278,309). Host vectors; y, gamma
 * in canonical order (length o). NULL for all = cold start (SolverState.zeros,
 * solver.py:118-127). mu is needed for the one-time warm-start correction. */
int cf_plan_set_state(cf_plan* plan, double mu,
                      const double* x, const double* y, const double* z,
                      const double* lam, const double* gamma, const double* delta);
/* Keep b - r of every iteration so cf_plan_get_state can rebuild y (costs 8m
 * bytes per iteration; off by default, on for parity probing). */
int cf_plan_set_export(cf_plan* plan, int keep);
/* Export the full SolverState (solver.py:106-116) at the current iteration;
 * any output may be NULL. y/gamma are reconstructed in canonical order. */
int cf_plan_get_state(cf_plan* plan, double* x, double* y, double* z,
                      double* lam, double* gamma, double* delta, int64_t* iter);

/* ---------------------------------------------------------------- loop
 * cf_plan_iterate: n_iters iterations of solver.py:313-317 (x, y, z, duals)
 * with no report; for parity probing and benchmarking. */
int cf_plan_iterate(cf_plan* plan, double mu, int64_t n_iters);
/* compute_report (solver.py:206-242) at the current state; status is
 * CF_STATUS_RUNNING or CF_STATUS_DIVERGED (no termination test). */
int cf_plan_report(cf_plan* plan, double mu, cf_report* out);
/* The whole loop of solve() (solver.py:309-334) from the current state:
 * reports every check_every iterations and at max_iters, device-side
 * termination (check_termination, solver.py:245-272) with early exit.
 * trace: caller buffer of trace_cap reports (any size >= 0): the first
 * min(trace_cap, *n_reports) reports are written there; *n_reports = reports
 * of the whole solve (the last one is the SolveResult.report). The plan keeps
 * every report (growing one per check, like solver.py:310, 325), so a caller
 * with a small buffer fetches the rest with cf_plan_trace. x_out (n),
 * lam_out (m): host. */
int cf_plan_solve(cf_plan* plan, const cf_config* cfg,
                  double* x_out, double* lam_out,
                  cf_report* trace, int64_t trace_cap, int64_t* n_reports);
/* Reports [start, start + count) of the last cf_plan_solve on this plan. */
int cf_plan_trace(cf_plan* plan, int64_t start, int64_t count, cf_report* out);

/* ---------------------------------------------------------------- operators
 * Matrix-free products on device vectors (uv.py:106-131 composed):
 *   cf_apply_A : y = U(V^T x) = A x     (apply_U . apply_Vt)
 *   cf_apply_At: x = V(U^T y) = A^T y   (apply_V . apply_Ut)
 * Sums run sequentially in canonical order, bit-identical to np.bincount. */
int cf_apply_A(cf_plan* plan, const double* x_dev, double* y_dev);
int cf_apply_At(cf_plan* plan, const double* y_dev, double* x_dev);
/* cf_apply_At without the final stream synchronisation (ordered on the plan's stream) */
int cf_apply_At_async(cf_plan* plan, const double* y_dev, double* x_dev);
/* the part of cf_apply_At_async on the column tiles that START in [col_lo, col_hi): calling it
 * for consecutive ranges covers every column once, and after the call for [lo_r, lo_{r+1})
 * every column < lo_{r+1} is written (the sharded driver overlaps each range's reduction with
 * the next range's compute) */
int cf_apply_At_cols(cf_plan* plan, const double* y_dev, double* x_dev, int64_t col_lo, int64_t col_hi);
/* project_product (cones.py:103-110) of a device n-vector onto the plan's cone. */
int cf_project(cf_plan* plan, const double* w_dev, double* out_dev);

/* ---------------------------------------------------------------- batch
 * cf_batch_solve: many independent problems, each solved like cf_plan_solve
 * (the reference's batch mechanism is a process pool over solve(),
 * bench.py:96-106). The problems are passed as ONE block-diagonal problem:
 * problem p owns rows [row_off[p], row_off[p+1]) and columns
 * [col_off[p], col_off[p+1]) (host arrays of P+1, row_off[0] = col_off[0] = 0);
 * rows/cols/vals (o triplets, any order), b, c and the cone blocks are the
 * concatenation (no cone may cross a problem boundary). cfgs: one cf_config per
 * problem (its norm-dependent bounds from that problem's b, c). Outputs (host):
 * x_out (N), lam_out (M), final_reports / n_reports (P), and optionally the
 * first trace_cap reports of every problem in trace (P*trace_cap; NULL if 0).
 * One CTA per problem keeps it in shared memory; a problem that does not fit
 * returns CF_EINVAL. elapsed_ms: device time of the solve kernel. */
int cf_batch_solve(int64_t n_problems, const int64_t* row_off, const int64_t* col_off, int64_t o,
                   const int64_t* rows, const int64_t* cols, const double* vals,
                   const double* b, const double* c, int64_t n_blocks, const int64_t* block_sizes,
                   const cf_config* cfgs, double* x_out, double* lam_out,
                   cf_report* final_reports, int32_t* n_reports, cf_report* trace, int64_t trace_cap,
                   cf_problem_checks* checks, double* elapsed_ms);

/*
 * cf_cluster_solve: solve() (solver.py:275-334, cold start) of ONE mid-size
 * problem in a single launch of a thread-block cluster (up to 16 CTAs, iterates in
 * distributed shared memory; x and lam bit-identical to cf_plan_solve). Same
 * inputs and outputs as cf_batch_solve with P = 1 (trace: trace_cap reports).
 * *cluster_used = the cluster size, or 0 when the problem does not fit the
 * cluster's shared memory: then nothing was solved and the caller uses
 * cf_plan_create + cf_plan_solve. The reference has no such entry point; it
 * replaces the loop of solve() for problems like SURVEY config C1.
 */
int cf_cluster_solve(int64_t m, int64_t n, int64_t o, const int64_t* rows, const int64_t* cols,
                     const double* vals, const double* b, const double* c, int64_t n_blocks,
                     const int64_t* block_sizes, const cf_config* cfg, double* x_out, double* lam_out,
                     cf_report* final_report, int32_t* n_reports, cf_report* trace, int64_t trace_cap,
                     cf_problem_checks* checks, int32_t* cluster_used, double* elapsed_ms);

/* ---------------------------------------------------------------- row-sharded building blocks
 * Used by paper_2203_05027_b200/sharded.py (config C5: A's rows split over
 * ranks, one exchange per iteration). A rank's plan holds its row block and ALL
 * columns; per iteration the driver runs
 *   cf_apply_At(h) -> reduce-scatter -> cf_column_update on the rank's column
 *   slice -> all-gather x into the plan's x -> cf_plan_row_step.
 * Reports: cf_plan_row_parts + (cf_apply_At(lam) -> reduce-scatter ->
 * cf_column_parts), all-reduced, then the host assembles compute_report. */
#define CF_VEC_X 0
#define CF_VEC_Z 1
#define CF_VEC_DELTA 2
#define CF_VEC_LAM 3
#define CF_VEC_H 4
#define CF_VEC_AX 5
#define CF_VEC_B 6
#define CF_VEC_C 7
#define CF_VEC_FU 8
#define CF_VEC_DB 9
#define CF_VEC_BR 10   /* b - r (report iterations) */
/* device pointer and length of one of the plan's vectors */
int cf_plan_vector(cf_plan* plan, int which, double** ptr, int64_t* len);
/* per-column nonzero counts of the plan (n doubles, device) */
int cf_plan_column_counts(cf_plan* plan, double* cnt_dev);
/* the row pass of one iteration (y_update + lam/gamma updates, solver.py:179-183,194-195)
 * with the plan's current x; report=1 also keeps A x for cf_plan_row_parts */
int cf_plan_row_step(cf_plan* plan, double mu, int report);
/* Column-sharded building blocks (A's columns split over the ranks, all rows on every
 * rank; the exchange is one all-reduce of the m-vector A x): */
/* the plan's row norms d_i = sum a_ik^2 (uv.py:81 before the reciprocal) and max |a_ik|
 * over its own entries (device arrays of m); with A's columns split over ranks the
 * driver all-reduces them (sum / max) and sets them back, so fu, d*b and the
 * finiteness check use the whole rows */
int cf_plan_row_norms(cf_plan* plan, double* d_dev, double* amax_dev);
int cf_plan_set_row_norms(cf_plan* plan, const double* d_dev, const double* amax_dev);
/* the column pass of one iteration on the plan's columns (x_update + z_update + delta
 * update, solver.py:168-176,186-188,196) from the plan's h */
int cf_plan_col_step(cf_plan* plan, double mu);
/* y = A x on the plan (rows; the partial A_r x_r of a column slice), no host sync */
int cf_apply_A_async(cf_plan* plan, const double* x_dev, double* y_dev);
/* y_update + lam/gamma updates (solver.py:179-183,194-195) of every row of the plan from the
 * FULL A x in the plan's ax buffer (CF_VEC_AX, the all-reduced partials):
 * r = fu (d b + A x), lam += mu (r - b), h = (b - r) - lam / mu; report=1 keeps b - r for
 * cf_plan_row_parts */
int cf_plan_row_update(cf_plan* plan, double mu, int report);
/* row part of compute_report over the plan's rows: out = {sum (Ax-b)^2, max|Ax-b|,
 * max|Ax|, sum b*lam, nonfinite(lam)} (host array of 5) */
int cf_plan_row_parts(cf_plan* plan, double* out5);
/* column sharding with the row update sharded too: y_update + lam/gamma updates of rows
 * [r0, r1) only, from that slice of the full A x (reduce-scattered, ax_dev = r1 - r0
 * doubles); writes lam, h (and b - r when report) at those rows of the plan */
int cf_plan_row_update_range(cf_plan* plan, double mu, int report, int64_t r0, int64_t r1, const double* ax_dev);
/* cf_plan_row_parts over rows [r0, r1) from that slice of A x (host array of 5) */
int cf_plan_row_parts_range(cf_plan* plan, int64_t r0, int64_t r1, const double* ax_dev, double* out5);
/* Run the plan on an external h buffer (>= m doubles + 64 bytes; e.g. the NCCL all-gather
 * target of the sharded row update); the current h is copied over. NULL: back to the own. */
int cf_plan_bind_h(cf_plan* plan, double* h_ext);
/* x_update + z_update + delta update (solver.py:168-176,186-188,196) on a column slice
 * from the reduced A^T h: all device arrays of n; cone_ptr (device, n_blocks+1,
 * slice-local offsets) or NULL for the orthant; vterm (optional) replaces cnt*x + ath. */
int cf_column_update(int64_t n, const double* ath, const double* cnt, const double* c, double* x,
                     double* z, double* delta, double mu, int64_t n_blocks, const int32_t* cone_ptr,
                     void* stream);
/* cf_column_update fused with its collectives for the row-sharded step over NVLink peer
 * memory (SURVEY §8e "fused" row; replaces reduce-scatter -> cf_column_update ->
 * all-gather, solver.py:168-176,186-188,196). parts: device array of `world` pointers to
 * each rank's partial A^T h at this slice (P2P-readable, summed in rank order); x_dst:
 * device array of n_dst pointers to the x replicas at this slice, each receiving x+.
 * The caller orders the partials before and the replicas after with a cross-rank barrier. */
int cf_column_update_p2p(int64_t n, const double* const* parts, int32_t world, const double* cnt,
                         const double* c, double* x, double* z, double* delta, double mu, int64_t n_blocks,
                         const int32_t* cone_ptr, double* const* x_dst, int32_t n_dst, void* stream);
/* Peer memory for the fused step: a cudaMalloc'ed buffer (+64 bytes slack, zeroed) and its
 * 64-byte cudaIpcMemHandle_t; open / close a peer's buffer in this process. */
int cf_ipc_alloc(int64_t bytes, void** dev_ptr, void* handle64);
int cf_ipc_free(void* dev_ptr);
int cf_ipc_open(const void* handle64, void** dev_ptr);
int cf_ipc_close(void* dev_ptr);
/* Run the plan on an external x buffer (n doubles + 64 bytes, e.g. from cf_ipc_alloc, so
 * peers can store x+ into it); the current x is copied over. NULL: back to the plan's own
 * buffer (copied back). The external buffer stays the caller's. */
int cf_plan_bind_x(cf_plan* plan, double* x_ext);
/* column part of compute_report on a slice from the reduced A^T lam: out = {sum dual^2,
 * max|dual|, sum stat^2, max|stat|, max|A^T lam|, sum c*x, max|x-z|, nonfinite} (host, 8) */
int cf_column_parts(int64_t n, const double* atl, const double* c, const double* x, const double* z,
                    const double* delta, double* out8, void* stream);

/* ---------------------------------------------------------------- timing
 * CUDA-event time of the last cf_plan_iterate / cf_plan_solve loop (ms),
 * kernel launches issued by it, and the event time of row/col passes when
 * profiling was enabled with cf_plan_set_profiling(plan, 1). */
int cf_plan_last_timing(const cf_plan* plan, double* loop_ms, int64_t* launches,
                        double* row_pass_ms, double* col_pass_ms, int64_t* timed_iters);
/* enable = 0: off; 1: events around both passes of every iteration; k > 1: of every k-th
 * iteration only (the events break the passes' programmatic-launch overlap; last_timing
 * scales the sampled sums to the whole loop) */
int cf_plan_set_profiling(cf_plan* plan, int enable);
/* Synchronise the plan's stream. */
int cf_plan_sync(cf_plan* plan);

/* ---------------------------------------------------------------- NVLS (NVLink SHARP) fused step
 * SURVEY §2 K7 stage 2 / §8e: the row-sharded exchange done by the NVSwitch. A multicast
 * object (CUDA VMM, cuMulticastCreate) binds one buffer per rank; a multimem.ld_reduce of
 * the multicast address returns the sum of every rank's copy, a multimem.st writes every
 * rank's copy. Replaces reduce-scatter -> cf_column_update -> all-gather
 * (solver.py:168-176,186-188,196) like cf_column_update_p2p. */
typedef struct cf_mc cf_mc;
/* 1 when the current device supports multicast objects (CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED) */
int cf_mc_supported(int* supported);
/* create a multicast object of >= bytes per rank for `world` ranks; world > 1 also
 * exports a POSIX fd for the other ranks (cf_mc_import) */
int cf_mc_create(int64_t bytes, int32_t world, cf_mc** out, int* fd_out);
int cf_mc_import(int fd, int64_t bytes, int32_t world, cf_mc** out);
/* join with the current device (every rank), then bind + map: uc = this rank's copy,
 * mc = the multicast address (blocks until every rank has joined) */
int cf_mc_add_device(cf_mc* mc);
int cf_mc_bind(cf_mc* mc, void** uc_ptr, void** mc_ptr);
int cf_mc_destroy(cf_mc* mc);
/* cf_column_update on a slice with A^T h = multimem.ld_reduce(parts_mc) and x+ stored to
 * x (the slice) and through x_mc (every rank's replica; NULL: none) */
int cf_column_update_nvls(int64_t n, const double* parts_mc, const double* cnt, const double* c, double* x,
                          double* z, double* delta, double mu, int64_t n_blocks, const int32_t* cone_ptr,
                          double* x_mc, void* stream);
/* device-side team barrier: multimem.red.add 1 on the counter, wait until this rank's
 * copy reaches target (= world * epoch); stream-ordered, no host synchronisation */
int cf_mc_barrier(uint32_t* flag_mc, const uint32_t* flag_uc, uint32_t target, void* stream);

/* ---------------------------------------------------------------- instance generator (bench tooling)
 * Counter-based draws for the large synthetic configs, bit-identical to the numpy
 * restatement paper_2203_05027_b200/cfgen.py (which replaces the PCG64 stream of the
 * reference generator, generate.py:82-140, with H(seed, stream, k)). Asynchronous on
 * cuda_stream (a cudaStream_t, NULL = legacy default). */
/* out[i] = AS241 normal of draw start+i of `stream` */
int cf_gen_normal(uint64_t seed, uint64_t stream, int64_t start, int64_t count, double* out_dev, void* cuda_stream);
/* out[i] = draw start+i of stream 0, mod total (cell candidates) */
int cf_gen_cells(uint64_t seed, int64_t start, int64_t count, int64_t total, int64_t* out_dev, void* cuda_stream);
/* out[i] = draw start+i of `stream` >> 1 (non-negative sort keys) */
int cf_gen_keys(uint64_t seed, uint64_t stream, int64_t start, int64_t count, int64_t* out_dev, void* cuda_stream);

/* ---------------------------------------------------------------- CONEPROB text I/O (host)
 * Replaces parse_problem / write_problem (conefree/fileio.py:56-190) with a
 * multi-threaded native reader/writer. Errors reproduce
 * fileio.ParseError: CF_IO_PARSE with *err_line (0 = "file ended ...") and
 * the reference's message text; CF_IO_FALLBACK when the input is outside the
 * native subset (non-ASCII bytes, integers beyond int64) so the caller runs the
 * Python restatement (paper_2203_05027_b200/binio.py). */
typedef struct cf_text cf_text;
/* open a file (path) or an in-memory UTF-8 text (path == NULL) */
int cf_coneprob_open(const char* path, const char* text, int64_t len, cf_text** out);
void cf_coneprob_close(cf_text* t);
/* header, dimensions and CONES line (fileio.py:98-138): dims = {m, n, nnz, n_blocks} */
int cf_coneprob_header(cf_text* t, int64_t dims[4], int64_t* err_line, char* msg, int64_t cap);
/* the block sizes read by cf_coneprob_header (n_blocks int64) */
int cf_coneprob_sizes(const cf_text* t, int64_t* sizes);
/* entries, b, c and trailing content (fileio.py:140-190) into caller arrays;
 * threads <= 0: all host cores */
int cf_coneprob_body(cf_text* t, int64_t* rows, int64_t* cols, double* vals, double* b, double* c, int threads,
                     int64_t* err_line, char* msg, int64_t cap);
/* Python repr() of a float (fileio.py:52-53) into out (>= 32 bytes); returns the length */
int cf_format_double(double x, char* out);
/* write_problem (fileio.py:56-72) to a file; entries must already be in canonical order */
int cf_coneprob_write(const char* path, int64_t m, int64_t n, int64_t nnz, const int64_t* rows, const int64_t* cols,
                      const double* vals, const double* b, const double* c, int64_t n_blocks, const int64_t* sizes,
                      int threads);
/* write_solution (fileio.py:193-200) to a file: `head` (the STATUS and POBJ/DOBJ/ITERS
 * lines, newline-terminated) followed by x then lam, one repr() per line */
int cf_solution_write(const char* path, const char* head, const double* x, int64_t n, const double* lam, int64_t m,
                      int threads);

#ifdef __cplusplus
}
#endif
#endif /* CFB200_H */
