// Internal header of libcfb200: the plan object, error plumbing and the launch
// wrappers shared by the setup / loop / API translation units.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <string>
#include <vector>

#include "../../include/cfb200.h"

namespace cf {

// ---------------------------------------------------------------- geometry
constexpr int kThreads = 256;     // threads of the simple (non-pass) kernels
#ifndef CF_PCAP
#define CF_PCAP 3072
#endif
#ifndef CF_PSEG
#define CF_PSEG 256
#endif
constexpr int kTileNnz = CF_PCAP;  // nonzeros per tile (= pass::kPCap)
#ifndef CF_PCAP_LARGE
#define CF_PCAP_LARGE 8192
#endif
// Nonzeros per tile of a pass too large for the staged (Wide/Medium) dispatch: the
// direct engine loads idx/val straight from HBM, so a tile may hold more than the
// stage, and rows / columns longer than kTileNnz / kTileSeg then still fill all 8
// warp blocks of a tile (C3's row pass 0.237 -> 0.209 ms, the robust-LS column
// pass 0.48 -> 0.32 ms). The TMA ring stages every tile, so it keeps kTileNnz.
#if defined(CF_TMA) && CF_TMA
constexpr int kTileNnzLarge = CF_PCAP;
#else
constexpr int kTileNnzLarge = CF_PCAP_LARGE;
#endif
#ifndef CF_MEDIUM_TILES
#define CF_MEDIUM_TILES (148 * 12)
#endif
constexpr int kStagedMaxTiles = CF_MEDIUM_TILES;   // passes with more tiles per launch run unstaged
constexpr int kTileSeg = CF_PSEG;  // rows / columns per tile (= pass::kPSeg)
constexpr int kTileDiag = 256;    // longest segment inside a multi-segment tile (= pass::kMaxDiag)
// jagged-diagonal slack per tile-ranked tile: 8 warp blocks each aligned to 32 elements, +
// the tile's own alignment (cf_setup.cu build_jds)
constexpr int kTilePad = (kTileSeg / 32) * 32 + 32;
// pl = tile-local segment | length << kPlPermBits | block start << (kPlPermBits + 9)
constexpr int kPlPermBits = kTileSeg <= 256 ? 8 : 9;
constexpr int kSmallCone = kTileSeg;  // cones up to this size are projected inside the column tile
constexpr int kReportFieldsRow = 5;
constexpr int kReportFieldsCol = 8;
constexpr int kMaxGroups = 4;     // upper bound of pass::kGroups (partial buffer sizing)

// ---------------------------------------------------------------- errors
void set_error(const std::string& msg);
int cuda_fail(cudaError_t e, const char* what, const char* file, int line);

#define CF_CUDA(call)                                                       \
    do {                                                                    \
        cudaError_t _e = (call);                                            \
        if (_e != cudaSuccess) return ::cf::cuda_fail(_e, #call, __FILE__, __LINE__); \
    } while (0)
#define CF_TRY(call)                     \
    do {                                 \
        int _rc = (call);                \
        if (_rc != CF_OK) return _rc;    \
    } while (0)
#define CF_LAUNCHED() CF_CUDA(cudaGetLastError())

// Checked build (libcfb200_checked.so, -DCF_CHECKED=1): device-side bounds asserts on every
// index the passes and the on-chip solvers dereference, and guard canaries behind every
// device buffer, verified when the buffer is released (compute-sanitizer is not available
// on the GPU pool). Off in the product build: the macros compile to nothing.
#ifndef CF_CHECKED
#define CF_CHECKED 0
#endif
#if CF_CHECKED
#define CF_DASSERT(cond)                                                                              \
    do {                                                                                              \
        if (!(cond)) {                                                                                \
            printf("CF_CHECKED: %s failed at %s:%d (block %d thread %d)\n", #cond, __FILE__, __LINE__, \
                   (int)blockIdx.x, (int)threadIdx.x);                                                \
            __trap();                                                                                 \
        }                                                                                             \
    } while (0)
#else
#define CF_DASSERT(cond) \
    do {                 \
    } while (0)
#endif
constexpr size_t kGuardBytes = CF_CHECKED ? 4096 : 0;   // canary bytes behind a buffer (checked build)
void guard_fill(void* p, size_t used, size_t total);
void guard_check(const void* p, size_t used, size_t total);

// ---------------------------------------------------------------- device buffers
// Stream-ordered pool (cudaMallocAsync on the device's default pool with an unlimited release
// threshold): plans created one after another reuse already-mapped memory instead of paying
// cudaMalloc/cudaFree (and their implicit synchronisation) again. Allocation and release are
// ordered on the legacy stream and synchronised, so a buffer is usable on any stream at return.
cudaError_t pool_alloc(void** p, size_t bytes);
// host -> device upload of pageable arrays through cached pinned staging buffers (cf_h2d.cu)
struct H2DJob {
    void* dst;
    const void* src;
    size_t bytes;
};
int h2d_staged(const std::vector<H2DJob>& jobs, cudaStream_t stream);
// process-wide cached pinned host buffer, held (locked) for the lifetime of the object
class PinnedScratch {
  public:
    PinnedScratch();
    ~PinnedScratch();
    void* get(size_t bytes);   // nullptr on failure; valid until the object dies
    PinnedScratch(const PinnedScratch&) = delete;
    PinnedScratch& operator=(const PinnedScratch&) = delete;
};
void pool_free(void* p);
template <class T>
struct DevBuf {
    T* p = nullptr;
    size_t n = 0;
    DevBuf() = default;
    DevBuf(const DevBuf&) = delete;
    DevBuf& operator=(const DevBuf&) = delete;
    ~DevBuf() { release(); }
    int alloc(size_t count) {
        release();
        if (count == 0) count = 1;  // keep a valid pointer for empty dims
        // +64 bytes: the pass engine's bulk copies read 16-byte-aligned supersets
        cudaError_t e = pool_alloc(reinterpret_cast<void**>(&p), count * sizeof(T) + 64 + kGuardBytes);
        if (e != cudaSuccess) {
            p = nullptr;
            cudaGetLastError();
            set_error(std::string("cudaMalloc of ") + std::to_string(count * sizeof(T)) +
                      " bytes failed: " + cudaGetErrorString(e));
            return CF_ENOMEM;
        }
        n = count;
        if (kGuardBytes) guard_fill(p, count * sizeof(T), count * sizeof(T) + 64 + kGuardBytes);
        return CF_OK;
    }
    void release() {
        if (p && kGuardBytes) guard_check(p, n * sizeof(T), n * sizeof(T) + 64 + kGuardBytes);
        if (p) pool_free(p);
        p = nullptr;
        n = 0;
    }
};

}  // namespace cf

// ---------------------------------------------------------------- the plan
// Device image of one ProblemInstance after build_uv (uv.py:64-98): the
// canonical nonzero list held twice, as CSC (= canonical order) and CSR
// (rows, columns ascending inside a row), plus the iterate vectors of the
// reduced two-pass iteration.
struct cf_plan {
    int64_t m = 0, n = 0, o = 0;
    bool batch_mode = false;        // built for cf_batch_solve: one CSR panel, no pass tiles
    cudaStream_t stream = nullptr;
    bool own_stream = false;

    // CSC (canonical order, uv.py:76)
    cf::DevBuf<int32_t> colptr, rowidx;
    cf::DevBuf<double> valc;
    // CSR
    cf::DevBuf<int32_t> rowptr, colidx;
    cf::DevBuf<double> valr;
    cf::DevBuf<int32_t> csr2csc;  // canonical position of each CSR entry

    // problem vectors and cached diagonals (fu_diag uv.py:81; d*b for the row pass)
    cf::DevBuf<double> b, c, fu, db, amax;
    cf::DevBuf<double> dn;   // row norms d_i (the row pass recomputes fu and d b from d and b)

    // cones (cones.py:39-59) and column tiling
    bool all_unit = true;
    int64_t n_blocks = 0;
    cf::DevBuf<int32_t> cone_ptr;      // block offsets (n_blocks+1), only when !all_unit
    cf::DevBuf<int32_t> tile_start;    // column tile starts (col_tiles+1)
    cf::DevBuf<int32_t> tile_cone;     // first cone of each column tile
    cf::DevBuf<int32_t> tile_big;      // big-cone id of a tile, -1 otherwise
    cf::DevBuf<int32_t> big_cone;      // cone index of each big cone
    int64_t n_big = 0;
    int32_t warp_cone = 0;             // uniform cone size in {2,4,...,32} with no big cones (warp epilogue), else 0
    cf::DevBuf<int4> row_tb, col_tb;   // tile table {first segment, first nonzero, normal (1) / long (0), 0}
    // jagged-diagonal copies of the CSR panels (rj_*) and of the CSC (cj_*) read by the passes
    cf::DevBuf<int32_t> rj_idx, cj_idx;
    cf::DevBuf<double> rj_val, cj_val;
    cf::DevBuf<uint32_t> rj_pl, cj_pl;  // per segment position: perm (rank -> segment) | length << 5 | block start << 14
    int64_t row_tiles = 0, col_tiles = 0;
    bool row_large_tiles = false, col_large_tiles = false;   // cut at kTileNnzLarge (never staged)
    // row-pass column panels: the CSR is stored panel-major (segment = panel*m + row)
    // so each row-pass launch gathers only one panel's slice of x (L2-resident)
    int32_t n_panels = 1;
    int64_t panel_cols = 0;
    std::vector<int64_t> row_panel_tile;   // first row tile of each panel (n_panels+1)
    std::vector<int32_t> col_tile_start;   // first segment of each column tile (host copy, col_tiles+1)
    // prefix counts of tile-ranked (aligned, unstageable) tiles: a launch over tiles [t0, t1)
    // may stage them iff the count over the range is 0
    std::vector<int32_t> row_unpacked, col_unpacked;
    // column-pass row bands: with h larger than ~48 MB the column pass runs band by band
    // (segment = band*n + col, each band's slice of h L2-resident), carrying the partial
    // column sums in atcarry; only the last band runs the epilogue
    int32_t n_bands = 1;
    int64_t band_rows = 0;
    std::vector<int64_t> col_band_tile;    // first column tile of each band (n_bands+1)
    // mixed cone sizes in runs (e.g. K4 blocks then an orthant): the column pass launches
    // each run of tiles with its own epilogue (1: orthant, 2..32: warp cones of that size,
    // 0: the shared-memory group epilogue); empty = one launch per band
    struct ColRun {
        int64_t t0, t1;
        int32_t cls;
    };
    std::vector<ColRun> col_runs;
    cf::DevBuf<double> atcarry;            // partial A^T h / A^T lam between bands (n)
    // banded CSC, only while the column JDS is built (released afterwards)
    cf::DevBuf<int32_t> bcolptr, browidx;
    cf::DevBuf<double> bvalc;
    cf::DevBuf<double> wbuf;           // w = x+ - delta/mu for big-cone columns

    // iterate state: x, z, delta (n); lam, h (m); br = b - r (m) when kept
    cf::DevBuf<double> x, z, delta, lam, h, br, ax;
    bool keep_br = false;
    bool br_valid = false;
    int64_t iter = 0;                  // iterations applied since the last set_state
    double export_mu = 1.0;            // mu of the last iterations (y export after a warm start)
    int since_warm = 2;                // 0/1: next iteration needs warm-start correction
    cf::DevBuf<double> vterm1, rcorr, ccorr;   // warm-start corrections (A.3)
    cf::DevBuf<double> y0, gamma0, eps;        // init y/gamma and eps = gamma0 + U^T lam0

    // report machinery
    int32_t row_report_ctas = 0;
    cf::DevBuf<double> part_row, part_col;     // per-CTA partials
    cf::DevBuf<cf_report> report_slot;         // device report ring
    cf::DevBuf<int32_t> done;                  // device early-exit flag
    double* x_own = nullptr;                   // cf_plan_bind_x: the plan's own x while x.p is external
    double* h_own = nullptr;                   // cf_plan_bind_h: the plan's own h while h.p is external
    cf::DevBuf<int32_t> nf_flag;               // report: non-finite implicit y/gamma
    cf_report* host_reports = nullptr;         // pinned ring
    std::vector<cf_report> trace_all;          // every report of the last cf_plan_solve (grows per report)
    int64_t host_ring = 0;

    // timing
    cudaEvent_t ev0 = nullptr, ev1 = nullptr;
    double last_loop_ms = 0.0;
    int64_t last_launches = 0;
    int64_t last_timed_iters = 0;
    bool profiling = false;
    int32_t prof_stride = 1;               // events on every prof_stride-th iteration of a loop
    int64_t prof_iter = 0, prof_samples = 0;
    double prof_row_ms = 0.0, prof_col_ms = 0.0;   // summed over the sampled iterations
    std::vector<cudaEvent_t> prof_events;  // 3 per profiled iteration: start, after col pass, after row pass
    size_t prof_used = 0;
};

namespace cf {

// plan creation with an optional batch mode (cf_setup.cu)
int cf_plan_create_mode(int64_t m, int64_t n, int64_t o, const int64_t* rows, const int64_t* cols, const double* vals,
                        const double* b, const double* c, int64_t n_blocks, const int64_t* block_sizes,
                        int inputs_on_device, void* stream, cf_problem_checks* checks, int batch_mode,
                        cf_plan** out);

// ---------------------------------------------------------------- launch wrappers (cf_kernels.cu)
struct IterOpts {
    double mu = 1.0;
    bool report = false;         // write ax/br for the report of this iteration
    const double* vterm = nullptr;
    const double* ccorr = nullptr;
    const double* rcorr = nullptr;
};
// the column pass of one iteration (all row bands, cones, big cones)
int launch_col_only(cf_plan* p, const IterOpts& opt, const int32_t* done = nullptr, int64_t* launches = nullptr);
// row norms of the plan's entries / fu, d*b, amax from given row norms (column sharding)
int launch_row_norms(cf_plan* p, double* dout, double* amax);
int launch_set_row_diag(cf_plan* p, const double* din, const double* amax_in);
// RowIter's row epilogue from a full A x (column-sharded driver)
// row part of compute_report over rows [r0, r1) from the given A x slice (column sharding)
int launch_row_parts_range(cf_plan* p, int64_t r0, int64_t r1, const double* ax, double* out5_dev);
int launch_row_update(int64_t m, const double* ax, const double* b, const double* fu, const double* db, double* lam,
                      double* h, double* br, double mu, cudaStream_t st);
// the row pass of one iteration (all column panels)
int launch_row_only(cf_plan* p, const IterOpts& opt, const int32_t* done = nullptr, int64_t* launches = nullptr);
// one iteration (col pass + cones + row pass); returns kernel launches issued via *launches
int launch_iteration(cf_plan* p, const IterOpts& opt, const int32_t* done, int64_t* launches);
// y = A x (rows), x = A^T y (cols)
int launch_spmv_rows(cf_plan* p, const double* x, double* y);
int launch_spmv_cols(cf_plan* p, const double* y, double* x);
// x = A^T y on the column tiles that start in [col_lo, col_hi) (async, plan stream)
int launch_spmv_cols_range(cf_plan* p, const double* y, double* x, int64_t col_lo, int64_t col_hi);
// report of the current state into p->report_slot[slot]; termination per cfg (nullable)
int launch_report(cf_plan* p, double mu, bool ax_ready, const cf_config* cfg, int64_t k,
                  int64_t slot, const int32_t* done, int64_t* launches);
int launch_project(cf_plan* p, const double* w, double* out);
int launch_export(cf_plan* p, double mu, double* y, double* gamma);
int launch_warm_start(cf_plan* p, double mu);
// setup helpers
int launch_row_diag(cf_plan* p);
int max_col_report_ctas();
// row-sharded building blocks
int launch_col_update(int64_t n, const double* ath, const double* cnt, const double* c, double* x, double* z,
                      double* delta, double mu, int64_t n_blocks, const int32_t* cone_ptr, cudaStream_t st);
// the same update fed by `world` peer partials (summed in rank order) and storing x+ into
// every rank's x replica (P2P over NVLink): reduce-scatter + update + all-gather in one kernel
int launch_col_update_p2p(int64_t n, const double* const* parts, int world, const double* cnt, const double* c,
                          double* x, double* z, double* delta, double mu, int64_t n_blocks, const int32_t* cone_ptr,
                          double* const* x_dst, int n_dst, cudaStream_t st);
int col_parts_ctas(int64_t n);   // CTAs of launch_col_parts (its work buffer: 8 doubles each)
int launch_col_parts(int64_t n, const double* atl, const double* c, const double* x, const double* z,
                     const double* delta, double* out8_dev, double* work, cudaStream_t st);
int launch_row_parts(cf_plan* p, double* out5_dev);
int launch_counts(cf_plan* p, double* cnt);
// profiling: reset before a loop, fold the recorded per-pass event times after its final sync
void prof_reset(cf_plan* p);
void prof_collect(cf_plan* p);

}  // namespace cf
