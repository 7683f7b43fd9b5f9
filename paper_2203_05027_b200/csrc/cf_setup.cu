// Device setup: validate's triplet checks (model.py:152-201), build_uv
// (uv.py:64-98) and ConeWorkview.from_spec (cones.py:39-59).
//
// build_uv canonicalises the nonzeros with np.lexsort((rows, cols)) — column
// major, then row (uv.py:76). Here the canonical order comes from one CUB
// radix sort of the 64-bit key col*m + row (duplicates are adjacent after
// it, which is validate's duplicate check, model.py:167-175); the CSR copy
// is a second, stable radix sort of the canonical entries by row, so inside a
// row the entries stay in column order — the order np.bincount(row_of, ...)
// accumulates in (uv.py:10-12, :110), which makes fu_diag and every row sum
// bit-identical to the reference.
#include <cub/cub.cuh>

#include <algorithm>
#include <cmath>

#include "cf_common.h"

namespace cf {
namespace {

using ull = unsigned long long;

__device__ __forceinline__ void warp_add(ull* dst, ull v) {
    for (int off = 16; off > 0; off >>= 1) v += __shfl_down_sync(0xffffffffu, v, off);
    if ((threadIdx.x & 31) == 0 && v) atomicAdd(dst, v);
}

// counts[0] bad row, [1] bad col, [2] non-finite value, [3] zero value
__global__ void k_check_triplets(const int64_t* rows, const int64_t* cols, const double* vals, int64_t o,
                                 int64_t m, int64_t n, ull* counts) {
    ull br = 0, bc = 0, nf = 0, zv = 0;
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < o; k += (int64_t)gridDim.x * blockDim.x) {
        const int64_t r = rows[k], c = cols[k];
        const double v = vals[k];
        br += (r < 0 || r >= m);
        bc += (c < 0 || c >= n);
        nf += !isfinite(v);
        zv += (v == 0.0);
    }
    warp_add(counts + 0, br);
    warp_add(counts + 1, bc);
    warp_add(counts + 2, nf);
    warp_add(counts + 3, zv);
}

__global__ void k_check_finite(const double* v, int64_t len, ull* count) {
    ull nf = 0;
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < len; k += (int64_t)gridDim.x * blockDim.x)
        nf += !isfinite(v[k]);
    warp_add(count, nf);
}

__global__ void k_make_keys(const int64_t* rows, const int64_t* cols, int64_t o, int64_t m, uint64_t* keys,
                            int32_t* idx) {
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < o; k += (int64_t)gridDim.x * blockDim.x) {
        keys[k] = (uint64_t)cols[k] * (uint64_t)m + (uint64_t)rows[k];
        idx[k] = (int32_t)k;
    }
}

__global__ void k_count_dups(const uint64_t* keys, int64_t o, ull* count) {
    ull d = 0;
    for (int64_t k = 1 + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < o; k += (int64_t)gridDim.x * blockDim.x)
        d += (keys[k] == keys[k - 1]);
    warp_add(count, d);
}

// canonical (CSC) arrays from the sorted keys
__global__ void k_fill_csc(const uint64_t* keys, const int32_t* perm, const double* vals, int64_t o, int64_t m,
                           int32_t* rowidx, int32_t* colof, double* valc) {
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < o; k += (int64_t)gridDim.x * blockDim.x) {
        const uint64_t key = keys[k];
        rowidx[k] = (int32_t)(key % (uint64_t)m);
        colof[k] = (int32_t)(key / (uint64_t)m);
        valc[k] = vals[perm[k]];
    }
}

// segment pointers from a sorted segment-id array: ptr[s] = first k with seg_of[k] >= s
__global__ void k_ptr_from_sorted(const int32_t* seg_of, int64_t o, int64_t nseg, int32_t* ptr) {
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < o; k += (int64_t)gridDim.x * blockDim.x) {
        const int64_t s = seg_of[k];
        const int64_t sp = (k == 0) ? -1 : seg_of[k - 1];
        for (int64_t t = sp + 1; t <= s; ++t) ptr[t] = (int32_t)k;
        if (k == o - 1)
            for (int64_t t = s + 1; t <= nseg; ++t) ptr[t] = (int32_t)o;
    }
}

__global__ void k_iota(int32_t* v, int64_t len) {
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < len; k += (int64_t)gridDim.x * blockDim.x)
        v[k] = (int32_t)k;
}

__global__ void k_fill_csr(const int32_t* csr2csc, const int32_t* colof, const double* valc, int64_t o,
                           int32_t* colidx, double* valr) {
    for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < o; p += (int64_t)gridDim.x * blockDim.x) {
        const int32_t k = csr2csc[p];
        colidx[p] = colof[k];
        valr[p] = valc[k];
    }
}

inline unsigned grid1d(int64_t work, int threads = 256) {
    int64_t g = (work + threads - 1) / threads;
    if (g < 1) g = 1;
    if (g > 148 * 32) g = 148 * 32;
    return (unsigned)g;
}

inline int bits_for(uint64_t maxval) {
    int b = 1;
    while (b < 64 && (maxval >> b) != 0) ++b;
    return b;
}

int pick_tile(double avg_nnz) {
    const double target = 0.75 * kCap;
    int t = (int)(target / std::max(avg_nnz, 1e-9));
    t = std::max(32, std::min(kMaxSeg, t));
    return (t / 32) * 32;
}

// Column tiles aligned to cone boundaries (cones.py:39-59 offsets). A tile
// holds whole cones of size <= kSmallCone up to `cap` columns; a bigger cone
// is split over its own tiles and projected by k_big_cone.
int build_cone_tiles(cf_plan* p, const int64_t* sizes, int64_t nb) {
    int cap = p->cols_per_tile;
    for (int64_t q = 0; q < nb; ++q)
        if (sizes[q] <= kSmallCone) cap = std::max<int>(cap, (int)sizes[q]);
    p->cols_per_tile = cap;
    std::vector<int32_t> cone_ptr(nb + 1), ts, tc, tb, big;
    int64_t col = 0;
    for (int64_t q = 0; q < nb; ++q) {
        cone_ptr[q] = (int32_t)col;
        col += sizes[q];
    }
    cone_ptr[nb] = (int32_t)col;
    int64_t q = 0;
    col = 0;
    while (q < nb) {
        if (sizes[q] > kSmallCone) {
            const int32_t id = (int32_t)big.size();
            big.push_back((int32_t)q);
            for (int64_t s = 0; s < sizes[q]; s += cap) {
                ts.push_back((int32_t)(col + s));
                tc.push_back((int32_t)q);
                tb.push_back(id);
            }
            col += sizes[q];
            ++q;
        } else {
            ts.push_back((int32_t)col);
            tc.push_back((int32_t)q);
            tb.push_back(-1);
            int64_t cols = 0;
            while (q < nb && sizes[q] <= kSmallCone && cols + sizes[q] <= cap) {
                cols += sizes[q];
                ++q;
            }
            col += cols;
        }
    }
    ts.push_back((int32_t)col);
    tc.push_back((int32_t)nb);
    p->col_tiles = (int64_t)ts.size() - 1;
    p->n_big = (int64_t)big.size();
    CF_TRY(p->cone_ptr.alloc(nb + 1));
    CF_TRY(p->tile_start.alloc(ts.size()));
    CF_TRY(p->tile_cone.alloc(tc.size()));
    CF_TRY(p->tile_big.alloc(tb.size()));
    CF_TRY(p->big_cone.alloc(std::max<size_t>(1, big.size())));
    CF_CUDA(cudaMemcpyAsync(p->cone_ptr.p, cone_ptr.data(), cone_ptr.size() * 4, cudaMemcpyHostToDevice, p->stream));
    CF_CUDA(cudaMemcpyAsync(p->tile_start.p, ts.data(), ts.size() * 4, cudaMemcpyHostToDevice, p->stream));
    CF_CUDA(cudaMemcpyAsync(p->tile_cone.p, tc.data(), tc.size() * 4, cudaMemcpyHostToDevice, p->stream));
    CF_CUDA(cudaMemcpyAsync(p->tile_big.p, tb.data(), tb.size() * 4, cudaMemcpyHostToDevice, p->stream));
    if (!big.empty())
        CF_CUDA(cudaMemcpyAsync(p->big_cone.p, big.data(), big.size() * 4, cudaMemcpyHostToDevice, p->stream));
    // the host vectors die at return: make the copies complete first
    CF_CUDA(cudaStreamSynchronize(p->stream));
    return CF_OK;
}

int build(cf_plan* p, const int64_t* rows, const int64_t* cols, const double* vals, const double* bsrc,
          const double* csrc, int64_t nb, const int64_t* sizes, int on_device, cf_problem_checks* chk) {
    const int64_t m = p->m, n = p->n, o = p->o;
    cudaStream_t st = p->stream;
    DevBuf<int64_t> drows, dcols;
    DevBuf<double> dvals;
    if (!on_device) {
        CF_TRY(drows.alloc(o));
        CF_TRY(dcols.alloc(o));
        CF_TRY(dvals.alloc(o));
        if (o) {
            CF_CUDA(cudaMemcpyAsync(drows.p, rows, o * 8, cudaMemcpyHostToDevice, st));
            CF_CUDA(cudaMemcpyAsync(dcols.p, cols, o * 8, cudaMemcpyHostToDevice, st));
            CF_CUDA(cudaMemcpyAsync(dvals.p, vals, o * 8, cudaMemcpyHostToDevice, st));
        }
        rows = drows.p;
        cols = dcols.p;
        vals = dvals.p;
    }
    CF_TRY(p->b.alloc(m));
    CF_TRY(p->c.alloc(n));
    if (m) CF_CUDA(cudaMemcpyAsync(p->b.p, bsrc, m * 8, on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, st));
    if (n) CF_CUDA(cudaMemcpyAsync(p->c.p, csrc, n * 8, on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, st));

    // ---- validate (model.py:152-201)
    DevBuf<ull> counts;
    CF_TRY(counts.alloc(8));
    CF_CUDA(cudaMemsetAsync(counts.p, 0, 8 * sizeof(ull), st));
    if (o) k_check_triplets<<<grid1d(o), 256, 0, st>>>(rows, cols, vals, o, m, n, counts.p);
    if (m) k_check_finite<<<grid1d(m), 256, 0, st>>>(p->b.p, m, counts.p + 5);
    if (n) k_check_finite<<<grid1d(n), 256, 0, st>>>(p->c.p, n, counts.p + 6);
    CF_LAUNCHED();
    ull h_counts[8] = {0};
    CF_CUDA(cudaMemcpyAsync(h_counts, counts.p, 8 * sizeof(ull), cudaMemcpyDeviceToHost, st));
    CF_CUDA(cudaStreamSynchronize(st));
    chk->bad_row = (int64_t)h_counts[0];
    chk->bad_col = (int64_t)h_counts[1];
    chk->nonfinite_val = (int64_t)h_counts[2];
    chk->zero_val = (int64_t)h_counts[3];
    chk->nonfinite_b = (int64_t)h_counts[5];
    chk->nonfinite_c = (int64_t)h_counts[6];
    chk->duplicates = 0;
    if (h_counts[0] || h_counts[1]) {
        set_error("invalid problem: triplet index out of range");
        return CF_EPROBLEM;  // keys would be meaningless
    }

    // ---- canonical order: radix sort of col*m + row (uv.py:76)
    CF_TRY(p->colptr.alloc(n + 1));
    CF_TRY(p->rowidx.alloc(o));
    CF_TRY(p->valc.alloc(o));
    CF_TRY(p->rowptr.alloc(m + 1));
    CF_TRY(p->colidx.alloc(o));
    CF_TRY(p->valr.alloc(o));
    CF_TRY(p->csr2csc.alloc(o));
    DevBuf<int32_t> colof;
    CF_TRY(colof.alloc(o));
    if (o) {
        DevBuf<uint64_t> k_a, k_b;
        DevBuf<int32_t> i_a, i_b;
        CF_TRY(k_a.alloc(o));
        CF_TRY(k_b.alloc(o));
        CF_TRY(i_a.alloc(o));
        CF_TRY(i_b.alloc(o));
        k_make_keys<<<grid1d(o), 256, 0, st>>>(rows, cols, o, m, k_a.p, i_a.p);
        CF_LAUNCHED();
        const int end_bit = bits_for((uint64_t)m * (uint64_t)n - 1);
        cub::DoubleBuffer<uint64_t> kb(k_a.p, k_b.p);
        cub::DoubleBuffer<int32_t> ib(i_a.p, i_b.p);
        size_t tmp_bytes = 0;
        CF_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tmp_bytes, kb, ib, (int64_t)o, 0, end_bit, st));
        DevBuf<unsigned char> tmp;
        CF_TRY(tmp.alloc(tmp_bytes));
        CF_CUDA(cub::DeviceRadixSort::SortPairs(tmp.p, tmp_bytes, kb, ib, (int64_t)o, 0, end_bit, st));
        const uint64_t* skeys = kb.Current();
        const int32_t* sperm = ib.Current();
        k_count_dups<<<grid1d(o), 256, 0, st>>>(skeys, o, counts.p + 4);
        k_fill_csc<<<grid1d(o), 256, 0, st>>>(skeys, sperm, vals, o, m, p->rowidx.p, colof.p, p->valc.p);
        CF_LAUNCHED();
        ull dups = 0;
        CF_CUDA(cudaMemcpyAsync(&dups, counts.p + 4, sizeof(ull), cudaMemcpyDeviceToHost, st));
        CF_CUDA(cudaStreamSynchronize(st));
        chk->duplicates = (int64_t)dups;
        if (dups || chk->nonfinite_val || chk->zero_val || chk->nonfinite_b || chk->nonfinite_c) {
            set_error("invalid problem: validate() found violations");
            return CF_EPROBLEM;
        }
        CF_CUDA(cudaMemsetAsync(p->colptr.p, 0, (n + 1) * 4, st));
        k_ptr_from_sorted<<<grid1d(o), 256, 0, st>>>(colof.p, o, n, p->colptr.p);
        CF_LAUNCHED();

        // ---- CSR: stable sort of canonical entries by row
        cub::DoubleBuffer<uint32_t> rb(reinterpret_cast<uint32_t*>(i_a.p), reinterpret_cast<uint32_t*>(i_b.p));
        CF_CUDA(cudaMemcpyAsync(rb.Current(), p->rowidx.p, o * 4, cudaMemcpyDeviceToDevice, st));
        // k_a / k_b reused as int32 scratch for the permutation
        int32_t* pa = reinterpret_cast<int32_t*>(k_a.p);
        int32_t* pb = reinterpret_cast<int32_t*>(k_b.p);
        k_iota<<<grid1d(o), 256, 0, st>>>(pa, o);
        CF_LAUNCHED();
        cub::DoubleBuffer<int32_t> pbuf(pa, pb);
        const int row_bits = bits_for((uint64_t)std::max<int64_t>(m - 1, 1));
        size_t tmp2 = 0;
        CF_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tmp2, rb, pbuf, (int64_t)o, 0, row_bits, st));
        if (tmp2 > tmp_bytes) CF_TRY(tmp.alloc(tmp2));
        CF_CUDA(cub::DeviceRadixSort::SortPairs(tmp.p, tmp2, rb, pbuf, (int64_t)o, 0, row_bits, st));
        CF_CUDA(cudaMemcpyAsync(p->csr2csc.p, pbuf.Current(), o * 4, cudaMemcpyDeviceToDevice, st));
        k_fill_csr<<<grid1d(o), 256, 0, st>>>(p->csr2csc.p, colof.p, p->valc.p, o, p->colidx.p, p->valr.p);
        CF_CUDA(cudaMemsetAsync(p->rowptr.p, 0, (m + 1) * 4, st));
        k_ptr_from_sorted<<<grid1d(o), 256, 0, st>>>(reinterpret_cast<const int32_t*>(rb.Current()), o, m,
                                                     p->rowptr.p);
        CF_LAUNCHED();
        CF_CUDA(cudaStreamSynchronize(st));  // scratch buffers are released at scope exit
    } else {
        if (chk->nonfinite_b || chk->nonfinite_c) {
            set_error("invalid problem: validate() found violations");
            return CF_EPROBLEM;
        }
        CF_CUDA(cudaMemsetAsync(p->colptr.p, 0, (n + 1) * 4, st));
        CF_CUDA(cudaMemsetAsync(p->rowptr.p, 0, (m + 1) * 4, st));
    }

    // ---- cached diagonals (uv.py:81-82; fv is recomputed in-kernel from colptr)
    CF_TRY(p->fu.alloc(m));
    CF_TRY(p->db.alloc(m));
    CF_TRY(launch_row_diag(p));

    // ---- tiles
    p->rows_per_tile = pick_tile(m ? (double)o / (double)m : 1.0);
    p->cols_per_tile = pick_tile(n ? (double)o / (double)n : 1.0);
    p->row_tiles = (m + p->rows_per_tile - 1) / p->rows_per_tile;
    p->n_blocks = nb;
    int64_t maxsize = 0;
    for (int64_t q = 0; q < nb; ++q) maxsize = std::max(maxsize, sizes[q]);
    p->all_unit = (nb == 0 || maxsize == 1);
    if (p->all_unit) {
        p->col_tiles = (n + p->cols_per_tile - 1) / p->cols_per_tile;
        CF_TRY(p->tile_big.alloc(1));
        CF_TRY(p->tile_cone.alloc(1));
        CF_TRY(p->cone_ptr.alloc(1));
    } else {
        CF_TRY(build_cone_tiles(p, sizes, nb));
        if (p->n_big) CF_TRY(p->wbuf.alloc(n));
    }

    // ---- iterate state (SolverState.zeros, solver.py:118-127) and report buffers
    CF_TRY(p->x.alloc(n));
    CF_TRY(p->z.alloc(n));
    CF_TRY(p->delta.alloc(n));
    CF_TRY(p->lam.alloc(m));
    CF_TRY(p->h.alloc(m));
    CF_TRY(p->br.alloc(m));
    CF_TRY(p->ax.alloc(m));
    CF_CUDA(cudaMemsetAsync(p->x.p, 0, std::max<int64_t>(n, 1) * 8, st));
    CF_CUDA(cudaMemsetAsync(p->z.p, 0, std::max<int64_t>(n, 1) * 8, st));
    CF_CUDA(cudaMemsetAsync(p->delta.p, 0, std::max<int64_t>(n, 1) * 8, st));
    CF_CUDA(cudaMemsetAsync(p->lam.p, 0, std::max<int64_t>(m, 1) * 8, st));
    CF_CUDA(cudaMemsetAsync(p->h.p, 0, std::max<int64_t>(m, 1) * 8, st));
    CF_CUDA(cudaMemsetAsync(p->br.p, 0, std::max<int64_t>(m, 1) * 8, st));
    p->row_report_ctas = (int32_t)std::min<int64_t>(std::max<int64_t>((m + 255) / 256, 1), 148 * 4);
    CF_TRY(p->part_row.alloc((size_t)kReportFieldsRow * p->row_report_ctas));
    CF_TRY(p->part_col.alloc((size_t)kReportFieldsCol * std::max<int64_t>(p->col_tiles, 1)));
    p->host_ring = 64;
    CF_TRY(p->report_slot.alloc(p->host_ring));
    CF_TRY(p->done.alloc(1));
    CF_CUDA(cudaMemsetAsync(p->done.p, 0, 4, st));
    CF_CUDA(cudaMallocHost(&p->host_reports, p->host_ring * sizeof(cf_report)));
    CF_CUDA(cudaEventCreate(&p->ev0));
    CF_CUDA(cudaEventCreate(&p->ev1));
    CF_CUDA(cudaStreamSynchronize(st));
    p->iter = 0;
    p->since_warm = 2;
    return CF_OK;
}

}  // namespace
}  // namespace cf

extern "C" int cf_plan_create(int64_t m, int64_t n, int64_t o, const int64_t* rows, const int64_t* cols,
                              const double* vals, const double* b, const double* c, int64_t n_blocks,
                              const int64_t* block_sizes, int inputs_on_device, void* stream,
                              cf_problem_checks* checks, cf_plan** out) {
    using namespace cf;
    if (!out) {
        set_error("cf_plan_create: out is NULL");
        return CF_EINVAL;
    }
    *out = nullptr;
    cf_problem_checks local{};
    if (!checks) checks = &local;
    *checks = cf_problem_checks{};
    if (m < 0 || n < 0 || o < 0 || n_blocks < 0) {
        set_error("cf_plan_create: negative size");
        return CF_EINVAL;
    }
    if (m >= (int64_t)INT32_MAX || n >= (int64_t)INT32_MAX || o >= (int64_t)INT32_MAX) {
        set_error("cf_plan_create: m, n and o must be < 2^31 (int32 tile indices)");
        return CF_EINVAL;
    }
    if ((o && (!rows || !cols || !vals)) || (m && !b) || (n && !c) || (n_blocks && !block_sizes)) {
        set_error("cf_plan_create: NULL input array");
        return CF_EINVAL;
    }
    int64_t total = 0;
    for (int64_t q = 0; q < n_blocks; ++q) {
        if (block_sizes[q] < 1) {
            set_error("cone block sizes must be >= 1");
            return CF_EINVAL;
        }
        total += block_sizes[q];
    }
    if (total != n) {
        set_error("cone sizes sum " + std::to_string(total) + " != n=" + std::to_string(n));
        return CF_EINVAL;
    }
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
        cudaGetLastError();
        set_error("cf_plan_create: no CUDA device visible (libcfb200 has no CPU path)");
        return CF_ECUDA;
    }
    cf_plan* p = new cf_plan();
    p->m = m;
    p->n = n;
    p->o = o;
    if (stream) {
        p->stream = (cudaStream_t)stream;
    } else {
        cudaError_t e = cudaStreamCreateWithFlags(&p->stream, cudaStreamNonBlocking);
        if (e != cudaSuccess) {
            delete p;
            return cuda_fail(e, "cudaStreamCreate", __FILE__, __LINE__);
        }
        p->own_stream = true;
    }
    const int rc = build(p, rows, cols, vals, b, c, n_blocks, block_sizes, inputs_on_device, checks);
    if (rc != CF_OK) {
        cf_plan_destroy(p);
        return rc;
    }
    *out = p;
    return CF_OK;
}
