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
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>

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
template <class SegT>
__global__ void k_ptr_from_sorted(const SegT* seg_of, int64_t o, int64_t nseg, int32_t* ptr) {
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < o; k += (int64_t)gridDim.x * blockDim.x) {
        const int64_t s = (int64_t)seg_of[k];
        const int64_t sp = (k == 0) ? (int64_t)-1 : (int64_t)seg_of[k - 1];
        for (int64_t t = sp + 1; t <= s; ++t) ptr[t] = (int32_t)k;
        if (k == o - 1)
            for (int64_t t = s + 1; t <= nseg; ++t) ptr[t] = (int32_t)o;
    }
}

// column-pass segment of each canonical entry: band(row) * n + col
__global__ void k_band_keys(const int32_t* rowidx, const int32_t* colof, int64_t o, int64_t n, int64_t band_rows,
                            uint64_t* keys) {
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < o; k += (int64_t)gridDim.x * blockDim.x)
        keys[k] = (uint64_t)(rowidx[k] / band_rows) * (uint64_t)n + (uint64_t)colof[k];
}
// gather the canonical CSC entries into banded order
__global__ void k_fill_banded(const int32_t* perm, const int32_t* rowidx, const double* valc, int64_t o,
                              int32_t* browidx, double* bvalc) {
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < o; k += (int64_t)gridDim.x * blockDim.x) {
        const int32_t s = perm[k];
        browidx[k] = rowidx[s];
        bvalc[k] = valc[s];
    }
}

// row-pass segment of each canonical entry: panel(col) * m + row
__global__ void k_row_keys(const int32_t* rowidx, const int32_t* colof, int64_t o, int64_t m, int64_t panel_cols,
                           uint64_t* keys) {
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < o; k += (int64_t)gridDim.x * blockDim.x)
        keys[k] = (uint64_t)(colof[k] / panel_cols) * (uint64_t)m + (uint64_t)rowidx[k];
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

// Jagged-diagonal layout of one tile (see cf_pass.cuh). The tile's segments are ranked
// by length over the whole tile (descending, ties in segment order); warp block w is
// ranks [32w, 32w+32). pl[s0 + rank] = local segment | length << 8 | start_w << 17,
// and the k-th nonzero of rank r goes to base + start_w + sum_{j<k} width_j + (r mod 32),
// width_j = ranks of the block longer than j, start_w = the blocks before w each rounded
// up to 32 elements (so every full diagonal is aligned). base = tb.w, a multiple of 32.
// The pass recomputes the offsets from the lengths with warp ballots. A long tile
// (normal flag 0) is copied as is (canonical order) to base.
__global__ void __launch_bounds__(kTileSeg) k_build_jds(const int32_t* ptr, const int32_t* isrc,
                                                        const double* vsrc, const int4* tb, int32_t* idst,
                                                        double* vdst, uint32_t* pl) {
    constexpr int kW = kTileSeg / 32;
    __shared__ int lens[kTileSeg];
    __shared__ int perm[kTileSeg];
    __shared__ int rlen[kTileSeg];
    __shared__ int bsum[kW];
    __shared__ int boff[kW + 1];
    __shared__ int jo[kW][kTileDiag + 2];
    const int t = blockIdx.x;
    const int4 lo = tb[t], hi = tb[t + 1];
    const int s0 = lo.x, nseg = hi.x - lo.x, k0 = lo.y, k1 = hi.y, normal = lo.z, base = lo.w;
    if (!normal) {
        for (int k = threadIdx.x; k < k1 - k0; k += blockDim.x) {
            idst[base + k] = isrc[k0 + k];
            vdst[base + k] = vsrc[k0 + k];
        }
        if (threadIdx.x == 0) pl[s0] = 0;
        return;
    }
    const int q = threadIdx.x;
    const bool valid = q < nseg;
    const int len = valid ? ptr[s0 + q + 1] - ptr[s0 + q] : -1;
    lens[q] = len;
    __syncthreads();
    if (valid) {
        // rank over the tile (normal = 1) or inside the warp block (normal = 2: the tile runs
        // with a CTA barrier, which a tile-wide ranking would unbalance): longer first, ties in
        // segment order
        const int lo_q = normal == 2 ? (q & ~31) : 0, hi_q = normal == 2 ? min(nseg, lo_q + 32) : nseg;
        int rank = lo_q;
        for (int q2 = lo_q; q2 < hi_q; ++q2) {
            const int l2 = lens[q2];
            rank += (l2 > len) || (l2 == len && q2 < q);
        }
        perm[rank] = q;
        rlen[rank] = len;
    }
    __syncthreads();
    // thread r now stands for rank r
    const int r = threadIdx.x, w = r >> 5, l = r & 31;
    const bool rv = r < nseg;
    const int myl = rv ? rlen[r] : 0;
    int sum = myl;
    for (int off = 16; off > 0; off >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, off);
    if (l == 0) bsum[w] = sum;
    __syncthreads();
    if (threadIdx.x == 0) {
        boff[0] = 0;
        // tile-ranked tiles align every block to 32 elements (full diagonals are aligned
        // lines); block-ranked tiles (staged launches) stay packed so a tile fits a TileStage
        for (int bk = 0; bk < kW; ++bk)
            boff[bk + 1] = boff[bk] + (bk * 32 < nseg ? (normal == 1 ? (bsum[bk] + 31) / 32 * 32 : bsum[bk]) : 0);
    }
    __syncthreads();
    if (rv) pl[s0 + r] = (uint32_t)perm[r] | ((uint32_t)myl << kPlPermBits) | ((uint32_t)boff[w] << (kPlPermBits + 9));
    if (w * 32 < nseg) {
        const int mlen = rlen[w * 32];   // the block's longest
        // width of diagonal k = ranks of the block longer than k
        for (int k = l; k < mlen; k += 32) {
            int wd = 0;
            for (int r2 = 0; r2 < 32; ++r2) wd += (w * 32 + r2 < nseg) && rlen[w * 32 + r2] > k;
            jo[w][k + 1] = wd;
        }
        __syncwarp();
        if (l == 0) {
            jo[w][0] = boff[w];
            for (int k = 0; k < mlen; ++k) jo[w][k + 1] += jo[w][k];
        }
        __syncwarp();
        if (rv) {
            const int src0 = ptr[s0 + perm[r]];
            for (int kk = 0; kk < myl; ++kk) {
                const int dst = base + jo[w][kk] + l;
                idst[dst] = isrc[src0 + kk];
                vdst[dst] = vsrc[src0 + kk];
            }
        }
    }
}

// a tile takes consecutive segments while it stays within kTileSeg segments
// and kTileNnz nonzeros and holds no segment longer than kTileDiag; such a long
// segment gets a (long) tile of its own. `longs` lists the long segments in
// increasing order; the nonzero budget is found by binary search on ptr.
void tile_starts(const int32_t* ptr, int64_t s_begin, int64_t s_end, const std::vector<int64_t>& longs,
                 std::vector<int64_t>& starts, int32_t cap = kTileNnz) {
    size_t li = std::lower_bound(longs.begin(), longs.end(), s_begin) - longs.begin();
    int64_t s = s_begin;
    while (s < s_end) {
        while (li < longs.size() && longs[li] < s) ++li;
        starts.push_back(s);
        if (li < longs.size() && longs[li] == s) {   // long segment: a tile of its own
            ++s;
            continue;
        }
        int64_t e = std::min<int64_t>(s_end, s + kTileSeg);
        if (li < longs.size()) e = std::min<int64_t>(e, longs[li]);
        // last e with ptr[e] - ptr[s] <= cap (at least s + 1: a short segment fits alone)
        const int32_t* hi = std::upper_bound(ptr + s + 1, ptr + e + 1, ptr[s] + cap);
        s = std::max<int64_t>(s + 1, (int64_t)(hi - ptr) - 1);
    }
}

__global__ void k_long_segments(const int32_t* ptr, int64_t nseg, int32_t* out, int32_t cap, int32_t* count) {
    for (int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; s < nseg; s += (int64_t)gridDim.x * blockDim.x)
        if (ptr[s + 1] - ptr[s] > kTileDiag) {
            const int32_t k = atomicAdd(count, 1);
            if (k < cap) out[k] = (int32_t)s;
        }
}

// sorted indices of the segments longer than kTileDiag
int long_segments(cf_plan* p, const int32_t* ptr_dev, int64_t nseg, std::vector<int64_t>& out) {
    out.clear();
    if (nseg == 0) return CF_OK;
    DevBuf<int32_t> cnt;
    CF_TRY(cnt.alloc(1));
    int32_t cap = 1 << 16, h = 0;
    for (int attempt = 0; attempt < 2; ++attempt) {
        DevBuf<int32_t> list;
        CF_TRY(list.alloc(cap));
        CF_CUDA(cudaMemsetAsync(cnt.p, 0, 4, p->stream));
        k_long_segments<<<grid1d(nseg), 256, 0, p->stream>>>(ptr_dev, nseg, list.p, cap, cnt.p);
        CF_LAUNCHED();
        CF_CUDA(cudaMemcpyAsync(&h, cnt.p, 4, cudaMemcpyDeviceToHost, p->stream));
        CF_CUDA(cudaStreamSynchronize(p->stream));
        if (h <= cap) {
            std::vector<int32_t> v(h);
            if (h) CF_CUDA(cudaMemcpy(v.data(), list.p, (size_t)h * 4, cudaMemcpyDeviceToHost));
            out.assign(v.begin(), v.end());
            std::sort(out.begin(), out.end());
            return CF_OK;
        }
        cap = h;
    }
    set_error("long_segments: count changed between attempts");
    return CF_ECUDA;
}

// tile table {s0, k0, normal (1) / long (0), 0} from tile starts (+ the end segment)
void tile_table(const int32_t* ptr, const std::vector<int64_t>& starts, int64_t s_end, std::vector<int4>& tb) {
    tb.clear();
    for (size_t t = 0; t < starts.size(); ++t) {
        const int64_t s0 = starts[t], s1 = (t + 1 < starts.size()) ? starts[t + 1] : s_end;
        const int64_t nnz = ptr[s1] - ptr[s0];
        const int normal = !(s1 - s0 == 1 && nnz > kTileDiag);
        tb.push_back(make_int4((int)s0, ptr[s0], normal, 0));
    }
    tb.push_back(make_int4((int)s_end, ptr[s_end], 0, 0));
}

int build_jds(cf_plan* p, const int32_t* ptr, const int32_t* isrc, const double* vsrc, const std::vector<int4>& tb_in,
              int64_t nseg_total, DevBuf<int4>& dtb, DevBuf<int32_t>& idst, DevBuf<double>& vdst,
              DevBuf<uint32_t>& pl) {
    // JDS base of every tile: align32(k0 + kTilePad * (tile-ranked tiles before it) + 31 t)
    // leaves room for the per-block alignment slack of the tile-ranked tiles before it
    // (cf_common.h kTilePad); packed (block-ranked) tiles only need their own alignment
    std::vector<int4> tb(tb_in);
    int64_t aligned = 0;   // tile-ranked (aligned-block) tiles before t: only they need the slack
    for (size_t t = 0; t < tb.size(); ++t) {
        const int64_t b = ((int64_t)tb[t].y + (int64_t)kTilePad * aligned + 31 * (int64_t)t + 31) / 32 * 32;
        if (tb[t].z == 1) ++aligned;
        if (b > INT32_MAX - 64) {
            set_error("build_jds: padded nonzero positions exceed int32");
            return CF_EINVAL;
        }
        tb[t].w = (int)b;
    }
    const int64_t jds_len = (int64_t)tb.back().w + 32;
    CF_TRY(dtb.alloc(tb.size()));
    CF_CUDA(cudaMemcpyAsync(dtb.p, tb.data(), tb.size() * sizeof(int4), cudaMemcpyHostToDevice, p->stream));
    CF_TRY(idst.alloc(jds_len));
    CF_TRY(vdst.alloc(jds_len));
    // padding slots are never read by a lane; zero them so staged copies see defined bytes
    CF_CUDA(cudaMemsetAsync(idst.p, 0, (size_t)jds_len * 4, p->stream));
    CF_CUDA(cudaMemsetAsync(vdst.p, 0, (size_t)jds_len * 8, p->stream));
    CF_CUDA(cudaStreamSynchronize(p->stream));   // tb (a host copy) is released at return
    CF_TRY(pl.alloc(nseg_total));
    const int64_t ntiles = (int64_t)tb.size() - 1;
    if (ntiles > 0) {
        k_build_jds<<<(unsigned)ntiles, kTileSeg, 0, p->stream>>>(ptr, isrc, vsrc, dtb.p, idst.p, vdst.p, pl.p);
        CF_LAUNCHED();
    }
    return CF_OK;
}

int build_tiles(cf_plan* p, const int64_t* sizes, int64_t nb) {
    const int64_t m = p->m, n = p->n;
    const bool verbose = getenv("CF_VERBOSE") != nullptr;
    auto t_last = std::chrono::steady_clock::now();
    auto tick = [&](const char* what) {
        if (!verbose) return;
        const auto now = std::chrono::steady_clock::now();
        fprintf(stderr, "[cf tiles]   %-28s %8.2f ms\n", what, std::chrono::duration<double, std::milli>(now - t_last).count());
        t_last = now;
    };
    const int64_t nsr = (int64_t)p->n_panels * m;
    const int B = p->n_bands;
    const int64_t nsc = (int64_t)B * n;   // column-pass segments (band*n + col)
    const int32_t* cptr_dev = B > 1 ? p->bcolptr.p : p->colptr.p;
    std::vector<int64_t> rlong, clong;
    CF_TRY(long_segments(p, p->rowptr.p, nsr, rlong));
    CF_TRY(long_segments(p, cptr_dev, nsc, clong));
    // both pointer arrays in (cached) pinned memory
    PinnedScratch scratch;
    int32_t* rp = static_cast<int32_t*>(scratch.get((size_t)(nsr + 1 + nsc + 1) * 4));
    if (!rp) {
        set_error("build_tiles: pinned host allocation failed");
        return CF_ENOMEM;
    }
    int32_t* cpall = rp + nsr + 1;
    CF_CUDA(cudaMemcpyAsync(rp, p->rowptr.p, (size_t)(nsr + 1) * 4, cudaMemcpyDeviceToHost, p->stream));
    CF_CUDA(cudaMemcpyAsync(cpall, cptr_dev, (size_t)(nsc + 1) * 4, cudaMemcpyDeviceToHost, p->stream));
    CF_CUDA(cudaStreamSynchronize(p->stream));
    tick("ptr D2H + long segments");
    // rows, panel by panel (segment = panel*m + row)
    std::vector<int64_t> rstarts;
    rstarts.reserve(nsr / kTileSeg + 16);
    p->row_panel_tile.assign(p->n_panels + 1, 0);
    auto cut_rows = [&](int32_t cap) {
        rstarts.clear();
        for (int pn = 0; pn < p->n_panels; ++pn) {
            p->row_panel_tile[pn] = (int64_t)rstarts.size();
            tile_starts(rp, (int64_t)pn * m, (int64_t)(pn + 1) * m, rlong, rstarts, cap);
        }
        p->row_panel_tile[p->n_panels] = (int64_t)rstarts.size();
    };
    // a pass whose launches get more tiles than the staged dispatch takes runs
    // unstaged: cut it again with the larger nonzero budget
    // (env: CF_NO_LARGE_TILES off, CF_FORCE_LARGE_TILES on whatever the size -- tests)
    const bool large_ok = kTileNnzLarge > kTileNnz && !getenv("CF_NO_LARGE_TILES");
    const bool large_force = large_ok && getenv("CF_FORCE_LARGE_TILES");
    cut_rows(kTileNnz);
    p->row_large_tiles =
        large_force || (large_ok && (int64_t)rstarts.size() > (int64_t)kStagedMaxTiles * p->n_panels);
    if (p->row_large_tiles) cut_rows(kTileNnzLarge);
    std::vector<int4> rtb;
    tile_table(rp, rstarts, nsr, rtb);
    p->row_tiles = (int64_t)rtb.size() - 1;
    tick("row tiles (host)");
    // columns, band by band: the bands before the last only carry partial sums (plain
    // tiles); the last band runs the epilogue (cone-aligned tiles when not the orthant).
    // cp below is the LAST band's pointer array in column coordinates.
    std::vector<int64_t> cstarts;
    std::vector<int32_t> tcone, tbig, big, cone_ptr;
    auto cut_cols = [&](int32_t cap) {
        cstarts.clear();
        tcone.clear();
        tbig.clear();
        big.clear();
        cone_ptr.clear();
        p->col_band_tile.assign(B + 1, 0);
        for (int bd = 0; bd + 1 < B; ++bd) {
            p->col_band_tile[bd] = (int64_t)cstarts.size();
            tile_starts(cpall, (int64_t)bd * n, (int64_t)(bd + 1) * n, clong, cstarts, cap);
        }
        p->col_band_tile[B - 1] = (int64_t)cstarts.size();
        const int64_t last_off = (int64_t)(B - 1) * n;
        const int32_t* cp = cpall + last_off;
        std::vector<int64_t> clong_last;   // the last band's long segments in column coordinates
        for (int64_t s : clong)
            if (s >= last_off) clong_last.push_back(s - last_off);
        std::vector<int64_t> lstarts;
        if (p->all_unit) {
            tile_starts(cp, 0, n, clong_last, lstarts, cap);
        } else {
            cone_ptr.resize(nb + 1);
            int64_t col = 0;
            for (int64_t q = 0; q < nb; ++q) {
                cone_ptr[q] = (int32_t)col;
                col += sizes[q];
            }
            cone_ptr[nb] = (int32_t)col;
            int64_t q = 0;
            while (q < nb) {
                const int64_t c0 = cone_ptr[q];
                if (sizes[q] > kSmallCone) {
                    const size_t before = lstarts.size();
                    tile_starts(cp, c0, c0 + sizes[q], clong_last, lstarts, cap);
                    for (size_t t = before; t < lstarts.size(); ++t) {
                        tcone.push_back((int32_t)q);
                        tbig.push_back((int32_t)big.size());
                    }
                    big.push_back((int32_t)q);
                    ++q;
                    continue;
                }
                int64_t q1 = q + 1;
                auto cone_ok = [&](int64_t qq) {  // no column of the cone needs a long tile
                    for (int64_t c = cone_ptr[qq]; c < cone_ptr[qq] + sizes[qq]; ++c)
                        if (cp[c + 1] - cp[c] > kTileDiag) return false;
                    return true;
                };
                if (!cone_ok(q)) {  // cone with a very long column: treat like a big cone (k_big_cone)
                    const size_t before = lstarts.size();
                    tile_starts(cp, c0, c0 + sizes[q], clong_last, lstarts, cap);
                    for (size_t t = before; t < lstarts.size(); ++t) {
                        tcone.push_back((int32_t)q);
                        tbig.push_back((int32_t)big.size());
                    }
                    big.push_back((int32_t)q);
                    ++q;
                    continue;
                }
                while (q1 < nb && sizes[q1] <= kSmallCone && cone_ptr[q1] + sizes[q1] - c0 <= kTileSeg &&
                       cp[cone_ptr[q1] + sizes[q1]] - cp[c0] <= cap && cone_ok(q1))
                    ++q1;
                lstarts.push_back(c0);
                tcone.push_back((int32_t)q);
                tbig.push_back(-1);
                q = q1;
            }
            tcone.push_back((int32_t)nb);
        }
        for (int64_t s : lstarts) cstarts.push_back(s + last_off);
        p->col_band_tile[B] = (int64_t)cstarts.size();
    };
    cut_cols(kTileNnz);
    p->col_large_tiles = large_force || (large_ok && (int64_t)cstarts.size() > (int64_t)kStagedMaxTiles * B);
    if (p->col_large_tiles) cut_cols(kTileNnzLarge);
    std::vector<int4> ctb;
    tile_table(cpall, cstarts, nsc, ctb);
    p->col_tile_start.resize(ctb.size());
    for (size_t t = 0; t < ctb.size(); ++t) p->col_tile_start[t] = ctb[t].x;
    tick("col tiles (host)");
    p->col_tiles = (int64_t)ctb.size() - 1;
    p->n_big = (int64_t)big.size();
    p->warp_cone = 0;
    if (!p->all_unit && p->n_big == 0 && nb > 0 && !getenv("CF_GROUP_CONES")) {   // (env: force the group path)
        const int64_t s = sizes[0];
        bool uniform = s >= 2 && s <= 32 && (s & (s - 1)) == 0;
        for (int64_t q = 1; q < nb && uniform; ++q) uniform = sizes[q] == s;
        if (uniform) p->warp_cone = (int32_t)s;
    }
    // Tiles that run with a CTA barrier (staged launches of the small passes, the cone group
    // epilogue) keep the ranking inside each warp block (normal flag 2): ranking over the tile
    // would give one warp the longest block and make the others wait for it at the barrier
    // (1e6 nonzeros: 19.7 -> 25.4 us per iteration). The rest rank over the tile (flag 1).
    auto block_rank = [](std::vector<int4>& tb, int64_t t0, int64_t t1) {
        for (int64_t t = t0; t < t1; ++t)
            if (tb[t].z) tb[t].z = 2;
    };
    if (!p->row_large_tiles)
        for (int pn = 0; pn < p->n_panels; ++pn)
            if (p->row_panel_tile[pn + 1] - p->row_panel_tile[pn] <= kStagedMaxTiles)
                block_rank(rtb, p->row_panel_tile[pn], p->row_panel_tile[pn + 1]);
    // Cones of mixed sizes that come in runs (the robust-LS shape: K4 blocks, then an
    // orthant): a large pass launches each run of tiles whose cones all have one size with
    // the fused per-column (size 1) or warp-shuffle (2..32) epilogue, tile-ranked, and only
    // the tiles that mix sizes with the group epilogue (block-ranked, CTA barrier).
    p->col_runs.clear();
    if (!p->all_unit && p->warp_cone == 0 && p->n_big == 0 && B == 1 && nb > 0 && !getenv("CF_GROUP_CONES") &&
        !getenv("CF_NO_COL_RUNS") && p->col_tiles > kStagedMaxTiles && (int64_t)tcone.size() == p->col_tiles + 1) {
        std::vector<cf_plan::ColRun> runs;
        for (int64_t t = 0; t < p->col_tiles; ++t) {
            const int64_t q0 = tcone[t], q1 = tcone[t + 1];
            const int64_t s = sizes[q0];
            bool uniform = q1 > q0;
            for (int64_t q = q0 + 1; q < q1 && uniform; ++q) uniform = sizes[q] == s;
            const int32_t cls = !uniform ? 0 : (s == 1 ? 1 : ((s <= 32 && (s & (s - 1)) == 0) ? (int32_t)s : 0));
            if (!runs.empty() && runs.back().cls == cls)
                runs.back().t1 = t + 1;
            else
                runs.push_back({t, t + 1, cls});
        }
        int64_t fused = 0;
        for (const auto& r : runs)
            if (r.cls) fused += r.t1 - r.t0;
        // worth it when most tiles leave the barrier flow, in a few launches
        if (runs.size() <= 8 && 2 * fused >= p->col_tiles) p->col_runs = runs;
    }
    if (!p->col_runs.empty()) {
        for (const auto& r : p->col_runs)
            if (r.cls == 0) block_rank(ctb, r.t0, r.t1);
    } else if (!p->all_unit && p->warp_cone == 0) {
        block_rank(ctb, 0, (int64_t)ctb.size() - 1);
    } else if (!p->col_large_tiles) {
        for (int b = 0; b < B; ++b)
            if (p->col_band_tile[b + 1] - p->col_band_tile[b] <= kStagedMaxTiles)
                block_rank(ctb, p->col_band_tile[b], p->col_band_tile[b + 1]);
    }
    // stageable launch ranges: only block-ranked (packed) tiles fit a TileStage
    auto packed_prefix = [](const std::vector<int4>& tb, std::vector<int32_t>& pre) {
        pre.assign(tb.size(), 0);
        for (size_t t = 0; t + 1 < tb.size(); ++t) pre[t + 1] = pre[t] + (tb[t].z == 1 ? 1 : 0);
    };
    packed_prefix(rtb, p->row_unpacked);
    packed_prefix(ctb, p->col_unpacked);
    CF_TRY(build_jds(p, p->rowptr.p, p->colidx.p, p->valr.p, rtb, nsr, p->row_tb, p->rj_idx, p->rj_val, p->rj_pl));
    if (B > 1) {
        CF_TRY(build_jds(p, p->bcolptr.p, p->browidx.p, p->bvalc.p, ctb, nsc, p->col_tb, p->cj_idx, p->cj_val,
                         p->cj_pl));
        CF_CUDA(cudaStreamSynchronize(p->stream));
        p->bcolptr.release();
        p->browidx.release();
        p->bvalc.release();
        CF_TRY(p->atcarry.alloc(n));
    } else {
        CF_TRY(build_jds(p, p->colptr.p, p->rowidx.p, p->valc.p, ctb, n, p->col_tb, p->cj_idx, p->cj_val,
                         p->cj_pl));
    }
    if (verbose) CF_CUDA(cudaStreamSynchronize(p->stream));
    tick("jds build (device)");
    if (p->all_unit) {
        CF_TRY(p->tile_big.alloc(1));
        CF_TRY(p->tile_cone.alloc(1));
        CF_TRY(p->cone_ptr.alloc(1));
        CF_TRY(p->big_cone.alloc(1));
    } else {
        CF_TRY(p->cone_ptr.alloc(cone_ptr.size()));
        CF_TRY(p->tile_cone.alloc(tcone.size()));
        CF_TRY(p->tile_big.alloc(std::max<size_t>(1, tbig.size())));
        CF_TRY(p->big_cone.alloc(std::max<size_t>(1, big.size())));
        CF_CUDA(cudaMemcpyAsync(p->cone_ptr.p, cone_ptr.data(), cone_ptr.size() * 4, cudaMemcpyHostToDevice,
                                p->stream));
        CF_CUDA(cudaMemcpyAsync(p->tile_cone.p, tcone.data(), tcone.size() * 4, cudaMemcpyHostToDevice, p->stream));
        if (!tbig.empty())
            CF_CUDA(cudaMemcpyAsync(p->tile_big.p, tbig.data(), tbig.size() * 4, cudaMemcpyHostToDevice, p->stream));
        if (!big.empty())
            CF_CUDA(cudaMemcpyAsync(p->big_cone.p, big.data(), big.size() * 4, cudaMemcpyHostToDevice, p->stream));
        if (p->n_big) CF_TRY(p->wbuf.alloc(n));
    }
    CF_CUDA(cudaStreamSynchronize(p->stream));  // host vectors die at return
    return CF_OK;
}

// CF_VERBOSE=1: per-stage wall times of the setup on stderr
struct StageClock {
    bool on;
    cudaStream_t st;
    std::chrono::steady_clock::time_point t0, last;
    explicit StageClock(cudaStream_t s) : on(getenv("CF_VERBOSE") != nullptr), st(s) {
        t0 = last = std::chrono::steady_clock::now();
    }
    void mark(const char* what) {
        if (!on) return;
        cudaStreamSynchronize(st);
        const auto now = std::chrono::steady_clock::now();
        fprintf(stderr, "[cf setup] %-28s %8.2f ms (total %8.2f ms)\n", what,
                std::chrono::duration<double, std::milli>(now - last).count(),
                std::chrono::duration<double, std::milli>(now - t0).count());
        last = now;
    }
};

int build(cf_plan* p, const int64_t* rows, const int64_t* cols, const double* vals, const double* bsrc,
          const double* csrc, int64_t nb, const int64_t* sizes, int on_device, cf_problem_checks* chk) {
    const int64_t m = p->m, n = p->n, o = p->o;
    cudaStream_t st = p->stream;
    StageClock clk(st);
    DevBuf<int64_t> drows, dcols;
    DevBuf<double> dvals;
    if (!on_device) {
        CF_TRY(drows.alloc(o));
        CF_TRY(dcols.alloc(o));
        CF_TRY(dvals.alloc(o));
    }
    CF_TRY(p->b.alloc(m));
    CF_TRY(p->c.alloc(n));
    if (!on_device) {
        CF_TRY(h2d_staged({{drows.p, rows, (size_t)o * 8}, {dcols.p, cols, (size_t)o * 8}, {dvals.p, vals, (size_t)o * 8},
                           {p->b.p, bsrc, (size_t)m * 8}, {p->c.p, csrc, (size_t)n * 8}},
                          st));
        rows = drows.p;
        cols = dcols.p;
        vals = dvals.p;
    } else {
        if (m) CF_CUDA(cudaMemcpyAsync(p->b.p, bsrc, m * 8, cudaMemcpyDeviceToDevice, st));
        if (n) CF_CUDA(cudaMemcpyAsync(p->c.p, csrc, n * 8, cudaMemcpyDeviceToDevice, st));
    }

    clk.mark("inputs H2D");
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

    clk.mark("validate counters");
    // ---- canonical order: radix sort of col*m + row (uv.py:76)
    CF_TRY(p->colptr.alloc(n + 1));
    CF_TRY(p->rowidx.alloc(o));
    CF_TRY(p->valc.alloc(o));
    // column panels of the row pass: each panel's slice of x must stay L2-resident
    {
        double panel_mb = 48.0;
        if (const char* env = getenv("CF_PANEL_MB")) panel_mb = atof(env);
        const double xbytes = 8.0 * (double)n;
        int panels = (int)std::ceil(xbytes / (panel_mb * 1048576.0));
        if (panels < 1) panels = 1;
        if (panels > 64) panels = 64;
        if ((int64_t)panels * m >= (int64_t)INT32_MAX) panels = 1;  // tile segment ids are int32
        if (p->batch_mode) panels = 1;                                // the batched kernel reads plain CSR
        p->n_panels = panels;
        p->panel_cols = std::max<int64_t>(1, (n + panels - 1) / panels);
        // row bands of the column pass: each band's slice of h must stay L2-resident
        double band_mb = panel_mb;
        if (const char* env = getenv("CF_BAND_MB")) band_mb = atof(env);
        int bands = (int)std::ceil(8.0 * (double)m / (band_mb * 1048576.0));
        if (bands < 1) bands = 1;
        if (bands > 64) bands = 64;
        if ((int64_t)bands * n >= (int64_t)INT32_MAX) bands = 1;
        if (p->batch_mode || o == 0) bands = 1;
        p->n_bands = bands;
        p->band_rows = std::max<int64_t>(1, (m + bands - 1) / bands);
    }
    CF_TRY(p->rowptr.alloc((size_t)p->n_panels * m + 1));
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
        clk.mark("canonical sort");
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
        k_ptr_from_sorted<int32_t><<<grid1d(o), 256, 0, st>>>(colof.p, o, n, p->colptr.p);
        CF_LAUNCHED();

        clk.mark("csc fill + dup check");
        // ---- CSR panels: stable sort of canonical entries by (column panel, row); inside a
        //      segment the entries keep canonical (column) order
        const int64_t nseg_rows = (int64_t)p->n_panels * m;
        CF_CUDA(cudaMemsetAsync(p->rowptr.p, 0, (nseg_rows + 1) * 4, st));
        k_row_keys<<<grid1d(o), 256, 0, st>>>(p->rowidx.p, colof.p, o, m, p->panel_cols, k_a.p);
        k_iota<<<grid1d(o), 256, 0, st>>>(i_a.p, o);
        CF_LAUNCHED();
        cub::DoubleBuffer<uint64_t> rb(k_a.p, k_b.p);
        cub::DoubleBuffer<int32_t> pbuf(i_a.p, i_b.p);
        const int row_bits = bits_for((uint64_t)std::max<int64_t>(nseg_rows - 1, 1));
        size_t tmp2 = 0;
        CF_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tmp2, rb, pbuf, (int64_t)o, 0, row_bits, st));
        if (tmp2 > tmp_bytes) CF_TRY(tmp.alloc(tmp2));
        CF_CUDA(cub::DeviceRadixSort::SortPairs(tmp.p, tmp2, rb, pbuf, (int64_t)o, 0, row_bits, st));
        CF_CUDA(cudaMemcpyAsync(p->csr2csc.p, pbuf.Current(), o * 4, cudaMemcpyDeviceToDevice, st));
        k_fill_csr<<<grid1d(o), 256, 0, st>>>(p->csr2csc.p, colof.p, p->valc.p, o, p->colidx.p, p->valr.p);
        k_ptr_from_sorted<uint64_t><<<grid1d(o), 256, 0, st>>>(rb.Current(), o, nseg_rows, p->rowptr.p);
        CF_LAUNCHED();
        if (p->n_bands > 1) {
            // ---- banded CSC for the column pass: stable sort of canonical entries by (row band,
            //      column); inside a segment the entries keep canonical (row) order
            const int64_t nseg_cols = (int64_t)p->n_bands * n;
            CF_TRY(p->bcolptr.alloc(nseg_cols + 1));
            CF_TRY(p->browidx.alloc(o));
            CF_TRY(p->bvalc.alloc(o));
            CF_CUDA(cudaMemsetAsync(p->bcolptr.p, 0, (nseg_cols + 1) * 4, st));
            k_band_keys<<<grid1d(o), 256, 0, st>>>(p->rowidx.p, colof.p, o, n, p->band_rows, k_a.p);
            k_iota<<<grid1d(o), 256, 0, st>>>(i_a.p, o);
            CF_LAUNCHED();
            cub::DoubleBuffer<uint64_t> bb(k_a.p, k_b.p);
            cub::DoubleBuffer<int32_t> bp(i_a.p, i_b.p);
            const int band_bits = bits_for((uint64_t)std::max<int64_t>(nseg_cols - 1, 1));
            size_t tmp3 = 0;
            CF_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tmp3, bb, bp, (int64_t)o, 0, band_bits, st));
            if (tmp3 > std::max(tmp_bytes, tmp2)) CF_TRY(tmp.alloc(tmp3));
            CF_CUDA(cub::DeviceRadixSort::SortPairs(tmp.p, tmp3, bb, bp, (int64_t)o, 0, band_bits, st));
            k_fill_banded<<<grid1d(o), 256, 0, st>>>(bp.Current(), p->rowidx.p, p->valc.p, o, p->browidx.p,
                                                     p->bvalc.p);
            k_ptr_from_sorted<uint64_t><<<grid1d(o), 256, 0, st>>>(bb.Current(), o, nseg_cols, p->bcolptr.p);
            CF_LAUNCHED();
        }
        CF_CUDA(cudaStreamSynchronize(st));  // scratch buffers are released at scope exit
    } else {
        if (chk->nonfinite_b || chk->nonfinite_c) {
            set_error("invalid problem: validate() found violations");
            return CF_EPROBLEM;
        }
        CF_CUDA(cudaMemsetAsync(p->colptr.p, 0, (n + 1) * 4, st));
        CF_CUDA(cudaMemsetAsync(p->rowptr.p, 0, ((int64_t)p->n_panels * m + 1) * 4, st));
    }

    clk.mark("csr panel sort + fill");
    // ---- cached diagonals (uv.py:81-82; fv is recomputed in-kernel from colptr)
    CF_TRY(p->fu.alloc(m));
    CF_TRY(p->db.alloc(m));
    CF_TRY(p->amax.alloc(m));
    CF_TRY(p->dn.alloc(m));
    CF_TRY(launch_row_diag(p));

    // ---- cones (cones.py:39-59) and tiles
    p->n_blocks = nb;
    int64_t maxsize = 0;
    for (int64_t q = 0; q < nb; ++q) maxsize = std::max(maxsize, sizes[q]);
    p->all_unit = (nb == 0 || maxsize == 1);
    clk.mark("row diag");
    if (!p->batch_mode) {
        CF_TRY(build_tiles(p, sizes, nb));
    } else if (!p->all_unit) {
        std::vector<int32_t> cone_ptr(nb + 1, 0);
        for (int64_t q = 0; q < nb; ++q) cone_ptr[q + 1] = cone_ptr[q] + (int32_t)sizes[q];
        CF_TRY(p->cone_ptr.alloc(nb + 1));
        CF_CUDA(cudaMemcpyAsync(p->cone_ptr.p, cone_ptr.data(), (nb + 1) * 4, cudaMemcpyHostToDevice, st));
        CF_CUDA(cudaStreamSynchronize(st));
    }
    clk.mark("tiles + jds");

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
    CF_TRY(p->part_col.alloc((size_t)kReportFieldsCol * kMaxGroups * std::max(max_col_report_ctas(), 1)));
    p->host_ring = 64;
    CF_TRY(p->report_slot.alloc(p->host_ring));
    CF_TRY(p->done.alloc(1));
    CF_TRY(p->nf_flag.alloc(1));
    CF_CUDA(cudaMemsetAsync(p->nf_flag.p, 0, 4, st));
    CF_CUDA(cudaMemsetAsync(p->done.p, 0, 4, st));
    CF_CUDA(cudaMallocHost(&p->host_reports, p->host_ring * sizeof(cf_report)));
    CF_CUDA(cudaEventCreate(&p->ev0));
    CF_CUDA(cudaEventCreate(&p->ev1));
    CF_CUDA(cudaStreamSynchronize(st));
    clk.mark("state + report buffers");
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
    return cf::cf_plan_create_mode(m, n, o, rows, cols, vals, b, c, n_blocks, block_sizes, inputs_on_device, stream,
                                   checks, 0, out);
}

int cf::cf_plan_create_mode(int64_t m, int64_t n, int64_t o, const int64_t* rows, const int64_t* cols,
                            const double* vals, const double* b, const double* c, int64_t n_blocks,
                            const int64_t* block_sizes, int inputs_on_device, void* stream,
                            cf_problem_checks* checks, int batch_mode, cf_plan** out) {
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
    p->batch_mode = batch_mode != 0;
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
