// Probe: the column pass of C2 (n = 10M columns, Poisson(10) lengths, o ~ 1e8, h = 5M
// doubles = 40 MB) with a "CSR-stream" warp block instead of the jagged-diagonal one.
//
// A warp owns 32 consecutive segments (as in the JDS engine) but reads their nonzeros
// in CANONICAL order, 32 consecutive nonzeros per round (fully coalesced idx/val, every
// lane gathers), and forms each segment's sum with a systolic shuffle chain
// acc_l = (head_l ? init : acc_{l-1}) + p_l, which is exactly the sequential canonical
// order (bit-identical to np.bincount). Checked bit for bit against a one-thread-per-
// column sequential kernel, then timed with the LP column epilogue (x, z, delta, c).
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 --fmad=false -o scratch/csr_stream_probe scratch/csr_stream_probe.cu
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <cstring>
#include <algorithm>
#include <random>
#include <vector>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e)); exit(1); } } while (0)

__device__ __forceinline__ uint64_t pol_first() { uint64_t p; asm("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p)); return p; }
__device__ __forceinline__ uint64_t pol_last() { uint64_t p; asm("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p)); return p; }
__device__ __forceinline__ double ldg_hint(const double* p, uint64_t pol) {
    double v; asm("ld.global.nc.L1::no_allocate.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(v) : "l"(p), "l"(pol)); return v;
}
__device__ __forceinline__ int ldg_hint(const int* p, uint64_t pol) {
    int v; asm("ld.global.nc.L1::no_allocate.L2::cache_hint.s32 %0, [%1], %2;" : "=r"(v) : "l"(p), "l"(pol)); return v;
}
__device__ __forceinline__ void st_hint(double* p, double v, uint64_t pol) {
    asm volatile("st.global.L2::cache_hint.f64 [%0], %1, %2;" ::"l"(p), "d"(v), "l"(pol) : "memory");
}

// reference: one thread per column, sequential canonical sum
__global__ void k_ref(const int* ptr, const int* idx, const double* val, const double* g, double* out, int n) {
    for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < n; j += gridDim.x * blockDim.x) {
        double acc = 0.0;
        for (int k = ptr[j]; k < ptr[j + 1]; ++k) acc = __dadd_rn(acc, __dmul_rn(val[k], g[idx[k]]));
        out[j] = acc;
    }
}

// CSR-stream warp blocks. EPI: 0 = store the sums, 1 = LP column update (x, z, delta, c).
template <int EPI, int R>
__global__ void __launch_bounds__(256, 6) k_stream(const int* __restrict__ ptr, const int* __restrict__ idx,
                                                   const double* __restrict__ val, const double* __restrict__ g,
                                                   double* out, double* x, double* z, double* dl,
                                                   const double* __restrict__ c, int n) {
    const int lane = threadIdx.x & 31;
    const int wpb = blockDim.x >> 5;
    const int nblk = (n + 31) >> 5;
    const uint64_t pf = pol_first(), plast = pol_last();
    for (int blk = blockIdx.x * wpb + (threadIdx.x >> 5); blk < nblk; blk += gridDim.x * wpb) {
        const int s = blk * 32 + lane;
        const bool has = s < n;
        const int st = has ? __ldg(ptr + s) : 0;
        const int en = has ? __ldg(ptr + s + 1) : 0;
        const int base = __shfl_sync(0xffffffffu, st, 0);
        const int stop = __shfl_sync(0xffffffffu, en, min(31, n - 1 - blk * 32));
        double ev[4];
        if (EPI == 1 && has) {
            ev[0] = ldg_hint(x + s, pf); ev[1] = ldg_hint(z + s, pf); ev[2] = ldg_hint(dl + s, pf); ev[3] = ldg_hint(c + s, pf);
        }
        const int rst = has ? st - base : 0x7fffffff;   // my segment's start, block-relative
        double res = 0.0;                     // my segment's sum (0.0 for empty segments)
        double carry = 0.0;                   // acc of lane 31 of the previous round
        for (int r0 = 0; r0 < stop - base; r0 += 32 * R) {
            int jj[R];
            double vv[R], gv[R];
#pragma unroll
            for (int u = 0; u < R; ++u) {
                const int t = base + r0 + 32 * u + lane;
                const bool ok = t < stop;
                jj[u] = ok ? ldg_hint(idx + t, pf) : 0;
                vv[u] = ok ? ldg_hint(val + t, pf) : 0.0;
            }
#pragma unroll
            for (int u = 0; u < R; ++u) gv[u] = ldg_hint(g + jj[u], plast);
#pragma unroll
            for (int u = 0; u < R; ++u) {
                const int pos = r0 + 32 * u + lane;          // block-relative position of my element
                // q = last segment (lane) whose start <= pos: binary search over the sorted starts
                int q = 0;
#pragma unroll
                for (int step = 16; step > 0; step >>= 1) {
                    const int sq = __shfl_sync(0xffffffffu, rst, q + step);
                    if (q + step < 32 && sq <= pos) q += step;
                }
                const int sq = __shfl_sync(0xffffffffu, rst, q);
                const bool head = (sq == pos) || (base + pos >= stop);   // past the block: cut the chain
                const double p = __dmul_rn(vv[u], gv[u]);
                // systolic chain: acc_l = (head ? 0 : acc_{l-1}) + p_l, lane 0 continues from carry
                double acc = __dadd_rn(head ? 0.0 : carry, p);
                // number of steps = longest run of non-heads ending at any lane
                const unsigned H = __ballot_sync(0xffffffffu, head);
                const unsigned below = H & ((2u << lane) - 1u);   // heads at lanes <= me
                // lane l is final after (l - its head) steps, or l steps when it continues the carry
                const int dist = below ? lane - (31 - __clz(below)) : lane;
                const int steps = __reduce_max_sync(0xffffffffu, dist);
                for (int k = 1; k <= steps; ++k) {
                    const double prev = __shfl_up_sync(0xffffffffu, acc, 1);
                    if (!head && lane > 0) acc = __dadd_rn(prev, p);
                }
                // lane 0 of a non-head run already used carry; other lanes chained from lane-1
                carry = __shfl_sync(0xffffffffu, acc, 31);
                // my segment ends in this round? fetch its sum
                const int rend = en - base - 1;
                const int rr = r0 + 32 * u;
                const bool mine = has && en > st && rend >= rr && rend < rr + 32;
                const double got = __shfl_sync(0xffffffffu, acc, (rend - rr) & 31);
                if (mine) res = got;
            }
        }
        if (EPI == 0) {
            if (has) out[s] = res;
        } else if (has) {
            const int cnt = en - st;
            const double fv = 1.0 / (1.0 + (double)cnt);
            const double xj = ev[0], zj = ev[1], dj = ev[2], cj = ev[3];
            const double v = __dadd_rn(__dmul_rn((double)cnt, xj), res);
            const double xp = fv * (((v + zj) + dj) - cj);
            const double w = xp - dj;
            const double zp = w > 0.0 ? w : 0.0;
            st_hint(x + s, xp, plast);
            st_hint(z + s, zp, pf);
            st_hint(dl + s, dj + (zp - xp), pf);
        }
    }
}

int main(int argc, char** argv) {
    const int n = argc > 1 ? atoi(argv[1]) : 10000000;
    const int m = n / 2;
    std::mt19937_64 rng(1);
    std::poisson_distribution<int> pois(10.0);
    std::uniform_int_distribution<int> urow(0, m - 1);
    std::normal_distribution<double> nrm;
    std::vector<int> ptr(n + 1);
    ptr[0] = 0;
    for (int j = 0; j < n; ++j) ptr[j + 1] = ptr[j] + pois(rng);
    const int o = ptr[n];
    std::vector<int> idx(o);
    std::vector<double> val(o), h(m);
    for (int j = 0; j < n; ++j) {   // rows ascending within a column (canonical)
        std::vector<int> r(ptr[j + 1] - ptr[j]);
        for (auto& v : r) v = urow(rng);
        std::sort(r.begin(), r.end());
        for (size_t k = 0; k < r.size(); ++k) idx[ptr[j] + k] = r[k];
    }
    for (auto& v : val) v = nrm(rng);
    for (auto& v : h) v = nrm(rng);
    printf("n=%d m=%d o=%d\n", n, m, o);
    int *dptr, *didx;
    double *dval, *dh, *dout, *dref, *x, *z, *dl, *c;
    CK(cudaMalloc(&dptr, (n + 1) * 4)); CK(cudaMalloc(&didx, (size_t)o * 4 + 64));
    CK(cudaMalloc(&dval, (size_t)o * 8 + 64)); CK(cudaMalloc(&dh, (size_t)m * 8));
    CK(cudaMalloc(&dout, (size_t)n * 8)); CK(cudaMalloc(&dref, (size_t)n * 8));
    CK(cudaMalloc(&x, (size_t)n * 8)); CK(cudaMalloc(&z, (size_t)n * 8)); CK(cudaMalloc(&dl, (size_t)n * 8)); CK(cudaMalloc(&c, (size_t)n * 8));
    CK(cudaMemcpy(dptr, ptr.data(), (n + 1) * 4, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(didx, idx.data(), (size_t)o * 4, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(dval, val.data(), (size_t)o * 8, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(dh, h.data(), (size_t)m * 8, cudaMemcpyHostToDevice));
    CK(cudaMemset(x, 0, (size_t)n * 8)); CK(cudaMemset(z, 0, (size_t)n * 8)); CK(cudaMemset(dl, 0, (size_t)n * 8)); CK(cudaMemset(c, 0, (size_t)n * 8));
    k_ref<<<148 * 8, 256>>>(dptr, didx, dval, dh, dref, n);
    CK(cudaDeviceSynchronize());
    std::vector<double> a(n), b(n);
    CK(cudaMemcpy(a.data(), dref, (size_t)n * 8, cudaMemcpyDeviceToHost));
    int sms = 148;
    cudaEvent_t e0, e1;
    CK(cudaEventCreate(&e0)); CK(cudaEventCreate(&e1));
    auto run = [&](auto kern, const char* name, bool check) {
        kern<<<sms * 6, 256>>>(dptr, didx, dval, dh, dout, x, z, dl, c, n);
        CK(cudaDeviceSynchronize());
        if (check) {
            CK(cudaMemcpy(b.data(), dout, (size_t)n * 8, cudaMemcpyDeviceToHost));
            long bad = 0;
            for (int j = 0; j < n; ++j) if (memcmp(&a[j], &b[j], 8)) ++bad;
            printf("%s: bit-identical to the sequential kernel: %s (%ld differ)\n", name, bad ? "NO" : "yes", bad);
        }
        for (int i = 0; i < 3; ++i) kern<<<sms * 6, 256>>>(dptr, didx, dval, dh, dout, x, z, dl, c, n);
        CK(cudaEventRecord(e0));
        const int reps = 50;
        for (int i = 0; i < reps; ++i) kern<<<sms * 6, 256>>>(dptr, didx, dval, dh, dout, x, z, dl, c, n);
        CK(cudaEventRecord(e1)); CK(cudaEventSynchronize(e1));
        float ms; CK(cudaEventElapsedTime(&ms, e0, e1));
        printf("%-40s %.4f ms/pass  %.1f G gathers/s\n", name, ms / reps, o / (ms / reps * 1e-3) / 1e9);
    };
    run(k_stream<0, 2>, "stream R=2 sums only", true);
    run(k_stream<0, 4>, "stream R=4 sums only", true);
    run(k_stream<0, 8>, "stream R=8 sums only", true);
    run(k_stream<1, 2>, "stream R=2 + LP epilogue", false);
    run(k_stream<1, 4>, "stream R=4 + LP epilogue", false);
    run(k_stream<1, 8>, "stream R=8 + LP epilogue", false);
    return 0;
}
