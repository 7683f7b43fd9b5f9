// Probe: random fp64 gather throughput through the L1TEX path (LDG) vs the TMA unit
// (cp.async.bulk.tensor.2d tile::gather4, sm_100a), and both at once.
//
// Question: a pass is bound by ~1.03 L1TEX line requests per SM-cycle for
// its random gathers. Does TMA gather4 add request bandwidth on top of that?
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o scratch/tma_gather_probe scratch/tma_gather_probe.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <vector>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e)); exit(1); } } while (0)

__device__ __forceinline__ uint32_t hsh(uint32_t a) {
    a ^= a >> 16; a *= 0x7feb352dU; a ^= a >> 15; a *= 0x846ca68bU; a ^= a >> 16; return a;
}

// ---------------- LDG gathers: every thread, U independent loads per round
template <int U>
__global__ void k_ldg(const double* __restrict__ x, uint32_t nrows, int rounds, int ldg_warps, double* out) {
    const int w = threadIdx.x >> 5;
    if (w >= ldg_warps) return;
    uint32_t s = hsh(blockIdx.x * 1024 + threadIdx.x);
    double acc = 0;
    for (int r = 0; r < rounds; ++r) {
        double v[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            s = hsh(s + u);
            v[u] = __ldcg(x + 2 * (size_t)(s % nrows));
        }
#pragma unroll
        for (int u = 0; u < U; ++u) acc += v[u];
    }
    if (acc == 12345.678) out[0] = acc;
}

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

// ---------------- TMA gather4: lane 0 of each TMA warp keeps D gather4 in flight (4 rows of 16 B each)
template <int D>
__global__ void k_tma(const __grid_constant__ CUtensorMap tm, uint32_t nrows, int rounds, int ldg_warps,
                      const double* __restrict__ x, double* out, int ldg_rounds = 0, int tma_warps = 16) {
    __shared__ __align__(128) double buf[16][D][16];
    __shared__ __align__(8) uint64_t bar[16][D];
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    uint32_t s = hsh(blockIdx.x * 1024 + threadIdx.x + 77);
    double acc = 0;
    if (w < ldg_warps) {   // mixed mode: these warps do LDG gathers concurrently
        for (int r = 0; r < ldg_rounds; ++r) {
            double v[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) { s = hsh(s + u); v[u] = __ldcg(x + 2 * (size_t)(s % nrows)); }
#pragma unroll
            for (int u = 0; u < 8; ++u) acc += v[u];
        }
        if (acc == 12345.678) out[0] = acc;
        return;
    }
    if (w >= ldg_warps + tma_warps) return;
    if (lane == 0) {
        for (int d = 0; d < D; ++d)
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(smem_u32(&bar[w][d])));
        asm volatile("fence.mbarrier_init.release.cluster;");
        uint32_t phase[D];
        for (int d = 0; d < D; ++d) phase[d] = 0;
        for (int it = 0; it < rounds * D; ++it) {
            const int d = it % D;
            if (it >= D) {
                uint32_t ok = 0;
                while (!ok) {
                    asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                                 : "=r"(ok) : "r"(smem_u32(&bar[w][d])), "r"(phase[d]));
                }
                phase[d] ^= 1;
                acc += buf[w][d][0] + buf[w][d][2] + buf[w][d][4] + buf[w][d][6];
            }
            int32_t r0, r1, r2, r3;
            s = hsh(s + 1); r0 = s % nrows; s = hsh(s + 2); r1 = s % nrows;
            s = hsh(s + 3); r2 = s % nrows; s = hsh(s + 4); r3 = s % nrows;
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], 64;" :: "r"(smem_u32(&bar[w][d])));
            asm volatile(
                "cp.async.bulk.tensor.2d.shared::cta.global.tile::gather4.mbarrier::complete_tx::bytes "
                "[%0], [%1, {%2, %3, %4, %5, %6}], [%7];"
                :: "r"(smem_u32(&buf[w][d][0])), "l"(&tm), "r"(0), "r"(r0), "r"(r1), "r"(r2), "r"(r3),
                   "r"(smem_u32(&bar[w][d])) : "memory");
        }
        for (int d = 0; d < D; ++d) {
            uint32_t ok = 0;
            while (!ok) {
                asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                             : "=r"(ok) : "r"(smem_u32(&bar[w][d])), "r"(phase[d]));
            }
            acc += buf[w][d][0];
        }
        if (acc == 12345.678) out[0] = acc;
    }
}

typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                             const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                             CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main(int argc, char** argv) {
    const uint32_t nrows = argc > 1 ? atoi(argv[1]) : 2500000;   // rows of 16 B: 40 MB (L2-resident)
    const int sms = 148;
    double *x, *out;
    CK(cudaMalloc(&x, (size_t)nrows * 16));
    CK(cudaMalloc(&out, 64));
    CK(cudaMemset(x, 0, (size_t)nrows * 16));
    EncodeFn enc = nullptr;
    cudaDriverEntryPointQueryResult q;
    CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc, cudaEnableDefault, &q));
    CUtensorMap tm;
    cuuint64_t gdim[2] = {2, nrows};
    cuuint64_t gstride[1] = {16};
    cuuint32_t box[2] = {2, 1};
    cuuint32_t estr[2] = {1, 1};
    CUresult r = enc(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, x, gdim, gstride, box, estr,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE,
                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) { printf("encode failed %d\n", (int)r); return 1; }
    cudaEvent_t e0, e1;
    CK(cudaEventCreate(&e0)); CK(cudaEventCreate(&e1));
    auto timeit = [&](auto launch, double rows_total, const char* name) {
        launch(); CK(cudaDeviceSynchronize());
        CK(cudaEventRecord(e0));
        for (int i = 0; i < 10; ++i) launch();
        CK(cudaEventRecord(e1)); CK(cudaEventSynchronize(e1));
        float ms; CK(cudaEventElapsedTime(&ms, e0, e1));
        double gps = rows_total * 10 / (ms * 1e-3) / 1e9;
        printf("%-44s %8.3f ms/launch  %7.1f G rows/s  %.3f rows/SM/ns\n", name, ms / 10, gps, gps / sms);
    };
    // LDG only: 148 x 512 threads x rounds x 8
    for (int warps : {8, 16}) {
        const int rounds = 400;
        char nm[64]; snprintf(nm, 64, "LDG 8B gathers, %d warps/CTA", warps);
        timeit([&] { k_ldg<8><<<sms * 2, warps * 32>>>(x, nrows, rounds, warps, out); },
               2.0 * sms * warps * 32 * rounds * 8, nm);
    }
    // TMA only
    for (int warps : {4, 8, 16}) {
        const int rounds = 4000;
        char nm[64]; snprintf(nm, 64, "TMA gather4 (16 B rows), %d warps x D=8", warps);
        timeit([&] { k_tma<8><<<sms, warps * 32>>>(tm, nrows, rounds, 0, x, out); },
               1.0 * sms * warps * rounds * 8 * 4, nm);
    }
    // additivity: the same per-warp work alone and together (time ~ max -> separate paths; ~ sum -> shared)
    {
        const int rounds = 4000, ldg_rounds = 800;
        const double tma_rows = 1.0 * sms * 8 * rounds * 8 * 4;
        const double ldg_rows = 1.0 * sms * 8 * 32 * ldg_rounds * 8;
        timeit([&] { k_tma<8><<<sms, 16 * 32>>>(tm, nrows, rounds, 8, x, out, ldg_rounds, 0); }, ldg_rows,
               "alone: 8 LDG warps");
        timeit([&] { k_tma<8><<<sms, 16 * 32>>>(tm, nrows, rounds, 0, x, out, 0, 8); }, tma_rows,
               "alone: 8 TMA warps");
        timeit([&] { k_tma<8><<<sms, 16 * 32>>>(tm, nrows, rounds, 8, x, out, ldg_rounds, 8); },
               tma_rows + ldg_rows, "together: 8 LDG + 8 TMA warps");
    }
    return 0;
}
