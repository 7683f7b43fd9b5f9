// Probe: cost of one cluster-wide synchronisation for k_cluster (1024 threads per CTA),
// barrier.cluster (cg::cluster_group::sync) vs point-to-point mbarriers (each CTA: CTA
// barrier, then thread q of CTA... arrives remotely on every peer's mbarrier; every CTA
// waits on its own). 4000 synchronisations per launch; prints ns per sync.
#include <cooperative_groups.h>
#include <cuda_runtime.h>
#include <cstdio>
namespace cg = cooperative_groups;
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e)); exit(1); } } while (0)

__global__ void __launch_bounds__(1024, 1) k_barrier(int iters, int* out) {
    cg::cluster_group cl = cg::this_cluster();
    int acc = 0;
    for (int i = 0; i < iters; ++i) { cl.sync(); acc += i; }
    if (acc == -1) out[0] = acc;
}

__device__ __forceinline__ unsigned sm_addr(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }

__global__ void __launch_bounds__(1024, 1) k_mbar(int iters, int* out) {
    __shared__ __align__(8) unsigned long long bar[2];
    cg::cluster_group cl = cg::this_cluster();
    const int C = (int)cl.num_blocks(), q = (int)cl.block_rank(), t = threadIdx.x;
    if (t == 0) {
        for (int b = 0; b < 2; ++b) asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" :: "r"(sm_addr(&bar[b])), "r"(C));
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    cl.sync();
    for (int i = 0; i < iters; ++i) {
        const int b = i & 1;
        __syncthreads();   // this CTA's work (and remote stores) done
        if (t < C) {       // thread u arrives on CTA u's barrier
            unsigned remote;
            asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(remote) : "r"(sm_addr(&bar[b])), "r"(t));
            asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" :: "r"(remote) : "memory");
        }
        // everyone waits on the local barrier (parity of this buffer's use)
        const unsigned par = (unsigned)((i >> 1) & 1);
        unsigned ok = 0;
        while (!ok)
            asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                         : "=r"(ok) : "r"(sm_addr(&bar[b])), "r"(par) : "memory");
    }
    cl.sync();
    if (iters == -1) out[0] = 0;
}

int main() {
    int* out; CK(cudaMalloc(&out, 4));
    CK(cudaFuncSetAttribute(k_barrier, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    CK(cudaFuncSetAttribute(k_mbar, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    cudaEvent_t e0, e1; CK(cudaEventCreate(&e0)); CK(cudaEventCreate(&e1));
    const int iters = 4000;
    for (int C : {1, 2, 4, 8, 16}) {
        for (int kind = 0; kind < 2; ++kind) {
            cudaLaunchConfig_t lc{}; lc.gridDim = dim3(C); lc.blockDim = dim3(1024);
            cudaLaunchAttribute at[1]; at[0].id = cudaLaunchAttributeClusterDimension;
            at[0].val.clusterDim.x = C; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
            lc.attrs = at; lc.numAttrs = 1;
            auto go = [&] { if (kind == 0) CK(cudaLaunchKernelEx(&lc, k_barrier, iters, out)); else CK(cudaLaunchKernelEx(&lc, k_mbar, iters, out)); };
            go(); CK(cudaDeviceSynchronize());
            CK(cudaEventRecord(e0)); go(); CK(cudaEventRecord(e1)); CK(cudaEventSynchronize(e1));
            float ms; CK(cudaEventElapsedTime(&ms, e0, e1));
            printf("C=%2d %-22s %7.1f ns per sync\n", C, kind ? "mbarrier p2p" : "barrier.cluster", ms * 1e6 / iters);
        }
    }
    return 0;
}
