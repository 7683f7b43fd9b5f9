// Probe: does the random-gather sector rate depend on how many lanes of a warp instruction are active?
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#define CK(x) do{cudaError_t e=(x); if(e!=cudaSuccess){printf("CUDA %s @%d\n",cudaGetErrorString(e),__LINE__); return 1;}}while(0)
__device__ __forceinline__ uint32_t hsh(uint64_t k){ k^=k>>33; k*=0xff51afd7ed558ccdULL; k^=k>>33; k*=0xc4ceb9fe1a85ec53ULL; k^=k>>33; return (uint32_t)k; }
__device__ __forceinline__ double ld_g(const double* p){ double v; asm volatile("ld.global.nc.L1::no_allocate.f64 %0,[%1];":"=d"(v):"l"(p)); return v;}

// every warp runs `iters` gather instructions; lanes >= active are predicated off
__global__ void __launch_bounds__(256) lanefill(const double* x, uint32_t n, int iters, int active, double* out){
  const int lane = threadIdx.x & 31;
  uint64_t seed=((uint64_t)blockIdx.x<<40) + ((uint64_t)threadIdx.x << 20);
  double acc = 0;
  const bool on = lane < active;
  for (int it = 0; it < iters; it += 8) {
    double v[8];
#pragma unroll
    for (int u = 0; u < 8; u++) v[u] = on ? ld_g(x + (hsh(seed + it + u) % n)) : 0.0;
#pragma unroll
    for (int u = 0; u < 8; u++) acc += v[u];
  }
  if (acc == 1234.5) out[0] = acc;
}

int main(){
  uint32_t n=5000000; double* x; CK(cudaMalloc(&x, n*8ull)); cudaMemset(x,0,n*8ull); double* out; CK(cudaMalloc(&out,64));
  cudaEvent_t e0,e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int ctas_per_sm : {6, 8}) for (int active : {32, 24, 16, 8}) {
    int iters = 2048; float best=1e9;
    for(int rep=0;rep<3;rep++){ cudaEventRecord(e0); lanefill<<<148*ctas_per_sm, 256>>>(x,n,iters,active,out);
      cudaEventRecord(e1); CK(cudaEventSynchronize(e1)); float ms; cudaEventElapsedTime(&ms,e0,e1); if(rep&&ms<best)best=ms; }
    double rows=148.0*ctas_per_sm*8*active*(double)iters, instr=148.0*ctas_per_sm*8*(double)iters;
    double cyc = best*1e-3*1.9e9;
    printf("ctas/SM=%d active=%2d: %.3f ms  %.3f gathers/SM-cycle  %.3f instr/SM-cycle\n", ctas_per_sm, active, best, rows/148/cyc, instr/148/cyc);
  }
  return 0;
}
