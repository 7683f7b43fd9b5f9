// Probe 4: random-gather throughput vs memory-level parallelism (threads/SM x loads in flight).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__device__ __forceinline__ uint32_t hsh(uint64_t k){ k^=k>>33; k*=0xff51afd7ed558ccdULL; k^=k>>33; k*=0xc4ceb9fe1a85ec53ULL; k^=k>>33; return (uint32_t)k; }
template<int U>
__global__ void g(const double* __restrict__ x, uint32_t n, int iters, double* out){
  double acc=0; uint64_t base=((uint64_t)blockIdx.x*blockDim.x+threadIdx.x)*iters*U;
  for(int t=0;t<iters;t++){
    uint32_t j[U]; double v[U];
    #pragma unroll
    for(int u=0;u<U;u++) j[u]=hsh(base+t*U+u)%n;
    #pragma unroll
    for(int u=0;u<U;u++) v[u]=__ldg(x+j[u]);
    #pragma unroll
    for(int u=0;u<U;u++) acc+=v[u];
  }
  if(acc==1234.5) out[0]=acc;
}
template<int U> void run(double* x, uint32_t n, int thr, double* out){
  cudaEvent_t e0,e1; cudaEventCreate(&e0); cudaEventCreate(&e1); float best=1e9; int iters=4096/U;
  for(int r=0;r<3;r++){ cudaEventRecord(e0); g<U><<<148,thr>>>(x,n,iters,out); cudaEventRecord(e1); cudaEventSynchronize(e1); float ms; cudaEventElapsedTime(&ms,e0,e1); if(r&&ms<best)best=ms;}
  double gathers=148.0*thr*iters*U; printf("thr/SM=%4d unroll=%2d inflight/SM<=%5d: %6.1f Ggather/s  (%.2f /SM-cycle@1.9G)\n",thr,U,thr*U,gathers/best/1e6,gathers/best/1e6/148/1.9);
}
int main(){ double* x; cudaMalloc(&x, 80ull<<20); cudaMemset(x,0,80ull<<20); double* out; cudaMalloc(&out,64); uint32_t n=5000000;
  for(int thr: {256,512,1024}){ run<4>(x,n,thr,out); run<8>(x,n,thr,out); run<16>(x,n,thr,out);} return 0; }
