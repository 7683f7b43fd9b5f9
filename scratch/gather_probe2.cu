// Probe 2: is random-gather throughput bound per SM (L1TEX wavefronts) or chip-wide (L2)?
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#define CK(x) do{cudaError_t e=(x); if(e!=cudaSuccess){printf("CUDA %s @%d\n",cudaGetErrorString(e),__LINE__); return 1;}}while(0)
__device__ __forceinline__ uint32_t hsh(uint64_t k){ k^=k>>33; k*=0xff51afd7ed558ccdULL; k^=k>>33; k*=0xc4ceb9fe1a85ec53ULL; k^=k>>33; return (uint32_t)k; }
template<typename T, int MODE>
__global__ void g(const T* __restrict__ x, uint32_t n, long long per_thread, double* out){
  double acc=0; uint64_t base=((uint64_t)blockIdx.x*blockDim.x+threadIdx.x)*per_thread;
  #pragma unroll 8
  for(long long t=0;t<per_thread;t++){
    uint32_t j=hsh(base+t)%n;
    T v;
    if(MODE==0) v=x[j]; else if (MODE==1) v=__ldcg(x+j); else v=__ldg(x+j);
    if constexpr (sizeof(T)==16) acc += ((double*)&v)[0]; else acc+=(double)v;
  }
  if(acc==1234.5) out[0]=acc;
}
template<typename T,int MODE> int run(const char* name, void* x, uint32_t n, int ctas, int thr, long long pt, double* out){
  cudaEvent_t e0,e1; cudaEventCreate(&e0); cudaEventCreate(&e1); float best=1e9;
  for(int r=0;r<4;r++){ cudaEventRecord(e0); g<T,MODE><<<ctas,thr>>>((const T*)x,n,pt,out); cudaEventRecord(e1); CK(cudaEventSynchronize(e1)); float ms; cudaEventElapsedTime(&ms,e0,e1); if(r&&ms<best)best=ms;}
  double gathers=(double)ctas*thr*pt; printf("%-10s n=%u ctas=%d thr=%d: %.3f ms  %.1f Ggather/s  %.3f gathers/SMcycle@1.9G\n",name,n,ctas,thr,best,gathers/best/1e6, gathers/best/1e6/ (ctas<148?ctas:148)/1.9);
  return 0;
}
int main(){
  void* x; CK(cudaMalloc(&x, 160ll<<20)); cudaMemset(x,0,160ll<<20); double* out; CK(cudaMalloc(&out,64));
  uint32_t n=4000000; // 32 MB of doubles: L2 resident
  for(int ctas: {37,74,148}) run<double,0>("f64",x,n,ctas,1024,2000,out);
  run<double,0>("f64",x,n,148*2,1024,2000,out);
  run<double,1>("f64.cg",x,n,148*2,1024,2000,out);
  run<double,2>("f64.nc",x,n,148*2,1024,2000,out);
  run<float,0>("f32",x,n,148*2,1024,2000,out);
  run<double2,0>("f64x2",x,n/2,148*2,1024,2000,out);
  run<double,0>("f64 n=16K",x,16384,148*2,1024,2000,out);
  run<double,0>("f64 n=10M",x,10000000,148*2,1024,2000,out);
  return 0;
}
