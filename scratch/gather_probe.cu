// Probe: streaming + random-gather throughput on B200 (informs K1/K2 design).
#include <cstdio>
#include <cstdint>
#include <vector>
#include <random>
#include <cuda_runtime.h>
#define CK(x) do{cudaError_t e=(x); if(e!=cudaSuccess){printf("CUDA %s @%d\n",cudaGetErrorString(e),__LINE__); return 1;}}while(0)

__device__ __forceinline__ uint64_t pol_first(){ uint64_t p; asm("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;":"=l"(p)); return p;}
__device__ __forceinline__ uint64_t pol_last(){ uint64_t p; asm("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;":"=l"(p)); return p;}
__device__ __forceinline__ double ld_last(const double* p){ double v; asm volatile("ld.global.nc.L2::cache_hint.f64 %0,[%1],%2;":"=d"(v):"l"(p),"l"(pol_last())); return v;}
__device__ __forceinline__ int ld_first_i(const int* p){ int v; asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.s32 %0,[%1],%2;":"=r"(v):"l"(p),"l"(pol_first())); return v;}
__device__ __forceinline__ double ld_first_d(const double* p){ double v; asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.f64 %0,[%1],%2;":"=d"(v):"l"(p),"l"(pol_first())); return v;}

// out[k] -> sum of val[k]*x[idx[k]] over chunks; each thread strided
template<int MODE>
__global__ void gather_k(const int* __restrict__ idx, const double* __restrict__ val, const double* __restrict__ x, long long o, double* out){
  double acc=0; long long stride=(long long)gridDim.x*blockDim.x;
  for(long long k=blockIdx.x*(long long)blockDim.x+threadIdx.x;k<o;k+=stride){
    if(MODE==0){ acc += val[k]*x[idx[k]]; }
    else if(MODE==1){ acc += ld_first_d(val+k)*ld_last(x+ld_first_i(idx+k)); }
    else { acc += ld_first_d(val+k)*(double)ld_first_i(idx+k); } // stream only
  }
  if(acc==1234.5) out[0]=acc;
}
__global__ void copy_k(const double4* a, double4* b, long long n){ long long s=(long long)gridDim.x*blockDim.x; for(long long i=blockIdx.x*(long long)blockDim.x+threadIdx.x;i<n;i+=s) b[i]=a[i]; }

int main(){
  int dev=0; cudaDeviceProp pr; CK(cudaGetDeviceProperties(&pr,dev));
  printf("%s SMs=%d L2=%d MB persistMax=%d MB\n",pr.name,pr.multiProcessorCount,pr.l2CacheSize>>20,pr.persistingL2CacheMaxSize>>20);
  long long o=100000000; 
  int* idx; double* val; double* x; double* out;
  CK(cudaMalloc(&idx,o*4)); CK(cudaMalloc(&val,o*8)); CK(cudaMalloc(&out,64));
  long long nmax=10000000; CK(cudaMalloc(&x,nmax*8));
  std::vector<int> h(o); std::mt19937_64 g(1);
  cudaEvent_t e0,e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  // copy bandwidth
  { long long nb=1ll<<30; double4 *a,*b; CK(cudaMalloc(&a,nb)); CK(cudaMalloc(&b,nb)); cudaMemset(a,0,nb);
    for(int r=0;r<3;r++){ cudaEventRecord(e0); copy_k<<<148*8,256>>>(a,b,nb/32); cudaEventRecord(e1); cudaEventSynchronize(e1); float ms; cudaEventElapsedTime(&ms,e0,e1); printf("copy 1GiB: %.3f ms  %.1f GB/s\n",ms,2.0*nb/ms/1e6);} cudaFree(a); cudaFree(b);}
  for(long long n : {1000000ll, 5000000ll, 10000000ll}){
    for(long long k=0;k<o;k++) h[k]=(int)(g()%n);
    CK(cudaMemcpy(idx,h.data(),o*4,cudaMemcpyHostToDevice)); cudaMemset(val,0,o*8); cudaMemset(x,0,n*8);
    for(int mode=0;mode<3;mode++) for(int grid : {148*8, 148*16}){
      float best=1e9;
      for(int r=0;r<4;r++){ cudaEventRecord(e0);
        if(mode==0) gather_k<0><<<grid,256>>>(idx,val,x,o,out); else if(mode==1) gather_k<1><<<grid,256>>>(idx,val,x,o,out); else gather_k<2><<<grid,256>>>(idx,val,x,o,out);
        cudaEventRecord(e1); CK(cudaEventSynchronize(e1)); float ms; cudaEventElapsedTime(&ms,e0,e1); if(r>0&&ms<best)best=ms; }
      printf("n=%lld (x %lld MB) mode=%d grid=%d: %.3f ms  stream %.1f GB/s  gathers %.1f G/s\n",n,n*8>>20,mode,grid,best,12.0*o/best/1e6,o/best/1e6);
    }
  }
  return 0;
}
