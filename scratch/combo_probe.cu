// Probe: do TMA tile::gather4 and LSU gathers add up? (random fp64 rows from a 40 MB vector)
#include <cstdio>
#include <cstdint>
#include <cuda.h>
#include <cuda_runtime.h>
#define CK(x) do{cudaError_t e=(x); if(e!=cudaSuccess){printf("CUDA %s @%d\n",cudaGetErrorString(e),__LINE__); return 1;}}while(0)
__device__ __forceinline__ uint32_t hsh(uint64_t k){ k^=k>>33; k*=0xff51afd7ed558ccdULL; k^=k>>33; k*=0xc4ceb9fe1a85ec53ULL; k^=k>>33; return (uint32_t)k; }
__device__ __forceinline__ uint32_t smem_u32(const void* p){ return (uint32_t)__cvta_generic_to_shared(p);}
__device__ __forceinline__ void mbar_init(uint64_t* b, int cnt){ asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;"::"r"(smem_u32(b)),"r"(cnt)); }
__device__ __forceinline__ void mbar_expect(uint64_t* b, uint32_t bytes){ asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;"::"r"(smem_u32(b)),"r"(bytes):"memory"); }
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t phase){
  asm volatile("{\n.reg .pred p;\nW: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W;\n}\n"::"r"(smem_u32(b)),"r"(phase):"memory"); }
__device__ __forceinline__ double ld_g(const double* p){ double v; asm volatile("ld.global.nc.L1::no_allocate.f64 %0,[%1];":"=d"(v):"l"(p)); return v;}

#define STAGES 4
#define PER_STAGE 32
// warps [0, tmaw) issue gather4 (lanes 0..31 each one gather4 per stage); others LSU-gather
__global__ void __launch_bounds__(1024) combo(const __grid_constant__ CUtensorMap tm, const double* x, uint32_t nrows,
    int tmaw, int titers, int liters, double* out){
  __shared__ __align__(128) double buf[2][STAGES][PER_STAGE][8][2];
  __shared__ __align__(8) uint64_t bar[2][STAGES];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) { for (int t = 0; t < 2; t++) for(int s=0;s<STAGES;s++) mbar_init(&bar[t][s],1); asm volatile("fence.mbarrier_init.release.cluster;"); }
  __syncthreads();
  uint64_t seed=((uint64_t)blockIdx.x<<40) + ((uint64_t)threadIdx.x << 20);
  if (w < tmaw) {
    for(int it=0; it<titers; it++){
      int s=it%STAGES; uint32_t ph=(it/STAGES)&1;
      if(it>=STAGES){ mbar_wait(&bar[w][s], ph^1); }
      __syncwarp();
      if(lane==0) mbar_expect(&bar[w][s], PER_STAGE*4*16);
      __syncwarp();
      int r0=hsh(seed+it*4+0)%nrows, r1=hsh(seed+it*4+1)%nrows, r2=hsh(seed+it*4+2)%nrows, r3=hsh(seed+it*4+3)%nrows;
      asm volatile("cp.async.bulk.tensor.2d.shared::cta.global.tile::gather4.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5, %6}], [%7];"
        ::"r"(smem_u32(&buf[w][s][lane][0][0])),"l"(&tm),"r"(0),"r"(r0),"r"(r1),"r"(r2),"r"(r3),"r"(smem_u32(&bar[w][s])):"memory");
    }
    for(int it=titers; it<titers+STAGES; it++){ int s=it%STAGES; uint32_t ph=(it/STAGES)&1; if(it>=STAGES) mbar_wait(&bar[w][s],ph^1);}
    if(buf[w][0][lane][0][0]==1234.5) out[0]=1;
  } else {
    double acc = 0;
    for (int it = 0; it < liters; it += 8) {
      double v[8];
#pragma unroll
      for (int u = 0; u < 8; u++) v[u] = ld_g(x + 2ull * (hsh(seed + it + u) % nrows));
#pragma unroll
      for (int u = 0; u < 8; u++) acc += v[u];
    }
    if (acc == 1234.5) out[0] = acc;
  }
}

typedef CUresult (*encode_t)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
int main(){
  uint32_t nrows=2500000; double* x; CK(cudaMalloc(&x, nrows*16ull)); cudaMemset(x,0,nrows*16ull); double* out; CK(cudaMalloc(&out,64));
  encode_t enc; cudaDriverEntryPointQueryResult q; CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled",(void**)&enc,cudaEnableDefault,&q));
  CUtensorMap tm; cuuint64_t gdim[2]={2,nrows}; cuuint64_t gstr[1]={16}; cuuint32_t box[2]={2,1}; cuuint32_t es[2]={1,1};
  CUresult r=enc(&tm,CU_TENSOR_MAP_DATA_TYPE_FLOAT64,2,x,gdim,gstr,box,es,CU_TENSOR_MAP_INTERLEAVE_NONE,CU_TENSOR_MAP_SWIZZLE_NONE,CU_TENSOR_MAP_L2_PROMOTION_NONE,CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  printf("encode rc=%d\n",(int)r);
  CK(cudaFuncSetAttribute(combo, cudaFuncAttributeMaxDynamicSharedMemorySize, 0));
  cudaEvent_t e0,e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  struct Cfg { int threads, tmaw, titers, liters; };
  Cfg cfgs[] = {{1024,0,0,4096},{1024,1,4096,0},{1024,2,4096,0},{1024,1,4096,4096},{1024,2,4096,4096},{1024,2,8192,4096},{512,1,4096,4096},{1024,2,2048,4096}};
  for (auto c : cfgs) {
    float best=1e9;
    for(int rep=0;rep<3;rep++){ cudaEventRecord(e0); combo<<<148, c.threads>>>(tm,x,nrows,c.tmaw,c.titers,c.liters,out);
      cudaEventRecord(e1); CK(cudaEventSynchronize(e1)); float ms; cudaEventElapsedTime(&ms,e0,e1); if(rep&&ms<best)best=ms; }
    double trows=148.0*c.tmaw*32*4*(double)c.titers, lrows=148.0*(c.threads/32-c.tmaw)*32*(double)c.liters;
    double cyc = best*1e-3*1.9e9;
    printf("thr=%d tmaw=%d titers=%d liters=%d: %.3f ms  tma %.3f + lsu %.3f = %.3f rows/SM-cycle@1.9G\n", c.threads,c.tmaw,c.titers,c.liters,best,
      trows/148/cyc, lrows/148/cyc, (trows+lrows)/148/cyc);
  }
  return 0;
}
