// Probe 3: random-row gather throughput via TMA tile::gather4 and via 16-byte cp.async.bulk,
// vs the LSU path's ~1 sector/SM-cycle.
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

#define STAGES 8
#define PER_STAGE 32   // gather4 ops (or bulk copies) per stage, issued by lanes 0..31

template<int MODE>
__global__ void __launch_bounds__(32) tma_gather(const __grid_constant__ CUtensorMap tm, const double* x, uint32_t nrows, int iters, double* out){
  __shared__ __align__(128) double buf[STAGES][PER_STAGE][8][2];
  __shared__ __align__(8) uint64_t bar[STAGES];
  int lane=threadIdx.x;
  if(lane==0){ for(int s=0;s<STAGES;s++) mbar_init(&bar[s],1); asm volatile("fence.mbarrier_init.release.cluster;"); }
  __syncwarp();
  uint64_t seed=((uint64_t)blockIdx.x<<32);
  const uint32_t stage_bytes = MODE==0 ? PER_STAGE*4*16 : PER_STAGE*16;
  for(int it=0; it<iters; it++){
    int s=it%STAGES; uint32_t ph=(it/STAGES)&1;
    if(it>=STAGES){ mbar_wait(&bar[s], ph^1); }
    __syncwarp();
    if(lane==0) mbar_expect(&bar[s], stage_bytes);
    __syncwarp();
    if(MODE==0){
      int r0=hsh(seed+it*128+lane*4+0)%nrows, r1=hsh(seed+it*128+lane*4+1)%nrows, r2=hsh(seed+it*128+lane*4+2)%nrows, r3=hsh(seed+it*128+lane*4+3)%nrows;
      asm volatile("cp.async.bulk.tensor.2d.shared::cta.global.tile::gather4.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5, %6}], [%7];"
        ::"r"(smem_u32(&buf[s][lane][0][0])),"l"(&tm),"r"(0),"r"(r0),"r"(r1),"r"(r2),"r"(r3),"r"(smem_u32(&bar[s])):"memory");
    } else {
      uint32_t r=hsh(seed+it*32+lane)%nrows;
      asm volatile("cp.async.bulk.shared::cta.global.mbarrier::complete_tx::bytes [%0], [%1], 16, [%2];"
        ::"r"(smem_u32(&buf[s][lane][0][0])),"l"(x+2ull*r),"r"(smem_u32(&bar[s])):"memory");
    }
  }
  for(int it=iters; it<iters+STAGES; it++){ int s=it%STAGES; uint32_t ph=(it/STAGES)&1; if(it>=STAGES) mbar_wait(&bar[s],ph^1);} 
  if(buf[0][lane][0][0]==1234.5) out[0]=1;
}

typedef CUresult (*encode_t)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
int main(){
  uint32_t nrows=2000000; double* x; CK(cudaMalloc(&x, nrows*16ull)); cudaMemset(x,0,nrows*16ull); double* out; CK(cudaMalloc(&out,64));
  encode_t enc; cudaDriverEntryPointQueryResult q; CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled",(void**)&enc,cudaEnableDefault,&q));
  CUtensorMap tm; cuuint64_t gdim[2]={2,nrows}; cuuint64_t gstr[1]={16}; cuuint32_t box[2]={2,1}; cuuint32_t es[2]={1,1};
  CUresult r=enc(&tm,CU_TENSOR_MAP_DATA_TYPE_FLOAT64,2,x,gdim,gstr,box,es,CU_TENSOR_MAP_INTERLEAVE_NONE,CU_TENSOR_MAP_SWIZZLE_NONE,CU_TENSOR_MAP_L2_PROMOTION_NONE,CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  printf("encode rc=%d\n",(int)r);
  cudaEvent_t e0,e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for(int mode=0; mode<2; mode++) for(int cps : {1,2,4,8}){
    int ctas=148*cps, iters=4000; float best=1e9;
    for(int rep=0;rep<3;rep++){ cudaEventRecord(e0); if(mode==0) tma_gather<0><<<ctas,32>>>(tm,x,nrows,iters,out); else tma_gather<1><<<ctas,32>>>(tm,x,nrows,iters,out);
      cudaEventRecord(e1); CK(cudaEventSynchronize(e1)); float ms; cudaEventElapsedTime(&ms,e0,e1); if(rep&&ms<best)best=ms; }
    double rows=(double)ctas*iters*PER_STAGE*(mode==0?4:1);
    printf("%s ctas/SM=%d: %.3f ms  %.1f G rows/s  %.3f rows/SM-cycle@1.9G\n", mode==0?"gather4":"bulk16 ", cps, best, rows/best/1e6, rows/best/1e6/148/1.9);
  }
  return 0;
}
