// Probe: cost of streaming idx/val next to random gathers — TMA bulk vs LDG vs cp.async.
// Each element: idx (i32) + val (f64) streamed, x[idx] gathered (x L2-resident), acc += val*x.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#define CK(x) do{cudaError_t e=(x); if(e!=cudaSuccess){printf("CUDA %s @%d\n",cudaGetErrorString(e),__LINE__); return 1;}}while(0)

constexpr int T = 2048;          // elements per tile
constexpr int NC = 512;          // consumer threads
constexpr int S = 4;             // stages
struct alignas(128) Stage { int idx[T]; double val[T]; };

__device__ __forceinline__ uint32_t sa(const void* p){ return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* b, int c){ asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;"::"r"(sa(b)),"r"(c):"memory"); }
__device__ __forceinline__ void mbar_tx(uint64_t* b, uint32_t n){ asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;"::"r"(sa(b)),"r"(n):"memory"); }
__device__ __forceinline__ void mbar_arrive(uint64_t* b){ asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];"::"r"(sa(b)):"memory"); }
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t ph){ asm volatile("{\n.reg .pred P;\nW%=:\nmbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n@!P bra W%=;\n}\n"::"r"(sa(b)),"r"(ph):"memory"); }
__device__ __forceinline__ uint64_t polf(){ uint64_t p; asm("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;":"=l"(p)); return p; }
__device__ __forceinline__ void bulk(void* d, const void* s, uint32_t n, uint64_t* b){ asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;"::"r"(sa(d)),"l"(s),"r"(n),"r"(sa(b)),"l"(polf()):"memory"); }
__device__ __forceinline__ double gat(const double* p){ double v; asm("ld.global.nc.L1::no_allocate.f64 %0, [%1];":"=d"(v):"l"(p)); return v; }

// MODE 0: TMA stream + gather; 1: TMA stream only; 2: gather only (idx from hash, val const)
template<int MODE, int NC=512, int T=2048, int S=4>
__global__ void __launch_bounds__(NC+32) k_tma(const int* idx, const double* val, const double* x, int ntiles, double* out){
  struct alignas(128) Stage { int idx[T]; double val[T]; };
  extern __shared__ __align__(128) unsigned char sm[];
  Stage* st=(Stage*)sm; uint64_t* full=(uint64_t*)(sm+S*sizeof(Stage)); uint64_t* empty=full+S;
  int my=(ntiles-(int)blockIdx.x+gridDim.x-1)/gridDim.x;
  if(threadIdx.x==0){ for(int s=0;s<S;s++){ mbar_init(&full[s],1); mbar_init(&empty[s],NC/32);} asm volatile("fence.mbarrier_init.release.cluster;":::"memory"); }
  __syncthreads();
  if(threadIdx.x>=NC){
    if(threadIdx.x==NC && MODE!=2){
      for(int i=0;i<my;i++){ int s=i%S; if(i>=S) mbar_wait(&empty[s],((i/S)-1)&1);
        long t=(long)blockIdx.x+(long)i*gridDim.x;
        mbar_tx(&full[s],T*12); bulk(st[s].idx,idx+t*T,T*4,&full[s]); bulk(st[s].val,val+t*T,T*8,&full[s]); }
    }
    return;
  }
  double acc=0;
  for(int i=0;i<my;i++){ int s=i%S;
    if(MODE!=2) mbar_wait(&full[s],(i/S)&1);
    long t=(long)blockIdx.x+(long)i*gridDim.x;
    #pragma unroll
    for(int u=0;u<T/NC;u++){ int e=threadIdx.x+u*NC;
      if(MODE==0) acc+=st[s].val[e]*gat(x+st[s].idx[e]);
      else if(MODE==1) acc+=st[s].val[e]+st[s].idx[e];
      else { uint32_t j=(uint32_t)((t*T+e)*2654435761u)%5000000u; acc+=gat(x+j); }
    }
    __syncwarp(); if(MODE!=2 && (threadIdx.x&31)==0) mbar_arrive(&empty[s]);
  }
  if(acc==1234.5) out[0]=acc;
}
// MODE 0: LDG stream + gather; 1: LDG stream only
template<int MODE>
__global__ void __launch_bounds__(NC,1) k_ldg(const int* idx, const double* val, const double* x, int ntiles, double* out){
  double acc=0;
  for(long t=blockIdx.x;t<ntiles;t+=gridDim.x){
    int j[T/NC]; double v[T/NC];
    #pragma unroll
    for(int u=0;u<T/NC;u++){ long e=t*T+threadIdx.x+u*NC; j[u]=__ldcs(idx+e); v[u]=__ldcs(val+e); }
    #pragma unroll
    for(int u=0;u<T/NC;u++){ if(MODE==0) acc+=v[u]*gat(x+j[u]); else acc+=v[u]+j[u]; }
  }
  if(acc==1234.5) out[0]=acc;
}
template<int MODE>
__global__ void __launch_bounds__(NC,1) k_ldg_rt(const int* idx, const double* val, const double* x, int ntiles, double* out){
  __shared__ int si[NC*4]; __shared__ double sv[NC*4];
  double acc=0;
  for(long t=blockIdx.x;t<ntiles;t+=gridDim.x){
    int j[T/NC]; double v[T/NC];
    #pragma unroll
    for(int u=0;u<T/NC;u++){ long e=t*T+threadIdx.x+u*NC; j[u]=__ldcs(idx+e); v[u]=__ldcs(val+e); }
    #pragma unroll
    for(int u=0;u<T/NC;u++){ si[threadIdx.x+u*NC]=j[u]; sv[threadIdx.x+u*NC]=v[u]; }
    __syncwarp();
    #pragma unroll
    for(int u=0;u<T/NC;u++){ j[u]=si[threadIdx.x+u*NC]; v[u]=sv[threadIdx.x+u*NC]; }
    #pragma unroll
    for(int u=0;u<T/NC;u++){ acc+=v[u]*gat(x+j[u]); }
    __syncwarp();
  }
  if(acc==1234.5) out[0]=acc;
}
// cp.async 16B stream (consumers copy their own next tile, double buffer) + gather
__device__ __forceinline__ void cpa16(void* d,const void* s){ asm volatile("cp.async.cg.shared.global.L2::cache_hint [%0], [%1], 16, %2;"::"r"(sa(d)),"l"(s),"l"(polf()):"memory"); }
template<int MODE>
__global__ void __launch_bounds__(NC,1) k_cpa(const int* idx, const double* val, const double* x, int ntiles, double* out){
  extern __shared__ __align__(128) unsigned char sm[];
  Stage* st=(Stage*)sm;
  int my=(ntiles-(int)blockIdx.x+gridDim.x-1)/gridDim.x;
  auto issue=[&](int i){ if(i<my){ long t=(long)blockIdx.x+(long)i*gridDim.x; Stage& s=st[i%S];
      for(int c=threadIdx.x;c<T/4;c+=NC) cpa16(&s.idx[c*4], idx+t*T+c*4);
      for(int c=threadIdx.x;c<T/2;c+=NC) cpa16(&s.val[c*2], val+t*T+c*2);}
    asm volatile("cp.async.commit_group;":::"memory"); };
  for(int i=0;i<S-1;i++) issue(i);
  double acc=0;
  for(int i=0;i<my;i++){ int s=i%S;
    asm volatile("cp.async.wait_group %0;"::"n"(S-2):"memory"); __syncthreads();
    #pragma unroll
    for(int u=0;u<T/NC;u++){ int e=threadIdx.x+u*NC; if(MODE==0) acc+=st[s].val[e]*gat(x+st[s].idx[e]); else acc+=st[s].val[e]+st[s].idx[e]; }
    __syncthreads();
    issue(i+S-1);
  }
  if(acc==1234.5) out[0]=acc;
}

template<class F> float tm(F f){ cudaEvent_t a,b; cudaEventCreate(&a); cudaEventCreate(&b); float best=1e9; for(int r=0;r<5;r++){ cudaEventRecord(a); f(); cudaEventRecord(b); cudaEventSynchronize(b); float ms; cudaEventElapsedTime(&ms,a,b); if(r&&ms<best)best=ms;} return best; }

int main(){
  const long N=100l*1000*1000; const int ntiles=N/T; const int nx=5000000;
  int* idx; double* val; double* x; double* out;
  CK(cudaMalloc(&idx,N*4)); CK(cudaMalloc(&val,N*8)); CK(cudaMalloc(&x,nx*8)); CK(cudaMalloc(&out,64));
  // random idx
  int* h=(int*)malloc(N*4); uint64_t s=88172645463325252ull; for(long i=0;i<N;i++){ s^=s<<13; s^=s>>7; s^=s<<17; h[i]=(int)(s%nx);}
  CK(cudaMemcpy(idx,h,N*4,cudaMemcpyHostToDevice)); cudaMemset(val,0,N*8); cudaMemset(x,0,nx*8);
  int sms; cudaDeviceGetAttribute(&sms,cudaDevAttrMultiProcessorCount,0);
  size_t smt=S*sizeof(Stage)+2*S*8;
  cudaFuncSetAttribute(k_tma<0>,cudaFuncAttributeMaxDynamicSharedMemorySize,(int)smt);
  cudaFuncSetAttribute(k_tma<1>,cudaFuncAttributeMaxDynamicSharedMemorySize,(int)smt);
  cudaFuncSetAttribute(k_tma<2>,cudaFuncAttributeMaxDynamicSharedMemorySize,(int)smt);
  cudaFuncSetAttribute(k_cpa<0>,cudaFuncAttributeMaxDynamicSharedMemorySize,(int)smt);
  cudaFuncSetAttribute(k_cpa<1>,cudaFuncAttributeMaxDynamicSharedMemorySize,(int)smt);
  printf("tiles %d, smem %zu\n",ntiles,smt);
  printf("tma stream+gather : %.3f ms\n", tm([&]{k_tma<0><<<sms,NC+32,smt>>>(idx,val,x,ntiles,out);}));
  {
    size_t s2=2*(2048*12+128)+64; cudaFuncSetAttribute(k_tma<0,512,2048,2>,cudaFuncAttributeMaxDynamicSharedMemorySize,(int)s2);
    printf("tma S=2 T=2048 NC=512 1cta: %.3f ms\n", tm([&]{k_tma<0,512,2048,2><<<sms,NC+32,s2>>>(idx,val,x,ntiles,out);}));
    size_t s3=4*(1024*12+128)+64; cudaFuncSetAttribute(k_tma<0,256,1024,4>,cudaFuncAttributeMaxDynamicSharedMemorySize,(int)s3);
    printf("tma S=4 T=1024 NC=256 2cta: %.3f ms\n", tm([&]{k_tma<0,256,1024,4><<<2*sms,256+32,s3>>>(idx,val,x,ntiles*2,out);}));
    printf("tma S=4 T=1024 NC=256 3cta: %.3f ms\n", tm([&]{k_tma<0,256,1024,4><<<3*sms,256+32,s3>>>(idx,val,x,ntiles*2,out);}));
    size_t s4=4*(512*12+128)+64; cudaFuncSetAttribute(k_tma<0,128,512,4>,cudaFuncAttributeMaxDynamicSharedMemorySize,(int)s4);
    printf("tma S=4 T=512 NC=128 4cta: %.3f ms\n", tm([&]{k_tma<0,128,512,4><<<4*sms,128+32,s4>>>(idx,val,x,ntiles*4,out);}));
    printf("ldg + smem roundtrip: %.3f ms\n", tm([&]{k_ldg_rt<0><<<sms,NC>>>(idx,val,x,ntiles,out);}));
  }
  printf("tma stream only   : %.3f ms\n", tm([&]{k_tma<1><<<sms,NC+32,smt>>>(idx,val,x,ntiles,out);}));
  printf("ldg stream+gather : %.3f ms\n", tm([&]{k_ldg<0><<<sms,NC>>>(idx,val,x,ntiles,out);}));
  printf("ldg stream+gather 2CTA: %.3f ms\n", tm([&]{k_ldg<0><<<2*sms,NC>>>(idx,val,x,ntiles,out);}));
  cudaFuncSetAttribute(k_ldg<0>,cudaFuncAttributeMaxDynamicSharedMemorySize,200000);
  for (int kb : {16, 64, 98, 128, 160, 190})
    printf("ldg stream+gather smem %d KB: %.3f ms\n", kb, tm([&]{k_ldg<0><<<sms,NC,kb*1024>>>(idx,val,x,ntiles,out);}));
  printf("ldg stream only   : %.3f ms\n", tm([&]{k_ldg<1><<<sms,NC>>>(idx,val,x,ntiles,out);}));
  printf("cpa stream+gather : %.3f ms\n", tm([&]{k_cpa<0><<<sms,NC,smt>>>(idx,val,x,ntiles,out);}));
  printf("cpa stream only   : %.3f ms\n", tm([&]{k_cpa<1><<<sms,NC,smt>>>(idx,val,x,ntiles,out);}));
  CK(cudaGetLastError()); CK(cudaDeviceSynchronize());
  return 0;
}
