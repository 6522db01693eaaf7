// Per-SM streaming bandwidth probe: cp.async.bulk ring (chunk, stages) vs LDG.128, for G CTAs.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__device__ __forceinline__ uint32_t sa(const void* p){return (uint32_t)__cvta_generic_to_shared(p);}
__global__ void k_bulk(const double* src, long long per_cta, int chunk, int stages, double* out){
  extern __shared__ __align__(128) unsigned char sm[];
  uint64_t* bar=(uint64_t*)sm; double* buf=(double*)(sm+128);
  const double* s=src+blockIdx.x*per_cta; int nch=per_cta/chunk; int tid=threadIdx.x;
  if(tid==0){for(int q=0;q<stages;++q) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;"::"r"(sa(&bar[q])));
    asm volatile("fence.mbarrier_init.release.cluster;");}
  __syncthreads();
  auto issue=[&](int q){int st=q%stages; asm volatile("fence.proxy.async.shared::cta;");
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;"::"r"(sa(&bar[st])),"r"(chunk*8));
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"::"r"(sa(buf+(size_t)st*chunk)),"l"(s+(size_t)q*chunk),"r"(chunk*8),"r"(sa(&bar[st])):"memory");};
  if(tid==0) for(int q=0;q<stages&&q<nch;++q) issue(q);
  double acc=0;
  for(int q=0;q<nch;++q){int st=q%stages; uint32_t par=(q/stages)&1;
    asm volatile("{.reg .pred P1; W%=: mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1; @!P1 bra W%=;}"::"r"(sa(&bar[st])),"r"(par):"memory");
    const double* b=buf+(size_t)st*chunk; for(int i=tid;i<chunk;i+=blockDim.x) acc+=b[i];
    __syncthreads(); if(tid==0&&q+stages<nch) issue(q+stages);}
  if(acc==12345.678) out[0]=acc;
}
__global__ void k_ldg(const double* src, long long per_cta, double* out){
  const double2* s=(const double2*)(src+blockIdx.x*per_cta); long long n2=per_cta/2; double acc=0;
  #pragma unroll 8
  for(long long i=threadIdx.x;i<n2;i+=blockDim.x){double2 v=__ldg(s+i); acc+=v.x+v.y;}
  if(acc==12345.678) out[0]=acc;
}
int main(){
  long long total=1LL<<30; double* src; double* out; cudaMalloc(&src,total*8); cudaMalloc(&out,8); cudaMemset(src,0,total*8);
  cudaEvent_t a,b; cudaEventCreate(&a); cudaEventCreate(&b);
  int Gs[]={16,64,148,296};
  for(int G: Gs){
    long long per=(total/G)/8192*8192;
    int chunks[]={4096,8192,16384}; int stg[]={2,3,4,6,8};
    for(int ch: chunks) for(int st: stg){ size_t smem=128+(size_t)ch*8*st; if(smem>227*1024) continue;
      cudaFuncSetAttribute(k_bulk,cudaFuncAttributeMaxDynamicSharedMemorySize,smem);
      k_bulk<<<G,256,smem>>>(src,per,ch,st,out); cudaEventRecord(a);
      k_bulk<<<G,256,smem>>>(src,per,ch,st,out); cudaEventRecord(b); cudaEventSynchronize(b);
      float ms; cudaEventElapsedTime(&ms,a,b); printf("bulk G=%3d chunk=%6dB stages=%d: %7.1f GB/s total, %6.1f GB/s per CTA\n",G,ch*8,st,per*G*8/ms/1e6,per*8/ms/1e6);}
    for(int th: {256,512,1024}){ k_ldg<<<G,th>>>(src,per,out); cudaEventRecord(a); k_ldg<<<G,th>>>(src,per,out); cudaEventRecord(b); cudaEventSynchronize(b);
      float ms; cudaEventElapsedTime(&ms,a,b); printf("ldg  G=%3d threads=%4d: %7.1f GB/s total, %6.1f GB/s per CTA\n",G,th,per*G*8/ms/1e6,per*8/ms/1e6);}
  }
  printf("err %s\n",cudaGetErrorString(cudaGetLastError()));
}
