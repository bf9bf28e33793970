// Microbenchmarks to size the radix-sort design on B200 (scratch; not product code).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#define CK(x) do{cudaError_t e=(x); if(e!=cudaSuccess){printf("CUDA %s at %d\n", cudaGetErrorString(e), __LINE__); return 1;}}while(0)

__device__ __forceinline__ uint32_t hsh(uint32_t x){ x^=x>>16; x*=0x7feb352d; x^=x>>15; x*=0x846ca68b; x^=x>>16; return x; }

template<int MODE>
__global__ void k_smem_atomic(uint32_t* out, int iters){
  __shared__ uint32_t h[256*8];
  for(int i=threadIdx.x;i<256*8;i+=blockDim.x) h[i]=0;
  __syncthreads();
  uint32_t s = hsh(threadIdx.x + blockIdx.x*blockDim.x);
  uint32_t acc=0;
  for(int it=0; it<iters; ++it){
    s = s*1664525u + 1013904223u;
    uint32_t d = s>>24;
    if(MODE==0) atomicAdd(&h[d],1u);
    else if(MODE==1) acc += atomicAdd(&h[d],1u);
    else if(MODE==2){ unsigned p=__match_any_sync(0xffffffffu,d); acc+=p; }
    else if(MODE==3){ atomicAdd(&h[(threadIdx.x>>5&7)*256+d],1u);} // warp-private (8 copies)
    else if(MODE==4){ d = (s>>31)? 7u : (s>>24); atomicAdd(&h[d],1u);} // 50% skew
    else if(MODE==5){ d = 7u; atomicAdd(&h[d],1u);} // all same
  }
  __syncthreads();
  if(threadIdx.x==0) out[blockIdx.x]=h[threadIdx.x]+acc;
}

__global__ void k_read(const uint4* __restrict__ p, size_t n, uint32_t* out){
  uint32_t x=0;
  for(size_t i=blockIdx.x*(size_t)blockDim.x+threadIdx.x;i<n;i+=(size_t)gridDim.x*blockDim.x){ uint4 v=__ldg(p+i); x^=v.x^v.y^v.z^v.w; }
  if(x==0x12345678) out[0]=x;
}
__global__ void k_copy(const uint4* __restrict__ p, uint4* __restrict__ q, size_t n){
  for(size_t i=blockIdx.x*(size_t)blockDim.x+threadIdx.x;i<n;i+=(size_t)gridDim.x*blockDim.x){ q[i]=p[i]; }
}
__global__ void k_gred(uint32_t* h, int iters, uint32_t mask){
  uint32_t s = hsh(threadIdx.x + blockIdx.x*blockDim.x);
  for(int it=0; it<iters; ++it){ s = s*1664525u + 1013904223u; atomicAdd(&h[(s>>8)&mask],1u); }
}

int main(){
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  uint32_t* out; CK(cudaMalloc(&out, 1<<24));
  cudaEvent_t a,b; cudaEventCreate(&a); cudaEventCreate(&b);
  const char* names[]={"atomicAdd smem noret","atomicAdd smem ret","match_any","warp-private atomics","50% skew atomics","all-same atomics"};
  for(int mode=0; mode<6; ++mode){
    for(int bs: {256,512,1024}){
      int iters=4096; int grid=sms*(2048/bs);
      float ms=0;
      for(int r=0;r<3;++r){
        cudaEventRecord(a);
        switch(mode){case 0:k_smem_atomic<0><<<grid,bs>>>(out,iters);break;case 1:k_smem_atomic<1><<<grid,bs>>>(out,iters);break;case 2:k_smem_atomic<2><<<grid,bs>>>(out,iters);break;case 3:k_smem_atomic<3><<<grid,bs>>>(out,iters);break;case 4:k_smem_atomic<4><<<grid,bs>>>(out,iters);break;default:k_smem_atomic<5><<<grid,bs>>>(out,iters);}
        cudaEventRecord(b); CK(cudaEventSynchronize(b)); cudaEventElapsedTime(&ms,a,b);
      }
      double ops=(double)grid*bs*iters;
      printf("%-24s bs=%4d: %.3f ms  %.1f Gop/s  %.3f op/clk/SM @1.9GHz\n", names[mode], bs, ms, ops/ms/1e6, ops/(ms*1e-3)/sms/1.9e9);
    }
  }
  size_t bytes=(size_t)4<<30; uint4 *p,*q; CK(cudaMalloc(&p,bytes)); CK(cudaMalloc(&q,bytes)); cudaMemset(p,1,bytes); cudaMemset(q,0,bytes);
  for(int g: {sms*2, sms*4, sms*8}){ float ms; for(int r=0;r<3;++r){cudaEventRecord(a); k_read<<<g,512>>>(p,bytes/16,out); cudaEventRecord(b); cudaEventSynchronize(b);} cudaEventElapsedTime(&ms,a,b); printf("read grid=%d %.1f GB/s\n", g, bytes/ms/1e6);}
  for(int g: {sms*2, sms*4, sms*8}){ float ms; for(int r=0;r<3;++r){cudaEventRecord(a); k_copy<<<g,512>>>(p,q,bytes/16); cudaEventRecord(b); cudaEventSynchronize(b);} cudaEventElapsedTime(&ms,a,b); printf("copy grid=%d %.1f GB/s (r+w)\n", g, 2*bytes/ms/1e6);}
  for(uint32_t mask: {255u, 65535u, (1u<<24)-1}){ float ms; int it=1024; int g=sms*4; for(int r=0;r<3;++r){cudaEventRecord(a); k_gred<<<g,512>>>(out,it,mask); cudaEventRecord(b); cudaEventSynchronize(b);} cudaEventElapsedTime(&ms,a,b); printf("global RED mask=%u %.1f Gop/s\n", mask, (double)g*512*it/ms/1e6);}
  CK(cudaGetLastError());
  return 0;
}
