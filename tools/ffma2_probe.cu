#include <cstdio>
#include <cuda_runtime.h>
typedef unsigned long long u64;
__device__ __forceinline__ u64 fma2(u64 a, u64 b, u64 c){ u64 d; asm volatile("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c)); return d;}
template<int CH>
__global__ void sc(float* out, float a, float b, int iters){
  float x[CH];
  for(int i=0;i<CH;i++) x[i]=threadIdx.x*1e-3f+i;
  for(int it=0;it<iters;it++){
#pragma unroll
    for(int i=0;i<CH;i++) asm volatile("fma.rn.f32 %0, %0, %1, %2;" : "+f"(x[i]) : "f"(a), "f"(b));
  }
  float s=0; for(int i=0;i<CH;i++) s+=x[i]; if(s==1.2345f) out[0]=s;
}
template<int CH>
__global__ void pk(float* out, u64 a, u64 b, int iters){
  u64 x[CH];
  for(int i=0;i<CH;i++) x[i]=threadIdx.x+i;
  for(int it=0;it<iters;it++){
#pragma unroll
    for(int i=0;i<CH;i++) x[i]=fma2(x[i],a,b);
  }
  u64 s=0; for(int i=0;i<CH;i++) s^=x[i]; if(s==12345) out[0]=s;
}
int main(){
  float* o; cudaMalloc(&o,4);
  int dev; cudaGetDevice(&dev); cudaDeviceProp p; cudaGetDeviceProperties(&p,dev);
  int blocks=p.multiProcessorCount*8, thr=256, iters=4096;
  cudaEvent_t e0,e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for(int rep=0;rep<3;rep++){
    float ms;
    sc<8><<<blocks,thr>>>(o,1.0001f,0.5f,iters);
    cudaEventRecord(e0); sc<8><<<blocks,thr>>>(o,1.0001f,0.5f,iters); cudaEventRecord(e1); cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms,e0,e1);
    double lanes=(double)blocks*thr*iters*8;
    printf("scalar FFMA: %.2f T lane-fma/s\n", lanes/ms/1e9);
    pk<8><<<blocks,thr>>>(o,0x3f8000003f800000ull,0x3f0000003f000000ull,iters);
    cudaEventRecord(e0); pk<8><<<blocks,thr>>>(o,0x3f8000003f800000ull,0x3f0000003f000000ull,iters); cudaEventRecord(e1); cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms,e0,e1);
    printf("FFMA2: %.2f T lane-fma/s (x2 per instr)\n", lanes*2/ms/1e9);
  }
  printf("SMs %d\n", p.multiProcessorCount);
}
