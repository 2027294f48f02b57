// FP64 pipe microbenchmark: DMMA.8x8x4 (mma.sync f64) and DFMA throughput on sm_100a.
#include <cstdio>
#include <cuda_runtime.h>
template<int NACC>
__global__ void dmma_loop(double* out, int iters, double seed){
  double acc[NACC][2];
  double a = seed + threadIdx.x*1e-3, b = seed*0.5 - threadIdx.x*1e-3;
#pragma unroll
  for(int i=0;i<NACC;i++){acc[i][0]=0;acc[i][1]=0;}
  for(int it=0; it<iters; ++it){
#pragma unroll
    for(int i=0;i<NACC;i++){
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
        : "+d"(acc[i][0]),"+d"(acc[i][1]) : "d"(a),"d"(b));
    }
  }
  double s=0;
#pragma unroll
  for(int i=0;i<NACC;i++) s+=acc[i][0]+acc[i][1];
  if(s==12345.678) out[threadIdx.x]=s;
}
template<int NACC>
__global__ void dfma_loop(double* out, int iters, double seed){
  double acc[NACC];
  double a = seed + threadIdx.x*1e-3, b = 0.999999;
#pragma unroll
  for(int i=0;i<NACC;i++) acc[i]=i;
  for(int it=0; it<iters; ++it){
#pragma unroll
    for(int i=0;i<NACC;i++) acc[i]=fma(acc[i],b,a);
  }
  double s=0;
#pragma unroll
  for(int i=0;i<NACC;i++) s+=acc[i];
  if(s==12345.678) out[threadIdx.x]=s;
}
int main(){
  double* out; cudaMalloc(&out, 1<<20);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t e0,e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int iters=20000;
  for(int warps : {4,8,16,32}){
    for(int rep=0;rep<2;rep++){
      int threads=warps*32;
      cudaEventRecord(e0);
      dmma_loop<8><<<sms*2,threads>>>(out,iters,1.0);
      cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms,e0,e1);
      double flops = 2.0*sms*threads/32.0*iters*8*512;
      if(rep) printf("DMMA warps/blk=%d x2 blk/SM: %.2f TFLOP/s (%.3f ms)\n", warps, flops/ms/1e9, ms);
    }
  }
  for(int warps : {4,8,16,32}){
    for(int rep=0;rep<2;rep++){
      int threads=warps*32;
      cudaEventRecord(e0);
      dfma_loop<8><<<sms*2,threads>>>(out,iters,1.0);
      cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms,e0,e1);
      double flops = 2.0*sms*threads*(double)iters*8*2;
      if(rep) printf("DFMA warps/blk=%d x2 blk/SM: %.2f TFLOP/s (%.3f ms)\n", warps, flops/ms/1e9, ms);
    }
  }
  printf("err=%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
