// Microbenchmark: issue rates of fp64 DADD/DMUL, fp32 FFMA, packed FFMA2 on this GPU.
// Used once to derive the ALU roofline denominators quoted in DESIGN.md.
#include <cstdio>
#include <cuda_runtime.h>
#define ITERS 4096
__global__ void dfma_k(double* o, double a, double b){
  double x0=threadIdx.x, x1=x0+1, x2=x0+2, x3=x0+3, x4=x0+4, x5=x0+5, x6=x0+6, x7=x0+7;
  for(int i=0;i<ITERS;i++){
    x0=__dmul_rn(x0,a); x1=__dmul_rn(x1,a); x2=__dmul_rn(x2,a); x3=__dmul_rn(x3,a);
    x4=__dadd_rn(x4,b); x5=__dadd_rn(x5,b); x6=__dadd_rn(x6,b); x7=__dadd_rn(x7,b);
  }
  o[blockIdx.x*blockDim.x+threadIdx.x]=x0+x1+x2+x3+x4+x5+x6+x7;
}
__global__ void ffma_k(float* o, float a, float b){
  float x0=threadIdx.x, x1=x0+1, x2=x0+2, x3=x0+3, x4=x0+4, x5=x0+5, x6=x0+6, x7=x0+7;
  for(int i=0;i<ITERS;i++){
    x0=fmaf(x0,a,b); x1=fmaf(x1,a,b); x2=fmaf(x2,a,b); x3=fmaf(x3,a,b);
    x4=fmaf(x4,a,b); x5=fmaf(x5,a,b); x6=fmaf(x6,a,b); x7=fmaf(x7,a,b);
  }
  o[blockIdx.x*blockDim.x+threadIdx.x]=x0+x1+x2+x3+x4+x5+x6+x7;
}
__device__ __forceinline__ unsigned long long pk(float a,float b){unsigned long long r; asm("mov.b64 %0,{%1,%2};":"=l"(r):"f"(a),"f"(b)); return r;}
__global__ void ffma2_k(float* o, float a, float b){
  unsigned long long A=pk(a,a), B=pk(b,b);
  float t=threadIdx.x;
  unsigned long long x0=pk(t,t+1),x1=pk(t+2,t+3),x2=pk(t+4,t+5),x3=pk(t+6,t+7),x4=pk(t,t),x5=pk(t+1,t),x6=pk(t+2,t),x7=pk(t+3,t);
  for(int i=0;i<ITERS;i++){
    asm volatile("fma.rn.f32x2 %0,%0,%1,%2;":"+l"(x0):"l"(A),"l"(B));
    asm volatile("fma.rn.f32x2 %0,%0,%1,%2;":"+l"(x1):"l"(A),"l"(B));
    asm volatile("fma.rn.f32x2 %0,%0,%1,%2;":"+l"(x2):"l"(A),"l"(B));
    asm volatile("fma.rn.f32x2 %0,%0,%1,%2;":"+l"(x3):"l"(A),"l"(B));
    asm volatile("fma.rn.f32x2 %0,%0,%1,%2;":"+l"(x4):"l"(A),"l"(B));
    asm volatile("fma.rn.f32x2 %0,%0,%1,%2;":"+l"(x5):"l"(A),"l"(B));
    asm volatile("fma.rn.f32x2 %0,%0,%1,%2;":"+l"(x6):"l"(A),"l"(B));
    asm volatile("fma.rn.f32x2 %0,%0,%1,%2;":"+l"(x7):"l"(A),"l"(B));
  }
  unsigned long long s=x0^x1^x2^x3^x4^x5^x6^x7;
  o[blockIdx.x*blockDim.x+threadIdx.x]=__int_as_float((int)s);
}
template<class F> float timeit(F f){
  cudaEvent_t a,b; cudaEventCreate(&a); cudaEventCreate(&b);
  f(); cudaDeviceSynchronize();
  cudaEventRecord(a); for(int r=0;r<5;r++) f(); cudaEventRecord(b); cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms,a,b); return ms/5;
}
int main(){
  int sms; cudaDeviceGetAttribute(&sms,cudaDevAttrMultiProcessorCount,0);
  int blocks=sms*8, thr=256; float* o; cudaMalloc(&o, (size_t)blocks*thr*8);
  double lanes=(double)blocks*thr*ITERS*8;
  float t1=timeit([&]{dfma_k<<<blocks,thr>>>((double*)o,1.0000001,1e-9);});
  float t2=timeit([&]{ffma_k<<<blocks,thr>>>(o,1.0000001f,1e-9f);});
  float t3=timeit([&]{ffma2_k<<<blocks,thr>>>(o,1.0000001f,1e-9f);});
  printf("sms=%d\n",sms);
  printf("fp64 DMUL/DADD: %.3f T lane-ops/s\n", lanes/t1/1e9);
  printf("fp32 FFMA     : %.3f T lane-ops/s\n", lanes/t2/1e9);
  printf("fp32 FFMA2    : %.3f T instr-lanes/s (x2 flops-lanes)\n", lanes/t3/1e9);
  return 0;
}
