// Pipe throughput probe: ex2.approx.f32 (0), ex2.approx.f16x2 (1), ex2.approx.ftz.bf16x2 (2),
// cvt.rn.bf16x2.f32 (3), FFMA (4), DFMA (5)
#include <cstdio>
#include <cuda_fp16.h>
#include <cuda_bf16.h>
__device__ __forceinline__ float ex2f(float x){float y;asm volatile("ex2.approx.ftz.f32 %0,%1;":"=f"(y):"f"(x));return y;}
__device__ __forceinline__ unsigned ex2h(unsigned x){unsigned y;asm volatile("ex2.approx.f16x2 %0,%1;":"=r"(y):"r"(x));return y;}
__device__ __forceinline__ unsigned ex2b(unsigned x){unsigned y;asm volatile("ex2.approx.ftz.bf16x2 %0,%1;":"=r"(y):"r"(x));return y;}
__device__ __forceinline__ unsigned pk(float lo, float hi){unsigned r;asm volatile("cvt.rn.bf16x2.f32 %0,%1,%2;":"=r"(r):"f"(hi),"f"(lo));return r;}
template<int MODE> __global__ void k(float* out, int iters){
  float a[8]; unsigned u[8];
  for(int i=0;i<8;i++){a[i]=-0.001f*(threadIdx.x+i); u[i]=0xB800B800u+i;}
  for(int it=0;it<iters;it++){
#pragma unroll
    for(int i=0;i<8;i++){ if(MODE==0) a[i]=ex2f(a[i])-1.0f; else if(MODE==1) u[i]=ex2h(u[i])^0x8000u; else if(MODE==2) u[i]=ex2b(u[i])^0x8000u;
      else if(MODE==3) { u[i]=pk(a[i], __uint_as_float(u[i])); }
      else if(MODE==4) { a[i]=fmaf(a[i], 1.0001f, -0.5f); } }
  }
  if (MODE==5) {
    double d[8]; for(int i=0;i<8;i++) d[i]=a[i];
    for(int it=0;it<iters;it++){
#pragma unroll
      for(int i=0;i<8;i++) d[i]=fma(d[i], 1.0000001, -0.25);
    }
    for(int i=0;i<8;i++) a[i]=(float)d[i];
  }
  float s=0; for(int i=0;i<8;i++) s+=a[i]+(float)u[i];
  out[blockIdx.x*blockDim.x+threadIdx.x]=s;
}
int main(){
  float* o; cudaMalloc(&o, 148*8*1024*4);
  int iters=4096;
  for(int mode=0;mode<6;mode++){
    cudaEvent_t e0,e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    for(int rep=0;rep<2;rep++){
      cudaEventRecord(e0);
      if(mode==0) k<0><<<148*8,1024>>>(o,iters); else if(mode==1) k<1><<<148*8,1024>>>(o,iters); else if(mode==2) k<2><<<148*8,1024>>>(o,iters);
      else if(mode==3) k<3><<<148*8,1024>>>(o,iters); else if(mode==4) k<4><<<148*8,1024>>>(o,iters);
      else k<5><<<148*8,1024>>>(o,iters/4);
      cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms,e0,e1);
      double ops=148.0*8*1024*(mode==5?iters/4:iters)*8; // instructions (lanes)
      int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
      if(rep) printf("mode %d: %.3f ms, %.2f lane-instr/clk/SM (at %d MHz)\n", mode, ms, ops/(ms*1e-3)/(clk*1e3)/148, clk/1000);
    }
  }
  return 0;
}
