// Pipe-throughput microbenchmark (B200 roofline denominators):
// MUFU.RCP, MUFU.LG2+EX2, FFMA (scalar), FFMA2 (packed) per clock per SM.
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ float rcpa(float x){float y; asm volatile("rcp.approx.ftz.f32 %0,%1;":"=f"(y):"f"(x)); return y;}
__device__ __forceinline__ float lg2a(float x){float y; asm volatile("lg2.approx.ftz.f32 %0,%1;":"=f"(y):"f"(x)); return y;}
template<int MODE> __global__ void k(float* out, int iters, long long* cyc) {
  float a[8]; float2 b[8];
  for (int i=0;i<8;++i){ a[i]=1.0f+threadIdx.x*1e-3f+i; b[i]=make_float2(a[i],a[i]+1);}
  long long t0=clock64();
  for (int it=0; it<iters; ++it) {
#pragma unroll
    for (int i=0;i<8;++i) {
      if (MODE==0) a[i]=rcpa(a[i]);
      else if (MODE==1) a[i]=lg2a(a[i]);
      else if (MODE==2) a[i]=fmaf(a[i],1.0001f,0.5f);
      else b[i]=__ffma2_rn(b[i],make_float2(1.0001f,1.0001f),make_float2(0.5f,0.5f));
    }
  }
  long long t1=clock64();
  float s=0; for(int i=0;i<8;++i) s+=a[i]+b[i].x+b[i].y;
  out[blockIdx.x*blockDim.x+threadIdx.x]=s;
  if(threadIdx.x==0&&blockIdx.x==0) *cyc=t1-t0;
}
int main(){
  float* o; long long* c; cudaMalloc(&o, 148*8*1024*4); cudaMalloc(&c,8);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  const char* names[4]={"MUFU.RCP","MUFU.LG2","FFMA","FFMA2(x2 lanes)"};
  for (int mode=0; mode<4; ++mode) {
    int iters=4096; int blocks=sms*4, threads=512;
    cudaEvent_t e0,e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    for (int rep=0; rep<2; ++rep) {
      cudaEventRecord(e0);
      if(mode==0) k<0><<<blocks,threads>>>(o,iters,c);
      if(mode==1) k<1><<<blocks,threads>>>(o,iters,c);
      if(mode==2) k<2><<<blocks,threads>>>(o,iters,c);
      if(mode==3) k<3><<<blocks,threads>>>(o,iters,c);
      cudaEventRecord(e1); cudaEventSynchronize(e1);
    }
    float ms; cudaEventElapsedTime(&ms,e0,e1); long long cy; cudaMemcpy(&cy,c,8,cudaMemcpyDeviceToHost);
    double ops=(double)blocks*threads*iters*8*(mode==3?2:1);
    double per_clk_sm = ops/ (double)cy / sms; // using clock64 of block 0 (all blocks resident concurrently)
    printf("%-16s %.3e ops/s  %.1f ops/clk/SM (by clock64)  sms=%d clk_khz=%d ms=%.3f\n", names[mode], ops/(ms*1e-3), per_clk_sm, sms, clk, ms);
  }
  return 0;
}
