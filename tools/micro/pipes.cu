// Microbenchmark of the sm_100a issue/pipe model for the instruction classes
// the IsoQuant kernels use: FFMA, FFMA2 (fma.rn.f32x2), FSET (set.ge), LOP3,
// FMNMX, HADD2.F32 (cvt.f32.f16) alone and interleaved 1:1 on independent
// chains.  Prints warp-instructions per clock per SMSP.
#include <cstdio>
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#define N 8
__device__ __forceinline__ void op_ffma(float& a) { asm volatile("fma.rn.f32 %0, %0, 0f3F7FBE77, 0f38D1B717;" : "+f"(a)); }
__device__ __forceinline__ void op_ffma2(unsigned long long& a) {
  asm volatile("{.reg .b64 m; .reg .b64 c; mov.b64 m, 0x3F7FBE773F7FBE77; mov.b64 c, 0x38D1B71738D1B717; fma.rn.f32x2 %0, %0, m, c;}" : "+l"(a));
}
__device__ __forceinline__ void op_fset(float& a) { asm volatile("set.ge.f32.f32 %0, %0, 0f3F000000;" : "+f"(a)); }
__device__ __forceinline__ void op_lop(unsigned& a) { asm volatile("lop3.b32 %0, %0, 0x80000000, 0x3F800000, 0x6a;" : "+r"(a)); }
__device__ __forceinline__ void op_fmnmx(float& a) { asm volatile("max.f32 %0, %0, 0f3E800000;" : "+f"(a)); }
__device__ __forceinline__ void op_cvt(float& a, unsigned short h) { asm volatile("{.reg .f32 t; cvt.f32.f16 t, %1; add.f32 %0, %0, t;}" : "+f"(a) : "h"(h)); }

template <int A, int B>  // op ids: 0 ffma, 1 ffma2, 2 fset, 3 lop3, 4 fmnmx, 5 none
__global__ void k(float* out, int iters, long long* clk) {
  float f[N], g[N]; unsigned u[N]; unsigned long long p[N];
  for (int i = 0; i < N; ++i) { f[i] = threadIdx.x + i; g[i] = f[i] * 0.5f; u[i] = threadIdx.x * 7 + i; p[i] = (unsigned long long)u[i] * 0x100000001ull; }
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < N; ++i) {
      if (A == 0) op_ffma(f[i]); if (A == 1) op_ffma2(p[i]); if (A == 2) op_fset(f[i]); if (A == 3) op_lop(u[i]); if (A == 4) op_fmnmx(f[i]);
      if (B == 0) op_ffma(g[i]); if (B == 1) op_ffma2(p[i ^ 1]); if (B == 2) op_fset(g[i]); if (B == 3) op_lop(u[i]); if (B == 4) op_fmnmx(g[i]);
    }
  }
  long long t1 = clock64();
  float r = 0;
  for (int i = 0; i < N; ++i) r += f[i] + g[i] + (float)u[i] + (float)(p[i] & 0xffff);
  out[blockIdx.x * blockDim.x + threadIdx.x] = r;
  if (threadIdx.x == 0 && blockIdx.x == 0) *clk = t1 - t0;
}
template <int A, int B> void run(const char* name, float* out, long long* clk, int warps) {
  int iters = 2048;
  k<A, B><<<148, warps * 32>>>(out, iters, clk);
  cudaDeviceSynchronize();
  k<A, B><<<148, warps * 32>>>(out, iters, clk);
  cudaDeviceSynchronize();
  long long c; cudaMemcpy(&c, clk, 8, cudaMemcpyDeviceToHost);
  double instr = (double)iters * N * ((A != 5) + (B != 5)) * warps;  // warp-instructions per SM
  printf("%-14s warps/SM %2d: %.3f warp-instr/clk/SMSP\n", name, warps, instr / c / 4.0);
}
int main() {
  float* out; long long* clk; cudaMalloc(&out, 148 * 1024 * 4); cudaMalloc(&clk, 8);
  for (int w : {16, 32}) {
    run<0, 5>("FFMA", out, clk, w);
    run<1, 5>("FFMA2", out, clk, w);
    run<2, 5>("FSET", out, clk, w);
    run<3, 5>("LOP3", out, clk, w);
    run<4, 5>("FMNMX", out, clk, w);
    run<0, 2>("FFMA+FSET", out, clk, w);
    run<1, 2>("FFMA2+FSET", out, clk, w);
    run<1, 3>("FFMA2+LOP3", out, clk, w);
    run<0, 1>("FFMA+FFMA2", out, clk, w);
    run<2, 3>("FSET+LOP3", out, clk, w);
    run<0, 0>("FFMA+FFMA", out, clk, w);
  }
  return 0;
}
