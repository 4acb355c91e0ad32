// Microbenchmark: FP32 FMA throughput per SM per clock for scalar FFMA vs
// packed FFMA2, and for FFMA2 interleaved with an ALU op (FSET), to learn
// the pipe model the kernels are tuned against.  Prints FMAs/clk/SM.
#include <cstdio>
#include <cuda_runtime.h>
template <int MODE>
__global__ void k(float* out, int iters, long long* clk) {
  float2 a[8]; float s[8];
  for (int i = 0; i < 8; ++i) { a[i] = make_float2(threadIdx.x * 1e-3f + i, i * 0.5f); s[i] = a[i].x; }
  const float2 m = make_float2(0.999f, 1.001f), c = make_float2(1e-4f, 2e-4f);
  float acc = 0.f;
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (MODE == 0) s[i] = fmaf(s[i], 0.999f, 1e-4f);
      if (MODE == 1) a[i] = __ffma2_rn(a[i], m, c);
      if (MODE == 2) { a[i] = __ffma2_rn(a[i], m, c); acc += (a[i].x >= 0.5f) ? 1.0f : 0.0f; }
    }
  }
  long long t1 = clock64();
  float r = acc;
  for (int i = 0; i < 8; ++i) r += s[i] + a[i].x + a[i].y;
  out[blockIdx.x * blockDim.x + threadIdx.x] = r;
  if (threadIdx.x == 0 && blockIdx.x == 0) *clk = t1 - t0;
}
int main() {
  float* out; long long* clk; cudaMalloc(&out, 148 * 1024 * 4 * 8); cudaMalloc(&clk, 8);
  int iters = 4096;
  for (int mode = 0; mode < 3; ++mode) {
    for (int warps : {8, 16, 32}) {
      cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
      auto launch = [&]() {
        if (mode == 0) k<0><<<148, warps * 32>>>(out, iters, clk);
        if (mode == 1) k<1><<<148, warps * 32>>>(out, iters, clk);
        if (mode == 2) k<2><<<148, warps * 32>>>(out, iters, clk);
      };
      launch(); cudaDeviceSynchronize();
      cudaEventRecord(e0); launch(); cudaEventRecord(e1); cudaEventSynchronize(e1);
      long long c; cudaMemcpy(&c, clk, 8, cudaMemcpyDeviceToHost);
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      double fmas_per_thread = (double)iters * 8 * (mode == 0 ? 1 : 2);
      double per_sm_clk = fmas_per_thread * warps * 32 / (double)c;
      printf("mode %d (%s) warps/SM %2d: %.1f FMA/clk/SM (clock64 %lld cycles, %.3f ms)\n", mode,
             mode == 0 ? "FFMA" : mode == 1 ? "FFMA2" : "FFMA2+FSET+FADD", warps, per_sm_clk, c, ms);
    }
  }
  return 0;
}
