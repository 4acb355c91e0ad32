// Issue/pipe rates of the instruction classes a stage-1 decision can be
// built from, on sm_100a: warp-instructions per clock per SMSP for each op
// alone (8 independent chains per thread) and for pairs of ops interleaved
// 1:1.  Register operands (not immediates) unless the name says imm.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/pipes2 tools/micro/pipes2.cu && /tmp/pipes2
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#define N 8

struct St {
  float f[N];
  uint32_t u[N];
  unsigned long long p[N];
  float k0, k1;
  uint32_t ku;
  unsigned long long kp;
};

// each op updates chain i of its own register class
#define OP(id, s, i)                                                                                              \
  do {                                                                                                            \
    if (id == 0) asm volatile("fma.rn.f32 %0, %0, %1, %2;" : "+f"(s.f[i]) : "f"(s.k0), "f"(s.k1));                 \
    if (id == 1) asm volatile("fma.rn.f32x2 %0, %0, %1, %2;" : "+l"(s.p[i]) : "l"(s.kp), "l"(s.kp));               \
    if (id == 2) asm volatile("set.ge.f32.f32 %0, %0, %1;" : "+f"(s.f[i]) : "f"(s.k0));                            \
    if (id == 3) asm volatile("lop3.b32 %0, %0, %1, %2, 0x6a;" : "+r"(s.u[i]) : "r"(s.ku), "r"(s.ku));             \
    if (id == 4) asm volatile("max.f32 %0, %0, %1;" : "+f"(s.f[i]) : "f"(s.f[(i + 3) % N]));                                   \
    if (id == 5) asm volatile("add.f32 %0, %0, %1;" : "+f"(s.f[i]) : "f"(s.k0));                                   \
    if (id == 6) asm volatile("add.rn.f32x2 %0, %0, %1;" : "+l"(s.p[i]) : "l"(s.kp));                              \
    if (id == 7)                                                                                                  \
      asm volatile("{.reg .f32 t; .reg .b16 h; mov.b32 {h, _}, %0; cvt.f32.f16 t, h; mov.b32 %0, t;}"               \
                   : "+r"(s.u[i]));                                                                               \
    if (id == 8) asm volatile("{.reg .f32 t; mov.b32 t, %0; cvt.rn.f16x2.f32 %0, t, %1;}" : "+r"(s.u[i]) : "f"(s.k0));             \
    if (id == 9) asm volatile("shfl.sync.idx.b32 %0, %0, %0, 0x1f, 0xffffffff;" : "+r"(s.u[i]));                   \
    if (id == 10) asm volatile("prmt.b32 %0, %0, %1, %2;" : "+r"(s.u[i]) : "r"(s.ku), "r"(s.ku));                  \
    if (id == 11) asm volatile("fma.rn.sat.f32 %0, %0, %1, %2;" : "+f"(s.f[i]) : "f"(s.k0), "f"(s.k1));            \
    if (id == 12) asm volatile("min.u32 %0, %0, %1;" : "+r"(s.u[i]) : "r"(s.u[(i + 3) % N]));                                  \
    if (id == 13)                                                                                                 \
      asm volatile("{.reg .pred q; setp.ge.f32 q, %0, %1; selp.f32 %0, %1, %0, q;}" : "+f"(s.f[i]) : "f"(s.k0));  \
    if (id == 14) asm volatile("mul.rn.f32x2 %0, %0, %1;" : "+l"(s.p[i]) : "l"(s.kp));                             \
    if (id == 15) asm volatile("shf.r.wrap.b32 %0, %0, %1, 7;" : "+r"(s.u[i]) : "r"(s.ku));                        \
    if (id == 16) asm volatile("fma.rn.f16x2 %0, %0, %1, %1;" : "+r"(s.u[i]) : "r"(s.ku));                         \
    if (id == 17) asm volatile("fma.rm.f32x2 %0, %0, %1, %2;" : "+l"(s.p[i]) : "l"(s.kp), "l"(s.kp));              \
    if (id == 18) asm volatile("add.u32 %0, %0, %1;" : "+r"(s.u[i]) : "r"(s.ku));                                  \
    if (id == 19) asm volatile("fma.rn.f32 %0, %0, 0f3F7FBE77, 0f38D1B717;" : "+f"(s.f[i]));                       \
    if (id == 20) asm volatile("ld.shared.u32 %0, [%0];" : "+r"(s.u[i]));                                          \
    if (id == 21) asm volatile("{.reg .f32 t; mov.b32 t, %0; set.ge.u32.f32 %0, t, %1;}" : "+r"(s.u[i]) : "f"(s.k0));              \
    if (id == 22) asm volatile("{.reg .f32 t; cvt.rn.f32.s32 t, %0; mov.b32 %0, t;}" : "+r"(s.u[i]));                             \
    if (id == 23) asm volatile("mov.b32 %0, %0;" : "+r"(s.u[i]));                                                  \
    if (id == 24)                                                                                                 \
      asm volatile("{.reg .b16 l, h; .reg .f32 t; mov.b32 {l, h}, %0; add.rn.f32.f16 t, h, 0f80000000; mov.b32 %0, t;}" \
                   : "+r"(s.u[i]));                                                                               \
    if (id == 25)                                                                                                 \
      asm volatile("{.reg .b16 l, h; mov.b32 {l, h}, %1; fma.rn.f32.f16 %0, h, h, %0;}" : "+f"(s.f[i]) : "r"(s.u[i])); \
  } while (0)

__shared__ uint32_t sh[1024];

template <int A, int B>
__global__ void k(float* out, int iters, long long* clk) {
  St s;
  for (int i = 0; i < N; ++i) {
    s.f[i] = threadIdx.x + i;
    s.u[i] = (threadIdx.x * 4 + i * 4) & 1023;
    s.p[i] = (unsigned long long)(threadIdx.x + i) * 0x100000001ull;
  }
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) sh[i] = (i * 4 + 4) & 4092;
  __syncthreads();
  s.k0 = 0.999f + threadIdx.x * 1e-9f;
  s.k1 = 1e-4f;
  s.ku = 0x3F800000u + threadIdx.x;
  s.kp = 0x3F7FBE773F7FBE77ull;
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < N; ++i) {
      OP(A, s, i);
      if (B >= 0) OP(B, s, (i ^ 1));
    }
  }
  long long t1 = clock64();
  float r = 0;
  for (int i = 0; i < N; ++i) r += s.f[i] + (float)s.u[i] + (float)(s.p[i] & 0xffff);
  out[blockIdx.x * blockDim.x + threadIdx.x] = r;
  if (threadIdx.x == 0 && blockIdx.x == 0) *clk = t1 - t0;
}

template <int A, int B>
void run(const char* name, float* out, long long* clk, int warps) {
  int iters = 1024;
  k<A, B><<<148, warps * 32>>>(out, iters, clk);
  cudaDeviceSynchronize();
  k<A, B><<<148, warps * 32>>>(out, iters, clk);
  cudaError_t e = cudaDeviceSynchronize();
  long long c;
  cudaMemcpy(&c, clk, 8, cudaMemcpyDeviceToHost);
  double instr = (double)iters * N * (1 + (B >= 0)) * warps;   // warp-instructions per SM
  printf("%-22s warps/SM %2d: %.3f warp-instr/clk/SMSP %s\n", name, warps, instr / c / 4.0,
         e ? cudaGetErrorString(e) : "");
}

#define R1(a, nm) run<a, -1>(nm, out, clk, w)
#define R2(a, b, nm) run<a, b>(nm, out, clk, w)
int main() {
  float* out;
  long long* clk;
  cudaMalloc(&out, 148 * 1024 * 4);
  cudaMalloc(&clk, 8);
  for (int w : {16, 32}) {
    R1(0, "FFMA reg");
    R1(19, "FFMA imm");
    R1(1, "FFMA2");
    R1(14, "FMUL2");
    R1(6, "FADD2");
    R1(17, "FFMA2.RM");
    R1(5, "FADD");
    R1(2, "FSET.BF");
    R1(21, "FSET (mask)");
    R1(13, "FSETP+FSEL");
    R1(3, "LOP3");
    R1(4, "FMNMX");
    R1(12, "IMNMX");
    R1(18, "IADD");
    R1(7, "HADD2.F32 (cvt)");
    R1(8, "F2FP pack");
    R1(9, "SHFL.IDX");
    R1(20, "LDS.32");
    R1(10, "PRMT");
    R1(11, "FFMA.SAT");
    R1(15, "SHF");
    R1(16, "HFMA2");
    R1(22, "I2F");
    R1(24, "FHADD");
    R1(25, "FHFMA");
    R2(1, 24, "FFMA2+FHADD");
    R2(1, 25, "FFMA2+FHFMA");
    R2(3, 24, "LOP3+FHADD");
    R2(13, 5, "FSETP+FSEL+FADD");
    R2(2, 14, "FSET+FMUL2");
    R2(1, 2, "FFMA2+FSET");
    R2(1, 3, "FFMA2+LOP3");
    R2(1, 9, "FFMA2+SHFL");
    R2(1, 4, "FFMA2+FMNMX");
    R2(1, 5, "FFMA2+FADD");
    R2(1, 7, "FFMA2+HADD2.F32");
    R2(1, 8, "FFMA2+F2FP");
    R2(3, 9, "LOP3+SHFL");
    R2(2, 3, "FSET+LOP3");
    R2(2, 4, "FSET+FMNMX");
    R2(3, 4, "LOP3+FMNMX");
    R2(5, 3, "FADD+LOP3");
    R2(0, 3, "FFMA+LOP3");
    R2(0, 4, "FFMA+FMNMX");
    R2(4, 4, "FMNMX+FMNMX");
    R2(10, 3, "PRMT+LOP3");
    R2(15, 3, "SHF+LOP3");
    R2(18, 3, "IADD+LOP3");
    R2(12, 3, "IMNMX+LOP3");
    R2(1, 12, "FFMA2+IMNMX");
    R2(1, 18, "FFMA2+IADD");
    R2(9, 20, "SHFL+LDS");
  }
  return 0;
}
