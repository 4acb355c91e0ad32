// Standalone check of the tcgen05 (UMMA) building blocks the stage-2 sketch
// kernel uses: TMEM allocation, SWIZZLE_NONE K-major shared-memory
// descriptors, the kind::f16 instruction descriptor (M=128, N=128, fp32
// accumulate), tcgen05.commit -> mbarrier, and 32x32b TMEM loads.
// One CTA of 4 warps computes D[128x128] = A[128xK] * B[128xK]^T (fp16 in,
// fp32 out) and the host compares it with an fp64 product.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o umma_check umma_check.cu && ./umma_check
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <cstdint>
#include <vector>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

constexpr int M = 128, N = 128, K = 128;

#ifndef SW128
#define SW128 1
#endif
#if SW128
// K-major SWIZZLE_128B: atoms of 8 rows x 128 B (64 fp16 of K), rows at
// 128 B, 16-B chunk j of row r stored at j ^ (r % 8); atoms of a K slab are
// stacked along M at SBO = 1024 B, K slabs (64 elements) at M/8 * 1024 B.
constexpr uint32_t LBO = 0, SBO = 1024, SLAB = (M / 8) * 1024;
__host__ __device__ inline uint32_t cm_off(int r, int k) {
  return (k / 64) * SLAB + (r / 8) * 1024 + (r % 8) * 128 + ((((k % 64) / 8) ^ (r % 8)) * 16) + (k % 8) * 2;
}
constexpr uint64_t LAYOUT = 2;
#else
// core-matrix (8 rows x 16 B) K-major layout without swizzle:
// element (r, k) at byte (r/8)*SBO + (k/8)*LBO + (r%8)*16 + (k%8)*2
constexpr uint32_t LBO = 128, SBO = (K / 8) * 128;
__host__ __device__ inline uint32_t cm_off(int r, int k) {
  return (r / 8) * SBO + (k / 8) * LBO + (r % 8) * 16 + (k % 8) * 2;
}
constexpr uint64_t LAYOUT = 0;
#endif
// byte offset of the K-step s (16 fp16) from the operand base
__host__ __device__ inline uint32_t kstep_off(int s) {
#if SW128
  return (s * 16 / 64) * SLAB + (s * 16 % 64) * 2;
#else
  return s * 2 * LBO;
#endif
}

__device__ inline uint64_t sdesc(uint32_t saddr) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)((LBO >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((SBO >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;  // version 1 (sm100)
  d |= LAYOUT << 61;       // base offset 0, lbo mode 0
  return d;
}

__global__ void k(const uint8_t* a_img, const uint8_t* b_img, float* d_out, unsigned long long* clk) {
  extern __shared__ __align__(1024) uint8_t smem[];
  uint8_t* sa = smem;
  uint8_t* sb = smem + M * K * 2;
  __shared__ uint32_t tmem_base;
  __shared__ __align__(8) uint64_t bar;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  for (int i = tid; i < M * K * 2 / 16; i += blockDim.x) {
    reinterpret_cast<uint4*>(sa)[i] = reinterpret_cast<const uint4*>(a_img)[i];
    reinterpret_cast<uint4*>(sb)[i] = reinterpret_cast<const uint4*>(b_img)[i];
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     (uint32_t)__cvta_generic_to_shared(&tmem_base)),
                 "n"(128));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"((uint32_t)__cvta_generic_to_shared(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");   // generic smem writes -> async proxy
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = tmem_base;
  unsigned long long t0 = clock64();
  if (tid == 0) {
    const uint32_t idesc = (1u << 4) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
    const uint32_t a0 = (uint32_t)__cvta_generic_to_shared(sa), b0 = (uint32_t)__cvta_generic_to_shared(sb);
    for (int s = 0; s < K / 16; ++s) {
      const uint64_t da = sdesc(a0 + kstep_off(s)), db = sdesc(b0 + kstep_off(s));
      const uint32_t acc = s > 0;
      asm volatile(
          "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
          "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem),
          "l"(da), "l"(db), "r"(idesc), "r"(acc));
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
        (uint32_t)__cvta_generic_to_shared(&bar)));
  }
  // wait for the commit (phase 0)
  {
    uint32_t ok = 0;
    long spins = 0;
    while (!ok) {
      asm volatile(
          "{\n.reg .pred p;\nmbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\nselp.u32 %0, 1, 0, p;\n}\n"
          : "=r"(ok)
          : "r"((uint32_t)__cvta_generic_to_shared(&bar)));
      if (++spins > (1l << 26)) __trap();
    }
  }
  asm volatile("tcgen05.fence::after_thread_sync;");
  unsigned long long t1 = clock64();
  // warp w reads TMEM lanes 32w..32w+31 (row = lane), 32 columns per load
  for (int c0 = 0; c0 < N; c0 += 32) {
    uint32_t v[32];
    const uint32_t addr = tmem + ((uint32_t)(32 * warp) << 16) + c0;
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
        "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
          "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]),
          "=r"(v[15]), "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]),
          "=r"(v[22]), "=r"(v[23]), "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]),
          "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
        : "r"(addr));
    asm volatile("tcgen05.wait::ld.sync.aligned;");
    const int row = 32 * warp + lane;
    for (int j = 0; j < 32; ++j) d_out[row * N + c0 + j] = __uint_as_float(v[j]);
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(128));
  if (tid == 0) *clk = t1 - t0;
}

int main() {
  std::vector<__half> A(M * K), B(N * K);
  srand(1);
  for (auto& x : A) x = __float2half((rand() / (float)RAND_MAX - 0.5f) * 4.0f);
  for (auto& x : B) x = __float2half((rand() / (float)RAND_MAX - 0.5f) * 4.0f);
  std::vector<uint8_t> ai(M * K * 2), bi(N * K * 2);
  for (int r = 0; r < M; ++r)
    for (int kk = 0; kk < K; ++kk) *reinterpret_cast<__half*>(&ai[cm_off(r, kk)]) = A[r * K + kk];
  for (int r = 0; r < N; ++r)
    for (int kk = 0; kk < K; ++kk) *reinterpret_cast<__half*>(&bi[cm_off(r, kk)]) = B[r * K + kk];
  uint8_t *da, *db;
  float* dd;
  unsigned long long* dclk;
  cudaMalloc(&da, ai.size()); cudaMalloc(&db, bi.size()); cudaMalloc(&dd, M * N * 4); cudaMalloc(&dclk, 8);
  cudaMemcpy(da, ai.data(), ai.size(), cudaMemcpyHostToDevice);
  cudaMemcpy(db, bi.data(), bi.size(), cudaMemcpyHostToDevice);
  const int smem = 2 * M * K * 2 + 1024;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  k<<<1, 128, smem>>>(da, db, dd, dclk);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) { printf("CUDA error %s\n", cudaGetErrorString(e)); return 1; }
  std::vector<float> D(M * N);
  unsigned long long clk;
  cudaMemcpy(D.data(), dd, M * N * 4, cudaMemcpyDeviceToHost);
  cudaMemcpy(&clk, dclk, 8, cudaMemcpyDeviceToHost);
  double maxerr = 0, maxref = 0;
  for (int i = 0; i < M; ++i)
    for (int j = 0; j < N; ++j) {
      double ref = 0;
      for (int kk = 0; kk < K; ++kk) ref += (double)__half2float(A[i * K + kk]) * (double)__half2float(B[j * K + kk]);
      maxerr = fmax(maxerr, fabs(ref - D[i * N + j]));
      maxref = fmax(maxref, fabs(ref));
    }
  printf("umma_check SW128=%d M=%d N=%d K=%d: max |err| %.3e (max |ref| %.3e), mma+commit %llu cycles -> %s\n", SW128, M, N, K,
         maxerr, maxref, clk, maxerr <= 1e-3 * maxref ? "PASS" : "FAIL");
  printf("D[0][0..3] = %f %f %f %f\n", D[0], D[1], D[2], D[3]);
  return maxerr <= 1e-3 * maxref ? 0 : 2;
}
