// sm_100a kernels of the IsoQuant stage-1 path (Algorithm 1,
// P:229-258).  The path is an elementwise map with O(d) work per O(d) bytes
// and no reuse: it is bound by HBM bandwidth and, at fp16, close to the
// instruction-issue ceiling.  No tensor cores.  See DESIGN.md "Kernels".
//
// Encoder kernels (quantize K1, fused roundtrip K3) are persistent and
// warp-specialised: one producer warp streams tiles of TILE_V contiguous rows
// of x from HBM into a ring of shared-memory stages with 1-D TMA bulk copies
// (cp.async.bulk + mbarrier complete_tx), so the bytes in flight do not cost
// registers; NWC compute warps read their rows from shared memory, release
// the stage, compute in registers and store results with 128-bit streaming
// stores.  The decoder (K2) reads only d*b/8 + 4 bytes per row and is bound
// by its stores; it loads codes directly.
//
// Thread mapping inside a compute warp: a row of d elements of dtype T is cut
// into 16-byte chunks (EPC = 4 fp32 / 8 fp16 elements); G consecutive lanes
// serve one row, lane `sub` owning chunks sub, sub+G, ... (CPL chunks), so
// every warp-wide access of a chunk index is contiguous.  Each lane owns an
// even number of blocks; blocks are processed two at a time with packed
// fp32x2 FMAs (FFMA2): the pair (block A, block B) shares every instruction
// of the rotation.  A lane's blocks never change, so their 4x4 (2x2)
// operators stay in registers for the whole kernel ("the entire
// block can often remain in registers from input load through output store").
#pragma once
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "iq_internal.h"

namespace iq {

constexpr unsigned kFull = 0xffffffffu;
constexpr int kNWC = 8;                 // compute warps per encoder CTA
constexpr int kEncThreads = 32 * (kNWC + 1);
constexpr int kStageBytes = 16384;      // one TMA stage
constexpr int kStages = 6;              // ring depth per CTA
constexpr int kEncSmem = kStages * kStageBytes + 2 * kStages * 8 + 64;
constexpr int kThreads = 256;           // decoder / statistics CTAs

template <class T> struct DT;
template <> struct DT<float> { static constexpr int EPC = 4; };
template <> struct DT<__half> { static constexpr int EPC = 8; };

template <class T, int D, int VAR>
struct Geo {
  static constexpr int EPC = DT<T>::EPC;
  static constexpr int PW = (VAR == IQ_VARIANT_PLANAR2D) ? 2 : 4;   // block width
  static constexpr int CHUNKS = D / EPC;
  // each lane needs >= 2*PW coordinates so that blocks pair up for FFMA2
  static constexpr int CPL_MIN = (2 * PW + EPC - 1) / EPC;
  static constexpr int G = (CHUNKS / CPL_MIN) < 32 ? (CHUNKS / CPL_MIN) : 32;
  static constexpr int CPL = CHUNKS / G;
  static constexpr int VPW = 32 / G;
  static constexpr int EPL = CPL * EPC;          // coordinates per lane
  static constexpr int NPAIR = EPL / (2 * PW);   // block pairs per lane
  static constexpr int ROWB = D * (int)sizeof(T);
  static constexpr int TILE_V = kStageBytes / ROWB;        // rows per TMA stage
  static constexpr int U = TILE_V / (kNWC * VPW);          // rows per lane group per stage
  static_assert(D % EPC == 0 && (G & (G - 1)) == 0 && CHUNKS % G == 0, "unsupported d");
  static_assert(EPL % (2 * PW) == 0, "lane must own whole block pairs");
  static_assert(U >= 1 && TILE_V % (kNWC * VPW) == 0, "stage too small for the warp layout");
  // decoder: rows per lane group per iteration (16-B stores in flight)
  static constexpr int UD = (4 / CPL) > 0 ? (4 / CPL) : 1;
};

// ---------------------------------------------------------------- PTX helpers
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
// 1-D TMA bulk copy global -> shared, completion counted on `bar` (bytes).
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar,
                                         uint64_t policy) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(policy)
      : "memory");
}
__device__ __forceinline__ uint64_t policy_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint4 lds128(const void* p) {
  uint4 r;
  asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "r"(smem_u32(p)));
  return r;
}
__device__ __forceinline__ void st_stream(void* p, const uint4& v) {
  __stcs(reinterpret_cast<uint4*>(p), v);
}
__device__ __forceinline__ float sqrt_approx(float x) {
  float r;
  asm("sqrt.approx.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}
__device__ __forceinline__ float rsqrt_approx(float x) {
  float r;
  asm("rsqrt.approx.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}

// ----------------------------------------------------------- dtype <-> fp32
template <class T> __device__ __forceinline__ void to_f32(const uint4& r, float* f);
template <> __device__ __forceinline__ void to_f32<float>(const uint4& r, float* f) {
  f[0] = __uint_as_float(r.x); f[1] = __uint_as_float(r.y);
  f[2] = __uint_as_float(r.z); f[3] = __uint_as_float(r.w);
}
template <> __device__ __forceinline__ void to_f32<__half>(const uint4& r, float* f) {
  const uint32_t w[4] = {r.x, r.y, r.z, r.w};
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const float2 t = __half22float2(*reinterpret_cast<const __half2*>(&w[k]));
    f[2 * k] = t.x; f[2 * k + 1] = t.y;
  }
}
template <class T> __device__ __forceinline__ uint4 from_f32(const float* f);
template <> __device__ __forceinline__ uint4 from_f32<float>(const float* f) {
  return make_uint4(__float_as_uint(f[0]), __float_as_uint(f[1]), __float_as_uint(f[2]),
                    __float_as_uint(f[3]));
}
template <> __device__ __forceinline__ uint4 from_f32<__half>(const float* f) {
  uint32_t w[4];
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    __half2 h = __floats2half2_rn(f[2 * k], f[2 * k + 1]);  // round-to-nearest-even [R15]
    w[k] = *reinterpret_cast<uint32_t*>(&h);
  }
  return make_uint4(w[0], w[1], w[2], w[3]);
}

// ------------------------------------------------------------ packed fp32x2
__device__ __forceinline__ float2 f2(float a, float b) { return make_float2(a, b); }
__device__ __forceinline__ float2 fma2(float2 a, float2 b, float2 c) { return __ffma2_rn(a, b, c); }
__device__ __forceinline__ float2 mul2(float2 a, float2 b) { return __fmul2_rn(a, b); }

// Lane coordinate of element j of block A / B in block pair k (lane-local
// coordinates are chunk-major: coordinate c*EPC + e is element e of the
// lane's chunk c).
template <int PW> __device__ __forceinline__ constexpr int coordA(int k, int j) { return 2 * PW * k + j; }
template <int PW> __device__ __forceinline__ constexpr int coordB(int k, int j) { return 2 * PW * k + PW + j; }

// Paired block operator: M2[i*PW+j] = (M_A[i][j], M_B[i][j]).
// forward y = M x (+0-started dot products: a rotated coordinate is never -0,
// so the sign test below classifies +-0 exactly like the count definition).
template <int PW>
__device__ __forceinline__ void rot_fwd2(const float2* M2, const float2* x, float2* y) {
#pragma unroll
  for (int i = 0; i < PW; ++i) {
    float2 a = fma2(M2[PW * i], x[0], f2(0.0f, 0.0f));
#pragma unroll
    for (int j = 1; j < PW; ++j) a = fma2(M2[PW * i + j], x[j], a);
    y[i] = a;
  }
}
// inverse v = M^T c: the inverse sandwich conj(q_L) v q_R is exactly M^T
// (Proposition); R(-theta) = R(theta)^T.
template <int PW>
__device__ __forceinline__ void rot_inv2(const float2* M2, const float2* c, float2* v) {
#pragma unroll
  for (int j = 0; j < PW; ++j) {
    float2 a = mul2(M2[j], c[0]);
#pragma unroll
    for (int i = 1; i < PW; ++i) a = fma2(M2[PW * i + j], c[i], a);
    v[j] = a;
  }
}

// --------------------------------------------------------------- quantizer Q
// code = #{k : y >= t_k} over the symmetric fp32 thresholds (ties go up,
// out-of-range clamps) [R3][R4]:
//   y >= 0 : code = h + m,          m = #{i >= 1 : y >= tau_i}
//   y <  0 : code = h - 1 - m,      m = #{i >= 1 : |y| > tau_i}
// For positive floats |y| > tau <=> nextdown(|y|) >= tau, and nextdown is
// "bits - 1", so key = bits(|y|) - s (s = sign bit) turns both cases into
// key >= tau (compared as floats; key is a non-negative float).  With H = h,
// h - 1 - m = m ^ (h - 1) and h + m = m ^ h, so code = m ^ (h - s).
// Decision in fp32, the kernel's precision [R14b].
__device__ __forceinline__ uint32_t sign_of(float y) { return __float_as_uint(y) >> 31; }
__device__ __forceinline__ float key_of(float y) {
  const uint32_t b = __float_as_uint(y);
  return __uint_as_float(b - (b >> 31) * 0x80000001u);
}

// Signed centroid values of a coordinate pair (roundtrip without codes):
// c = cpos[0] + sum_i [key >= tau_i] * (cpos[i] - cpos[i-1]), sign of y.
template <int BITS>
__device__ __forceinline__ float2 qvalue2(float2 y, const KCodebook& cb) {
  constexpr int H = 1 << (BITS - 1);
  const float ka = key_of(y.x), kb = key_of(y.y);
  float2 c = f2(cb.cpos[0], cb.cpos[0]);
#pragma unroll
  for (int i = 1; i < H; ++i) {
    const float2 g = f2(ka >= cb.tau[i] ? 1.0f : 0.0f, kb >= cb.tau[i] ? 1.0f : 0.0f);
    c = fma2(g, f2(cb.delta[i], cb.delta[i]), c);
  }
  return f2(__uint_as_float(__float_as_uint(c.x) ^ (__float_as_uint(y.x) & 0x80000000u)),
            __uint_as_float(__float_as_uint(c.y) ^ (__float_as_uint(y.y) & 0x80000000u)));
}

// Code (and, through the shared-memory table s_cpos, the signed centroid).
template <int BITS>
__device__ __forceinline__ uint32_t qcode(float y, const KCodebook& cb) {
  constexpr int H = 1 << (BITS - 1);
  const float k = key_of(y);
  uint32_t m = 0;
#pragma unroll
  for (int i = 1; i < H; ++i) m += (k >= cb.tau[i]) ? 1u : 0u;
  return m ^ (uint32_t)(H - (int)sign_of(y));
}
// signed centroid from the code: C[code], symmetric table in shared memory
__device__ __forceinline__ float centroid_of(uint32_t code, const float* s_cent) { return s_cent[code]; }

// ------------------------------------------------------------- bit packing
// A lane's chunk contributes B = EPC*BITS consecutive bits of the row's
// LSB-first bitstream [R7].  G lanes form a segment of G*B bits = W words.
constexpr int max_sources(int G, int B) {
  int mx = 0;
  for (int w = 0; w < G * B / 32; ++w) {
    const int s0 = 32 * w / B, s1 = (32 * w + 31) / B;
    if (s1 - s0 + 1 > mx) mx = s1 - s0 + 1;
  }
  return mx;
}

// Word `sub` of the segment (valid for sub < W), gathered by shuffles from
// the lanes whose bits overlap it.
template <int G, int B>
__device__ __forceinline__ uint32_t gather_word(uint32_t bits, int sub, int vbase) {
  if constexpr (B == 32) {
    return bits;
  } else {
    constexpr int NS = max_sources(G, B);
    const int s0 = (32 * sub) / B;
    uint32_t word = 0;
#pragma unroll
    for (int j = 0; j < NS; ++j) {
      const int s = s0 + j;
      const uint32_t v = __shfl_sync(kFull, bits, vbase + (s < G ? s : G - 1));
      const int shift = s * B - 32 * sub;
      if (s < G && shift < 32) word |= (shift >= 0) ? (v << shift) : (v >> (-shift));
    }
    return word;
  }
}

// The B bits of lane `sub` from the segment's words (word t held by lane t).
template <int G, int B>
__device__ __forceinline__ uint32_t scatter_bits(uint32_t word, int sub, int vbase) {
  if constexpr (B == 32) {
    return word;
  } else {
    constexpr int W = G * B / 32;
    const int off = sub * B;
    const int w0 = off >> 5, sh = off & 31;
    const uint32_t lo = __shfl_sync(kFull, word, vbase + w0);
    const uint32_t hi = __shfl_sync(kFull, word, vbase + (w0 + 1 < W ? w0 + 1 : W - 1));
    uint32_t r = (sh == 0) ? lo : ((lo >> sh) | (hi << (32 - sh)));
    return r & ((1u << B) - 1u);
  }
}

// Load a lane's paired operators: pair k = blocks A (lane coords 2PWk..) and
// B (2PWk+PW..).  Lane coordinate c*EPC+e <-> global coordinate
// (sub + c*G)*EPC + e, so block index = global coordinate / PW.
template <class Gm>
__device__ __forceinline__ void load_ops(const float* __restrict__ mat, int sub,
                                         float2 (&P)[Gm::NPAIR][Gm::PW * Gm::PW]) {
  constexpr int PW = Gm::PW, EPC = Gm::EPC, G = Gm::G, NPB = PW * PW;
#pragma unroll
  for (int k = 0; k < Gm::NPAIR; ++k) {
    const int la = coordA<PW>(k, 0), lb = coordB<PW>(k, 0);
    const int ga = (sub + (la / EPC) * G) * EPC + la % EPC;
    const int gb = (sub + (lb / EPC) * G) * EPC + lb % EPC;
    const float* ma = mat + (size_t)(ga / PW) * NPB;
    const float* mb = mat + (size_t)(gb / PW) * NPB;
#pragma unroll
    for (int q = 0; q < NPB; ++q) P[k][q] = f2(__ldg(ma + q), __ldg(mb + q));
  }
}

// --------------------------------------------------------- encoder (K1/K3)
// MODE 0: quantize (codes + norms).  MODE 1: fused roundtrip (y; codes and
// norms too when `codes` is non-null).
template <class T, int D, int BITS, int VAR, int MODE>
__global__ void __launch_bounds__(kEncThreads)
k_encode(const float* __restrict__ mat, const KCodebook cb, int64_t n, const T* x, T* y,
         uint8_t* __restrict__ codes, float* __restrict__ norms) {
  using Gm = Geo<T, D, VAR>;
  constexpr int EPC = Gm::EPC, G = Gm::G, CPL = Gm::CPL, VPW = Gm::VPW, U = Gm::U;
  constexpr int PW = Gm::PW, NPAIR = Gm::NPAIR, EPL = Gm::EPL, TILE_V = Gm::TILE_V;
  constexpr int B = EPC * BITS, W = G * B / 32, RB = D * BITS / 8;
  constexpr int L = 1 << BITS;
  static_assert((G * B) % 32 == 0, "segment must be whole words");

  extern __shared__ __align__(128) uint8_t smem[];
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + kStages * kStageBytes);
  uint64_t* empty = full + kStages;
  float* s_cent = reinterpret_cast<float*>(empty + kStages);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], kNWC);
    }
    fence_mbar_init();
  }
  if (threadIdx.x < L) s_cent[threadIdx.x] = cb.cent[threadIdx.x];
  __syncthreads();

  const int64_t ntiles = (n + TILE_V - 1) / TILE_V;

  if (warp == kNWC) {  // ---------------- producer: TMA bulk loads into the ring
    if (lane == 0) {
      const uint64_t pol = policy_evict_first();
      int s = 0;
      uint32_t ph = 0;
      for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
        mbar_wait(&empty[s], ph ^ 1);
        const int64_t v0 = t * TILE_V;
        const int64_t nv = (n - v0) < TILE_V ? (n - v0) : TILE_V;
        const uint32_t bytes = (uint32_t)(nv * Gm::ROWB);
        mbar_arrive_expect_tx(&full[s], bytes);
        bulk_g2s(smem + s * kStageBytes, x + v0 * D, bytes, &full[s], pol);
        if (++s == kStages) { s = 0; ph ^= 1; }
      }
    }
    return;
  }

  // ---------------------------------------------------- compute warps
  const int sub = lane & (G - 1);
  const int vbase = lane & ~(G - 1);
  const int vslot = lane / G;
  float2 P[NPAIR][PW * PW];
  load_ops<Gm>(mat, sub, P);
  const bool emit = (MODE == 0) || (codes != nullptr);

  int s = 0;
  uint32_t ph = 0;
  for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
    mbar_wait(&full[s], ph);
    const uint8_t* st = smem + s * kStageBytes;
    uint4 raw[U][CPL];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int vl = (warp * U + u) * VPW + vslot;   // row within the tile
#pragma unroll
      for (int i = 0; i < CPL; ++i)
        raw[u][i] = lds128(st + (size_t)vl * Gm::ROWB + (sub + i * G) * 16);
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[s]);           // stage may be refilled
    if (++s == kStages) { s = 0; ph ^= 1; }

#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t vec = t * TILE_V + (warp * U + u) * VPW + vslot;
      const bool valid = vec < n;
      float v[EPL];
#pragma unroll
      for (int i = 0; i < CPL; ++i) to_f32<T>(raw[u][i], v + i * EPC);
      // Alg.1 l.1: rho = ||x||, xbar = x / max(rho, eps)  [R5]
      float2 ss2 = f2(0.0f, 0.0f);
#pragma unroll
      for (int e = 0; e < EPL; e += 2) ss2 = fma2(f2(v[e], v[e + 1]), f2(v[e], v[e + 1]), ss2);
      float ss = ss2.x + ss2.y;
#pragma unroll
      for (int o = G / 2; o >= 1; o >>= 1) ss += __shfl_xor_sync(kFull, ss, o);
      const float rho = sqrt_approx(ss);
      const float inv = rsqrt_approx(fmaxf(ss, 1e-24f));
      const float2 inv2 = f2(inv, inv), rho2 = f2(rho, rho);

      float out[EPL];
      uint32_t cw[CPL];
#pragma unroll
      for (int i = 0; i < CPL; ++i) cw[i] = 0;
#pragma unroll
      for (int k = 0; k < NPAIR; ++k) {
        float2 xb[PW], yb[PW], cq[PW], rb[PW];
#pragma unroll
        for (int j = 0; j < PW; ++j) xb[j] = mul2(f2(v[coordA<PW>(k, j)], v[coordB<PW>(k, j)]), inv2);
        rot_fwd2<PW>(P[k], xb, yb);                          // v~ = T(v)   (Alg.1 l.5/9/13)
        if (emit) {
#pragma unroll
          for (int j = 0; j < PW; ++j) {
            const uint32_t ca = qcode<BITS>(yb[j].x, cb), cbb = qcode<BITS>(yb[j].y, cb);
            const int la = coordA<PW>(k, j), lb = coordB<PW>(k, j);
            cw[la / EPC] += ca << ((la % EPC) * BITS);
            cw[lb / EPC] += cbb << ((lb % EPC) * BITS);
            if (MODE == 1) cq[j] = f2(centroid_of(ca, s_cent), centroid_of(cbb, s_cent));
          }
        } else {
#pragma unroll
          for (int j = 0; j < PW; ++j) cq[j] = qvalue2<BITS>(yb[j], cb);   // v^ = Q(v~)
        }
        if (MODE == 1) {
          rot_inv2<PW>(P[k], cq, rb);                        // v_rec = T^-1(v^)
#pragma unroll
          for (int j = 0; j < PW; ++j) {
            const float2 o = mul2(rb[j], rho2);              // x^ = rho * v_rec
            out[coordA<PW>(k, j)] = o.x;
            out[coordB<PW>(k, j)] = o.y;
          }
        }
      }
#pragma unroll
      for (int i = 0; i < CPL; ++i) {
        if (MODE == 1 && valid) st_stream(y + vec * D + (sub + i * G) * EPC, from_f32<T>(out + i * EPC));
        if (emit) {
          const uint32_t word = gather_word<G, B>(cw[i], sub, vbase);
          if (valid && sub < W)
            *reinterpret_cast<uint32_t*>(codes + vec * RB + 4 * (i * W + sub)) = word;
        }
      }
      if (emit && valid && sub == 0) norms[vec] = rho;
    }
  }
}

// ---------------------------------------------------------------- decoder (K2)
template <class T, int D, int BITS, int VAR>
__global__ void __launch_bounds__(kThreads)
k_decode(const float* __restrict__ mat, const KCodebook cb, int64_t n,
         const uint8_t* __restrict__ codes, const float* __restrict__ norms, T* __restrict__ y) {
  using Gm = Geo<T, D, VAR>;
  constexpr int EPC = Gm::EPC, G = Gm::G, CPL = Gm::CPL, VPW = Gm::VPW, U = Gm::UD;
  constexpr int PW = Gm::PW, NPAIR = Gm::NPAIR, EPL = Gm::EPL;
  constexpr int B = EPC * BITS, W = G * B / 32, RB = D * BITS / 8;
  constexpr int L = 1 << BITS;

  __shared__ float s_cent[L];
  if (threadIdx.x < L) s_cent[threadIdx.x] = cb.cent[threadIdx.x];
  __syncthreads();

  const int lane = threadIdx.x & 31;
  const int sub = lane & (G - 1);
  const int vbase = lane & ~(G - 1);
  const int vslot = lane / G;
  float2 P[NPAIR][PW * PW];
  load_ops<Gm>(mat, sub, P);

  const int64_t warp = ((int64_t)blockIdx.x * kThreads + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * kThreads) >> 5;
  const int64_t ntiles = (n + VPW * U - 1) / (VPW * U);
  for (int64_t tile = warp; tile < ntiles; tile += nwarps) {
    uint32_t wd[U][CPL];
    float rho[U];
    int64_t vec[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      vec[u] = tile * (VPW * U) + u * VPW + vslot;
      const bool valid = vec[u] < n;
#pragma unroll
      for (int i = 0; i < CPL; ++i)
        wd[u][i] = (valid && sub < W)
            ? __ldcs(reinterpret_cast<const unsigned int*>(codes + vec[u] * RB + 4 * (i * W + sub)))
            : 0u;
      rho[u] = valid ? __ldcs(norms + vec[u]) : 0.0f;
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      uint32_t bits[CPL];
#pragma unroll
      for (int i = 0; i < CPL; ++i) bits[i] = scatter_bits<G, B>(wd[u][i], sub, vbase);
      const float2 rho2 = f2(rho[u], rho[u]);
      float out[EPL];
#pragma unroll
      for (int k = 0; k < NPAIR; ++k) {
        float2 cq[PW], rb[PW];
#pragma unroll
        for (int j = 0; j < PW; ++j) {
          const int la = coordA<PW>(k, j), lb = coordB<PW>(k, j);
          const uint32_t ca = (bits[la / EPC] >> ((la % EPC) * BITS)) & (L - 1);
          const uint32_t cbb = (bits[lb / EPC] >> ((lb % EPC) * BITS)) & (L - 1);
          cq[j] = f2(s_cent[ca], s_cent[cbb]);             // v^ = C[code]
        }
        rot_inv2<PW>(P[k], cq, rb);                         // T^-1
#pragma unroll
        for (int j = 0; j < PW; ++j) {
          const float2 o = mul2(rb[j], rho2);               // x^ = rho * ...
          out[coordA<PW>(k, j)] = o.x;
          out[coordB<PW>(k, j)] = o.y;
        }
      }
      if (vec[u] < n) {
#pragma unroll
        for (int i = 0; i < CPL; ++i)
          st_stream(y + vec[u] * D + (sub + i * G) * EPC, from_f32<T>(out + i * EPC));
      }
    }
  }
}

// ------------------------------------------------ reconstruction statistics
template <class T>
__global__ void __launch_bounds__(kThreads)
k_error_sums(int64_t nchunks, const T* __restrict__ x, const T* __restrict__ y, double* sums) {
  constexpr int EPC = DT<T>::EPC;
  float se = 0.0f, sx = 0.0f;
  double dse = 0.0, dsx = 0.0;
  int cnt = 0;
  for (int64_t c = (int64_t)blockIdx.x * kThreads + threadIdx.x; c < nchunks;
       c += (int64_t)gridDim.x * kThreads) {
    float a[EPC], b[EPC];
    to_f32<T>(__ldcs(reinterpret_cast<const uint4*>(x + c * EPC)), a);
    to_f32<T>(__ldcs(reinterpret_cast<const uint4*>(y + c * EPC)), b);
#pragma unroll
    for (int e = 0; e < EPC; ++e) {
      const float t = a[e] - b[e];
      se = fmaf(t, t, se);
      sx = fmaf(a[e], a[e], sx);
    }
    if (++cnt == 64) { dse += se; dsx += sx; se = sx = 0.0f; cnt = 0; }
  }
  dse += se; dsx += sx;
#pragma unroll
  for (int o = 16; o >= 1; o >>= 1) {
    dse += __shfl_xor_sync(kFull, dse, o);
    dsx += __shfl_xor_sync(kFull, dsx, o);
  }
  if ((threadIdx.x & 31) == 0) {
    atomicAdd(sums, dse);
    atomicAdd(sums + 1, dsx);
  }
}

}  // namespace iq
