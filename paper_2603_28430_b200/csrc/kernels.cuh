// sm_100a kernels of the IsoQuant stage-1 path (Algorithm 1,
// P:229-258).  The path is an elementwise map with O(d) work per O(d) bytes
// and no reuse, so it is bound by HBM bandwidth (and, at fp16, close to the
// instruction-issue ceiling): no tensor cores, no shared-memory staging of
// the data; 128-bit streaming loads/stores, parameters in registers, the
// codebook in the constant bank, warp shuffles for the norm and for code
// packing.  See DESIGN.md "Kernels".
//
// Thread mapping: a vector of d elements of dtype T is split into 16-byte
// chunks (EPC = 4 fp32 or 8 fp16 elements).  G = min(32, d/EPC) consecutive
// lanes serve one vector; lane `sub` owns chunks sub, sub+G, ... (CPL chunks),
// so every warp-wide access of a chunk index is contiguous.  A warp holds
// VPW = 32/G vectors and each iteration of the persistent loop handles U
// vectors per lane group (U*CPL 16-byte loads in flight per lane).  The
// blocks a lane rotates never change, so their operators stay in registers
// for the whole kernel ("the entire block can often remain in
// registers from input load through output store").
#pragma once
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "iq_internal.h"

namespace iq {

constexpr unsigned kFull = 0xffffffffu;
constexpr int kThreads = 256;

template <class T> struct DT;
template <> struct DT<float> { static constexpr int EPC = 4; };
template <> struct DT<__half> { static constexpr int EPC = 8; };

template <class T, int D>
struct Geo {
  static constexpr int EPC = DT<T>::EPC;
  static constexpr int CHUNKS = D / EPC;
  static constexpr int G = CHUNKS < 32 ? CHUNKS : 32;
  static constexpr int CPL = CHUNKS / G;
  static constexpr int VPW = 32 / G;
  static constexpr int U = (4 / CPL) > 0 ? (4 / CPL) : 1;
  static_assert(D % EPC == 0 && (G & (G - 1)) == 0 && CHUNKS % G == 0, "unsupported d");
};

// ---------------------------------------------------------------- memory ops
__device__ __forceinline__ uint4 ld_stream(const void* p) {
  return __ldcs(reinterpret_cast<const uint4*>(p));
}
__device__ __forceinline__ void st_stream(void* p, const uint4& v) {
  __stcs(reinterpret_cast<uint4*>(p), v);
}

template <class T> __device__ __forceinline__ void to_f32(const uint4& r, float* f);
template <> __device__ __forceinline__ void to_f32<float>(const uint4& r, float* f) {
  f[0] = __uint_as_float(r.x); f[1] = __uint_as_float(r.y);
  f[2] = __uint_as_float(r.z); f[3] = __uint_as_float(r.w);
}
template <> __device__ __forceinline__ void to_f32<__half>(const uint4& r, float* f) {
  const uint32_t w[4] = {r.x, r.y, r.z, r.w};
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    __half2 h = *reinterpret_cast<const __half2*>(&w[k]);
    float2 t = __half22float2(h);
    f[2 * k] = t.x; f[2 * k + 1] = t.y;
  }
}

template <class T> __device__ __forceinline__ uint4 from_f32(const float* f);
template <> __device__ __forceinline__ uint4 from_f32<float>(const float* f) {
  return make_uint4(__float_as_uint(f[0]), __float_as_uint(f[1]),
                    __float_as_uint(f[2]), __float_as_uint(f[3]));
}
template <> __device__ __forceinline__ uint4 from_f32<__half>(const float* f) {
  uint32_t w[4];
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    __half2 h = __floats2half2_rn(f[2 * k], f[2 * k + 1]);  // RN-even [R15]
    w[k] = *reinterpret_cast<uint32_t*>(&h);
  }
  return make_uint4(w[0], w[1], w[2], w[3]);
}

// ----------------------------------------------------------- block operator
// PW x PW operator M (row-major): forward y = M v, inverse v = M^T c.
// 4-D: M = L(q_L) R(conj q_R) (Full) / L(q_L) (Fast); the inverse sandwich
// conj(q_L) v q_R is exactly M^T (Proposition).  2-D: M = R(theta),
// inverse R(-theta) = R(theta)^T.  Every dot product starts from +0
// so that a rotated coordinate is never -0 (the decision below then treats
// +-0 like the count definition does: both go to the upper half [R3]).
template <int PW>
__device__ __forceinline__ void rot_fwd(const float* M, const float* v, float* y) {
#pragma unroll
  for (int i = 0; i < PW; ++i) {
    float a = 0.0f;
#pragma unroll
    for (int j = 0; j < PW; ++j) a = fmaf(M[PW * i + j], v[j], a);
    y[i] = a;
  }
}
template <int PW>
__device__ __forceinline__ void rot_inv(const float* M, const float* c, float* v) {
#pragma unroll
  for (int j = 0; j < PW; ++j) {
    float a = 0.0f;
#pragma unroll
    for (int i = 0; i < PW; ++i) a = fmaf(M[PW * i + j], c[i], a);
    v[j] = a;
  }
}

// --------------------------------------------------------------- quantizer Q
// code = #{k : y >= t_k} over the symmetric fp32 thresholds (ties up, clamp):
//   y >= 0 : code = h + #{m >= 1 : y >= tau_m}
//   y <  0 : code = h - 1 - #{m >= 1 : |y| > tau_m}
// |y| > tau for positive floats <=> bits(|y|) - 1 >= bits(tau) (IEEE order of
// non-negative floats = integer order), so one integer key serves both
// signs.  Decision in fp32, the kernel's precision [R14b].
template <int BITS>
__device__ __forceinline__ float quant_value(float y, const KCodebook& cb) {
  constexpr int H = 1 << (BITS - 1);
  const bool neg = y < 0.0f;
  const uint32_t key = (__float_as_uint(y) & 0x7fffffffu) - (neg ? 1u : 0u);
  float c = cb.cpos[0];
#pragma unroll
  for (int m = 1; m < H; ++m) c = (key >= cb.tau_bits[m]) ? cb.cpos[m] : c;
  return neg ? -c : c;
}

template <int BITS>
__device__ __forceinline__ uint32_t quant_code(float y, const KCodebook& cb, float* value) {
  constexpr int H = 1 << (BITS - 1);
  const bool neg = y < 0.0f;
  const uint32_t key = (__float_as_uint(y) & 0x7fffffffu) - (neg ? 1u : 0u);
  float c = cb.cpos[0];
  uint32_t m = 0;
#pragma unroll
  for (int i = 1; i < H; ++i) {
    const bool ge = key >= cb.tau_bits[i];
    c = ge ? cb.cpos[i] : c;
    m += ge ? 1u : 0u;
  }
  *value = neg ? -c : c;
  return neg ? (uint32_t)(H - 1) - m : (uint32_t)H + m;
}

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

// The B bits of lane `sub` from the segment's words (word t held by lane t).
template <int G, int B>
__device__ __forceinline__ uint32_t scatter_bits(uint32_t word, int sub, int vbase) {
  constexpr int W = G * B / 32;
  const int off = sub * B;
  const int w0 = off >> 5, sh = off & 31;
  const uint32_t lo = __shfl_sync(kFull, word, vbase + w0);
  uint32_t r;
  if constexpr (B == 32) {
    r = lo;
  } else {
    const uint32_t hi = __shfl_sync(kFull, word, vbase + (w0 + 1 < W ? w0 + 1 : W - 1));
    r = (sh == 0) ? lo : ((lo >> sh) | (hi << (32 - sh)));
    r &= (1u << B) - 1u;
  }
  return r;
}

// --------------------------------------------------------- encoder (K1/K3)
// MODE 0: quantize (codes + norms).  MODE 1: fused roundtrip (y; codes and
// norms too when `codes` is non-null).
template <class T, int D, int BITS, int VAR, int MODE>
__global__ void __launch_bounds__(kThreads)
k_encode(const float* __restrict__ mat, const KCodebook cb, int64_t n,
         const T* x, T* y, uint8_t* __restrict__ codes, float* __restrict__ norms) {
  using Gm = Geo<T, D>;
  constexpr int EPC = Gm::EPC, G = Gm::G, CPL = Gm::CPL, VPW = Gm::VPW, U = Gm::U;
  constexpr int PW = (VAR == IQ_VARIANT_PLANAR2D) ? 2 : 4;
  constexpr int BPC = EPC / PW, NPB = PW * PW;
  constexpr int B = EPC * BITS, W = G * B / 32, RB = D * BITS / 8;
  static_assert((G * B) % 32 == 0, "segment must be whole words");

  const int lane = threadIdx.x & 31;
  const int sub = lane & (G - 1);
  const int vbase = lane & ~(G - 1);
  const int vslot = lane / G;

  float P[CPL][BPC * NPB];
#pragma unroll
  for (int i = 0; i < CPL; ++i) {
    const float4* src = reinterpret_cast<const float4*>(mat + (size_t)(sub + i * G) * EPC * PW);
#pragma unroll
    for (int k = 0; k < BPC * NPB / 4; ++k) {
      const float4 t = __ldg(src + k);
      P[i][4 * k] = t.x; P[i][4 * k + 1] = t.y; P[i][4 * k + 2] = t.z; P[i][4 * k + 3] = t.w;
    }
  }
  const bool emit = (MODE == 0) || (codes != nullptr);

  const int64_t warp = ((int64_t)blockIdx.x * kThreads + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * kThreads) >> 5;
  const int64_t ntiles = (n + VPW * U - 1) / (VPW * U);
  for (int64_t tile = warp; tile < ntiles; tile += nwarps) {
    uint4 raw[U][CPL];
    int64_t vec[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      vec[u] = tile * (VPW * U) + u * VPW + vslot;
#pragma unroll
      for (int i = 0; i < CPL; ++i)
        raw[u][i] = (vec[u] < n) ? ld_stream(x + vec[u] * D + (sub + i * G) * EPC)
                                 : make_uint4(0, 0, 0, 0);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      float v[CPL][EPC];
      float ss = 0.0f;
#pragma unroll
      for (int i = 0; i < CPL; ++i) {
        to_f32<T>(raw[u][i], v[i]);
#pragma unroll
        for (int e = 0; e < EPC; ++e) ss = fmaf(v[i][e], v[i][e], ss);
      }
#pragma unroll
      for (int o = G / 2; o >= 1; o >>= 1) ss += __shfl_xor_sync(kFull, ss, o);
      const float rho = sqrtf(ss);                          // Alg.1 l.1
      const float inv = __frcp_rn(fmaxf(rho, 1e-12f));      // 1 / max(rho, eps) [R5]
      const bool valid = vec[u] < n;
#pragma unroll
      for (int i = 0; i < CPL; ++i) {
        float out[EPC];
        uint32_t cbits = 0;
#pragma unroll
        for (int b = 0; b < BPC; ++b) {
          float xb[PW], yb[PW], cq[PW];
#pragma unroll
          for (int e = 0; e < PW; ++e) xb[e] = v[i][b * PW + e] * inv;
          rot_fwd<PW>(&P[i][b * NPB], xb, yb);              // v~ = T(v)
#pragma unroll
          for (int e = 0; e < PW; ++e) {
            if (emit) {
              const uint32_t code = quant_code<BITS>(yb[e], cb, &cq[e]);
              cbits |= code << ((b * PW + e) * BITS);
            } else {
              cq[e] = quant_value<BITS>(yb[e], cb);         // v^ = Q(v~)
            }
          }
          if (MODE == 1) {
            float rb[PW];
            rot_inv<PW>(&P[i][b * NPB], cq, rb);            // v_rec = T^-1(v^)
#pragma unroll
            for (int e = 0; e < PW; ++e) out[b * PW + e] = rho * rb[e];   // x^ = rho * ...
          }
        }
        if (MODE == 1 && valid) st_stream(y + vec[u] * D + (sub + i * G) * EPC, from_f32<T>(out));
        if (emit) {
          const uint32_t word = gather_word<G, B>(cbits, sub, vbase);
          if (valid && sub < W)
            *reinterpret_cast<uint32_t*>(codes + vec[u] * RB + 4 * (i * W + sub)) = word;
        }
      }
      if (emit && valid && sub == 0) norms[vec[u]] = rho;
    }
  }
}

// ---------------------------------------------------------------- decoder (K2)
template <class T, int D, int BITS, int VAR>
__global__ void __launch_bounds__(kThreads)
k_decode(const float* __restrict__ mat, const KCodebook cb, int64_t n,
         const uint8_t* __restrict__ codes, const float* __restrict__ norms, T* __restrict__ y) {
  using Gm = Geo<T, D>;
  constexpr int EPC = Gm::EPC, G = Gm::G, CPL = Gm::CPL, VPW = Gm::VPW, U = Gm::U;
  constexpr int PW = (VAR == IQ_VARIANT_PLANAR2D) ? 2 : 4;
  constexpr int BPC = EPC / PW, NPB = PW * PW;
  constexpr int B = EPC * BITS, W = G * B / 32, RB = D * BITS / 8;
  constexpr int L = 1 << BITS;

  __shared__ float s_cent[L];
  if (threadIdx.x < L) s_cent[threadIdx.x] = cb.cent[threadIdx.x];
  __syncthreads();

  const int lane = threadIdx.x & 31;
  const int sub = lane & (G - 1);
  const int vbase = lane & ~(G - 1);
  const int vslot = lane / G;

  float P[CPL][BPC * NPB];
#pragma unroll
  for (int i = 0; i < CPL; ++i) {
    const float4* src = reinterpret_cast<const float4*>(mat + (size_t)(sub + i * G) * EPC * PW);
#pragma unroll
    for (int k = 0; k < BPC * NPB / 4; ++k) {
      const float4 t = __ldg(src + k);
      P[i][4 * k] = t.x; P[i][4 * k + 1] = t.y; P[i][4 * k + 2] = t.z; P[i][4 * k + 3] = t.w;
    }
  }

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
#pragma unroll
      for (int i = 0; i < CPL; ++i) {
        const uint32_t bits = scatter_bits<G, B>(wd[u][i], sub, vbase);
        float out[EPC];
#pragma unroll
        for (int b = 0; b < BPC; ++b) {
          float cq[PW], rb[PW];
#pragma unroll
          for (int e = 0; e < PW; ++e)
            cq[e] = s_cent[(bits >> ((b * PW + e) * BITS)) & (L - 1)];   // v^ = C[code]
          rot_inv<PW>(&P[i][b * NPB], cq, rb);                          // T^-1
#pragma unroll
          for (int e = 0; e < PW; ++e) out[b * PW + e] = rho[u] * rb[e];  // x^ = rho * ...
        }
        if (vec[u] < n) st_stream(y + vec[u] * D + (sub + i * G) * EPC, from_f32<T>(out));
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
    to_f32<T>(ld_stream(x + c * EPC), a);
    to_f32<T>(ld_stream(y + c * EPC), b);
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
