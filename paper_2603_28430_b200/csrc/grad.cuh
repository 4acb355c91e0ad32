// Learning the block rotations (NEXT row 4 of SURVEY section 8(f); PAPER.md
// "Parameterization and Learning": q = u / ||u|| with free u, so
// that optimisation stays Euclidean).  The paper leaves the objective open;
// DESIGN.md reading R29 takes the stage-1 distortion on normalised rows,
//   L = sum_rows || T xbar - Q(T xbar) ||^2      (= the normalised MSE, T orthogonal),
// whose gradient with respect to each block operator M_b is exact almost
// everywhere (Q is piecewise constant):
//   dL/dM_b = 2 sum_rows e_b xbar_b^T,   e = T xbar - Q(T xbar).
// This kernel streams the rows once (TMA ring as in the encoders), forms e
// per block in registers and accumulates the PW x PW outer products; lanes,
// warps (shared-memory atomics) and CTAs (fp64 global atomics) are reduced at
// the end.  The chain rule to the quaternion / angle parameters is a host
// step (params.cpp, iq_rot_grad_from_operator_grad).
#pragma once
#include "kernels.cuh"

namespace iq {

template <class T, int D, int BITS, int VAR>
struct GGeo {
  using Gm = Geo<T, D, BITS, VAR, 4>;            // 8 coordinates per lane, operators in registers
  static constexpr int GSM_OFF = Gm::ENC_SMEM;   // per-CTA sums [D / PW][PW * PW] floats
  static constexpr int SMEM = GSM_OFF + D * Gm::PW * 4;
};

template <class T, int D, int BITS, int VAR>
__global__ void __launch_bounds__(GGeo<T, D, BITS, VAR>::Gm::CTA_THREADS, 1)
k_distortion_grad(const float* __restrict__ mat, const KCodebook cb, int64_t n, const T* x,
                  double* __restrict__ grad, double* __restrict__ loss) {
  using GG = GGeo<T, D, BITS, VAR>;
  using Gm = typename GG::Gm;
  constexpr int NWC = Gm::NWC;
  constexpr int EPC = Gm::EPC, G = Gm::G, CPL = Gm::CPL, VPW = Gm::VPW, U = Gm::U;
  constexpr int PW = Gm::PW, NBL = Gm::NBL, EPL = Gm::EPL, TILE_V = Gm::TILE_V;
  constexpr int STAGE = Gm::ENC_STAGE, NST = Gm::ENC_STAGES, NPB = PW * PW;
  static_assert(!Gm::OPS_SMEM, "operators in registers");

  extern __shared__ __align__(128) uint8_t smem[];
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + NST * STAGE);
  uint64_t* empty = full + NST;
  float* gsm = reinterpret_cast<float*>(smem + GG::GSM_OFF);
  ring_init<NST, NWC>(full, empty);
  for (int i = threadIdx.x; i < D * PW; i += blockDim.x) gsm[i] = 0.0f;
  __syncthreads();

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t ntiles = (n + TILE_V - 1) / TILE_V;

  if (warp == NWC) {  // ---------------- producer: TMA bulk loads into the ring
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
        bulk_g2s(smem + s * STAGE, x + v0 * D, bytes, &full[s], pol);
        if (++s == NST) { s = 0; ph ^= 1; }
      }
    }
    return;
  }

  const int sub = lane & (G - 1);
  const int vslot = lane / G;
  float P[NBL][NPB];
  load_ops<Gm>(mat, sub, P);
  float acc[NBL][NPB];
#pragma unroll
  for (int b = 0; b < NBL; ++b)
#pragma unroll
    for (int k = 0; k < NPB; ++k) acc[b][k] = 0.0f;
  float lsum = 0.0f;

  int s = 0;
  uint32_t ph = 0;
  for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
    mbar_wait_warp(&full[s], ph, lane);
    const uint8_t* st = smem + s * STAGE;
    const int ss_ = s;
    if (++s == NST) { s = 0; ph ^= 1; }
    const int64_t v0 = t * TILE_V;
    const int nv = (n - v0) < TILE_V ? (int)(n - v0) : TILE_V;
#pragma unroll 1
    for (int u = 0; u < U; u += 2) {
      uint4 ra[CPL], rb[CPL];
      const int vl = (warp * U + u) * VPW + vslot;
#pragma unroll
      for (int i = 0; i < CPL; ++i) {
        ra[i] = lds128(st + vl * Gm::ROWB + (sub + i * G) * 16);
        rb[i] = lds128(st + (vl + VPW) * Gm::ROWB + (sub + i * G) * 16);
      }
      if (vl >= nv) {                       // stale stage bytes past the end: zero rows
#pragma unroll
        for (int i = 0; i < CPL; ++i) ra[i] = make_uint4(0u, 0u, 0u, 0u);
      }
      if (vl + VPW >= nv) {
#pragma unroll
        for (int i = 0; i < CPL; ++i) rb[i] = make_uint4(0u, 0u, 0u, 0u);
      }
      float2 v[EPL];
#pragma unroll
      for (int i = 0; i < CPL; ++i) to_pairs<T>(ra[i], rb[i], v + i * EPC);
      float2 ss = mul2(v[0], v[0]);
#pragma unroll
      for (int e = 1; e < EPL; ++e) ss = fma2(v[e], v[e], ss);
      if (u + 2 == U) {
        __syncwarp();
        if (lane == 0) mbar_arrive_after(&empty[ss_], ss.x + ss.y);
      }
#pragma unroll
      for (int o = G / 2; o >= 1; o >>= 1)
        ss = add2(ss, f2(__shfl_xor_sync(kFull, ss.x, o), __shfl_xor_sync(kFull, ss.y, o)));
      const float2 inv = f2(rsqrt_ftz(fmaxf(ss.x, 1e-24f)), rsqrt_ftz(fmaxf(ss.y, 1e-24f)));   // 1/max(rho, eps)
      // rows beyond the tile's end contribute nothing (zero xbar, masked e)
      const float2 ok = f2(vl < nv ? 1.0f : 0.0f, vl + VPW < nv ? 1.0f : 0.0f);
#pragma unroll
      for (int b = 0; b < NBL; ++b) {
        float2 xb[PW], yb[PW];
#pragma unroll
        for (int j = 0; j < PW; ++j) xb[j] = mul2(v[b * PW + j], inv);     // xbar (Alg.1 l.1)
        rot_fwd<PW>(P[b], xb, yb);                                      // ybar = T xbar
#pragma unroll
        for (int i = 0; i < PW; ++i) {
          uint32_t d0, d1;
          const float2 c = quantize_pair_u<BITS, true, false>(yb[i], cb, d0, d1);   // Q(ybar)
          const float2 e = f2((yb[i].x - c.x) * ok.x, (yb[i].y - c.y) * ok.y);
          lsum = fmaf(e.x, e.x, fmaf(e.y, e.y, lsum));
#pragma unroll
          for (int j = 0; j < PW; ++j)                                    // e_i xbar_j
            acc[b][PW * i + j] = fmaf(e.x, xb[j].x, fmaf(e.y, xb[j].y, acc[b][PW * i + j]));
        }
      }
    }
  }
  // ---- reduction: lanes that own the same blocks (row slots), warps, CTAs
#pragma unroll
  for (int o = G; o < 32; o <<= 1) {
#pragma unroll
    for (int b = 0; b < NBL; ++b)
#pragma unroll
      for (int k = 0; k < NPB; ++k) acc[b][k] += __shfl_xor_sync(kFull, acc[b][k], o);
  }
#pragma unroll
  for (int o = 16; o >= 1; o >>= 1) lsum += __shfl_xor_sync(kFull, lsum, o);
  if (lane < G) {
#pragma unroll
    for (int b = 0; b < NBL; ++b) {
      const int lc = b * PW;
      const int gc = (sub + (lc / EPC) * G) * EPC + lc % EPC;   // first coordinate of the block
#pragma unroll
      for (int k = 0; k < NPB; ++k) atomicAdd(&gsm[(gc / PW) * NPB + k], acc[b][k]);
    }
  }
  if (lane == 0 && loss) atomicAdd(loss, (double)lsum);
  asm volatile("bar.sync 1, %0;" ::"r"(NWC * 32) : "memory");   // compute warps only
  for (int i = threadIdx.x; i < D * PW; i += NWC * 32) atomicAdd(&grad[i], 2.0 * (double)gsm[i]);
}

}  // namespace iq
