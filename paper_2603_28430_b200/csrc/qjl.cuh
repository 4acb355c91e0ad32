// Stage-2 residual sketch fused with the stage-1 encoder (NEXT row 1 of
// SURVEY section 8(f); PAPER.md section "Compatibility with Residual
// Correction": r = x - x^_mse, projected with a quantized
// Johnson-Lindenstrauss transform).  DESIGN.md readings R20-R24.
//
// One persistent CTA per SM streams 128-row tiles of x through a TMA ring
// (as the stage-1 encoders do).  Per tile:
//   compute warps  : stage 1 for their rows (codes + norms, identical to
//                    iq_quantize), x^ = rho T^-1(C[code]) in fp32, the
//                    residual r = x - x^, gamma = ||r||, and r scaled by
//                    256 / max(rho, eps) split into fp16 hi + lo parts written
//                    to the UMMA A tiles (K-major, 128-byte swizzle);
//   MMA warp       : one elected thread issues tcgen05.mma kind::f16,
//                    M = 128, N = m, K = d, twice (hi, lo) into one of two
//                    TMEM accumulators: z = S (r_hi + r_lo) in fp32;
//   compute warps  : (one tile later) tcgen05.ld the accumulator, pack the
//                    sign bits [z >= 0] LSB-first and store them.
// S (m x d fp16, the sketch) stays in shared memory for the whole kernel.
// The GEMM is 2 * 2 d^2 flop per row (d = 128: 65.5 kflop), far below the
// tensor peak; the kernel is bound by the stage-1 arithmetic and HBM.
#pragma once
#include "kernels.cuh"

namespace iq {

template <class T, int D, int BITS, int VAR, bool SETS = false>
struct QGeo {
  using Gm = Geo<T, D, BITS, VAR, 6>;            // stage-1 lane geometry of the code-emitting kernels
#ifndef IQ_QJL_ROTD
#define IQ_QJL_ROTD 1
#endif
#ifndef IQ_QJL_NOWAIT_PROBE
#define IQ_QJL_NOWAIT_PROBE 0   // timing probe only: compute warps do not wait for the A tile (racy)
#endif
#ifndef IQ_QJL_MASKSPLIT
#define IQ_QJL_MASKSPLIT 1   // fp16 hi by mantissa truncation (LOP3) instead of RN + convert back
#endif
#ifndef IQ_QJL_TCWAIT
#define IQ_QJL_TCWAIT 0   // compute-warp waits on tcgen05.commit barriers without a suspend hint
#endif
#ifndef IQ_QJL_PASSES
#define IQ_QJL_PASSES (Q::ROTD ? 3 : 2)   // MMA passes per tile (timing probes override it)
#endif
#ifdef IQ_QJL_NWC
  static constexpr int NWC0 = IQ_QJL_NWC;
#else
  // measured: 16 warps for 16-bit rows at b <= 3 (the rotated-domain
  // residual fits the 96-register cap without spills), 8 at b = 4 and for
  // fp32 (whose inverse-rotation path would spill)
  static constexpr int NWC0 = (sizeof(T) == 2 && BITS <= 3) ? 16 : 8;
#endif
  // compute warps: a multiple of 4 (TMEM lane quadrants), each with at least
  // one row pair per lane group of the 128-row tile
  static constexpr int NWC = NWC0 < 128 / (2 * Gm::VPW) ? NWC0 : 128 / (2 * Gm::VPW);
  static constexpr int CTA_THREADS = 32 * (NWC + 2);   // + TMA producer + MMA warp
  static constexpr int TILE = 128;               // rows per tile = UMMA M
  static constexpr int M = D;                    // sketch rows (m = d, R20)
  static constexpr int ROWB = D * (int)sizeof(T);
  static constexpr int STAGE = TILE * ROWB;      // 32 KB (fp16) / 64 KB (fp32 at d = 128)
  static constexpr int NST = 2;
  // 16-bit rows: residual in the rotated domain, r' = T x - rho C[code]
  // (no inverse rotation), against S' = S M^T as fp16 hi + lo (3 MMA passes)
  // (parameter sets [R31]: the direct form, whose B operand S is the same
  // for every set; S' = S M^T would be per set)
  static constexpr bool ROTD = !SETS && sizeof(T) == 2 && IQ_QJL_ROTD;
  static constexpr int A_BYTES = TILE * D * 2;   // one fp16 operand tile (hi or lo)
  static constexpr int S_BYTES = M * D * 2;
  static constexpr int B_BYTES = ROTD ? 2 * S_BYTES : S_BYTES;   // the B image(s) in shared memory
  static constexpr int A_OFF = NST * STAGE;      // 1024-aligned (STAGE is)
  static constexpr int S_OFF = A_OFF + 2 * A_BYTES;
  static constexpr int BAR_OFF = S_OFF + B_BYTES;
  static constexpr int OPS_OFF = BAR_OFF + 256;   // stage-1 operators (when Gm::OPS_SMEM)
  static constexpr int SMEM = OPS_OFF + Gm::OPS_BYTES + 1024;   // + slack to align the base to 1024
  static constexpr int CW = M / (NWC / 4);        // sketch columns per epilogue warp
  static constexpr int TMEM_COLS = (2 * M) <= 32 ? 32 : (2 * M) <= 64 ? 64 : (2 * M) <= 128 ? 128 : 256;
  static constexpr int U = TILE / (NWC * Gm::VPW);   // rows per lane group per tile
  static_assert(U % 2 == 0, "row pairs");
  static_assert(D == 64 || D == 128, "sketch kernel: d in {64, 128}");
  static_assert(NWC % 4 == 0 && (CW == 16 || CW % 32 == 0), "epilogue split");
};

// ------------------------------------------------------------ tcgen05 helpers
// Shared-memory matrix descriptor, K-major with 128-byte swizzle: start
// address, SBO = 1024 B between 8-row atoms, version 1 (sm_100), layout 2.
__device__ __forceinline__ uint64_t umma_desc_sw128(uint32_t saddr) {
  return (uint64_t)((saddr >> 4) & 0x3FFF) | ((uint64_t)(1024 >> 4) << 32) | ((uint64_t)1 << 46) |
         ((uint64_t)2 << 61);
}
// byte offset of K-step s (16 fp16) inside an operand with `rows` rows
__host__ __device__ constexpr uint32_t umma_kstep_off(int s, int rows) {
  return (uint32_t)((s * 16 / 64) * (rows / 8) * 1024 + (s * 16 % 64) * 2);
}
__device__ __forceinline__ void umma_f16(uint32_t tmem_d, uint64_t da, uint64_t db, uint32_t idesc,
                                         uint32_t accumulate) {
  asm volatile(
      "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem_d),
      "l"(da), "l"(db), "r"(idesc), "r"(accumulate));
}
__device__ __forceinline__ void umma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                   smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void fence_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

// 32 (or 16) consecutive fp32 columns of this thread's TMEM lane -> sign
// word: bit j = [z_j >= 0], taken from the float sign bit (R22; a -0 result
// needs every product to be -0, which the zero row does not produce).
__device__ __forceinline__ uint32_t tmem_sign_word32(uint32_t taddr) {
  uint32_t v[32];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
        "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]),
        "=r"(v[15]), "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]),
        "=r"(v[22]), "=r"(v[23]), "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]),
        "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
  // funnel the sign bits in, one SHF per bit: acc = (acc << 1) | (v_j >> 31)
  // from j = 31 down, so bit j of acc is the sign of column j
  uint32_t neg = 0;
#pragma unroll
  for (int j = 31; j >= 0; --j) neg = __funnelshift_l(v[j], neg, 1);
  return ~neg;
}
__device__ __forceinline__ uint32_t tmem_sign_word16(uint32_t taddr) {
  uint32_t v[16];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
        "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]),
        "=r"(v[15])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
  uint32_t neg = 0;
#pragma unroll
  for (int j = 15; j >= 0; --j) neg = __funnelshift_l(v[j], neg, 1);
  return ~neg & 0xFFFFu;
}

// store fp16 hi / lo of a lane's EPC consecutive coordinates of tile row r
// (coordinates k0 .. k0+EPC-1) into the A operand tiles
template <int EPC>
__device__ __forceinline__ void store_residual(uint8_t* a_hi, uint8_t* a_lo, uint32_t off, const float* rs) {
  uint32_t h[EPC / 2], l[EPC / 2];
#pragma unroll
  for (int e = 0; e < EPC; e += 2) {
#if IQ_QJL_MASKSPLIT
    // hi = r truncated to 11 significant bits (exact in fp16 for |r| >=
    // 2^-14), lo = r - hi exact in fp32 then rounded: r to ~2^-21 relative
    const float h0 = __uint_as_float(__float_as_uint(rs[e]) & 0xFFFFE000u);
    const float h1 = __uint_as_float(__float_as_uint(rs[e + 1]) & 0xFFFFE000u);
    h[e / 2] = pack2<__half>(h0, h1);
    l[e / 2] = pack2<__half>(rs[e] - h0, rs[e + 1] - h1);
#else
    const __half2 hh = __floats2half2_rn(rs[e], rs[e + 1]);
    const float2 hf = __half22float2(hh);
    const __half2 ll = __floats2half2_rn(rs[e] - hf.x, rs[e + 1] - hf.y);
    h[e / 2] = *reinterpret_cast<const uint32_t*>(&hh);
    l[e / 2] = *reinterpret_cast<const uint32_t*>(&ll);
#endif
  }
  if constexpr (EPC == 8) {
    *reinterpret_cast<uint4*>(a_hi + off) = make_uint4(h[0], h[1], h[2], h[3]);
    *reinterpret_cast<uint4*>(a_lo + off) = make_uint4(l[0], l[1], l[2], l[3]);
  } else {
    *reinterpret_cast<uint2*>(a_hi + off) = make_uint2(h[0], h[1]);
    *reinterpret_cast<uint2*>(a_lo + off) = make_uint2(l[0], l[1]);
  }
}

template <class T, int D, int BITS, int VAR, bool SETS = false>
__global__ void __launch_bounds__(QGeo<T, D, BITS, VAR, SETS>::CTA_THREADS, 1)
k_quantize_qjl(const float* __restrict__ mat, const KCodebook cb, int64_t n, const T* x,
               const uint8_t* __restrict__ s_img, uint8_t* __restrict__ codes, float* __restrict__ norms,
               uint8_t* __restrict__ qjl, float* __restrict__ rnorms) {
  using Q = QGeo<T, D, BITS, VAR, SETS>;
  using Gm = typename Q::Gm;
  constexpr int NWC = Q::NWC, TILE = Q::TILE, M = Q::M, U = Q::U, NST = Q::NST;
  constexpr int EPC = Gm::EPC, G = Gm::G, CPL = Gm::CPL, VPW = Gm::VPW;
  constexpr int PW = Gm::PW, NBL = Gm::NBL, EPL = Gm::EPL;
  constexpr int B = Gm::B, W = Gm::W, RB = Gm::RB;
  constexpr bool GRID = BITS >= IQ_GRID_MIN_BITS;

  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024 - (smem_u32(smem_raw) & 1023)) & 1023);   // 1024-aligned base
  uint8_t* a_hi = smem + Q::A_OFF;
  uint8_t* a_lo = a_hi + Q::A_BYTES;
  uint8_t* s_sm = smem + Q::S_OFF;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + Q::BAR_OFF);
  uint64_t* empty = full + NST;
  uint64_t* a_full = empty + NST;      // compute warps -> MMA: A tile written   (NWC arrivals)
  uint64_t* a_free = a_full + 1;       // MMA -> compute warps: A tile consumed  (commit)
  uint64_t* acc_full = a_free + 1;     // [2] MMA -> epilogue                    (commit)
  uint64_t* acc_empty = acc_full + 2;  // [2] epilogue -> MMA                    (NWC arrivals)
  uint64_t* s_bar = acc_empty + 2;     // S image loaded
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(s_bar + 1);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < NST; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], NWC); }
    mbar_init(a_full, NWC);
    mbar_init(a_free, 1);
    for (int b = 0; b < 2; ++b) { mbar_init(&acc_full[b], 1); mbar_init(&acc_empty[b], NWC); }
    mbar_init(s_bar, 1);
    fence_mbar_init();
  }
  if (warp == NWC + 1) {   // TMEM: two fp32 accumulators of M columns
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "n"(Q::TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const int64_t ntiles = (n + TILE - 1) / TILE;

  if (warp == NWC) {  // ------------------------------------------ TMA producer
    if (lane == 0) {
      const uint64_t pol = policy_evict_first();
      mbar_arrive_expect_tx(s_bar, Q::B_BYTES);
      bulk_g2s(s_sm, s_img, Q::B_BYTES, s_bar, policy_evict_last());     // every CTA reads S (S' hi, lo)
      int s = 0;
      uint32_t ph = 0;
      for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
        mbar_wait(&empty[s], ph ^ 1);
        const int64_t v0 = t * TILE;
        const int64_t nv = (n - v0) < TILE ? (n - v0) : TILE;
        const uint32_t bytes = (uint32_t)(nv * Q::ROWB);
        mbar_arrive_expect_tx(&full[s], bytes);
        bulk_g2s(smem + s * Q::STAGE, x + v0 * D, bytes, &full[s], pol);
        if (++s == NST) { s = 0; ph ^= 1; }
      }
    }
  } else if (warp == NWC + 1) {  // ------------------------------------ MMA issuer
    if (lane == 0) {
      // D[128 x M] (+)= A[128 x D] * S[M x D]^T: fp16 inputs, fp32 accumulate
      const uint32_t idesc = (1u << 4) | ((uint32_t)(M >> 3) << 17) | ((uint32_t)(TILE >> 4) << 24);
      const uint32_t ah = smem_u32(a_hi), al = smem_u32(a_lo), sb = smem_u32(s_sm);
      mbar_wait_tc(s_bar, 0);
      uint32_t j = 0;
      for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x, ++j) {
        const uint32_t b = j & 1;
        mbar_wait_tc(a_full, j & 1);
        mbar_wait_tc(&acc_empty[b], ((j >> 1) & 1) ^ 1);
        tc_fence_after();
        const uint32_t td = tmem + b * M;
        // A_hi B_hi + A_lo B_hi (+ A_hi B_lo with S' split in two)
#pragma unroll
        for (int part = 0; part < IQ_QJL_PASSES; ++part) {
          const uint32_t pa = part == 1 ? al : ah, pb = sb + (part == 2 ? Q::S_BYTES : 0);
#pragma unroll
          for (int s = 0; s < D / 16; ++s)
            umma_f16(td, umma_desc_sw128(pa + umma_kstep_off(s, TILE)), umma_desc_sw128(pb + umma_kstep_off(s, M)),
                     idesc, (part | s) != 0);
        }
        umma_commit(a_free);
        umma_commit(&acc_full[b]);
      }
    }
  } else {  // --------------------------------------------------------- compute warps
    const int sub = lane & (G - 1);
    const int vbase = lane & ~(G - 1);
    const int vslot = lane / G;
    float P[Gm::OPS_SMEM ? 1 : NBL][PW * PW];
    uint8_t* const ops = smem + Q::OPS_OFF;
    if constexpr (Gm::OPS_SMEM) {
      if (warp == 0 && lane < G) {
        float Pl[NBL][PW * PW];
        load_ops<Gm>(mat, sub, Pl);
        store_ops_smem<Gm>(ops, sub, Pl);
      }
      asm volatile("bar.sync 1, %0;" ::"r"(NWC * 32) : "memory");   // compute warps only
    } else {
      load_ops<Gm>(mat, sub, P);
    }
    const float ctab = cb.cent[lane & ((1 << BITS) - 1)];
    const float gtab = cb.gtab[lane];
    const float gval = cb.gval[lane];
    const uint32_t gcode = cb.gcode[lane];
    const int quad = warp & 3, part = warp >> 2;      // TMEM lane quadrant, column slice
    constexpr int CW = Q::CW;                         // columns per epilogue warp

    auto epilogue = [&](uint32_t jj, int64_t tt) {
      const uint32_t b = jj & 1;
#if IQ_QJL_TCWAIT
      mbar_wait_tc(&acc_full[b], (jj >> 1) & 1);        // completed by tcgen05.commit: no suspend hint
#else
      mbar_wait(&acc_full[b], (jj >> 1) & 1);           // suspend-hint wait (compute warps)
#endif
      tc_fence_after();
      const int row = 32 * quad + lane;
      const int64_t v = tt * TILE + row;
      const uint32_t ta = tmem + ((uint32_t)(32 * quad) << 16) + b * M + part * CW;
      uint32_t w[CW >= 32 ? CW / 32 : 1];
      if constexpr (CW == 16) {
        w[0] = tmem_sign_word16(ta);
      } else {
#pragma unroll
        for (int c = 0; c < CW / 32; ++c) w[c] = tmem_sign_word32(ta + 32 * c);
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&acc_empty[b]);
      if (v < n) {
        uint8_t* dst = qjl + v * (M / 8) + part * (CW / 8);
        if constexpr (CW == 16) *reinterpret_cast<uint16_t*>(dst) = (uint16_t)w[0];
        else if constexpr (CW == 32) *reinterpret_cast<uint32_t*>(dst) = w[0];
        else *reinterpret_cast<uint2*>(dst) = make_uint2(w[0], w[1]);
      }
    };

    int s = 0;
    uint32_t ph = 0, j = 0;
    int64_t tprev = -1;
    int cur_set = 0;                                   // operators of set 0 are loaded
    for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x, ++j) {
      // parameter sets [R31]: this tile's operators (tiles never straddle sets)
      if constexpr (SETS) switch_ops<Gm, NWC>(mat, cb, t * TILE, cur_set, sub, warp, lane, ops, P);
      mbar_wait_warp(&full[s], ph, lane);
      const uint8_t* st = smem + s * Q::STAGE;
      const int ss_ = s;
      if (++s == NST) { s = 0; ph ^= 1; }
      const int64_t v0 = t * TILE;
      const int nv = (n - v0) < TILE ? (int)(n - v0) : TILE;
      uint8_t* const ct = codes + v0 * RB;
      float* const nt = norms + v0;
      float* const gt = rnorms + v0;
#pragma unroll 1
      for (int u = 0; u < U; u += 2) {
        uint4 ra[CPL], rb[CPL];
        const int vl = (warp * U + u) * VPW + vslot;   // tile row of .x; .y is vl + VPW
#pragma unroll
        for (int i = 0; i < CPL; ++i) {
          ra[i] = lds128(st + vl * Q::ROWB + (sub + i * G) * 16);
          rb[i] = lds128(st + (vl + VPW) * Q::ROWB + (sub + i * G) * 16);
        }
        const bool oka = vl < nv, okb = vl + VPW < nv;
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
        const float2 rho = f2(sqrt_ftz(ss.x), sqrt_ftz(ss.y));
        const float2 rinv = f2(rsqrt_ftz(fmaxf(ss.x, 1e-24f)), rsqrt_ftz(fmaxf(ss.y, 1e-24f)));   // 1/max(rho, eps)
        const float2 nrho = f2(-rho.x, -rho.y);

        // ---- stage 1: codes (the iq_quantize rule) and x^ in fp32
        float2 out[EPL];
        uint32_t cwa[CPL], cwb[CPL];
#pragma unroll
        for (int i = 0; i < CPL; ++i) cwa[i] = cwb[i] = 0u;
        if constexpr (GRID) {
          const float2 sc = mul2(rinv, bc(cb.gscale));
#pragma unroll
          for (int b = 0; b < NBL; ++b) {
            float2 yb[PW], cq[PW];
            float Mb[PW * PW];
            fetch_op<Gm>(P, ops, sub, b, Mb);
            rot_fwd<PW>(Mb, v + b * PW, yb);              // T x (unnormalised)
#pragma unroll
            for (int jv = 0; jv < PW; ++jv) {
              const uint32_t ia = grid_index(yb[jv].x, sc.x, gtab, cb.gclamp);
              const uint32_t ib = grid_index(yb[jv].y, sc.y, gtab, cb.gclamp);
              const int e = (b * PW + jv) % EPC, c = (b * PW + jv) / EPC;
              cwa[c] |= grid_code<BITS>(ia, yb[jv].x, gcode) << (e * BITS);
              cwb[c] |= grid_code<BITS>(ib, yb[jv].y, gcode) << (e * BITS);
              cq[jv] = f2(grid_value(ia, yb[jv].x, gval), grid_value(ib, yb[jv].y, gval));
            }
            if constexpr (Q::ROTD) {                   // r' = T x - rho c
#pragma unroll
              for (int jv = 0; jv < PW; ++jv) out[b * PW + jv] = fma2(cq[jv], nrho, yb[jv]);
            } else {
              rot_inv<PW>(Mb, cq, out + b * PW);        // T^-1(C[code]); rho applied with r below
            }
          }
        } else {
          RowQ<BITS> q;
          make_rowq<BITS, false>(q, rho, cb);
          constexpr int BPCH = EPC / PW;
#pragma unroll
          for (int i = 0; i < CPL; ++i) {
            float2 yb[EPC], cq[EPC];
            float Mc[BPCH][PW * PW];
#pragma unroll
            for (int bb = 0; bb < BPCH; ++bb) {
              fetch_op<Gm>(P, ops, sub, i * BPCH + bb, Mc[bb]);
              rot_fwd<PW>(Mc[bb], v + i * EPC + bb * PW, yb + bb * PW);
            }
            encode_chunk<BITS, EPC>(yb, q, cwa[i], cwb[i]);
#pragma unroll
            for (int e = 0; e < EPC; ++e)
              cq[e] = f2(__shfl_sync(kFull, ctab, (int)(cwa[i] >> (e * BITS)), 1 << BITS),
                         __shfl_sync(kFull, ctab, (int)(cwb[i] >> (e * BITS)), 1 << BITS));
            if constexpr (Q::ROTD) {                     // r' = T x - rho c
#pragma unroll
              for (int e = 0; e < EPC; ++e) out[i * EPC + e] = fma2(cq[e], nrho, yb[e]);
            } else {
#pragma unroll
              for (int bb = 0; bb < BPCH; ++bb) rot_inv<PW>(Mc[bb], cq + bb * PW, out + i * EPC + bb * PW);
            }
          }
        }
        // codes + norms (bit-identical to iq_quantize)
#pragma unroll
        for (int i = 0; i < CPL; ++i) {
          if constexpr (IQ_BYTE_CODES && B % 8 == 0) {   // whole bytes: stored in place (k_encode)
            uint8_t* const pa = ct + vl * RB + (sub + i * G) * (B / 8);
            store_piece<B>(pa, cwa[i], (sub + i * G) & 1, oka);
            store_piece<B>(pa + VPW * RB, cwb[i], (sub + i * G) & 1, okb);
          } else {
            const uint32_t wa = gather_word<G, B>(cwa[i], sub, vbase);
            const uint32_t wb = gather_word<G, B>(cwb[i], sub, vbase);
            if (sub < W) {
              const int off = vl * RB + 4 * (i * W + sub);
              if (oka) *reinterpret_cast<uint32_t*>(ct + off) = wa;
              if (okb) *reinterpret_cast<uint32_t*>(ct + off + VPW * RB) = wb;
            }
          }
        }
        // ---- residual r = x - rho T^-1(C[code]) (R21) -- or r' = T r in the
        // rotated domain (ROTD); gamma = ||r|| = ||r'|| (R23)
        float2 g2 = bc(0.0f);
#pragma unroll
        for (int e = 0; e < EPL; ++e) {
          if constexpr (!Q::ROTD) out[e] = fma2(out[e], nrho, v[e]);
          g2 = fma2(out[e], out[e], g2);
        }
#pragma unroll
        for (int o = G / 2; o >= 1; o >>= 1)
          g2 = add2(g2, f2(__shfl_xor_sync(kFull, g2.x, o), __shfl_xor_sync(kFull, g2.y, o)));
        if (sub == 0) {
          if (oka) { nt[vl] = rho.x; gt[vl] = sqrt_ftz(g2.x); }
          if (okb) { nt[vl + VPW] = rho.y; gt[vl + VPW] = sqrt_ftz(g2.y); }
        }
        // ---- UMMA A operand: r * 256 / max(rho, eps) as fp16 hi + lo (sign(S r) is scale-free)
        const float2 sr = mul2(rinv, bc(256.0f));
        // the previous tile's MMAs must have consumed the A tiles (the
        // stage-1 work above overlaps them)
#if !IQ_QJL_NOWAIT_PROBE
#if IQ_QJL_TCWAIT
        if (u == 0) mbar_wait_tc(a_free, (j & 1) ^ 1);
#else
        if (u == 0) mbar_wait(a_free, (j & 1) ^ 1);
#endif
#endif
#pragma unroll
        for (int i = 0; i < CPL; ++i) {
          float ta[EPC], tb[EPC];
#pragma unroll
          for (int e = 0; e < EPC; ++e) {
            const float2 t2 = mul2(out[i * EPC + e], sr);
            ta[e] = t2.x;
            tb[e] = t2.y;
          }
          // (the offsets depend only on the lane and u: the compiler hoists them)
          const int k0 = (sub + i * G) * EPC;
          store_residual<EPC>(a_hi, a_lo, umma_sw128_off(vl, k0, 128), ta);
          store_residual<EPC>(a_hi, a_lo, umma_sw128_off(vl + VPW, k0, 128), tb);
        }
      }
      fence_async_smem();          // generic-proxy A writes -> tensor-core (async proxy) reads
      __syncwarp();
      if (lane == 0) mbar_arrive(a_full);
      if (tprev >= 0) epilogue(j - 1, tprev);
      tprev = t;
    }
    if (tprev >= 0) epilogue(j - 1, tprev);
  }
  tc_fence_before();
  __syncthreads();
  if (warp == NWC + 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(Q::TMEM_COLS));
  }
}

}  // namespace iq
