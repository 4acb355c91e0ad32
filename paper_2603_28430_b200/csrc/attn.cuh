// Fused KV-cache decode consumer (NEXT row 2 of SURVEY section 8(f);
// PAPER.md:460 "attention-logit preservation and inner-product error under
// the complete two-stage pipeline", "specialized kernels for fused
// KV-cache compression during autoregressive decoding").  DESIGN.md R25-R27.
//
// Attention logits straight from the packed cache, for H independent heads
// (one parameter handle, R13) of n_keys keys each and up to 16 queries per
// head (a GQA group or a batch of decode steps):
//   s[h][j][k] = <q_hj, x^_hk> = rho_hk <T q_hj, C[code_hk]>        (T orthogonal)
//              + sqrt(pi/2)/m gamma_hk <S q_hj, sign_hk>            (stage 2, optional)
// so no key is ever inverse-rotated: the queries are rotated once per head
// and the keys only decoded.  Warp roles of the persistent CTA (one per SM,
// each owning a contiguous range of 128-key tiles):
//   TMA producer (1 lane) : codes, norms (+ sketch bits, gammas) of a tile
//                           into a deep ring of small stages;
//   16 decoder warps      : C[code] as fp16 (width-L shuffle table) and +-1
//                           fp16 from the sketch bits (width-4 shuffle table
//                           of half2 pairs) into K-major 128B-swizzled UMMA A
//                           tiles (double-buffered), plus a per-buffer side
//                           table (rho, gamma, the head's query scales);
//   MMA issuer (1 lane)   : tcgen05.mma kind::f16, M = 128 keys, N = 16 query
//                           slots, K = d, into TMEM (stage-1 and stage-2
//                           accumulators, double-buffered);
//   4 epilogue warps      : tcgen05.ld (thread = key), scale, store
//                           s[h][j][k] (coalesced in k).
// At a head change the decoders drain the MMAs, rotate the new queries on
// the CUDA cores (T q: 16 FMA per block) and compute S q on the tensor cores
// (S staged through the drained A buffers).
#pragma once
#include "qjl.cuh"

namespace iq {

template <int D, int BITS>
struct AGeo {
  static constexpr int NQ = 16;                  // query slots (UMMA N)
  static constexpr int TILE = 128;               // keys per tile (UMMA M)
  static constexpr int RB = D * BITS / 8;        // code bytes per key
  // K-split: the A operand of a tile is built and consumed in chunks of KCH
  // coordinates (one 128 x KCH fp16 K-major operand each, accumulated into
  // one TMEM accumulator), so d = 256 / 512 keys fit the same buffers
  static constexpr int KCH = D < 128 ? D : 128;
  static constexpr int KC = D / KCH;             // chunks per tile
  // stage-2 term: d <= 128, and d = 256 at b <= 3 (the widest key tiles and
  // pair tables leave no shared memory for the sketch operands beyond that)
  static constexpr bool ST2OK = D <= 128 || (D == 256 && BITS <= 3);
  static constexpr int NPART = ST2OK ? 2 : 1;    // A parts per buffer: stage 1 [, stage 2]
  static constexpr int QB = ST2OK ? D / 8 : 0;   // sketch bytes per key
  // ring stage: codes [TILE][RB] | norms [TILE] | sketch [TILE][QB] | gammas [TILE]
  static constexpr int C_OFF = 0;
  static constexpr int N_OFF = (TILE * RB + 15) / 16 * 16;
  static constexpr int Q_OFF = N_OFF + TILE * 4;
  static constexpr int G_OFF = Q_OFF + TILE * QB;
  static constexpr int STAGE = (G_OFF + (ST2OK ? TILE * 4 : 0) + 127) / 128 * 128;
  static constexpr int A_BYTES = TILE * KCH * 2; // one fp16 A operand chunk
  static constexpr int B_BYTES = NQ * D * 2;     // one fp16 B tile (queries, all of K)
  static constexpr int MT = D <= 128 ? 1 : D / 128;   // 128-row tiles of S (m = d sketch rows)
  static constexpr int S_TILE = 128 * D * 2;     // one of them as an A operand (rows >= m zero)
  static constexpr int S_BYTES = MT * S_TILE;    // all of S, staged in the drained A buffers
  static constexpr int A_OFF = 0;                // [2 buffers][NPART]
  static constexpr int B_OFF = A_OFF + 2 * NPART * A_BYTES;
  static constexpr int QT_OFF = B_OFF + NPART * B_BYTES;   // sigma q as fp16 [NQ][D] (B of the S q MMA)
  static constexpr int NACC = 4;                 // accumulator / side-table buffers (TMEM is cheap)
  static constexpr int SIDE_OFF = QT_OFF + (ST2OK ? B_BYTES : 0);   // per accumulator: rho[128], gamma[128], scales[2][16]
  static constexpr int SIDE_BYTES = (2 * TILE + 2 * NQ) * 4;
  static constexpr int QS_OFF = SIDE_OFF + NACC * SIDE_BYTES;   // the current head's scales [2][16]
  // lookup tables replicated across the 32 banks (entry e of lane l at
  // e * stride + 4 l, so every lane reads its own bank): a code PAIR -> half2
  // (C[c0], C[c1]), and 4 sketch bits -> 4 halves of +-1 (two words)
  static constexpr int PAIRS = 1 << (2 * BITS);
  static constexpr int PT_OFF = QS_OFF + 2 * NQ * 4;
  static constexpr int ST_OFF = PT_OFF + PAIRS * 128;
  static constexpr int BAR_OFF = ST_OFF + (ST2OK ? 16 * 256 : 0);
  static constexpr int RING_OFF = (BAR_OFF + 512 + 127) / 128 * 128;
  static constexpr int RING_MAX = 227 * 1024 - RING_OFF - 1024;
  static constexpr int NST = (RING_MAX / STAGE) < 16 ? (RING_MAX / STAGE) : 16;
  static constexpr int SMEM = RING_OFF + NST * STAGE + 1024;
#ifndef IQ_ATTN_NWD
#define IQ_ATTN_NWD 16
#endif
  // decoder warps: 8 at d = 64 (24 % faster there: 367 -> 278 us for 256 x
  // 32768 keys), 16 otherwise (8 or 12 are slower at d >= 128; measured)
  static constexpr int NWD = D <= 64 ? 8 : IQ_ATTN_NWD;
  static constexpr int NWE = 4;                  // epilogue warps (one per TMEM lane quadrant)
  static constexpr int W_PROD = NWD + NWE, W_MMA = NWD + NWE + 1;
  static constexpr int CTA_THREADS = 32 * (NWD + NWE + 2);
  static constexpr int CGROUPS = KCH / 32;       // 32-coordinate groups per key and chunk
  static constexpr int TMEM_COLS = 256;          // [NACC][stage 1, stage 2] x NQ, + MT NQ for S q
  static constexpr int SQ_COL = 2 * NACC * NQ;
  static_assert(D == 64 || D == 128 || D == 256 || D == 512, "attention consumer: d in {64, 128, 256, 512}");
  static_assert(NST >= 3, "ring too shallow");
  static_assert(!ST2OK || S_BYTES <= 4 * A_BYTES, "S staging");
  static_assert(SQ_COL + MT * NQ <= TMEM_COLS, "TMEM");
};

__device__ __forceinline__ void tmem_ld16(uint32_t taddr, uint32_t (&v)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
        "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]),
        "=r"(v[15])
      : "r"(taddr));
}

template <class TQ, int D, int BITS, int VAR>
__global__ void __launch_bounds__(AGeo<D, BITS>::CTA_THREADS, 1)
k_attn_scores(const float* __restrict__ mat, const KCodebook cb, int heads, int64_t n_keys,
              const uint8_t* __restrict__ codes, const float* __restrict__ norms,
              const uint8_t* __restrict__ sketch, const float* __restrict__ gammas,
              const uint8_t* __restrict__ s_img, int n_q, const TQ* __restrict__ q, float* __restrict__ scores) {
  using A = AGeo<D, BITS>;
  constexpr int TILE = A::TILE, NQ = A::NQ, NWD = A::NWD, NST = A::NST, RB = A::RB, QB = A::QB;
  constexpr int KC = A::KC, KCH = A::KCH, NPART = A::NPART, CGROUPS = A::CGROUPS;
  constexpr int PW = (VAR == IQ_VARIANT_PLANAR2D) ? 2 : 4;
  constexpr int L = 1 << BITS;
  const bool st2 = A::ST2OK && sketch != nullptr;

  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024 - (smem_u32(smem_raw) & 1023)) & 1023);
  uint8_t* a_base = smem + A::A_OFF;            // A[buf][part] at a_base + (NPART buf + part) A_BYTES
  uint8_t* b_base = smem + A::B_OFF;            // B[part]
  float* qs = reinterpret_cast<float*>(smem + A::QS_OFF);   // [2][NQ]: 1/sigma_j, 8/sigma_j
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + A::BAR_OFF);
  uint64_t* empty = full + NST;
  uint64_t* a_full = empty + NST;      // [4] decoders -> MMA
  uint64_t* a_free = a_full + 4;       // [4] MMA -> decoders (A buffer consumed)
  uint64_t* acc_full = a_free + 4;     // [NACC] MMA -> epilogue
  uint64_t* acc_empty = acc_full + A::NACC;   // [NACC] epilogue -> MMA, decoders (accumulator, side table free)
  uint64_t* side_full = acc_empty + A::NACC;  // [NACC] decoders -> epilogue: side table written
  uint64_t* s_bar = side_full + A::NACC;      // S image staged (per head change)
  uint64_t* sq_bar = s_bar + 1;        // S q MMA done
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(sq_bar + 1);
  uint8_t* ring = smem + A::RING_OFF;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < NST; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], NWD); }
    for (int b = 0; b < 4; ++b) { mbar_init(&a_full[b], NWD); mbar_init(&a_free[b], 1); }
    for (int c = 0; c < A::NACC; ++c) {
      mbar_init(&acc_full[c], 1); mbar_init(&acc_empty[c], A::NWE);
      mbar_init(&side_full[c], (2 * TILE) / 32);   // the warps that write rho / gamma / scales
    }
    mbar_init(s_bar, 1);
    mbar_init(sq_bar, 1);
    fence_mbar_init();
  }
  if (warp == A::W_MMA) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "n"(A::TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const int64_t tph = (n_keys + TILE - 1) / TILE;   // tiles per head
  const int64_t ntiles = tph * heads;
  // each CTA takes a contiguous range of tiles, so it changes heads (and
  // re-prepares its queries) about once, not on every tile
  const int64_t per_cta = (ntiles + gridDim.x - 1) / gridDim.x;
  const int64_t t_begin = blockIdx.x * per_cta;
  const int64_t t_end = (t_begin + per_cta) < ntiles ? (t_begin + per_cta) : ntiles;
  // A operand buffers in flight: without the stage-2 term its part of each
  // double buffer is free, so stage 1 runs four single-part buffers deep
  // (more decoded tiles queued ahead of the tensor pipe's completion latency)
  const uint32_t nab = (A::ST2OK && !st2) ? 2u * NPART : 2u;
  const uint32_t a_stride = (A::ST2OK && !st2) ? (uint32_t)A::A_BYTES : (uint32_t)(NPART * A::A_BYTES);

  if (warp == A::W_PROD) {  // ---------------------------------------- TMA producer
    if (lane == 0) {
      const uint64_t pol = policy_evict_first();
      int s = 0;
      uint32_t ph = 0;
      int64_t h = t_begin / tph, k0 = (t_begin - h * tph) * TILE;   // advanced incrementally
      for (int64_t t = t_begin; t < t_end; ++t, k0 += TILE) {
        if (k0 >= n_keys) { k0 = 0; ++h; }
        mbar_wait(&empty[s], ph ^ 1);
        const int64_t nk = (n_keys - k0) < TILE ? (n_keys - k0) : TILE;
        const int64_t row0 = h * n_keys + k0;
        // whole 16-byte units; a ragged remainder is read from global memory
        const uint32_t cb16 = (uint32_t)(nk * RB) & ~15u, nb16 = (uint32_t)(nk * 4) & ~15u;
        const uint32_t qb16 = st2 ? ((uint32_t)(nk * QB) & ~15u) : 0u, gb16 = st2 ? nb16 : 0u;
        const uint32_t tot = cb16 + nb16 + qb16 + gb16;
        uint8_t* stg = ring + s * A::STAGE;
        if (tot == 0) {
          mbar_arrive(&full[s]);
        } else {
          mbar_arrive_expect_tx(&full[s], tot);
          if (cb16) bulk_g2s(stg + A::C_OFF, codes + row0 * RB, cb16, &full[s], pol);
          if (nb16) bulk_g2s(stg + A::N_OFF, norms + row0, nb16, &full[s], pol);
          if (qb16) bulk_g2s(stg + A::Q_OFF, sketch + row0 * QB, qb16, &full[s], pol);
          if (gb16) bulk_g2s(stg + A::G_OFF, gammas + row0, gb16, &full[s], pol);
        }
        if (++s == NST) { s = 0; ph ^= 1; }
      }
    }
  } else if (warp == A::W_MMA) {  // ------------------------------------------ MMA issuer
    if (lane == 0) {
      const uint32_t idesc = (1u << 4) | ((uint32_t)(NQ >> 3) << 17) | ((uint32_t)(TILE >> 4) << 24);
      const uint32_t ab = smem_u32(a_base), bb = smem_u32(b_base);
      uint32_t j = 0, jj = 0;                    // tiles, A-operand chunks
      for (int64_t t = t_begin; t < t_end; ++t, ++j) {
        const uint32_t c = j % A::NACC, u = j / A::NACC;
        mbar_wait_tc(&acc_empty[c], (u & 1) ^ 1);
#pragma unroll 1
        for (int kc = 0; kc < KC; ++kc, ++jj) {
          const uint32_t b = jj % nab;
          mbar_wait_tc(&a_full[b], (jj / nab) & 1);
          tc_fence_after();
#pragma unroll 1
          for (int part = 0; part < (st2 ? 2 : 1); ++part) {
            const uint32_t ta = ab + b * a_stride + part * A::A_BYTES, tb = bb + part * A::B_BYTES;
            const uint32_t td = tmem + (2 * c + part) * NQ;
#pragma unroll
            for (int s = 0; s < KCH / 16; ++s)
              umma_f16(td, umma_desc_sw128(ta + umma_kstep_off(s, TILE)),
                       umma_desc_sw128(tb + umma_kstep_off(kc * (KCH / 16) + s, NQ)), idesc, (kc | s) != 0);
          }
          umma_commit(&a_free[b]);
        }
        umma_commit(&acc_full[c]);
      }
    }
  } else if (warp >= NWD) {  // --------------------------------------------- epilogue
    const int quad = warp & 3;                   // TMEM lane quadrant (warp id % 4)
    const int row = 32 * quad + lane;
    const float cpi = 1.2533141373155003f / (float)D;   // sqrt(pi/2) / m, m = d (R20)
    uint32_t j = 0;
    int64_t h = t_begin / tph, k0 = (t_begin - h * tph) * TILE;
    for (int64_t t = t_begin; t < t_end; ++t, ++j, k0 += TILE) {
      if (k0 >= n_keys) { k0 = 0; ++h; }
      const uint32_t c = j % A::NACC, u = j / A::NACC;
      mbar_wait(&acc_full[c], u & 1);            // suspend-hint wait: the epilogue is off the critical path
      tc_fence_after();
      uint32_t v1[16], v2[16];
      const uint32_t ta = tmem + ((uint32_t)(32 * quad) << 16);
      tmem_ld16(ta + (2 * c) * NQ, v1);
      if (st2) tmem_ld16(ta + (2 * c + 1) * NQ, v2);
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
      tc_fence_before();
      mbar_wait(&side_full[c], u & 1);            // ordinary release/acquire for the side table
      const float* side = reinterpret_cast<const float*>(smem + A::SIDE_OFF + c * A::SIDE_BYTES);
      const int64_t k = k0 + row;
      if (k < n_keys) {
        const float rho = side[row], gam = side[TILE + row], cg = cpi * gam;
        float* out = scores + h * (int64_t)n_q * n_keys + k;
        // query slots in groups of four; n_q is uniform, so the early exit
        // leaves no per-slot branches
#pragma unroll
        for (int g4 = 0; g4 < NQ / 4; ++g4) {
          if (4 * g4 >= n_q) break;
#pragma unroll
          for (int c4 = 0; c4 < 4; ++c4) {
            const int jq = 4 * g4 + c4;
            float sv = __uint_as_float(v1[jq]) * side[2 * TILE + jq] * rho;
            if (st2) sv = fmaf(__uint_as_float(v2[jq]) * side[2 * TILE + NQ + jq], cg, sv);
            if (jq < n_q) __stcs(out, sv);
            out += n_keys;
          }
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&acc_empty[c]);   // accumulator and side table c are free
    }
  } else {  // ------------------------------------------------------------- decoders
    // build the replicated lookup tables (once per CTA)
    for (int e = threadIdx.x; e < A::PAIRS * 32; e += NWD * 32) {
      const int pr = e >> 5, l = e & 31;
      const __half2 hv = __floats2half2_rn(cb.cent[pr & (L - 1)], cb.cent[pr >> BITS]);
      *reinterpret_cast<__half2*>(smem + A::PT_OFF + pr * 128 + 4 * l) = hv;
    }
    for (int e = threadIdx.x; A::ST2OK && e < 16 * 32; e += NWD * 32) {   // bit set = +1 (R22); stage 2 only
      const int nib = e >> 5, l = e & 31;
      uint32_t w[2];
#pragma unroll
      for (int k = 0; k < 2; ++k)
        w[k] = ((nib >> (2 * k)) & 1 ? 0x3C00u : 0xBC00u) | ((nib >> (2 * k + 1)) & 1 ? 0x3C000000u : 0xBC000000u);
      *reinterpret_cast<uint2*>(smem + A::ST_OFF + nib * 256 + 8 * l) = make_uint2(w[0], w[1]);
    }
    asm volatile("bar.sync 1, %0;" ::"r"(NWD * 32) : "memory");
    // table address = (index * stride | lane offset) + base: the OR needs the
    // lane offset below the stride; the (warp-uniform) base is added after
    const uint32_t pt_base = smem_u32(smem + A::PT_OFF), st_base = smem_u32(smem + A::ST_OFF);
    const uint32_t pt_lane = 4 * lane, st_lane = 8 * lane;
    uint32_t nprep = 0;                          // query preparations so far (s_bar / sq_bar parity)

    // rotate the head's queries into the B tiles: q' = T q (stage 1) and
    // S q (stage 2), fp16 with per-query power-of-two scales
    auto load_queries = [&](int64_t h) {
      const TQ* qh = q + h * (int64_t)n_q * D;
      const float* mset = mat + (size_t)(h % cb.n_sets) * cb.set_stride;   // the head's set [R31]
      if (A::ST2OK && st2 && threadIdx.x == 0) {   // stage S in the drained A buffers
        mbar_arrive_expect_tx(s_bar, A::S_BYTES);
        bulk_g2s(a_base, s_img, A::S_BYTES, s_bar, policy_evict_last());
      }
      // per-query norms: warp w sums query w (lanes stride d)
      for (int jq = warp; jq < NQ; jq += NWD) {
        float ss = 0.0f;
        if (jq < n_q)
          for (int i = lane; i < D; i += 32) { const float v = (float)qh[jq * D + i]; ss = fmaf(v, v, ss); }
#pragma unroll
        for (int o = 16; o >= 1; o >>= 1) ss += __shfl_xor_sync(kFull, ss, o);
        if (lane == 0) {
          // sigma = 2^(8 - ceil(log2 ||q||)): |T q| <= ||q|| -> |sigma T q| <= 256;
          // the stage-2 tile holds S sigma q / 8 (|.| <~ 4 sqrt(d) 256 / 8)
          int e = 0;
          frexpf(sqrtf(ss), &e);
          qs[jq] = ldexpf(1.0f, e - 8);                 // 1 / sigma
          qs[NQ + jq] = ldexpf(1.0f, e - 5);            // 8 / sigma
        }
      }
      asm volatile("bar.sync 1, %0;" ::"r"(NWD * 32) : "memory");
      // stage 1: thread handles (query jq, block b)
      for (int w = threadIdx.x; w < NQ * (D / PW); w += NWD * 32) {
        const int jq = w / (D / PW), b = w % (D / PW);
        float xv[PW], yv[PW];
        const float sg = 1.0f / qs[jq];
#pragma unroll
        for (int c = 0; c < PW; ++c) xv[c] = jq < n_q ? (float)qh[jq * D + b * PW + c] * sg : 0.0f;
#pragma unroll
        for (int r = 0; r < PW; ++r) {
          float a = 0.0f;
#pragma unroll
          for (int c = 0; c < PW; ++c) a = fmaf(__ldg(mset + (size_t)b * PW * PW + r * PW + c), xv[c], a);
          yv[r] = a;
        }
#pragma unroll
        for (int r = 0; r < PW; ++r)
          *reinterpret_cast<__half*>(b_base + umma_sw128_off(jq, b * PW + r, NQ)) = __float2half_rn(yv[r]);
      }
      if (A::ST2OK && st2) {
        // stage 2: S q on the tensor cores.  B = sigma q as fp16 (queries x d),
        // A = S (128 x d, rows >= m zero), D = S (sigma q)^T in TMEM; thread i
        // of warps 0..3 then holds (S sigma q_j)_i for the 16 query slots and
        // writes (S sigma q_j)_i / 8 into the stage-2 B tile (row j, column i)
        for (int w = threadIdx.x; w < NQ * D; w += NWD * 32) {
          const int jq = w / D, k = w % D;
          const float v = jq < n_q ? (float)qh[jq * D + k] / qs[jq] : 0.0f;
          *reinterpret_cast<__half*>(smem + A::QT_OFF + umma_sw128_off(jq, k, NQ)) = __float2half_rn(v);
        }
        fence_async_smem();
        asm volatile("bar.sync 1, %0;" ::"r"(NWD * 32) : "memory");
        if (threadIdx.x == 0) {
          mbar_wait_tc(s_bar, nprep & 1);
          tc_fence_after();
          const uint32_t idesc = (1u << 4) | ((uint32_t)(NQ >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
          const uint32_t sa = smem_u32(a_base), qb = smem_u32(smem + A::QT_OFF);
#pragma unroll
          for (int mt = 0; mt < A::MT; ++mt)           // sketch rows 128 mt .. 128 mt + 127
#pragma unroll
            for (int s = 0; s < D / 16; ++s)
              umma_f16(tmem + A::SQ_COL + mt * NQ, umma_desc_sw128(sa + mt * A::S_TILE + umma_kstep_off(s, 128)),
                       umma_desc_sw128(qb + umma_kstep_off(s, NQ)), idesc, s != 0);
          umma_commit(sq_bar);
        }
        mbar_wait_tc(sq_bar, nprep & 1);
        tc_fence_after();
        if (warp < 4) {
#pragma unroll 1
          for (int mt = 0; mt < A::MT; ++mt) {
            uint32_t v[16];
            tmem_ld16(tmem + ((uint32_t)(32 * warp) << 16) + A::SQ_COL + mt * NQ, v);
            asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
            const int i = 128 * mt + 32 * warp + lane;
            if (i < D) {
#pragma unroll
              for (int jq = 0; jq < NQ; ++jq)
                *reinterpret_cast<__half*>(b_base + A::B_BYTES + umma_sw128_off(jq, i, NQ)) =
                    __float2half_rn(__uint_as_float(v[jq]) * 0.125f);
            }
          }
        }
        tc_fence_before();
      }
      ++nprep;
      fence_async_smem();
      asm volatile("bar.sync 1, %0;" ::"r"(NWD * 32) : "memory");   // B tiles, qs and the A buffers ready
    };

    __builtin_assume(threadIdx.x < NWD * 32);
    // per-thread constants of the decode mapping (thread g -> key g / CGROUPS,
    // 32-coordinate group g % CGROUPS of every chunk): stage word offsets
    // (chunk 0), A-operand chunk offsets
    constexpr int NG = (TILE * CGROUPS + NWD * 32 - 1) / (NWD * 32);   // groups per thread and chunk
    uint32_t coff[NG], qoff[NG], aoff[NG][4];
#pragma unroll
    for (int gi = 0; gi < NG; ++gi) {
      const int g = threadIdx.x + gi * NWD * 32;
      const int gr = g / CGROUPS, gs = g % CGROUPS;
      coff[gi] = (uint32_t)(gr * RB + gs * BITS * 4);
      qoff[gi] = (uint32_t)(gr * A::QB + gs * 4);
#pragma unroll
      for (int c8 = 0; c8 < 4; ++c8) aoff[gi][c8] = umma_sw128_off(gr, gs * 32 + c8 * 8, TILE);
    }
    int s = 0;
    uint32_t ph = 0, j = 0, jj = 0;
    int64_t hcur = -1;
    float qs_mine = 0.0f;                        // qs[threadIdx.x] of the current head (threads < 2 NQ)
    int64_t h = t_begin / tph, k0 = (t_begin - h * tph) * TILE;
    for (int64_t t = t_begin; t < t_end; ++t, ++j, k0 += TILE) {
      if (k0 >= n_keys) { k0 = 0; ++h; }
      if (h != hcur) {
        // drain: the last MMA issued (chunk jj - 1) completes after every
        // earlier one, so the B tiles and both A buffers are free
        if (jj > 0) mbar_wait_tc(&a_free[(jj - 1) % nab], ((jj - 1) / nab) & 1);
        load_queries(h);
        hcur = h;
        if (threadIdx.x < 2 * NQ) qs_mine = qs[threadIdx.x];
      }
      mbar_wait(&full[s], ph);
      const uint8_t* stg = ring + s * A::STAGE;
      const int ss_ = s;
      if (++s == NST) { s = 0; ph ^= 1; }
      const int64_t nk = (n_keys - k0) < TILE ? (n_keys - k0) : TILE;
      const int64_t hrow0 = h * n_keys + k0;
      const uint32_t cb16 = (uint32_t)(nk * RB) & ~15u, nb16 = (uint32_t)(nk * 4) & ~15u;
      const uint32_t qb16 = (uint32_t)(nk * A::QB) & ~15u;
      const bool full_tile = nk == TILE;         // TILE * (RB, 4, QB) are 16-byte multiples
      // every chunk's code words (BITS per 32-coordinate group) and sketch
      // words, contiguous in the stage (consecutive lanes read consecutive
      // words: no bank conflicts); the stage is released once they are in
      uint32_t cw[KC][NG][BITS], sw[KC][NG];
      float dep = 0.0f;
#pragma unroll
      for (int kc = 0; kc < KC; ++kc) {
#pragma unroll
        for (int gi = 0; gi < NG; ++gi) {
          const int g = threadIdx.x + gi * NWD * 32;
          const int gr = g / CGROUPS, gs = kc * CGROUPS + g % CGROUPS;
          const bool gv = g < TILE * CGROUPS && gr < nk;
          if (full_tile && g < TILE * CGROUPS) {   // everything is in the stage
#pragma unroll
            for (int i = 0; i < BITS; ++i) cw[kc][gi][i] = lds32(stg + A::C_OFF + coff[gi] + kc * (CGROUPS * BITS * 4) + 4 * i);
          } else {
#pragma unroll
            for (int i = 0; i < BITS; ++i) {
              const uint32_t off = (uint32_t)(gr * RB + (gs * BITS + i) * 4);
              cw[kc][gi][i] = !gv ? 0u : (off + 4 <= cb16) ? lds32(stg + A::C_OFF + off)
                                                            : __ldg(reinterpret_cast<const uint32_t*>(codes + hrow0 * RB + off));
            }
          }
#pragma unroll
          for (int i = 0; i < BITS; ++i) dep += __uint_as_float(cw[kc][gi][i] & 0x007FFFFFu);
        }
      }
#pragma unroll
      for (int kc = 0; kc < KC; ++kc) {
#pragma unroll
        for (int gi = 0; gi < NG; ++gi) {
          sw[kc][gi] = 0u;
          if (A::ST2OK && st2) {
            const int g = threadIdx.x + gi * NWD * 32;
            const int gr = g / CGROUPS, gs = kc * CGROUPS + g % CGROUPS;   // sketch word gs of the key
            const bool gv = g < TILE * CGROUPS && gr < nk;
            if (full_tile && g < TILE * CGROUPS) {
              sw[kc][gi] = lds32(stg + A::Q_OFF + qoff[gi] + kc * CGROUPS * 4);
            } else {
              const uint32_t off = (uint32_t)(gr * A::QB + gs * 4);
              sw[kc][gi] = !gv ? 0u : (off + 4 <= qb16) ? lds32(stg + A::Q_OFF + off)
                                                       : __ldg(reinterpret_cast<const uint32_t*>(sketch + hrow0 * A::QB + off));
            }
            dep += __uint_as_float(sw[kc][gi] & 0x007FFFFFu);
          }
        }
      }
      // rho and gamma of the tile's keys for the side table
      float rg = 0.0f;
      if (threadIdx.x < 2 * TILE) {
        const int r = threadIdx.x & (TILE - 1);
        const bool isg = threadIdx.x >= TILE;
        if (r < nk && (!isg || st2))
          rg = (full_tile || (uint32_t)(r * 4 + 4) <= nb16) ? ldsf(stg + (isg ? A::G_OFF : A::N_OFF) + r * 4)
                                                            : __ldg((isg ? gammas : norms) + hrow0 + r);
        dep += rg;
      }
      __syncwarp();
      if (lane == 0) mbar_arrive_after(&empty[ss_], dep);
      const uint32_t ca = j % A::NACC;
      mbar_wait_tc(&acc_empty[ca], ((j / A::NACC) & 1) ^ 1);   // side table read by the epilogue of tile j - NACC
      float* side = reinterpret_cast<float*>(smem + A::SIDE_OFF + ca * A::SIDE_BYTES);
      if (threadIdx.x < 2 * TILE) side[threadIdx.x] = rg;
      if (threadIdx.x < 2 * NQ) side[2 * TILE + threadIdx.x] = qs_mine;
      if (threadIdx.x < 2 * TILE) {
        __syncwarp();
        if (lane == 0) mbar_arrive(&side_full[ca]);
      }
#pragma unroll
      for (int kc = 0; kc < KC; ++kc, ++jj) {
        const uint32_t b = jj % nab;
        mbar_wait_tc(&a_free[b], ((jj / nab) & 1) ^ 1);     // A[b] consumed by the MMAs of chunk jj - nab
        uint8_t* a1 = a_base + b * a_stride;
        uint8_t* a2 = a1 + A::A_BYTES;
#pragma unroll
        for (int gi = 0; gi < NG; ++gi) {
          const int g = threadIdx.x + gi * NWD * 32;
          if (g >= TILE * CGROUPS) continue;
          // stage 1: C[code] as fp16, two coordinates per lookup: the pair's
          // 2 BITS-bit field is shifted to bit 7 and OR-ed into this lane's
          // column of the pair table (one SHF + LOP3 + LDS per pair)
#pragma unroll
          for (int c8 = 0; c8 < 4; ++c8) {
            uint32_t hw[4];
#pragma unroll
            for (int e = 0; e < 8; e += 2) {
              const int b0 = (c8 * 8 + e) * BITS;
              constexpr uint32_t MSK = (uint32_t)(A::PAIRS - 1) << 7;
              uint32_t f;
              if (b0 % 32 + 2 * BITS <= 32) {
                const int sh = b0 % 32 - 7;
                f = sh >= 0 ? (cw[kc][gi][b0 / 32] >> sh) : (cw[kc][gi][b0 / 32] << -sh);
              } else {
                f = __funnelshift_r(cw[kc][gi][b0 / 32], cw[kc][gi][b0 / 32 + 1], b0 % 32) << 7;
              }
              hw[e / 2] = lds32_addr(((f & MSK) | pt_lane) + pt_base);
            }
            *reinterpret_cast<uint4*>(a1 + aoff[gi][c8]) = make_uint4(hw[0], hw[1], hw[2], hw[3]);
          }
          if (A::ST2OK && st2) {  // stage 2: +-1 from the sketch bits, four per lookup
#pragma unroll
            for (int c8 = 0; c8 < 4; ++c8) {
              uint32_t hw[4];
#pragma unroll
              for (int e = 0; e < 2; ++e) {
                const int b0 = c8 * 8 + 4 * e;
                const uint32_t f = b0 >= 8 ? (sw[kc][gi] >> (b0 - 8)) : (sw[kc][gi] << (8 - b0));
                const uint2 t2 = lds64_addr(((f & (15u << 8)) | st_lane) + st_base);
                hw[2 * e] = t2.x;
                hw[2 * e + 1] = t2.y;
              }
              *reinterpret_cast<uint4*>(a2 + aoff[gi][c8]) = make_uint4(hw[0], hw[1], hw[2], hw[3]);
            }
          }
        }
        fence_async_smem();
        __syncwarp();
        if (lane == 0) mbar_arrive(&a_full[b]);
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == A::W_MMA) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(A::TMEM_COLS));
  }
}

}  // namespace iq
