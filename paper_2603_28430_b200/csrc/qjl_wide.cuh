// Stage-2 residual sketch at the paper's wider heads, d in {256, 512}
// (NEXT row 1 of SURVEY section 8(f); PAPER.md "Compatibility with Residual
// Correction"; widths from P:373; readings R20-R24).
//
// At d >= 256 the sketch S (m = d rows, R20) no longer fits shared memory
// next to a 128-row residual tile (S is 128 / 512 KB of fp16), and the
// contraction dominates: 4 d m flop per row (1 Mflop at d = 512) puts the
// pass on the tensor-core roofline.  iq_quantize_qjl therefore runs two
// kernels here: the stage-1 quantizer (k_encode MODE 0, codes + norms
// bit-identical to iq_quantize), then this sketch kernel, which rebuilds
// the residual from x, the codes and the norms it just wrote, K-chunk by
// K-chunk, and streams S through shared memory:
//
//   S          : the K-major 128-byte-swizzled UMMA image in K-chunks of
//                64 coordinates (m rows x 128 B), by TMA: resident at
//                d = 256 (128 KB, loaded once per CTA), streamed from L2
//                through a two-stage ring at d = 512 (evict-last);
//   16 warps   : for every (row pair, 8-coordinate piece) of the chunk:
//                x (128-bit loads, one work item ahead), codes -> C[code]
//                (width-L shuffle table), x^ = rho M^T C[code] (block
//                operators from shared memory), r = x - x^ (R21),
//                gamma^2 += r^2 (R23), r * 256 / max(rho, eps) split into
//                fp16 hi + lo, stored as the chunk's UMMA A tiles (K-major,
//                128-byte swizzle);
//   MMAs       : d = 256: issued by one thread of the LAST warp to finish
//                the chunk (a shared-memory arrival counter), so no warp is
//                parked on the tensor pipe; d = 512 (tensor-bound): a
//                dedicated MMA warp (and a TMA warp refilling the S ring): z (+)= A_hi S_k^T + A_lo S_k^T, M = 128
//                rows, N = m (one or two N = 256 instructions per K-step),
//                fp32 in TMEM; the same thread refills the S ring;
//   epilogue   : tcgen05.ld, sign bits [z >= 0] packed LSB-first (R22).
// The residual arithmetic is the fused d <= 128 kernel's direct form
// (qjl.cuh, fp32 rows), so the two agree on the readings.
#pragma once
#include "qjl.cuh"

namespace iq {

template <class T, int D, int BITS, int VAR>
struct WGeo {
  static constexpr int PW = (VAR == IQ_VARIANT_PLANAR2D) ? 2 : 4;   // block width
  static constexpr int M = D;                    // sketch rows (R20)
  static constexpr int TILE = 128;               // rows per tile = UMMA M
  static constexpr int NPC = M / 256;            // N = 256 MMA pieces per K-step
  static constexpr int NWC = 16;                 // compute warps: (row pair, piece) = thread; no dedicated MMA warp
  static constexpr int KC = 64;                  // coordinates per K-chunk (one 128-byte swizzle atom)
  static constexpr int NKC = D / KC;
  static constexpr int B_STAGE = M * 128;        // one K-chunk of S: m rows x 64 fp16
  // d = 256: all of S (128 KB) stays resident (loaded once per CTA), 16
  // warps (4 per sub-partition: 128 registers); d = 512: S (512 KB) streams
  // from L2 through a two-stage ring refilled by a dedicated TMA warp (the
  // refill must not wait for a compute warp to reach a polling point)
  static constexpr bool RES = NKC * B_STAGE <= 128 * 1024;
  // streamed S also gets a dedicated MMA warp (d = 512, where the tensor
  // pipe is the bottleneck and must never wait for a compute warp to reach
  // its arrival: 1.85-1.95 ms vs 2.1 ms with the last-arriver issue)
  static constexpr bool MMAW = !RES;
  static constexpr int CTA_THREADS = 32 * (NWC + (RES ? 0 : 2));
  static constexpr int RB = D * BITS / 8;        // code bytes per row
  static constexpr int NB = RES ? NKC : 2;        // S stages
  static constexpr int A_TILE = TILE * 128;      // one fp16 operand chunk (hi or lo): 16 KB
  static constexpr int NA = 2;                   // A ring depth (hi + lo per stage)
  static constexpr int NACC = 2 * M <= 512 ? 2 : 1;   // TMEM accumulators of M columns
  static constexpr int NQ = PW * PW / 4;         // float4 per block operator
  static constexpr int BPP = 8 / PW;             // blocks per 8-coordinate piece
  static constexpr int OPS_BYTES = D * PW * 4;   // every block operator (D / PW blocks x PW^2 floats)
  static constexpr int A_OFF = NB * B_STAGE;     // 1024-aligned (B_STAGE is)
  static constexpr int OPS_OFF = A_OFF + NA * 2 * A_TILE;
  static constexpr int BAR_OFF = OPS_OFF + OPS_BYTES;
  static constexpr int SMEM = BAR_OFF + 256 + 1024;   // + slack to align the base to 1024
  static constexpr int CW = M / (NWC / 4);       // epilogue columns per warp
  static constexpr int XV = sizeof(T) == 4 ? 2 : 1;   // 16-byte loads per 8 coordinates
  static_assert(D == 256 || D == 512, "wide sketch kernel: d in {256, 512}");
  static_assert(CW % 64 == 0 && NKC > NA && NKC % 2 == 0, "epilogue split, ring depth, chunk pairs");
  static_assert(SMEM <= 227 * 1024, "shared memory");
};

// TMA prefetch of a contiguous global range into L2 (no shared memory, no
// completion tracking): the next tile's rows are on chip by the time the
// compute threads' loads ask for them
__device__ __forceinline__ void prefetch_l2(const void* p, uint32_t bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"(bytes) : "memory");
}

__device__ __forceinline__ float rcp_approx(float x) {
  float r;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}

template <class T, int D, int BITS, int VAR>
__global__ void __launch_bounds__(WGeo<T, D, BITS, VAR>::CTA_THREADS, 1)
k_qjl_sketch(const float* __restrict__ mat, const KCodebook cb, int64_t n, const T* __restrict__ x,
             const uint8_t* __restrict__ s_img, const uint8_t* __restrict__ codes, const float* __restrict__ norms,
             uint8_t* __restrict__ qjl, float* __restrict__ rnorms) {
  using W = WGeo<T, D, BITS, VAR>;
  constexpr int NWC = W::NWC, TILE = W::TILE, M = W::M, NKC = W::NKC, NB = W::NB, NA = W::NA;
  constexpr int PW = W::PW, NQ = W::NQ, BPP = W::BPP, NACC = W::NACC, RB = W::RB;
  constexpr int L = 1 << BITS;

  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024 - (smem_u32(smem_raw) & 1023)) & 1023);   // 1024-aligned base
  uint8_t* b_ring = smem;
  uint8_t* a_ring = smem + W::A_OFF;     // stage s: hi at 2 s A_TILE, lo at (2 s + 1) A_TILE
  float4* ops = reinterpret_cast<float4*>(smem + W::OPS_OFF);
  uint64_t* b_full = reinterpret_cast<uint64_t*>(smem + W::BAR_OFF);
  uint64_t* b_empty = b_full + NB;       // streaming only (tcgen05.commit)
  uint64_t* a_empty = b_empty + NB;      // MMAs of the stage done (tcgen05.commit)
  uint64_t* acc_full = a_empty + NA;     // MMAs of the tile done (tcgen05.commit)
  uint64_t* acc_empty = acc_full + NACC; // epilogue read the accumulator (NWC arrivals)
  uint64_t* a_full = acc_empty + NACC;   // [NA] compute warps -> MMA warp (MMAW only; NWC arrivals)
  uint32_t* arrivals = reinterpret_cast<uint32_t*>(a_full + NA);   // [NA] warps done with the stage (no MMAW)
  uint32_t* tmem_slot = arrivals + NA;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t ntiles = (n + TILE - 1) / TILE;
  const int64_t my_tiles = blockIdx.x < ntiles ? (ntiles - 1 - blockIdx.x) / gridDim.x + 1 : 0;
  const uint32_t total = (uint32_t)(my_tiles * NKC);   // K-chunks this CTA produces
  const uint64_t pol = policy_evict_last();            // S is re-read by every CTA: keep it in L2
  // streamed S: CTA i walks the K-chunks starting at chunk i mod NKC, so at
  // any moment the 148 CTAs read different parts of S (the same 64 KB from
  // every SM at once is an L2 hot spot: measured 1.5-2.6 ms, unstable)
  const int rot = W::RES ? 0 : (int)(blockIdx.x % NKC);
  if (threadIdx.x == 0) {
    for (int s = 0; s < NB; ++s) { mbar_init(&b_full[s], 1); mbar_init(&b_empty[s], 1); }
    for (int s = 0; s < NA; ++s) { mbar_init(&a_empty[s], 1); mbar_init(&a_full[s], NWC); arrivals[s] = 0; }
    for (int b = 0; b < NACC; ++b) { mbar_init(&acc_full[b], 1); mbar_init(&acc_empty[b], NWC); }
    fence_mbar_init();
    // the first NB chunks of S (all of it when resident)
    const uint32_t first = W::RES ? (uint32_t)NB : (total < (uint32_t)NB ? total : (uint32_t)NB);
    for (uint32_t k = 0; k < first; ++k) {
      mbar_arrive_expect_tx(&b_full[k], W::B_STAGE);
      bulk_g2s(b_ring + k * W::B_STAGE, s_img + (size_t)((k + rot) % NKC) * W::B_STAGE, W::B_STAGE, &b_full[k], pol);
    }
  }
  // every block operator, as float4 q of block b of piece p at
  // (u * NQ + q) * (D / 8) + p with b = p * BPP + u: the 8 pieces of a chunk
  // (consecutive lanes) read consecutive float4s
  for (int i = threadIdx.x; i < D / PW * NQ; i += blockDim.x) {
    const int b = i / NQ, q = i % NQ;
    ops[((b % BPP) * NQ + q) * (D / 8) + b / BPP] = __ldg(reinterpret_cast<const float4*>(mat) + i);
  }
  if (warp == 0) {   // TMEM: 512 columns (NACC accumulators of M columns)
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(tmem_slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  // D[128 x 256] (+)= A[128 x 16] * B[256 x 16]^T per instruction: fp16, fp32 accumulate
  constexpr uint32_t idesc = (1u << 4) | ((uint32_t)(256 >> 3) << 17) | ((uint32_t)(TILE >> 4) << 24);
  // the MMAs of chunk c (K-chunk k of accumulator b), by the last warp to finish it
  auto issue = [&](uint32_t c, int k, uint32_t b, bool last_of_tile) {
    const int sa = c % NA, sb = W::RES ? k : (int)(c % NB);
    mbar_wait_tc(&b_full[sb], W::RES ? 0u : (c / NB) & 1);
    tc_fence_after();
    const uint32_t ah = smem_u32(a_ring + 2 * sa * W::A_TILE), al = ah + W::A_TILE;
    const uint32_t bs = smem_u32(b_ring + sb * W::B_STAGE);
#pragma unroll
    for (int part = 0; part < 2; ++part)          // A_hi S^T + A_lo S^T
#pragma unroll
      for (int s = 0; s < W::KC / 16; ++s)
#pragma unroll
        for (int pc = 0; pc < W::NPC; ++pc)
          umma_f16(tmem + b * M + pc * 256, umma_desc_sw128((part ? al : ah) + 32 * s),
                   umma_desc_sw128(bs + pc * 256 * 128 + 32 * s), idesc, (k | part | s) != 0);
    umma_commit(&a_empty[sa]);
    if constexpr (!W::RES) umma_commit(&b_empty[sb]);
    if (last_of_tile) umma_commit(&acc_full[b]);
  };

  if constexpr (!W::RES) {
    if (warp == NWC) {   // ------------------------------ streamed S: the TMA refill warp
      if (lane == 0) {
        for (uint32_t u = NB; u < total; ++u) {   // chunk u reuses the stage of chunk u - NB
          const int st = u % NB;
          mbar_wait_tc(&b_empty[st], ((u / NB) & 1) ^ 1);   // completed by tcgen05.commit
          mbar_arrive_expect_tx(&b_full[st], W::B_STAGE);
          bulk_g2s(b_ring + st * W::B_STAGE, s_img + (size_t)((u + rot) % NKC) * W::B_STAGE, W::B_STAGE,
                   &b_full[st], pol);
        }
      }
    }
  }
  if constexpr (W::MMAW) {
    if (warp == NWC + 1) {   // ------------------------------ streamed S: the MMA warp
      if (lane == 0) {
        uint32_t c = 0, j = 0;
        for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x, ++j) {
          const uint32_t b = j % NACC;
          mbar_wait_tc(&acc_empty[b], ((j / NACC) & 1) ^ 1);
          for (int k = 0; k < NKC; ++k, ++c) {
            mbar_wait_tc(&a_full[c % NA], (c / NA) & 1);
            issue(c, k, b, k == NKC - 1);
          }
        }
      }
    }
  }
  if (warp < NWC) {    // ------------------------------------------------ compute warps
  const int tid = threadIdx.x;
  const int pc = tid & 7;                 // 8-coordinate piece of the chunk
  const int rp = tid >> 3;                // row pair: tile rows rp and rp + 64
  const float ctab = cb.cent[lane & (L - 1)];   // C[k] in lane k of each group of L lanes
  const int quad = warp & 3, part = warp >> 2;  // epilogue: TMEM lane quadrant, column slice
  constexpr int CW = W::CW;
  // the piece's code bits: BITS bytes at byte offset (8 k + pc) BITS of the
  // row; 8 k BITS is a multiple of 4, so the word offset inside the chunk
  // and the shift depend on the piece only
  const int coff = pc * BITS;
  const int cshift = (coff & 3) * 8;
  const bool chi = BITS == 3 && (coff & 3) > 1;          // the 24 bits straddle two words
  const uint32_t offa = umma_sw128_off(rp, 8 * pc, TILE), offb = umma_sw128_off(rp + 64, 8 * pc, TILE);

  auto epilogue = [&](uint32_t jj, int64_t tt) {
    const uint32_t b = jj % NACC;
    mbar_wait_tc(&acc_full[b], (jj / NACC) & 1);   // completed by tcgen05.commit: no suspend hint
    tc_fence_after();
    const int row = 32 * quad + lane;
    const int64_t v = tt * TILE + row;
    const uint32_t ta = tmem + ((uint32_t)(32 * quad) << 16) + b * M + part * CW;
    uint32_t w[CW / 32];
#pragma unroll
    for (int c = 0; c < CW / 32; ++c) w[c] = tmem_sign_word32(ta + 32 * c);
    tc_fence_before();
    __syncwarp();
    if (lane == 0) mbar_arrive(&acc_empty[b]);
    if (v < n) {
      uint8_t* dst = qjl + v * (M / 8) + part * (CW / 8);
#pragma unroll
      for (int c = 0; c < CW / 32; c += 2) *reinterpret_cast<uint2*>(dst + 4 * c) = make_uint2(w[c], w[c + 1]);
    }
  };

  // raw loads of one (tile, chunk) work item, issued one item ahead
  struct Raw {
    uint4 xa[W::XV], xb[W::XV];
    uint32_t ca0, ca1, cb0, cb1;   // code words (the second only when the piece straddles)
    float rho_a, rho_b;            // loaded with the tile's first chunk
  };
  auto fetch = [&](int64_t t, int k, Raw& f) {
    if (t >= ntiles) return;
    const int64_t ra = t * TILE + rp, rb = ra + 64;
    const int64_t la = ra < n ? ra : n - 1, lb = rb < n ? rb : n - 1;   // clamped for the ragged tail
    const int q = ((k + rot) % NKC) * 8 + pc;                           // coordinates 8 q .. 8 q + 7
#pragma unroll
    for (int i = 0; i < W::XV; ++i) {
      f.xa[i] = __ldg(reinterpret_cast<const uint4*>(x + la * D + 8 * q) + i);
      f.xb[i] = __ldg(reinterpret_cast<const uint4*>(x + lb * D + 8 * q) + i);
    }
    const uint32_t* wa = reinterpret_cast<const uint32_t*>(codes + la * RB + ((q * BITS) & ~3));
    const uint32_t* wb = reinterpret_cast<const uint32_t*>(codes + lb * RB + ((q * BITS) & ~3));
    f.ca0 = __ldg(wa);
    f.cb0 = __ldg(wb);
    f.ca1 = chi ? __ldg(wa + 1) : 0u;
    f.cb1 = chi ? __ldg(wb + 1) : 0u;
    if (k == 0) {
      f.rho_a = __ldg(norms + la);
      f.rho_b = __ldg(norms + lb);
    }
  };
  auto unpack8 = [&](const uint4* u, float* v) {
    if constexpr (sizeof(T) == 4) {
      v[0] = __uint_as_float(u[0].x); v[1] = __uint_as_float(u[0].y);
      v[2] = __uint_as_float(u[0].z); v[3] = __uint_as_float(u[0].w);
      v[4] = __uint_as_float(u[1].x); v[5] = __uint_as_float(u[1].y);
      v[6] = __uint_as_float(u[1].z); v[7] = __uint_as_float(u[1].w);
    } else {
      const uint32_t w[4] = {u[0].x, u[0].y, u[0].z, u[0].w};
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const float2 t2 = unpack2<T>(w[e]);
        v[2 * e] = t2.x;
        v[2 * e + 1] = t2.y;
      }
    }
  };

  uint32_t c = 0, j = 0;
  int64_t tprev = -1;
  float2 nrho = bc(0.0f), sr = bc(0.0f), g2 = bc(0.0f);
  // one K-chunk of the tile's A operand (hi, lo) from the raw item; the
  // warp that completes the chunk issues its MMAs
  auto chunk = [&](const Raw& cur, int k) {
    if (k == 0) {
      nrho = f2(-cur.rho_a, -cur.rho_b);
      // sign(S r) is scale-free: r * 256 / max(rho, eps) keeps the fp16 parts in range
      sr = f2(256.0f * rcp_approx(fmaxf(cur.rho_a, 1e-12f)), 256.0f * rcp_approx(fmaxf(cur.rho_b, 1e-12f)));
      g2 = bc(0.0f);
    }
    const int q = ((k + rot) % NKC) * 8 + pc;     // this step's K-chunk (rotated per CTA when S streams)
    const uint32_t wa = BITS == 3 ? __funnelshift_r(cur.ca0, cur.ca1, cshift) : cur.ca0 >> cshift;
    const uint32_t wb = BITS == 3 ? __funnelshift_r(cur.cb0, cur.cb1, cshift) : cur.cb0 >> cshift;
    float va[8], vb[8];
    unpack8(cur.xa, va);
    unpack8(cur.xb, vb);
    const int sa = c % NA;
    // the MMAs of the stage's last use are done.  Resident S (d = 256):
    // every lane waits, parked with a short suspend hint (the warp stays
    // converged for its shuffles: 0.74 -> 0.58 ms); streamed S (d = 512):
    // one lane waits (measured 15 % faster there)
    if constexpr (W::RES) {
      mbar_wait_short(&a_empty[sa], ((c / NA) & 1) ^ 1);
    } else {
      if (lane == 0) mbar_wait_tc(&a_empty[sa], ((c / NA) & 1) ^ 1);
      __syncwarp();
    }
    uint8_t* ah = a_ring + 2 * sa * W::A_TILE;
    uint8_t* al = ah + W::A_TILE;
    // the piece as two quads of coordinates (one 4-D block or two 2-D
    // blocks each): short live ranges, 8-byte operand stores
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      float2 cq[4], r[4];
#pragma unroll
      for (int e = 0; e < 4; ++e)                       // C[code], width-L shuffle table
        cq[e] = f2(__shfl_sync(kFull, ctab, (int)(wa >> ((4 * h + e) * BITS)), L),
                   __shfl_sync(kFull, ctab, (int)(wb >> ((4 * h + e) * BITS)), L));
#pragma unroll
      for (int u = 0; u < 4 / PW; ++u) {                // T^-1 per block: M^T c
        float Mb[PW * PW];
#pragma unroll
        for (int qq = 0; qq < NQ; ++qq) {
          const float4 t4 = ops[((h * (4 / PW) + u) * NQ + qq) * (D / 8) + q];
          Mb[4 * qq] = t4.x; Mb[4 * qq + 1] = t4.y; Mb[4 * qq + 2] = t4.z; Mb[4 * qq + 3] = t4.w;
        }
        rot_inv<PW>(Mb, cq + u * PW, r + u * PW);
      }
      uint32_t hw[2][2], lw[2][2];                      // [row A / B][coordinate pair]
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        r[e] = fma2(r[e], nrho, f2(va[4 * h + e], vb[4 * h + e]));   // r = x - rho T^-1(C[code])  (R21)
        g2 = fma2(r[e], r[e], g2);                      // gamma^2  (R23)
        r[e] = mul2(r[e], sr);
      }
#pragma unroll
      for (int e = 0; e < 4; e += 2) {
        // fp16 hi = r truncated to 11 significant bits (exact in fp16 for
        // |r| >= 2^-14, i.e. all but negligible coordinates), lo = r - hi
        // exactly in fp32, then rounded to fp16: r to ~2^-21 relative
        const float2 h0 = f2(__uint_as_float(__float_as_uint(r[e].x) & 0xFFFFE000u),
                             __uint_as_float(__float_as_uint(r[e].y) & 0xFFFFE000u));
        const float2 h1 = f2(__uint_as_float(__float_as_uint(r[e + 1].x) & 0xFFFFE000u),
                             __uint_as_float(__float_as_uint(r[e + 1].y) & 0xFFFFE000u));
        const float2 l0 = add2(r[e], f2(-h0.x, -h0.y)), l1 = add2(r[e + 1], f2(-h1.x, -h1.y));
        hw[0][e / 2] = pack2<__half>(h0.x, h1.x);
        hw[1][e / 2] = pack2<__half>(h0.y, h1.y);
        lw[0][e / 2] = pack2<__half>(l0.x, l1.x);
        lw[1][e / 2] = pack2<__half>(l0.y, l1.y);
      }
      *reinterpret_cast<uint2*>(ah + offa + 8 * h) = make_uint2(hw[0][0], hw[0][1]);
      *reinterpret_cast<uint2*>(ah + offb + 8 * h) = make_uint2(hw[1][0], hw[1][1]);
      *reinterpret_cast<uint2*>(al + offa + 8 * h) = make_uint2(lw[0][0], lw[0][1]);
      *reinterpret_cast<uint2*>(al + offb + 8 * h) = make_uint2(lw[1][0], lw[1][1]);
    }
    fence_async_smem();       // generic-proxy A writes -> tensor-core (async proxy) reads
    __syncwarp();
    if constexpr (W::MMAW) {
      if (lane == 0) mbar_arrive(&a_full[sa]);
      ++c;
      return;
    }
    // one accumulator: the previous tile's epilogue runs before this tile's
    // first chunk is handed over (its MMAs overwrite that accumulator)
    if (NACC == 1 && k == 0 && tprev >= 0) epilogue(j - 1, tprev);
    if (lane == 0) {
      __threadfence_block();
      const uint32_t old = atomicAdd(&arrivals[sa], 1u);
      if (old == (c / NA + 1) * NWC - 1) {          // the last warp of this chunk
        __threadfence_block();
        issue(c, k, j % NACC, k == NKC - 1);
      }
    }
    __syncwarp();
    ++c;
  };

  // L2 prefetch of the rows of tile t (x, codes, norms), one tile ahead
  auto prefetch_tile = [&](int64_t t) {
    if (t < ntiles && threadIdx.x == 0) {
      const int64_t v0 = t * TILE, nv = (n - v0) < TILE ? (n - v0) : TILE;
      prefetch_l2(x + v0 * D, (uint32_t)(nv * D * sizeof(T)));
      prefetch_l2(codes + v0 * RB, (uint32_t)((nv * RB + 15) & ~15));
      prefetch_l2(norms + v0, (uint32_t)((nv * 4 + 15) & ~15));
    }
  };
  prefetch_tile(blockIdx.x);
  Raw f0, f1;
  fetch(blockIdx.x, 0, f0);
  int cur_set = 0;                                       // the operators of set 0 are loaded
  for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x, ++j) {
    const int64_t ra = t * TILE + rp, rb = ra + 64;
    prefetch_tile(t + gridDim.x);
    // parameter sets [R31]: this tile's operators (tiles never straddle
    // sets), rewritten between two compute-warp barriers
    if (cb.n_sets > 1) {
      const int set = (int)((t * TILE / cb.set_rows) % cb.n_sets);
      if (set != cur_set) {
        cur_set = set;
        const float4* ms = reinterpret_cast<const float4*>(mat + (size_t)set * cb.set_stride);
        asm volatile("bar.sync 1, %0;" ::"r"(NWC * 32) : "memory");   // the old operators are no longer read
        for (int i = tid; i < D / PW * NQ; i += NWC * 32) {
          const int b = i / NQ, qq = i % NQ;
          ops[((b % BPP) * NQ + qq) * (D / 8) + b / BPP] = __ldg(ms + i);
        }
        asm volatile("bar.sync 1, %0;" ::"r"(NWC * 32) : "memory");
      }
    }
#pragma unroll 1
    for (int k = 0; k < NKC; k += 2) {               // ping-pong: the next item loads while this one computes
      fetch(t, k + 1, f1);
      chunk(f0, k);
      // two accumulators: the previous tile's epilogue once this tile's
      // first NA chunks are handed over (its accumulator is not reused
      // before the next tile)
      if ((NACC == 2 || W::MMAW) && k == NA - 1 && tprev >= 0) epilogue(j - 1, tprev);
      if (k + 2 < NKC) fetch(t, k + 2, f0);
      else fetch(t + gridDim.x, 0, f0);
      chunk(f1, k + 1);
      if ((NACC == 2 || W::MMAW) && k + 1 == NA - 1 && tprev >= 0) epilogue(j - 1, tprev);
    }
    // gamma = ||r|| over the row's 8 pieces (lanes pc = 0..7 of the group)
    float2 gs = g2;
#pragma unroll
    for (int o = 4; o >= 1; o >>= 1)
      gs = add2(gs, f2(__shfl_xor_sync(kFull, gs.x, o), __shfl_xor_sync(kFull, gs.y, o)));
    if (pc == 0) {
      if (ra < n) rnorms[ra] = sqrt_ftz(gs.x);
      if (rb < n) rnorms[rb] = sqrt_ftz(gs.y);
    }
    tprev = t;
  }
  if (tprev >= 0) epilogue(j - 1, tprev);
  }  // compute warps
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
  }
}

}  // namespace iq
