// sm_100a kernels of the IsoQuant stage-1 path (Algorithm 1,
// P:229-258).  The path is an elementwise map with O(d) work per O(d) bytes
// and no reuse: it is bound by HBM bandwidth and, at fp16, close to the
// instruction-issue ceiling.  No tensor cores.  See DESIGN.md "Kernels".
//
// All three kernels (quantize K1, dequantize K2, fused roundtrip K3) are
// persistent and warp-specialised.  One producer warp streams tiles of
// TILE_V contiguous rows from HBM into a ring of shared-memory stages with
// 1-D TMA bulk copies (cp.async.bulk + mbarrier complete_tx) — rows of x for
// K1/K3, rows of packed codes plus norms for K2 — so the bytes in flight do
// not cost registers.  NWC compute warps read their rows from shared memory,
// release the stage, compute in registers and write results with 128-bit
// streaming stores.
//
// Thread mapping inside a compute warp: a row of d elements of dtype T is cut
// into 16-byte chunks (EPC = 4 fp32 / 8 fp16 elements); G = min(32, d/EPC)
// consecutive lanes serve one row, lane `sub` owning chunks sub, sub+G, ...
// (CPL chunks), so every warp-wide access of a chunk index is contiguous.
// Each lane processes TWO rows at a time: coordinate e of row u0 and of row
// u1 form one packed fp32x2 register, and every step of the path — norm,
// rotation, quantizer, inverse rotation, rescale — is one FFMA2/FMUL2/FSET
// per pair, with the block operator as a broadcast scalar operand.  A lane's
// blocks never change, so their 4x4 (2x2) operators stay in registers for
// the whole kernel ("the entire block can often remain in
// registers from input load through output store").
#pragma once
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <type_traits>

#include "iq_internal.h"

namespace iq {

constexpr unsigned kFull = 0xffffffffu;
#ifndef IQ_RING_KB
#define IQ_RING_KB 96
#endif
#ifndef IQ_GRID_MIN_BITS
#define IQ_GRID_MIN_BITS 4   // bits at which the encoders use the grid decision [R19]
#endif
#ifndef IQ_OPS_SMEM
#define IQ_OPS_SMEM 1        // large-operator encoders read their operators from shared memory
#endif
#ifndef IQ_PDL
#define IQ_PDL 1             // programmatic dependent launch of the stage-1 encoders
#endif
#ifndef IQ_RING_WIDE_KB
#define IQ_RING_WIDE_KB 128  // TMA ring of the 16-warp encoders (measured: 128 KB > 200 KB, ~1-2%)
#endif
#ifndef IQ_STORE_CS
#define IQ_STORE_CS 1        // streaming (evict-first) 128-bit output stores
#endif
#ifndef IQ_NORM_SPLIT
#define IQ_NORM_SPLIT 0      // norm as two interleaved partial sums (experiment)
#endif
#ifndef IQ_NWC_WIDE
#define IQ_NWC_WIDE 16       // compute warps of the wide encoder CTAs
#endif
#ifndef IQ_NWC_NARROW
#define IQ_NWC_NARROW 8      // compute warps of the encoder CTAs with operators in registers
#endif
#ifndef IQ_B3_ALU
#define IQ_B3_ALU 1          // b = 3 fused value chain: FSETP + predicated FADD (else FSET + FFMA2)
#endif
#ifndef IQ_BYTE_CODES
#define IQ_BYTE_CODES 1      // byte-aligned code pieces stored in place (else gathered into words by shuffles)
#endif
#ifndef IQ_SIGN_SHF
#define IQ_SIGN_SHF 0        // code sign bits by funnel shifts (else FSET + FFMA2 positional count)
#endif
#ifndef IQ_K1_OPS_REG
#define IQ_K1_OPS_REG 1      // 16-bit quantizer at b = 3 with its operators in registers (8 compute warps; measured +5 %)
#endif
#ifndef IQ_GRID_PAIR
#define IQ_GRID_PAIR 0       // b = 4 grid decision with the two rows' FFMAs packed as FFMA2 (measured slower)
#endif
#ifndef IQ_FHADD
#define IQ_FHADD 0           // fp16 -> fp32 with the mixed-precision FHADD (else HADD2.F32)
#endif
#ifndef IQ_PAIR_UNROLL
#define IQ_PAIR_UNROLL 2     // two row pairs per loop iteration (K1 1.5-2 % faster, K3 unchanged; measured)
#endif
constexpr int kPairUnroll = IQ_PAIR_UNROLL;    // row pairs interleaved per iteration
constexpr int kThreads = 256;                  // statistics kernel CTAs

template <class T> struct DT;
template <> struct DT<float> { static constexpr int EPC = 4; };
template <> struct DT<__half> { static constexpr int EPC = 8; };
template <> struct DT<__nv_bfloat16> { static constexpr int EPC = 8; };

// two floats -> the packed 16-bit pair of T (round to nearest even [R15][R28])
template <class T> __device__ __forceinline__ uint32_t pack2(float lo, float hi);
template <> __device__ __forceinline__ uint32_t pack2<__half>(float lo, float hi) {
  __half2 h = __floats2half2_rn(lo, hi);
  return *reinterpret_cast<uint32_t*>(&h);
}
template <> __device__ __forceinline__ uint32_t pack2<__nv_bfloat16>(float lo, float hi) {
  __nv_bfloat162 h = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<uint32_t*>(&h);
}
// the packed 16-bit pair of T -> two floats (exact)
template <class T> __device__ __forceinline__ float2 unpack2(uint32_t w);
template <> __device__ __forceinline__ float2 unpack2<__half>(uint32_t w) {
#if IQ_FHADD
  // mixed-precision add f32 = f16 + (-0.0f): exact, one full-rate FMA-pipe
  // slot per value (HADD2.F32 takes two)
  float a, b;
  asm("{.reg .b16 l, h; mov.b32 {l, h}, %2;\n"
      "add.rn.f32.f16 %0, l, 0f80000000; add.rn.f32.f16 %1, h, 0f80000000;}"
      : "=f"(a), "=f"(b) : "r"(w));
  return make_float2(a, b);
#else
  return __half22float2(*reinterpret_cast<const __half2*>(&w));
#endif
}
template <> __device__ __forceinline__ float2 unpack2<__nv_bfloat16>(uint32_t w) {
  return make_float2(__uint_as_float(w << 16), __uint_as_float(w & 0xFFFF0000u));
}

constexpr int cgcd(int a, int b) { return b == 0 ? a : cgcd(b, a % b); }
constexpr int clcm(int a, int b) { return a / cgcd(a, b) * b; }

// Chunks per lane: the smallest power of two giving >= TPL coordinates per
// lane (fewer lanes per row = fewer shuffle levels and less per-row overhead
// per coordinate, at the price of operator registers), bounded so that <= 32
// lanes serve a row and a lane group's code bits fill whole 32-bit words.
template <int CHUNKS, int EPC, int BITS, int TPL>
constexpr int pick_cpl() {
  int cpl = 1;
  while (cpl * EPC < TPL && cpl * 2 <= CHUNKS) cpl *= 2;
  while (CHUNKS / cpl > 32) cpl *= 2;
  while (cpl > 1 && ((CHUNKS / cpl) * EPC * BITS) % 32 != 0) cpl /= 2;
  return cpl;
}

// Kernel kinds: 0 quantize (K1), 1 fused roundtrip (K3), 2 fused roundtrip +
// codes, 3 dequantize (K2), 4 distortion gradient, 6 the stage-2 sketch
// kernel's encoder (K3+codes' geometry), 5 quantize-on-append (K1's
// lane geometry, so it emits K1's codes and norms bit for bit; operators in
// registers because every lane group may use a different parameter set).  Coordinates per lane (TPL), measured on B200
// (DESIGN.md section 6): 16 for every encoder except the fp32 code-emitting
// ones (8); K1 and K3+codes share one geometry so that they emit
// bit-identical codes and norms; the decoder 8.
template <class T, int BITS, int KIND>
constexpr int pick_tpl() {
  constexpr bool f16 = sizeof(T) == 2;
#ifdef IQ_TPL_DEC
  if (KIND == 3) return IQ_TPL_DEC;
#endif
  if (KIND == 3) return (f16 && BITS == 4) ? 16 : 8;   // measured: 0.82 -> 0.89 at fp16 b = 4
  if (KIND == 4) return 8;                               // distortion gradient (grad.cuh)
#ifdef IQ_TPL_K3B4
  if (KIND == 1 && BITS == 4) return IQ_TPL_K3B4;
#endif
#ifdef IQ_TPL_K3
  if (KIND == 1) return IQ_TPL_K3;
#endif
  if (KIND == 1) return 16;
#ifdef IQ_TPL_EMIT
  return IQ_TPL_EMIT;
#endif
  return f16 ? 16 : 8;
}
// Where an encoder whose operators exceed 32 registers per lane keeps them
// (measured under the bench's sustained protocol):
// registers (8 compute warps) for the 16-bit fused kernel at every b, the
// 16-bit fused + codes kernel at b <= 3 and the 16-bit quantizer at b = 3
// (84.8 -> 80.7 us at d = 128) -- at the board's power cap the
// per-block operator re-reads from shared memory cost more clock than the
// 16-warp latency hiding buys (b = 3: 0.75 -> 0.79 of peak, b = 4: 0.715 ->
// 0.75 at d = 128 ... 512); shared memory (16 compute warps) for the other
// 16-bit encoders and the fp32 quantizer; registers (8 warps) otherwise.
template <class T, int BITS, int KIND>
constexpr bool pick_ops_smem() {
  if (!IQ_OPS_SMEM || (KIND >= 3 && KIND <= 5)) return false;   // decoder, gradient, append: registers
  // KIND 6: the stage-2 sketch kernel's stage-1 encoder (qjl.cuh), K3+codes'
  // lane geometry with its operators kept in shared memory (its 8 / 16 warps
  // also hold the residual tiles)
  if (sizeof(T) == 2) return !(KIND == 1 || (KIND == 2 && BITS <= 3) || (IQ_K1_OPS_REG && KIND == 0 && BITS == 3));
  return KIND == 0;
}

template <class T, int D, int BITS, int VAR, int KIND>
struct Geo {
  static constexpr bool ENC = KIND != 3;
  static constexpr int EPC = DT<T>::EPC;
  static constexpr int PW = (VAR == IQ_VARIANT_PLANAR2D) ? 2 : 4;   // block width
  static constexpr int CHUNKS = D / EPC;
  static constexpr int CPL = pick_cpl<CHUNKS, EPC, BITS, pick_tpl<T, BITS, KIND>()>();   // chunks per lane
  static constexpr int G = CHUNKS / CPL;                           // lanes per row
  static constexpr int VPW = 32 / G;                               // rows per warp
  static constexpr int EPL = CPL * EPC;                            // coordinates per lane
  static constexpr int NBL = EPL / PW;                             // blocks per lane
  static constexpr bool SMALL_OPS = NBL * PW * PW <= 32;
  // encoders whose operators do not fit 32 registers per lane keep them in
  // shared memory (lane-contiguous float4 columns, re-read per block) so that
  // 16 compute warps fit the register file
  static constexpr bool OPS_SMEM = ENC && !SMALL_OPS && pick_ops_smem<T, BITS, KIND>();
  static constexpr bool WIDE = ENC && (SMALL_OPS || OPS_SMEM);
  static constexpr int NWC = WIDE ? IQ_NWC_WIDE : (ENC ? IQ_NWC_NARROW : 8);   // compute warps per CTA
  static constexpr int CTA_THREADS = 32 * (NWC + 1);               // + 1 producer warp
  static constexpr int MIN_CTAS = (ENC || !SMALL_OPS) ? 1 : 2;
  static constexpr int OPS_BYTES = OPS_SMEM ? G * NBL * PW * PW * 4 : 0;
  static constexpr int RING = WIDE ? IQ_RING_WIDE_KB * 1024 - OPS_BYTES : IQ_RING_KB * 1024;   // TMA ring per CTA
  static constexpr int ROWB = D * (int)sizeof(T);                  // bytes per row of x
  static constexpr int RB = D * BITS / 8;                          // code bytes per row
  static constexpr int B = EPC * BITS;                             // code bits per chunk
  static constexpr int W = G * B / 32;                             // code words per segment
  // rows per stage: >= STAGE_KB of x and a whole number of row pairs per warp
  // (granule: whole row pairs per warp, and 16-byte aligned norm tiles)
  static constexpr int GR = clcm(2 * NWC * VPW, 4);
  // stage size (measured): 64 KB for the 16-bit quantizer at b >= 3, d >= 128
  // (2-5 % over 32 / 16 KB; worse at fp32 and b = 2), 32 KB for the other
  // b = 3 encoders, the b = 4 fused kernel and the b <= 2 fused kernels
  // (more rows per warp per mbarrier round trip; b = 2 fp16 sustained: fused
  // 95.7 -> 91.1 us, fused + codes 113.4 -> 104.2 us), else 16 KB
#ifdef IQ_STAGE_KB
  static constexpr int STAGE_KB = ENC ? IQ_STAGE_KB : 16;
#else
#ifndef IQ_DEC_STAGE_KB
#define IQ_DEC_STAGE_KB 0
#endif
  // decoder tiles: 32 KB of output rows at b <= 3 (1-8 % over 16 KB; d = 64
  // gains most), 16 KB at b = 4 (32 KB: 4-10 % slower)
  static constexpr int DEC_KB = IQ_DEC_STAGE_KB ? IQ_DEC_STAGE_KB : (BITS <= 3 ? 32 : 16);
  static constexpr int STAGE_KB = (KIND == 0 && sizeof(T) == 2 && BITS >= 3 && D >= 128) ? 64
                                  : (ENC && (BITS == 3 || (KIND == 1 && BITS == 4))) ? 32
                                  : ((KIND == 1 || KIND == 2) && BITS <= 2) ? 32
                                  : ENC ? 16 : DEC_KB;
#endif
  static constexpr int TV0 = (STAGE_KB * 1024 / ROWB) / GR * GR;
  static constexpr int TILE_V = TV0 > GR ? TV0 : GR;
  static constexpr int U = TILE_V / (NWC * VPW);                  // rows per lane group per stage
  static constexpr int ENC_STAGE = TILE_V * ROWB;
  static constexpr int ENC_STAGES = (RING / ENC_STAGE) < 2 ? 2 : (RING / ENC_STAGE) < 12 ? (RING / ENC_STAGE) : 12;
  static constexpr int OPS_OFF = (ENC_STAGES * ENC_STAGE + 2 * ENC_STAGES * 8 + 64 + 127) / 128 * 128;
  static constexpr int ENC_SMEM = OPS_OFF + OPS_BYTES;             // dynamic shared memory
  // decoder stage: codes tile (16-B aligned) followed by the norms tile
  static constexpr int DEC_CODES = (TILE_V * RB + 15) / 16 * 16;
  static constexpr int DEC_STAGE = (DEC_CODES + TILE_V * 4 + 127) / 128 * 128;
  static constexpr int DEC_STAGES = (RING / DEC_STAGE) < 8 ? (RING / DEC_STAGE) : 8;
  static_assert(D % EPC == 0 && (G & (G - 1)) == 0 && CHUNKS % G == 0, "unsupported d");
  static_assert(EPL % PW == 0, "lane must own whole blocks");
  static_assert(U % 2 == 0 && TILE_V % (2 * NWC * VPW) == 0, "rows pair up");
  static_assert((G * B) % 32 == 0, "code segment must be whole words");
  static_assert(ENC_STAGES >= 2 && DEC_STAGES >= 2, "ring too shallow");
};

// Shared-memory footprint: ring + full/empty barriers + the centroid table.
template <int STAGE, int NST>
constexpr int smem_bytes() { return NST * STAGE + 2 * NST * 8 + 64; }

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
// One try_wait with a suspend-time hint: the thread is parked in hardware
// until the phase completes or the hint elapses (no issue slots burnt).
__device__ __forceinline__ bool mbar_try_wait(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n.reg .pred p;\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, 1000000;\n"
      "selp.u32 %0, 1, 0, p;\n}\n"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}
// try_wait without a suspend-time hint (the hardware's default bounded wait):
// used for barriers completed by tcgen05.commit, whose waiters otherwise sit
// out the full suspend hint
__device__ __forceinline__ bool mbar_try_wait_nohint(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n.reg .pred p;\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
      "selp.u32 %0, 1, 0, p;\n}\n"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}
// try_wait with a short suspend-time hint (~256 ns): for barriers completed
// by tcgen05.commit that a whole warp waits on -- parks the lanes instead of
// spinning (shared-memory traffic next to the tensor pipe's operand reads)
// while bounding the oversleep
__device__ __forceinline__ bool mbar_try_wait_short(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n.reg .pred p;\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, 256;\n"
      "selp.u32 %0, 1, 0, p;\n}\n"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}
__device__ __forceinline__ void mbar_wait_short(uint64_t* bar, uint32_t parity) {
  while (!mbar_try_wait_short(bar, parity)) {
  }
}
#ifndef IQ_TC_SPIN
#define IQ_TC_SPIN 1
#endif
__device__ __forceinline__ void mbar_wait_tc(uint64_t* bar, uint32_t parity) {
#if IQ_TC_SPIN
  while (!mbar_try_wait_nohint(bar, parity)) {
  }
#else
  while (!mbar_try_wait(bar, parity)) {
  }
#endif
}
// Blocking wait.  The retry loop is C++ (compiler-visible), so the compiler
// places the warp's reconvergence point (BSSY/BSYNC) right after it, before
// the shared loads and shuffles that follow.
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  while (!mbar_try_wait(bar, parity)) {
  }
}
// Warp-wide consumer wait: every lane performs its own acquire of the TMA
// data.  (A rare wrong-row failure first blamed on an asm-internal retry loop
// was later traced to the stage-release race fixed in mbar_arrive_after.)
__device__ __forceinline__ void mbar_wait_warp(uint64_t* bar, uint32_t parity, int) {
  mbar_wait(bar, parity);
}

// Release a ring stage only after the values read from it have been
// CONSUMED: `dep` is computed from every register the stage's shared-memory
// loads wrote, and the arrive is predicated on it, so the arrive cannot be
// issued before those loads have returned their data.  (Arriving right after
// issuing the loads let the TMA refill of the stage overtake an in-flight
// load when a warp had only one row pair per stage: rows mixing two tiles'
// data, observed as ~1e-5 of rows with a wrong norm on a cold first launch.)
// The predicate must be an INTEGER compare: ptxas folds a float compare
// against NaN to a constant and drops the dependency.  Lane 0's registers
// suffice: a warp-wide LDS writes back all lanes together.
__device__ __forceinline__ void mbar_arrive_after(uint64_t* bar, float dep) {
  asm volatile(
      "{\n.reg .pred p;\n"
      "setp.ne.u32 p, %1, 0x7FC00001;\n"   // always true (a NaN payload no sum produces)
      "@p mbarrier.arrive.shared::cta.b64 _, [%0];\n}\n" ::"r"(smem_u32(bar)),
      "r"(__float_as_uint(dep))
      : "memory");
}

// Programmatic dependent launch (the launcher sets the PDL attribute): the
// prologue (barrier setup, operator loads from the immutable parameters)
// overlaps the previous kernel in the stream; global reads and writes of
// the data wait for it.  Both are no-ops without the attribute.
__device__ __forceinline__ void grid_dependency_wait() {
#if IQ_PDL
  asm volatile("griddepcontrol.wait;" ::: "memory");
#endif
}
__device__ __forceinline__ void grid_launch_dependents() {
#if IQ_PDL
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
#endif
}

// 1-D TMA bulk copy global -> shared, completion counted on `bar` (bytes).
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar,
                                         uint64_t policy) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint "
      "[%0], [%1], %2, [%3], %4;" ::"r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(policy)
      : "memory");
}
__device__ __forceinline__ uint64_t policy_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t policy_evict_last() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint4 lds128(const void* p) {
  uint4 r;
  asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "r"(smem_u32(p)));
  return r;
}
__device__ __forceinline__ uint32_t lds32(const void* p) {
  uint32_t r;
  asm volatile("ld.shared.u32 %0, [%1];" : "=r"(r) : "r"(smem_u32(p)));
  return r;
}
__device__ __forceinline__ uint32_t lds32_addr(uint32_t a) {
  uint32_t r;
  asm volatile("ld.shared.u32 %0, [%1];" : "=r"(r) : "r"(a));
  return r;
}
__device__ __forceinline__ uint2 lds64_addr(uint32_t a) {
  uint2 r;
  asm volatile("ld.shared.v2.u32 {%0,%1}, [%2];" : "=r"(r.x), "=r"(r.y) : "r"(a));
  return r;
}
__device__ __forceinline__ float ldsf(const void* p) {
  float r;
  asm volatile("ld.shared.f32 %0, [%1];" : "=f"(r) : "r"(smem_u32(p)));
  return r;
}
__device__ __forceinline__ void st_stream(void* p, const uint4& v) {
#if IQ_STORE_CS
  __stcs(reinterpret_cast<uint4*>(p), v);
#else
  *reinterpret_cast<uint4*>(p) = v;
#endif
}
// MUFU square root / reciprocal square root, flush-to-zero (no denormal
// fix-up code): the norm of a row with ||x||^2 < 2^-126 is flushed.
__device__ __forceinline__ float sqrt_ftz(float x) {
  float r;
  asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}
__device__ __forceinline__ float rsqrt_ftz(float x) {
  float r;
  asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}

// ------------------------------------------------------------ packed fp32x2
__device__ __forceinline__ float2 f2(float a, float b) { return make_float2(a, b); }
__device__ __forceinline__ float2 bc(float a) { return make_float2(a, a); }
__device__ __forceinline__ float2 fma2(float2 a, float2 b, float2 c) { return __ffma2_rn(a, b, c); }
__device__ __forceinline__ float2 mul2(float2 a, float2 b) { return __fmul2_rn(a, b); }
__device__ __forceinline__ float2 add2(float2 a, float2 b) { return __fadd2_rn(a, b); }

// chunk (16 B) of two rows -> EPC coordinate pairs (row u0 in .x, u1 in .y)
template <class T> __device__ __forceinline__ void to_pairs(const uint4& a, const uint4& b, float2* p);
template <> __device__ __forceinline__ void to_pairs<float>(const uint4& a, const uint4& b, float2* p) {
  p[0] = f2(__uint_as_float(a.x), __uint_as_float(b.x));
  p[1] = f2(__uint_as_float(a.y), __uint_as_float(b.y));
  p[2] = f2(__uint_as_float(a.z), __uint_as_float(b.z));
  p[3] = f2(__uint_as_float(a.w), __uint_as_float(b.w));
}
template <class T>
__device__ __forceinline__ void to_pairs16(const uint4& a, const uint4& b, float2* p) {
  const uint32_t wa[4] = {a.x, a.y, a.z, a.w}, wb[4] = {b.x, b.y, b.z, b.w};
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const float2 ta = unpack2<T>(wa[k]);
    const float2 tb = unpack2<T>(wb[k]);
    p[2 * k] = f2(ta.x, tb.x);
    p[2 * k + 1] = f2(ta.y, tb.y);
  }
}
template <> __device__ __forceinline__ void to_pairs<__half>(const uint4& a, const uint4& b, float2* p) {
  to_pairs16<__half>(a, b, p);
}
template <> __device__ __forceinline__ void to_pairs<__nv_bfloat16>(const uint4& a, const uint4& b, float2* p) {
  to_pairs16<__nv_bfloat16>(a, b, p);
}
// EPC coordinate pairs -> the two rows' 16-byte chunks (fp16: RN-even [R15])
template <class T> __device__ __forceinline__ void from_pairs(const float2* p, uint4& a, uint4& b);
template <> __device__ __forceinline__ void from_pairs<float>(const float2* p, uint4& a, uint4& b) {
  a = make_uint4(__float_as_uint(p[0].x), __float_as_uint(p[1].x), __float_as_uint(p[2].x),
                 __float_as_uint(p[3].x));
  b = make_uint4(__float_as_uint(p[0].y), __float_as_uint(p[1].y), __float_as_uint(p[2].y),
                 __float_as_uint(p[3].y));
}
template <class T>
__device__ __forceinline__ void from_pairs16(const float2* p, uint4& a, uint4& b) {
  uint32_t wa[4], wb[4];
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    wa[k] = pack2<T>(p[2 * k].x, p[2 * k + 1].x);
    wb[k] = pack2<T>(p[2 * k].y, p[2 * k + 1].y);
  }
  a = make_uint4(wa[0], wa[1], wa[2], wa[3]);
  b = make_uint4(wb[0], wb[1], wb[2], wb[3]);
}
template <> __device__ __forceinline__ void from_pairs<__half>(const float2* p, uint4& a, uint4& b) {
  from_pairs16<__half>(p, a, b);
}
template <> __device__ __forceinline__ void from_pairs<__nv_bfloat16>(const float2* p, uint4& a, uint4& b) {
  from_pairs16<__nv_bfloat16>(p, a, b);
}

// ----------------------------------------------------------- block operator
// M (row-major PW x PW): forward y = M v, inverse v = M^T c.  4-D: M =
// L(q_L) R(conj q_R) (Full) / L(q_L) (Fast); the inverse sandwich conj(q_L)
// v q_R is exactly M^T (Proposition).  2-D: M = R(theta) and
// R(-theta) = R(theta)^T.  Forward dot products start from +0, so a
// rotated coordinate is never -0 and the sign test of the quantizer
// classifies +-0 exactly like the count definition (both go up) [R3].
template <int PW>
__device__ __forceinline__ void rot_fwd(const float* M, const float2* x, float2* y) {
#pragma unroll
  for (int i = 0; i < PW; ++i) {
    float2 a = fma2(x[0], bc(M[PW * i]), bc(0.0f));
#pragma unroll
    for (int j = 1; j < PW; ++j) a = fma2(x[j], bc(M[PW * i + j]), a);
    y[i] = a;
  }
}
template <int PW>
__device__ __forceinline__ void rot_inv(const float* M, const float2* c, float2* v) {
#pragma unroll
  for (int j = 0; j < PW; ++j) {
    float2 a = mul2(c[0], bc(M[j]));
#pragma unroll
    for (int i = 1; i < PW; ++i) a = fma2(c[i], bc(M[PW * i + j]), a);
    v[j] = a;
  }
}

// --------------------------------------------------------------- quantizer Q
// Nearest-centroid code over the symmetric fp32 codebook [R1][R2]; a tie
// takes the larger-magnitude centroid and +-0 the positive side [R3];
// out-of-range values clamp [R4]; ybar = T(x / max(rho, eps)):
//   code = h + m (ybar >= 0)  or  h - 1 - m (ybar < 0),  m = #{i >= 1 : |ybar| >= tau_i}
// The kernels rotate the raw row, y = T(x), and compare |y| with per-row
// thresholds r*tau_i, r = max(rho, eps): |ybar| >= tau <=> |y| >= r*tau (T is
// linear, r > 0) [R14c].  |y| is a free operand modifier of the compare.
// With m < h: h + m = m ^ h and h - 1 - m = m ^ (h - 1), so code = m ^ (h - s),
// s = [y < 0] (a rotated coordinate is never -0, see rot_fwd).  Decisions are
// taken in fp32, the kernel's precision [R14b].
//
// Per-row quantizer constants for a pair of rows (row A in .x, row B in .y).
template <int BITS>
struct RowQ {
  static constexpr int H = 1 << (BITS - 1);
  float2 thr[H];   // thr[i] = r * tau_i, i >= 1
  float2 c0;       // rho * cpos[0]
  float2 dl[H];    // dl[i] = rho * delta_i, i >= 1
};

template <int BITS, bool VALUE>
__device__ __forceinline__ void make_rowq(RowQ<BITS>& q, float2 rho, const KCodebook& cb) {
  constexpr int H = 1 << (BITS - 1);
  const float2 r = f2(fmaxf(rho.x, 1e-12f), fmaxf(rho.y, 1e-12f));   // max(rho, eps) [R5]
#pragma unroll
  for (int i = 1; i < H; ++i) q.thr[i] = mul2(r, bc(cb.tau[i]));
  if (VALUE) {
    q.c0 = mul2(rho, bc(cb.cpos[0]));
#pragma unroll
    for (int i = 1; i < H; ++i) q.dl[i] = mul2(rho, bc(cb.delta[i]));
  }
}

__device__ __forceinline__ float sign_xor(float c, float y) {
  return __uint_as_float(__float_as_uint(c) ^ (__float_as_uint(y) & 0x80000000u));
}

// One coordinate pair through Q.  VALUE: returns rho * (signed centroid),
// accumulated as rho*cpos[0] + sum_i [key >= r*tau_i] * rho*delta_i.  CODE:
// the two codes (count in the low mantissa bits of 2^23 + sum of indicators).
template <int BITS, bool VALUE, bool CODE>
__device__ __forceinline__ float2 quantize_pair(float2 y, const RowQ<BITS>& q, uint32_t& code_a,
                                                uint32_t& code_b) {
  constexpr int H = 1 << (BITS - 1);
  const float ka = fabsf(y.x), kb = fabsf(y.y);                     // key = |y| [R3]
  float2 c = q.c0;
  float2 m = bc(8388608.0f);  // 2^23
#pragma unroll
  for (int i = 1; i < H; ++i) {
    if constexpr (VALUE && !CODE && BITS == 3 && IQ_B3_ALU) {
      // b = 3: conditional add on the ALU (FSETP + predicated FADD) instead of
      // the indicator FFMA2 -- shifts work off the FMA pipe (+3% measured)
      c.x = ka >= q.thr[i].x ? c.x + q.dl[i].x : c.x;
      c.y = kb >= q.thr[i].y ? c.y + q.dl[i].y : c.y;
      continue;
    }
    const float2 g = f2(ka >= q.thr[i].x ? 1.0f : 0.0f, kb >= q.thr[i].y ? 1.0f : 0.0f);
    if (VALUE) c = fma2(g, q.dl[i], c);
    if (CODE) m = add2(m, g);
  }
  if (CODE) {
    const uint32_t sa = __float_as_uint(y.x) >> 31, sb = __float_as_uint(y.y) >> 31;
    code_a = (__float_as_uint(m.x) ^ (uint32_t)(H - (int)sa)) & (2u * H - 1u);
    code_b = (__float_as_uint(m.y) ^ (uint32_t)(H - (int)sb)) & (2u * H - 1u);
  }
  if (VALUE) return f2(sign_xor(c.x, y.x), sign_xor(c.y, y.y));
  return c;
}

// Same decision on a normalised pair (ybar = T(xbar)) against the codebook as
// stored (constant-bank operands, no per-row registers): centroid values are
// unscaled, the caller multiplies by rho after T^-1.
template <int BITS, bool VALUE, bool CODE>
__device__ __forceinline__ float2 quantize_pair_u(float2 y, const KCodebook& cb, uint32_t& code_a,
                                                  uint32_t& code_b) {
  constexpr int H = 1 << (BITS - 1);
  const float ka = fabsf(y.x), kb = fabsf(y.y);
  float2 c = bc(cb.cpos[0]);
  float2 m = bc(8388608.0f);
#pragma unroll
  for (int i = 1; i < H; ++i) {
    const float2 g = f2(ka >= cb.tau[i] ? 1.0f : 0.0f, kb >= cb.tau[i] ? 1.0f : 0.0f);
    if (VALUE) c = fma2(g, bc(cb.delta[i]), c);
    if (CODE) m = add2(m, g);
  }
  if (CODE) {
    const uint32_t sa = __float_as_uint(y.x) >> 31, sb = __float_as_uint(y.y) >> 31;
    code_a = (__float_as_uint(m.x) ^ (uint32_t)(H - (int)sa)) & (2u * H - 1u);
    code_b = (__float_as_uint(m.y) ^ (uint32_t)(H - (int)sb)) & (2u * H - 1u);
  }
  if (VALUE) return f2(sign_xor(c.x, y.x), sign_xor(c.y, y.y));
  return c;
}

// Codes of one 16-byte chunk (EPC coordinates) for a pair of rows, formed
// positionally: with m_e = #{i : key_e >= r*tau_i} and s_e the sign bit, the
// code is m_e ^ (h - s_e) (see above), so the chunk's LSB-first code word is
// M ^ (C - S) with M = sum_e m_e 2^(e*BITS), S = sum_e s_e 2^(e*BITS),
// C = sum_e h 2^(e*BITS) (digit-wise, no carries: m_e < h, s_e <= 1 <= h).
// M and S are accumulated exactly in fp32 as 2^23 + sum of indicator *
// 2^(position) with FFMA2 (A coordinates per accumulator keep the sum below
// 2^23), then read back from the mantissa bits.
template <int BITS, int EPC>
__device__ __forceinline__ void encode_chunk(const float2* y, const RowQ<BITS>& q, uint32_t& wa,
                                             uint32_t& wb) {
  constexpr int H = 1 << (BITS - 1);
  constexpr int A = (BITS >= 3) ? 4 : EPC;             // coordinates per accumulator
  constexpr int NACC = EPC / A;
  float2 macc[NACC], sacc[NACC];
#pragma unroll
  for (int k = 0; k < NACC; ++k) macc[k] = sacc[k] = bc(8388608.0f);
#pragma unroll
  for (int e = 0; e < EPC; ++e) {
    const float w = (float)(1u << ((e % A) * BITS));
    const float ka = fabsf(y[e].x), kb = fabsf(y[e].y);               // key = |y| [R3]
#pragma unroll
    for (int i = 1; i < H; ++i)
      macc[e / A] = fma2(f2(ka >= q.thr[i].x ? 1.0f : 0.0f, kb >= q.thr[i].y ? 1.0f : 0.0f), bc(w),
                         macc[e / A]);
    if (!IQ_SIGN_SHF)
      sacc[e / A] = fma2(f2(y[e].x < 0.0f ? 1.0f : 0.0f, y[e].y < 0.0f ? 1.0f : 0.0f), bc(w), sacc[e / A]);
  }
  uint32_t ma = 0, mb = 0, sa = 0, sb = 0;
#pragma unroll
  for (int k = 0; k < NACC; ++k) {
    ma |= (__float_as_uint(macc[k].x) - 0x4B000000u) << (k * A * BITS);
    mb |= (__float_as_uint(macc[k].y) - 0x4B000000u) << (k * A * BITS);
    if (!IQ_SIGN_SHF) {
      sa |= (__float_as_uint(sacc[k].x) - 0x4B000000u) << (k * A * BITS);
      sb |= (__float_as_uint(sacc[k].y) - 0x4B000000u) << (k * A * BITS);
    }
  }
  if (IQ_SIGN_SHF) {
    // sign bits funnelled in from the top, last coordinate first: group e
    // ends with s_e in its top bit; shift it down to bit e * BITS and mask
    uint32_t fa = 0, fb = 0, msk = 0;
#pragma unroll
    for (int e = EPC - 1; e >= 0; --e) {
      fa = __funnelshift_l(__float_as_uint(y[e].x), fa, BITS);
      fb = __funnelshift_l(__float_as_uint(y[e].y), fb, BITS);
      msk |= 1u << (e * BITS);
    }
    sa = (fa >> (BITS - 1)) & msk;
    sb = (fb >> (BITS - 1)) & msk;
  }
  uint32_t c = 0;
#pragma unroll
  for (int e = 0; e < EPC; ++e) c |= (uint32_t)H << (e * BITS);
  wa = ma ^ (c - sa);
  wb = mb ^ (c - sb);
}

// Uniform-grid decision (reading R19, tables built in params.cpp): u =
// |y| * sc with y = T(x) unnormalised and sc = S / max(rho, eps), S = 2^k,
// formed inside the FFMAs (no separate scaling pass).  Cell j =
// min(floor(u), NC - 1) (FFMA.RM against 2^23 puts floor(u) in the low
// mantissa bits), one SHFL fetches the cell's threshold, and the index
// j + [u > nextdown(threshold)] selects the magnitude entry of gval / gcode;
// the shuffles read only the index's low five bits.  Per coordinate: FFMA.RM,
// IMNMX, SHFL, FFMA, LEA.HI -- independent of the number of thresholds (7 at
// b = 4).
__device__ __forceinline__ uint32_t grid_index(float y, float sc, float gtab, uint32_t gclamp) {
  uint32_t t = __float_as_uint(__fmaf_rd(fabsf(y), sc, 8388608.0f));
  t = min(t, gclamp);
  // the table holds nextdown(threshold): u >= threshold <=> nextdown - u < 0
  // on fp32 u, and the sign bit of that difference is the increment [R3, R19]
  const float dlt = __fmaf_rn(-fabsf(y), sc, __shfl_sync(kFull, gtab, (int)t));
  return t + (__float_as_uint(dlt) >> 31);
}
// The same for a coordinate pair (row A in .x, row B in .y, per-row scales):
// the two FFMAs run as packed FFMA2 (.RM and RN), bit-identical lane by
// lane to grid_index; one FMA-pipe instruction per pair instead of two.
__device__ __forceinline__ void grid_index2(float2 y, float2 sc, float gtab, uint32_t gclamp, uint32_t& ia,
                                            uint32_t& ib) {
  const float2 ay = f2(fabsf(y.x), fabsf(y.y));
  float2 u;
  asm("{.reg .b64 a, b, c, d;\n"
      "mov.b64 a, {%2, %3}; mov.b64 b, {%4, %5}; mov.b64 c, {%6, %6};\n"
      "fma.rm.f32x2 d, a, b, c;\n"
      "mov.b64 {%0, %1}, d;}"
      : "=f"(u.x), "=f"(u.y)
      : "f"(ay.x), "f"(ay.y), "f"(sc.x), "f"(sc.y), "f"(8388608.0f));
  const uint32_t ta = min(__float_as_uint(u.x), gclamp), tb = min(__float_as_uint(u.y), gclamp);
  const float2 thr = f2(__shfl_sync(kFull, gtab, (int)ta), __shfl_sync(kFull, gtab, (int)tb));
  const float2 dlt = fma2(f2(-ay.x, -ay.y), sc, thr);
  ia = ta + (__float_as_uint(dlt.x) >> 31);
  ib = tb + (__float_as_uint(dlt.y) >> 31);
}
// signed code of a grid index: (m | h) for ybar >= 0, h - 1 - m = (m | h) ^ (2h - 1) below
template <int BITS>
__device__ __forceinline__ uint32_t grid_code(uint32_t idx, float y, uint32_t gcode) {
  const uint32_t mh = (uint32_t)__shfl_sync(kFull, (int)gcode, (int)idx);
  return mh ^ ((uint32_t)((int)__float_as_uint(y) >> 31) & ((1u << BITS) - 1u));
}
// signed centroid of a grid index (C[code], unscaled)
__device__ __forceinline__ float grid_value(uint32_t idx, float y, float gval) {
  return sign_xor(__shfl_sync(kFull, gval, (int)idx), y);
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

// Store a lane's B code bits (B % 8 == 0) at byte address p of the row: one
// aligned store for 8 / 16 / 32 bits (p is B/8-aligned), an aligned 16-bit +
// 8-bit pair for 24 bits (odd: p odd, the byte goes first).
template <int B>
__device__ __forceinline__ void store_piece(uint8_t* p, uint32_t w, int odd, bool ok) {
  if constexpr (B == 8) {
    if (ok) *p = (uint8_t)w;
  } else if constexpr (B == 16) {
    if (ok) *reinterpret_cast<uint16_t*>(p) = (uint16_t)w;
  } else if constexpr (B == 32) {
    if (ok) *reinterpret_cast<uint32_t*>(p) = w;
  } else {
    static_assert(B == 24, "byte-aligned code pieces");
    uint8_t* const p16 = p + odd;
    uint8_t* const p8 = p + (odd ? 0 : 2);
    const uint16_t v16 = (uint16_t)(odd ? (w >> 8) : w);
    const uint8_t v8 = (uint8_t)(odd ? w : (w >> 16));
    if (ok) {
      *reinterpret_cast<uint16_t*>(p16) = v16;
      *p8 = v8;
    }
  }
}

// Load a lane's block operators: lane coordinate c*EPC + e is global
// coordinate (sub + c*G)*EPC + e; block b of the lane covers lane coordinates
// b*PW .. b*PW+PW-1 (blocks never straddle a chunk since PW divides EPC).
template <class Gm>
__device__ __forceinline__ void load_ops(const float* __restrict__ mat, int sub,
                                         float (&P)[Gm::NBL][Gm::PW * Gm::PW]) {
  constexpr int PW = Gm::PW, EPC = Gm::EPC, G = Gm::G, NPB = PW * PW;
#pragma unroll
  for (int b = 0; b < Gm::NBL; ++b) {
    const int lc = b * PW;
    const int gc = (sub + (lc / EPC) * G) * EPC + lc % EPC;
    const float4* m = reinterpret_cast<const float4*>(mat + (size_t)(gc / PW) * NPB);
#pragma unroll
    for (int q = 0; q < NPB / 4; ++q) {
      const float4 t = __ldg(m + q);
      P[b][4 * q] = t.x; P[b][4 * q + 1] = t.y; P[b][4 * q + 2] = t.z; P[b][4 * q + 3] = t.w;
    }
  }
}

// Operators in shared memory: float4 q of block b of lane `sub` lives at
// float4 index (b * NQ + q) * G + sub, so the G lanes of a row read 16 G
// contiguous bytes (the VPW row groups of a warp read the same addresses:
// broadcast, no bank conflicts).  Written once per CTA by compute warp 0.
template <class Gm>
__device__ __forceinline__ void store_ops_smem(uint8_t* ops, int sub, const float (&P)[Gm::NBL][Gm::PW * Gm::PW]) {
  constexpr int NQ = Gm::PW * Gm::PW / 4;
#pragma unroll
  for (int b = 0; b < Gm::NBL; ++b)
#pragma unroll
    for (int q = 0; q < NQ; ++q)
      reinterpret_cast<float4*>(ops)[(b * NQ + q) * Gm::G + sub] =
          make_float4(P[b][4 * q], P[b][4 * q + 1], P[b][4 * q + 2], P[b][4 * q + 3]);
}
// The operator of block b: the register copy, or (OPS_SMEM) a volatile
// shared-memory read right before use, which keeps it out of the loop-
// invariant register set.
template <class Gm>
__device__ __forceinline__ void fetch_op(const float (&P)[Gm::OPS_SMEM ? 1 : Gm::NBL][Gm::PW * Gm::PW],
                                         const uint8_t* ops, int sub, int b, float (&M)[Gm::PW * Gm::PW]) {
  constexpr int NQ = Gm::PW * Gm::PW / 4;
  if constexpr (Gm::OPS_SMEM) {
#pragma unroll
    for (int q = 0; q < NQ; ++q) {
      const uint4 t = lds128(ops + 16 * ((b * NQ + q) * Gm::G + sub));
      M[4 * q] = __uint_as_float(t.x); M[4 * q + 1] = __uint_as_float(t.y);
      M[4 * q + 2] = __uint_as_float(t.z); M[4 * q + 3] = __uint_as_float(t.w);
    }
  } else {
#pragma unroll
    for (int k = 0; k < Gm::PW * Gm::PW; ++k) M[k] = P[b][k];
  }
}

// Parameter sets (R31): reload the lane's operators when the tile's set
// differs from the loaded one.  Every compute warp walks the same tiles, so
// the branch is CTA-uniform; shared-memory operators are rewritten between
// two compute-warp barriers.  Tiles never straddle sets (set_rows is a
// multiple of 256, every TILE_V divides 256).
// Rewrite the shared-memory operators of a CTA with those of `ms`, one
// float4 at a time (rolled loops: it runs only at a set change and must not
// add register pressure to the hot loop).
template <class Gm>
__device__ __forceinline__ void reload_ops_smem(const float* __restrict__ ms, int sub, uint8_t* ops) {
  constexpr int PW = Gm::PW, EPC = Gm::EPC, G = Gm::G, NPB = PW * PW, NQ = NPB / 4;
#pragma unroll 1
  for (int b = 0; b < Gm::NBL; ++b) {
    const int lc = b * PW;
    const int gc = (sub + (lc / EPC) * G) * EPC + lc % EPC;
    const float4* m = reinterpret_cast<const float4*>(ms + (size_t)(gc / PW) * NPB);
#pragma unroll 1
    for (int q = 0; q < NQ; ++q) reinterpret_cast<float4*>(ops)[(b * NQ + q) * G + sub] = __ldg(m + q);
  }
}

template <class Gm, int NWC_BAR = Gm::NWC>
__device__ __forceinline__ void switch_ops(const float* __restrict__ mat, const KCodebook& cb, int64_t v0,
                                           int& cur_set, int sub, int warp, int lane, uint8_t* ops,
                                           float (&P)[Gm::OPS_SMEM ? 1 : Gm::NBL][Gm::PW * Gm::PW]) {
  if (cb.n_sets <= 1) return;
  const int set = (int)((v0 / cb.set_rows) % cb.n_sets);
  if (set == cur_set) return;
  cur_set = set;
  const float* ms = mat + (size_t)set * cb.set_stride;
  if constexpr (Gm::OPS_SMEM) {
    asm volatile("bar.sync 1, %0;" ::"r"(NWC_BAR * 32) : "memory");   // old operators no longer read
    if (warp == 0 && lane < Gm::G) reload_ops_smem<Gm>(ms, sub, ops);
    asm volatile("bar.sync 1, %0;" ::"r"(NWC_BAR * 32) : "memory");
  } else {
    load_ops<Gm>(ms, sub, P);
  }
}

// Ring setup shared by the three kernels.
template <int NST, int NWC>
__device__ __forceinline__ void ring_init(uint64_t* full, uint64_t* empty) {
  if (threadIdx.x == 0) {
    for (int s = 0; s < NST; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], NWC);
    }
    fence_mbar_init();
  }
}

// Stage 1 for one pair of rows once their norms are known (Alg.1 l.2-18):
// forward rotation, the decision, and -- per MODE -- the code words of each
// chunk (cwa / cwb: row A / row B) and / or the reconstruction x^ (out).
// Shared by the batch encoders (k_encode) and the append kernel (k_append),
// so both take bit-identical decisions.  v: the rows' coordinate pairs, ss:
// their squared norms before the lane-group reduction is applied to rho.
template <class T, int D, int BITS, int VAR, int MODE, int KIND = MODE>
__device__ __forceinline__ void encode_pair(
    const float2 (&v)[Geo<T, D, BITS, VAR, KIND>::EPL], float2 ss, float2 rho,
    const float (&P)[Geo<T, D, BITS, VAR, KIND>::OPS_SMEM ? 1 : Geo<T, D, BITS, VAR, KIND>::NBL]
                    [Geo<T, D, BITS, VAR, KIND>::PW * Geo<T, D, BITS, VAR, KIND>::PW],
    const uint8_t* ops, int sub, const KCodebook& cb, float ctab, float gtab, float gval, uint32_t gcode,
    float2 (&out)[Geo<T, D, BITS, VAR, KIND>::EPL], uint32_t (&cwa)[Geo<T, D, BITS, VAR, KIND>::CPL],
    uint32_t (&cwb)[Geo<T, D, BITS, VAR, KIND>::CPL]) {
  using Gm = Geo<T, D, BITS, VAR, KIND>;
  constexpr int EPC = Gm::EPC, CPL = Gm::CPL, PW = Gm::PW, NBL = Gm::NBL;
  constexpr bool emit = MODE != 1;
  constexpr bool value = MODE != 0;
  constexpr bool GRID = BITS >= IQ_GRID_MIN_BITS;          // uniform-grid decision [R19]
#pragma unroll
  for (int i = 0; i < CPL; ++i) cwa[i] = cwb[i] = 0u;
  if constexpr (GRID) {
    // u = |T x| * S / max(rho, eps): the normalisation (Alg.1 l.1) and
    // the power-of-two grid scale enter as the FFMAs' multiplier [R19]
    const float2 sc = f2(rsqrt_ftz(fmaxf(ss.x, 1e-24f)) * cb.gscale,
                         rsqrt_ftz(fmaxf(ss.y, 1e-24f)) * cb.gscale);
#pragma unroll
    for (int b = 0; b < NBL; ++b) {
      float2 yb[PW], cq[PW];
      float Mb[PW * PW];
      fetch_op<Gm>(P, ops, sub, b, Mb);
      rot_fwd<PW>(Mb, v + b * PW, yb);               // T(x)  (Alg.1 l.5/9/13)
#pragma unroll
      for (int j = 0; j < PW; ++j) {
        uint32_t ia, ib;
#if IQ_GRID_PAIR
        grid_index2(yb[j], sc, gtab, cb.gclamp, ia, ib);
#else
        ia = grid_index(yb[j].x, sc.x, gtab, cb.gclamp);
        ib = grid_index(yb[j].y, sc.y, gtab, cb.gclamp);
#endif
        if constexpr (emit) {
          const int e = (b * PW + j) % EPC, c = (b * PW + j) / EPC;
          cwa[c] |= grid_code<BITS>(ia, yb[j].x, gcode) << (e * BITS);
          cwb[c] |= grid_code<BITS>(ib, yb[j].y, gcode) << (e * BITS);
        }
        if constexpr (value)                         // v^ = C[code] (sign restored)
          cq[j] = f2(grid_value(ia, yb[j].x, gval), grid_value(ib, yb[j].y, gval));
      }
      if constexpr (value) {
        rot_inv<PW>(Mb, cq, out + b * PW);           // T^-1 (l.7/11/15)
#pragma unroll
        for (int j = 0; j < PW; ++j) out[b * PW + j] = mul2(out[b * PW + j], rho);   // x^ = rho * ...
      }
    }
  } else {
  // Decision rule (R14c).  SCALED: compare y = T(x) with per-row
  // thresholds r*tau, r = max(rho, eps) (saves normalising the row).
  // K1 (MODE 0) and K3+codes (MODE 2) always use it, so they emit
  // identical codes; MODE 2 then looks C[code] up in a shuffle table and
  // rescales after T^-1.  The value-only K3 (MODE 1) also builds
  // rho*C[code] directly (no rescale) for b <= 3; for b = 4 (seven
  // thresholds, register-bound) it normalises the row and compares with
  // the codebook as stored.
  constexpr bool SCALED = MODE != 1 || BITS <= 3;
  constexpr bool RESCALE = value && !SCALED;
  RowQ<BITS> q;
  float2 inv = bc(1.0f);
  if constexpr (SCALED) {
    make_rowq<BITS, MODE == 1>(q, rho, cb);
  } else {
    inv = f2(rsqrt_ftz(fmaxf(ss.x, 1e-24f)), rsqrt_ftz(fmaxf(ss.y, 1e-24f)));   // 1/max(rho, eps)
  }

  if constexpr (!emit) {                             // K3: values only
#pragma unroll
    for (int b = 0; b < NBL; ++b) {
      float2 yb[PW], cq[PW];
      float Mb[PW * PW];
      fetch_op<Gm>(P, ops, sub, b, Mb);
      if constexpr (SCALED) {
        rot_fwd<PW>(Mb, v + b * PW, yb);           // y = T(x)  (Alg.1 l.5/9/13, [R14c])
      } else {
        float2 xb[PW];
#pragma unroll
        for (int j = 0; j < PW; ++j) xb[j] = mul2(v[b * PW + j], inv);   // xbar (l.1)
        rot_fwd<PW>(Mb, xb, yb);                     // v~ = T(xbar)
      }
#pragma unroll
      for (int j = 0; j < PW; ++j) {
        uint32_t d0, d1;
        if constexpr (SCALED) cq[j] = quantize_pair<BITS, true, false>(yb[j], q, d0, d1);
        else cq[j] = quantize_pair_u<BITS, true, false>(yb[j], cb, d0, d1);
      }
      rot_inv<PW>(Mb, cq, out + b * PW);             // x^ = T^-1(rho * v^)  (l.7/11/15)
      if constexpr (RESCALE) {
#pragma unroll
        for (int j = 0; j < PW; ++j) out[b * PW + j] = mul2(out[b * PW + j], rho);
      }
    }
  } else {                                           // K1 / K3+codes
    constexpr int BPCH = EPC / PW;                   // blocks per chunk
#pragma unroll
    for (int i = 0; i < CPL; ++i) {
      float2 yb[EPC];
      float Mc[BPCH][PW * PW];
#pragma unroll
      for (int bb = 0; bb < BPCH; ++bb) {
        fetch_op<Gm>(P, ops, sub, i * BPCH + bb, Mc[bb]);
        rot_fwd<PW>(Mc[bb], v + i * EPC + bb * PW, yb + bb * PW);             // y = T(x)
      }
      encode_chunk<BITS, EPC>(yb, q, cwa[i], cwb[i]);                       // codes of Q(y)
      if constexpr (value) {
        float2 cq[EPC];
#pragma unroll
        for (int e = 0; e < EPC; ++e)                // v^ = C[code], width-L shuffle table
          cq[e] = f2(__shfl_sync(kFull, ctab, (int)(cwa[i] >> (e * BITS)), 1 << BITS),
                     __shfl_sync(kFull, ctab, (int)(cwb[i] >> (e * BITS)), 1 << BITS));
#pragma unroll
        for (int bb = 0; bb < BPCH; ++bb) {
          float2* o = out + i * EPC + bb * PW;
          rot_inv<PW>(Mc[bb], cq + bb * PW, o);             // T^-1
#pragma unroll
          for (int j = 0; j < PW; ++j) o[j] = mul2(o[j], rho);   // x^ = rho * ...
        }
      }
    }
  }
  }  // !GRID
}

// --------------------------------------------------------- encoder (K1/K3)
// MODE 0: quantize (codes + norms).  MODE 1: fused roundtrip (y only).
// MODE 2: fused roundtrip that also writes codes and norms.
template <class T, int D, int BITS, int VAR, int MODE, bool SETS = false>
__global__ void __launch_bounds__(Geo<T, D, BITS, VAR, MODE>::CTA_THREADS,
                                  Geo<T, D, BITS, VAR, MODE>::MIN_CTAS)
k_encode(const float* __restrict__ mat, const KCodebook cb, int64_t n, const T* x, T* y,
         uint8_t* __restrict__ codes, float* __restrict__ norms) {
  using Gm = Geo<T, D, BITS, VAR, MODE>;
  constexpr int NWC = Gm::NWC;
  constexpr int EPC = Gm::EPC, G = Gm::G, CPL = Gm::CPL, VPW = Gm::VPW, U = Gm::U;
  constexpr int PW = Gm::PW, NBL = Gm::NBL, EPL = Gm::EPL, TILE_V = Gm::TILE_V;
  constexpr int B = Gm::B, W = Gm::W, RB = Gm::RB;
  constexpr int STAGE = Gm::ENC_STAGE, NST = Gm::ENC_STAGES;

  extern __shared__ __align__(128) uint8_t smem[];
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + NST * STAGE);
  uint64_t* empty = full + NST;
  ring_init<NST, NWC>(full, empty);
  __syncthreads();

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t ntiles = (n + TILE_V - 1) / TILE_V;

  if (warp == NWC) {  // ---------------- producer: TMA bulk loads into the ring
    if (lane == 0) {
      grid_dependency_wait();             // the previous kernel's writes (PDL launch)
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
      grid_launch_dependents();           // every load issued: the next kernel may launch
    }
    return;
  }
  grid_dependency_wait();                 // before this CTA's first global write

  // ---------------------------------------------------- compute warps
  const int sub = lane & (G - 1);
  const int vbase = lane & ~(G - 1);
  const int vslot = lane / G;
  float P[Gm::OPS_SMEM ? 1 : NBL][PW * PW];
  uint8_t* const ops = smem + Gm::OPS_OFF;
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
  constexpr bool emit = MODE != 1;
  constexpr bool value = MODE != 0;
  const float ctab = cb.cent[lane & ((1 << BITS) - 1)];   // C[k] in lane k of each group of L
  const float gtab = cb.gtab[lane];
  const float gval = cb.gval[lane];
  const uint32_t gcode = cb.gcode[lane];

  int s = 0;
  uint32_t ph = 0;
  int cur_set = 0;                                       // operators of set 0 are loaded
  for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
    if constexpr (SETS) switch_ops<Gm>(mat, cb, t * TILE_V, cur_set, sub, warp, lane, ops, P);   // [R31]
    mbar_wait_warp(&full[s], ph, lane);
    const uint8_t* st = smem + s * STAGE;
    const int ss_ = s;
    if (++s == NST) { s = 0; ph ^= 1; }
    // per-tile bases: row offsets below stay 32-bit, bounds are tile-local
    const int64_t v0 = t * TILE_V;
    const int nv = (n - v0) < TILE_V ? (int)(n - v0) : TILE_V;
    T* const yt = value ? y + v0 * D : nullptr;
    uint8_t* const ct = emit ? codes + v0 * RB : nullptr;
    float* const nt = emit ? norms + v0 : nullptr;

    // one pair of rows at a time (rows u in .x, u+1 in .y): keeps the live
    // state of a single pair in registers so two CTAs fit per SM
#pragma unroll kPairUnroll
    for (int u = 0; u < U; u += 2) {
      uint4 ra[CPL], rb[CPL];
      const int vl = (warp * U + u) * VPW + vslot;   // row within the tile
#pragma unroll
      for (int i = 0; i < CPL; ++i) {
        ra[i] = lds128(st + vl * Gm::ROWB + (sub + i * G) * 16);
        rb[i] = lds128(st + (vl + VPW) * Gm::ROWB + (sub + i * G) * 16);
      }
      const bool oka = vl < nv, okb = vl + VPW < nv;
      float2 v[EPL];
#pragma unroll
      for (int i = 0; i < CPL; ++i) to_pairs<T>(ra[i], rb[i], v + i * EPC);
      // Alg.1 l.1: rho = ||x||_2
#if IQ_NORM_SPLIT
      // two interleaved partial sums: half the dependent FFMA2 chain
      float2 ss = mul2(v[0], v[0]), ss1 = mul2(v[1], v[1]);
#pragma unroll
      for (int e = 2; e < EPL; e += 2) {
        ss = fma2(v[e], v[e], ss);
        ss1 = fma2(v[e + 1], v[e + 1], ss1);
      }
      ss = add2(ss, ss1);
#else
      float2 ss = mul2(v[0], v[0]);
#pragma unroll
      for (int e = 1; e < EPL; ++e) ss = fma2(v[e], v[e], ss);
#endif
      if (u + 2 == U) {                                // last rows consumed: release the stage
        __syncwarp();
        if (lane == 0) mbar_arrive_after(&empty[ss_], ss.x + ss.y);
      }
#pragma unroll
      for (int o = G / 2; o >= 1; o >>= 1)
        ss = add2(ss, f2(__shfl_xor_sync(kFull, ss.x, o), __shfl_xor_sync(kFull, ss.y, o)));
      const float2 rho = f2(sqrt_ftz(ss.x), sqrt_ftz(ss.y));
      float2 out[EPL];
      uint32_t cwa[CPL], cwb[CPL];
      encode_pair<T, D, BITS, VAR, MODE>(v, ss, rho, P, ops, sub, cb, ctab, gtab, gval, gcode, out, cwa, cwb);
#pragma unroll
      for (int i = 0; i < CPL; ++i) {
        if constexpr (value) {
          uint4 oa, ob;
          from_pairs<T>(out + i * EPC, oa, ob);
          const int off = vl * D + (sub + i * G) * EPC;
          if (oka) st_stream(yt + off, oa);
          if (okb) st_stream(yt + off + VPW * D, ob);
        }
        if constexpr (emit && IQ_BYTE_CODES && B % 8 == 0) {
          // the lane's B code bits of chunk sub + i G are whole bytes of the
          // row (LSB-first [R7]): store them in place, no gather shuffles
          uint8_t* const pa = ct + vl * RB + (sub + i * G) * (B / 8);
          store_piece<B>(pa, cwa[i], (sub + i * G) & 1, oka);
          store_piece<B>(pa + VPW * RB, cwb[i], (sub + i * G) & 1, okb);
        } else if constexpr (emit) {
          const uint32_t wa = gather_word<G, B>(cwa[i], sub, vbase);
          const uint32_t wb = gather_word<G, B>(cwb[i], sub, vbase);
          if (sub < W) {
            const int off = vl * RB + 4 * (i * W + sub);
            if (oka) *reinterpret_cast<uint32_t*>(ct + off) = wa;
            if (okb) *reinterpret_cast<uint32_t*>(ct + off + VPW * RB) = wb;
          }
        }
      }
      if (emit && sub == 0) {
        if (oka) nt[vl] = rho.x;
        if (okb) nt[vl + VPW] = rho.y;
      }
    }
  }
}


// ------------------------------------------- quantize-on-append (KV cache)
// One new row per cache slot r (a (layer, head) pair, r = layer * heads +
// head) quantized straight into a strided cache during decoding (P:460,
// P:477): codes row r * cap + pos_r (RB bytes), norms[r * cap + pos_r], with
// the operators of parameter set r % n_sets [R31] and K1's lane geometry and
// decision code (encode_pair), so the codes and norms are bit-identical to
// iq_quantize of the same row with the same set.  One lane group per row,
// rows read with 128-bit loads (a decode step moves a few hundred rows: the
// kernel is latency-bound, not a bandwidth kernel).  A lane group whose row
// does not exist mirrors the last row (its shuffles need the whole warp) and
// stores nothing; a position outside [0, cap) stores nothing.
template <class T, int D, int BITS, int VAR>
__global__ void __launch_bounds__(256)
k_append(const float* __restrict__ mat, const KCodebook cb, int64_t n_rows, const T* __restrict__ x,
         uint8_t* __restrict__ codes, float* __restrict__ norms, int64_t cap, const int64_t* __restrict__ positions,
         int64_t position) {
  using Gm = Geo<T, D, BITS, VAR, 5>;
  constexpr int EPC = Gm::EPC, G = Gm::G, CPL = Gm::CPL, VPW = Gm::VPW, PW = Gm::PW, NBL = Gm::NBL;
  constexpr int EPL = Gm::EPL, B = Gm::B, W = Gm::W, RB = Gm::RB;
  static_assert(!Gm::OPS_SMEM, "append: operators in registers");
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int sub = lane & (G - 1), vbase = lane & ~(G - 1), vslot = lane / G;
  const int64_t r = ((int64_t)blockIdx.x * (blockDim.x >> 5) + warp) * VPW + vslot;
  if (((int64_t)blockIdx.x * (blockDim.x >> 5) + warp) * VPW >= n_rows) return;   // warp-uniform
  const int64_t rr = r < n_rows ? r : n_rows - 1;
  const int64_t pos = positions ? positions[rr] : position;
  const bool store = r < n_rows && pos >= 0 && pos < cap;
  const int set = cb.n_sets > 1 ? (int)(rr % cb.n_sets) : 0;
  float P[NBL][PW * PW];
  load_ops<Gm>(mat + (size_t)set * cb.set_stride, sub, P);
  const T* xr = x + rr * D;
  uint4 ra[CPL];
#pragma unroll
  for (int i = 0; i < CPL; ++i) ra[i] = __ldg(reinterpret_cast<const uint4*>(xr + (sub + i * G) * EPC));
  float2 v[EPL];
#pragma unroll
  for (int i = 0; i < CPL; ++i) to_pairs<T>(ra[i], ra[i], v + i * EPC);
  // Alg.1 l.1: rho = ||x||_2, in k_encode's summation order
#if IQ_NORM_SPLIT
  float2 ss = mul2(v[0], v[0]), ss1 = mul2(v[1], v[1]);
#pragma unroll
  for (int e = 2; e < EPL; e += 2) {
    ss = fma2(v[e], v[e], ss);
    ss1 = fma2(v[e + 1], v[e + 1], ss1);
  }
  ss = add2(ss, ss1);
#else
  float2 ss = mul2(v[0], v[0]);
#pragma unroll
  for (int e = 1; e < EPL; ++e) ss = fma2(v[e], v[e], ss);
#endif
#pragma unroll
  for (int o = G / 2; o >= 1; o >>= 1)
    ss = add2(ss, f2(__shfl_xor_sync(kFull, ss.x, o), __shfl_xor_sync(kFull, ss.y, o)));
  const float2 rho = f2(sqrt_ftz(ss.x), sqrt_ftz(ss.y));
  const float ctab = cb.cent[lane & ((1 << BITS) - 1)];
  float2 out[EPL];
  uint32_t cwa[CPL], cwb[CPL];
  encode_pair<T, D, BITS, VAR, 0, 5>(v, ss, rho, P, nullptr, sub, cb, ctab, cb.gtab[lane], cb.gval[lane],
                                     cb.gcode[lane], out, cwa, cwb);
  uint8_t* cr = codes + (rr * cap + pos) * RB;
#pragma unroll
  for (int i = 0; i < CPL; ++i) {
    if constexpr (IQ_BYTE_CODES && B % 8 == 0) {
      store_piece<B>(cr + (sub + i * G) * (B / 8), cwa[i], (sub + i * G) & 1, store);
    } else {
      const uint32_t w = gather_word<G, B>(cwa[i], sub, vbase);
      if (store && sub < W) *reinterpret_cast<uint32_t*>(cr + 4 * (i * W + sub)) = w;
    }
  }
  if (store && sub == 0) norms[rr * cap + pos] = rho.x;
}

// ---------------------------------------------------------------- decoder (K2)
// Ring stage = TILE_V rows of packed codes (RB bytes each) + their norms.
// One row per lane group at a time; coordinates are processed in adjacent
// pairs (e, e+1) so the inverse rotation is v_(j,j+1) = sum_i
// (M_ij, M_i,j+1) * c_i: row pairs of the row-major operator times a
// broadcast centroid, and the fp16 pack takes (v_j, v_j+1) as is.  The
// centroid lookup C[code] is a warp shuffle from a register table
// (lane k of every aligned group of L lanes holds C[k]); the shuffle's
// width-L source index does the masking of the code field.
template <class T, int D, int BITS, int VAR, bool SETS = false>
__global__ void __launch_bounds__(Geo<T, D, BITS, VAR, 3>::CTA_THREADS,
                                  Geo<T, D, BITS, VAR, 3>::MIN_CTAS)
k_decode(const float* __restrict__ mat, const KCodebook cb, int64_t n,
         const uint8_t* __restrict__ codes, const float* __restrict__ norms, T* __restrict__ y) {
  using Gm = Geo<T, D, BITS, VAR, 3>;
  constexpr int NWC = Gm::NWC;
  constexpr int EPC = Gm::EPC, G = Gm::G, CPL = Gm::CPL, VPW = Gm::VPW, U = Gm::U;
  constexpr int PW = Gm::PW, NBL = Gm::NBL, EPL = Gm::EPL, TILE_V = Gm::TILE_V;
  constexpr int B = Gm::B, RB = Gm::RB;
  constexpr int STAGE = Gm::DEC_STAGE, NST = Gm::DEC_STAGES, CODES_B = Gm::DEC_CODES;
  constexpr int L = 1 << BITS;

  extern __shared__ __align__(128) uint8_t smem[];
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + NST * STAGE);
  uint64_t* empty = full + NST;
  ring_init<NST, NWC>(full, empty);
  __syncthreads();

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t ntiles = (n + TILE_V - 1) / TILE_V;

  if (warp == NWC) {
    if (lane == 0) {
      grid_dependency_wait();             // the previous kernel's writes (PDL launch)
      const uint64_t pol = policy_evict_first();
      int s = 0;
      uint32_t ph = 0;
      for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
        mbar_wait(&empty[s], ph ^ 1);
        const int64_t v0 = t * TILE_V;
        const int64_t nv = (n - v0) < TILE_V ? (n - v0) : TILE_V;
        // bulk copies move whole 16-byte units; a ragged tail of the codes or
        // norms arrays is read directly from global memory by the consumers
        const uint32_t c16 = (uint32_t)(nv * RB) & ~15u, n16 = (uint32_t)(nv * 4) & ~15u;
        if (c16 + n16 == 0) {
          mbar_arrive(&full[s]);
        } else {
          mbar_arrive_expect_tx(&full[s], c16 + n16);
          if (c16) bulk_g2s(smem + s * STAGE, codes + v0 * RB, c16, &full[s], pol);
          if (n16) bulk_g2s(smem + s * STAGE + CODES_B, norms + v0, n16, &full[s], pol);
        }
        if (++s == NST) { s = 0; ph ^= 1; }
      }
      grid_launch_dependents();
    }
    return;
  }
  grid_dependency_wait();                 // before this CTA's first global access

  const int sub = lane & (G - 1);
  const int vslot = lane / G;
  float P[NBL][PW * PW];
  load_ops<Gm>(mat, sub, P);
  const float ctab = cb.cent[lane & (L - 1)];   // C[k] in lane k of each group of L

  int s = 0;
  uint32_t ph = 0;
  int cur_set = 0;
  for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
    if constexpr (SETS) switch_ops<Gm>(mat, cb, t * TILE_V, cur_set, sub, warp, lane, nullptr, P);   // [R31]
    mbar_wait_warp(&full[s], ph, lane);
    const uint8_t* st = smem + s * STAGE;
    const int64_t v0 = t * TILE_V;
    const int64_t nv = (n - v0) < TILE_V ? (n - v0) : TILE_V;
    uint32_t bits[U][CPL];
    float rho[U];
    if (nv == TILE_V && ((TILE_V * RB) % 16 == 0)) {   // full tile: everything is in smem
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int vl = (warp * U + u) * VPW + vslot;
#pragma unroll
        for (int i = 0; i < CPL; ++i) {
          const int bit0 = (i * G + sub) * B;        // this lane's bits in the row stream
          const int byte0 = vl * RB + (bit0 >> 5) * 4, sh = bit0 & 31;
          uint32_t r = lds32(st + byte0);
          if (B < 32 && sh + B > 32) r = __funnelshift_r(r, lds32(st + byte0 + 4), sh);
          else if (sh) r >>= sh;
          bits[u][i] = r;
        }
        rho[u] = ldsf(st + CODES_B + vl * 4);
      }
    } else {                                           // tail tile: direct loads
      const int64_t c16 = (nv * RB) & ~(int64_t)15, n16 = (nv * 4) & ~(int64_t)15;
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int vl = (warp * U + u) * VPW + vslot;
        const bool valid = vl < nv;
#pragma unroll
        for (int i = 0; i < CPL; ++i) {
          const int bit0 = (i * G + sub) * B;
          const int byte0 = vl * RB + (bit0 >> 5) * 4, sh = bit0 & 31;
          uint32_t lo = 0, hi = 0;
          if (valid) {
            lo = (byte0 + 4 <= c16) ? lds32(st + byte0)
                                    : __ldg(reinterpret_cast<const unsigned*>(codes + v0 * RB + byte0));
            if (B < 32 && sh + B > 32)
              hi = (byte0 + 8 <= c16) ? lds32(st + byte0 + 4)
                                      : __ldg(reinterpret_cast<const unsigned*>(codes + v0 * RB + byte0 + 4));
          }
          bits[u][i] = (B < 32 && sh + B > 32) ? __funnelshift_r(lo, hi, sh) : (lo >> sh);
        }
        rho[u] = valid ? ((vl * 4 + 4 <= n16) ? ldsf(st + CODES_B + vl * 4) : __ldg(norms + v0 + vl)) : 0.0f;
      }
    }
    {
      float dep = 0.0f;                                 // consume every loaded word
#pragma unroll
      for (int u = 0; u < U; ++u) {
        dep += rho[u];
#pragma unroll
        for (int i = 0; i < CPL; ++i) dep += __uint_as_float(bits[u][i] & 0x007FFFFFu);
      }
      __syncwarp();
      if (lane == 0) mbar_arrive_after(&empty[s], dep);
    }
    if (++s == NST) { s = 0; ph ^= 1; }

#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t v = v0 + (warp * U + u) * VPW + vslot;
      const float2 r2 = bc(rho[u]);
      float2 out[EPL / 2];
#pragma unroll
      for (int b = 0; b < NBL; ++b) {
        float c[PW];
#pragma unroll
        for (int j = 0; j < PW; ++j) {
          const int lc = b * PW + j;
          // v^ = C[code]: width-L shuffle masks the BITS-wide field itself
          c[j] = __shfl_sync(kFull, ctab, (int)(bits[u][lc / EPC] >> ((lc % EPC) * BITS)), L);
        }
#pragma unroll
        for (int jp = 0; jp < PW; jp += 2) {           // T^-1 on coordinate pairs
          float2 a = mul2(f2(P[b][jp], P[b][jp + 1]), bc(c[0]));
#pragma unroll
          for (int i = 1; i < PW; ++i) a = fma2(f2(P[b][PW * i + jp], P[b][PW * i + jp + 1]), bc(c[i]), a);
          out[(b * PW + jp) / 2] = mul2(a, r2);        // x^ = rho * ...
        }
      }
      if (v < n) {
#pragma unroll
        for (int i = 0; i < CPL; ++i) {
          uint4 o;
          if constexpr (EPC == 8) {
            uint32_t w[4];
#pragma unroll
            for (int k = 0; k < 4; ++k) w[k] = pack2<T>(out[i * 4 + k].x, out[i * 4 + k].y);
            o = make_uint4(w[0], w[1], w[2], w[3]);
          } else {
            o = make_uint4(__float_as_uint(out[i * 2].x), __float_as_uint(out[i * 2].y),
                           __float_as_uint(out[i * 2 + 1].x), __float_as_uint(out[i * 2 + 1].y));
          }
          st_stream(y + v * D + (size_t)(sub + i * G) * EPC, o);
        }
      }
    }
  }
}

// ------------------------------------------------ reconstruction statistics
template <class T> __device__ __forceinline__ void to_f32(const uint4& r, float* f);
template <> __device__ __forceinline__ void to_f32<float>(const uint4& r, float* f) {
  f[0] = __uint_as_float(r.x); f[1] = __uint_as_float(r.y);
  f[2] = __uint_as_float(r.z); f[3] = __uint_as_float(r.w);
}
template <class T> __device__ __forceinline__ void to_f32_16(const uint4& r, float* f) {
  const uint32_t w[4] = {r.x, r.y, r.z, r.w};
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const float2 t = unpack2<T>(w[k]);
    f[2 * k] = t.x; f[2 * k + 1] = t.y;
  }
}
template <> __device__ __forceinline__ void to_f32<__half>(const uint4& r, float* f) { to_f32_16<__half>(r, f); }
template <> __device__ __forceinline__ void to_f32<__nv_bfloat16>(const uint4& r, float* f) {
  to_f32_16<__nv_bfloat16>(r, f);
}

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
