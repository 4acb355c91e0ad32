// Internal declarations shared by the host parameter builder, the C ABI and
// the kernel launchers.  Not installed; the public ABI is include/isoquant.h.
#pragma once
#include <cstdint>
#include <string>
#include <vector>

#include "isoquant.h"

namespace iq {

constexpr int kMaxBits = 4;
constexpr int kMaxHalf = 1 << (kMaxBits - 1);  // h = L/2 <= 8

// Codebook as the kernels see it (passed by value as a kernel parameter, so
// it lives in the constant bank and is read through uniform registers).
// Symmetric [R2]: C_{h+m} = cpos[m], C_{h-1-m} = -cpos[m]; thresholds
// t_{h-1} = 0, t_{h-1+m} = tau[m] = -t_{h-1-m} for m = 1..h-1.
struct KCodebook {
  float cpos[kMaxHalf];        // positive centroids, ascending
  float tau[kMaxHalf];         // tau[0] = 0, tau[m] m>=1 positive thresholds
  uint32_t tau_bits[kMaxHalf]; // bit patterns of tau (non-negative floats)
  float cent[2 * kMaxHalf];    // all L centroids ascending (decode lookup)
  float delta[kMaxHalf];       // delta[m] m>=1: fp32 step with fl(cpos[m-1] + delta[m])
                               // == cpos[m] exactly, so an FMA chain over the
                               // decision indicators lands exactly on C[code]
  // Uniform-grid decision tables (reading R19).  u = |T x| * S /
  // max(rho, eps) (gscale S a power of two, formed inside FFMA) falls in cell
  // j = min(floor(u), NC - 1); each cell holds at most one positive threshold,
  // so the magnitude code is m_start(j) + [u > nextdown(tau S)] and, because
  // the upper part of cell j has the code of the start of cell j + 1, the
  // value / code lookup index is j + that increment.
  float gscale;                // S = 2^k
  uint32_t gclamp;             // bit pattern of 2^23 + (NC - 1)
  float gtab[32];              // [j] = nextdown(tau * S) of the threshold in cell j (else +inf)
  float gval[32];              // [j] = cpos[m_start(j)]
  uint32_t gcode[32];          // [j] = m_start(j) | h  (code magnitude, sign added later)
  // Parameter sets (R31): row r uses the operators of set
  // (r / set_rows) % n_sets, at mat + set * set_stride; n_sets = 1: one set.
  int64_t set_rows;
  int32_t n_sets;
  int32_t set_stride;
};

// Host-side parameter construction (params.cpp): the reference generator of
// DESIGN.md [R12] and the Lloyd-Max codebook [R1][R2].
struct HostParams {
  int d = 0, bits = 0, variant = 0;
  uint64_t seed = 0;
  int n_sets = 1;                  // parameter sets (R31): rot / mat hold n_sets copies
  int64_t set_rows = 0;
  std::vector<double> rot;        // canonical fp64 (see iq_export_params)
  std::vector<float> mat;         // device operator, fp32 (see iq_export_block_matrices)
  std::vector<float> centroids;   // [L] fp32 ascending
  std::vector<float> thresholds;  // [L-1] fp32 ascending
  KCodebook kcb{};
  // Stage-2 residual sketch (R20): S [m = d][d] of fp16-rounded
  // N(0,1) draws, row-major half bits, and the UMMA operand image (K-major,
  // 128-byte swizzle) the sketch kernel copies into shared memory.
  bool has_qjl = false;
  std::vector<uint16_t> qjl_half;
  std::vector<uint8_t> qjl_img;
  std::vector<uint8_t> qjl_img_a;   // the same S as a 128-row A operand (rows >= m zero)
  // S' = S M^T (M the fp32 block operators of mat): z = S r = S' (M r), so the
  // 16-bit sketch kernel works on the forward-rotated residual; fp16 hi and
  // lo parts (S' to ~2^-22), two K-major 128B-swizzled B images back to back
  std::vector<uint8_t> qjl_img_rot;
};

// n_sets - 1 further rotation sets (set s from seed + s, R31) appended to
// rot / mat; set_rows rows per set.
bool add_param_sets(HostParams* hp, int n_sets, int64_t set_rows, std::string* err);

// Sketch generator key and layout (params.cpp).
bool build_qjl(HostParams* hp, std::string* err);
bool qjl_supported(int d);   // GPU sketch: d in {64, 128} (fused kernel), {256, 512} (quantize + sketch kernel)
bool qjl_fused(int d);       // d in {64, 128}: one fused stage-1 + sketch kernel
// byte offset of element (row r, k) in a K-major 128B-swizzled UMMA operand
// with `rows` rows: K slabs of 64 fp16, 8-row atoms of 1024 B
#ifdef __CUDACC__
#define IQ_HD __host__ __device__
#else
#define IQ_HD
#endif
IQ_HD inline uint32_t umma_sw128_off(int r, int k, int rows) {
  return static_cast<uint32_t>((k / 64) * (rows / 8) * 1024 + (r / 8) * 1024 + (r % 8) * 128 +
                               ((((k % 64) / 8) ^ (r % 8)) * 16) + (k % 8) * 2);
}

// Returns false with a message on invalid input.  rot_in (nullable): explicit
// rotation parameters in the iq_export_params layout (normalised on input)
// instead of the seeded generator.
bool build_host_params(int d, int bits, int variant, uint64_t seed, HostParams* hp,
                       std::string* err, const double* rot_in = nullptr);
// dL/dM_b (row-major PW x PW per block) -> dL/d(rot) in the export layout,
// projected on the tangent space of the unit sphere (R30)
void operator_grad_to_rot(const HostParams& hp, const double* G, double* grad_rot);
size_t rotation_param_count(int d, int variant);
size_t block_matrix_count(int d, int variant);

// Kernel launchers (kernels.cu).  Each returns a cudaError_t as int.
struct LaunchArgs {
  const float* mat;   // device operator
  KCodebook cb;
  int64_t n;
  const void* x;
  void* y;
  uint8_t* codes;
  float* norms;
  const uint8_t* codes_in;
  const float* norms_in;
  // attention consumer (k_attn_scores)
  int heads;
  int n_q;
  const void* q;
  float* scores;
  const uint8_t* qjl_in;
  const float* rnorms_in;
  const uint8_t* qjl_img_a;
  const uint8_t* qjl_img_rot;
  double* grad;             // distortion gradient [block_matrix_count] (accumulated)
  double* loss;             // distortion sum (accumulated, nullable)
  double* sums;
  void* stream;
  const uint8_t* qjl_img;   // device UMMA image of S (stage 2)
  uint8_t* qjl;             // [n, d/8] sketch sign bits (stage 2)
  float* rnorms;            // [n] residual norms (stage 2)
  // quantize-on-append (k_append): cache of n rows x cap tokens
  int64_t cap;
  const int64_t* positions; // device [n] or null (then `position` for every row)
  int64_t position;
};

enum class Kernel { kQuantize = 0, kDequantize = 1, kRoundtrip = 2, kErrorSums = 3, kQuantizeQjl = 4, kAttnScores = 5, kDistortionGrad = 6, kAppend = 7, kQjlSketch = 8 };

// Dispatch to the template instance for (kernel, variant, dtype, d, bits).
// Returns: 0 ok, -1 unsupported configuration, else the CUDA error code.
int launch(Kernel k, int variant, int dtype, int d, int bits, const LaunchArgs& a);
bool attn_supported(int d);   // attention consumer: d in {64, 128, 256, 512} (stage 2: 64, 128)
bool gpu_supported(int d, int bits, int variant);

}  // namespace iq
