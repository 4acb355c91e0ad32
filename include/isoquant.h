/*
 * isoquant.h — C ABI of the B200-native IsoQuant stage-1 library
 * (libisoquant.so, built from paper_2603_28430_b200/csrc).
 *
 * What it computes: the stage-1 quantize -> dequantize path of IsoQuant
 * (arXiv 2603.28430), Algorithm 1:
 *   rho = ||x||_2,  xbar = x / max(rho, eps)
 *   per 4-D block v (Full/Fast) or 2-D pair u (planar):
 *     Full : v~ = q_L v conj(q_R), v^ = Q(v~), v_rec = conj(q_L) v^ q_R
 *     Fast : v~ = q_L v,           v^ = Q(v~), v_rec = conj(q_L) v^
 *     2D   : u~ = R(theta) u,      u^ = Q(u~), u_rec = R(-theta) u^
 *   x^ = rho * concat(v_rec)
 * Q is nearest-centroid coding against one shared Lloyd-Max codebook per
 * (d, bits); codes are b-bit, packed LSB-first per row.
 * Readings of points the paper leaves open are listed in DESIGN.md (R1..R18).
 *
 * Conventions for every entry point:
 *  - All functions are extern "C", never throw, never abort, and return an
 *    iq_status.  On failure a human-readable reason is available from
 *    iq_last_error_detail() (thread-local, valid until the next failing call
 *    on the same thread).
 *  - Arguments are validated synchronously BEFORE anything is launched.
 *  - Compute entry points (iq_quantize / iq_dequantize / iq_roundtrip /
 *    iq_error_sums) enqueue exactly ONE kernel on the caller's stream and
 *    return without synchronizing.  They never allocate.  Faults inside the
 *    kernel surface at the caller's next synchronization.  n == 0 returns
 *    IQ_OK and launches nothing.
 *  - Pointers named x, y, codes, norms, sums are DEVICE pointers on the
 *    params' device, which must be the calling thread's current CUDA device
 *    (else IQ_ERR_DEVICE_MISMATCH).  x and y must be 16-byte aligned, codes
 *    and norms 4-byte aligned for iq_quantize / iq_roundtrip and 16-byte
 *    aligned for iq_dequantize, whose kernel reads them with TMA bulk copies
 *    (else IQ_ERR_MISALIGNED).  The caller owns all
 *    tensors; the library keeps no reference after the call returns.
 *  - cuda_stream is a cudaStream_t passed as void* (NULL = legacy default).
 *  - Thread-safety: an iq_params handle is immutable after creation and may
 *    be used concurrently from any number of threads and streams.
 *  - NaN/Inf inputs and fp32 inputs with ||x||^2 beyond the fp32 range give
 *    unspecified (but memory-safe) outputs.
 *
 * Layouts (row-major, rows contiguous, no padding between rows):
 *  - x, y   : [n, d] of dtype (IQ_DTYPE_F32 = float, IQ_DTYPE_F16 = IEEE half,
 *             IQ_DTYPE_BF16 = bfloat16); kernels compute in fp32 for every dtype
 *  - codes  : [n, iq_code_bytes_per_vector(d, bits)] uint8; row r holds the
 *             bitstream in which bit (j*bits + m) is bit m of coordinate j's
 *             code, byte B holding stream bits 8B..8B+7 from its LSB up.
 *             A code is the index k in [0, 2^bits) of the centroid C_k
 *             (C ascending) nearest to the rotated normalised coordinate y:
 *             code = #{k : y >= t_k} for y >= 0 and #{k : y > t_k} for y < 0
 *             (a tie takes the larger-magnitude centroid, +-0 the positive
 *             side; out-of-range values clamp) — DESIGN.md reading R3.
 *  - norms  : [n] float, rho = ||x||_2 computed in fp32 (stored as is, not
 *             max(rho, eps)).
 */
#ifndef ISOQUANT_H_
#define ISOQUANT_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define IQ_ABI_VERSION 1

typedef enum iq_status {
  IQ_OK = 0,
  IQ_ERR_INVALID_ARGUMENT = 1, /* null handle/pointer, n < 0, bad enum value      */
  IQ_ERR_UNSUPPORTED = 2,      /* (d, bits, variant, dtype) outside the GPU set   */
  IQ_ERR_MISALIGNED = 3,       /* x/y not 16-B aligned, codes/norms not 4-B       */
  IQ_ERR_DEVICE_MISMATCH = 4,  /* current device != params device, or host-only  */
  IQ_ERR_CUDA = 5,             /* a CUDA runtime call failed (detail has text)    */
  IQ_ERR_OUT_OF_MEMORY = 6,    /* device/pinned allocation failed                 */
  IQ_ERR_BUFFER_TOO_SMALL = 7  /* an export buffer length is too small            */
} iq_status;

typedef enum iq_variant {
  IQ_VARIANT_FULL = 0,     /* T(v) = q_L v conj(q_R) */
  IQ_VARIANT_FAST = 1,     /* T(v) = q_L v */
  IQ_VARIANT_PLANAR2D = 2  /* u -> R(theta) u on pairs */
} iq_variant;

typedef enum iq_dtype {
  IQ_DTYPE_F32 = 0,
  IQ_DTYPE_F16 = 1,
  IQ_DTYPE_BF16 = 2   /* bfloat16 storage (R28; not in the paper) */
} iq_dtype;

typedef struct iq_params iq_params; /* opaque, immutable after creation */

/* Library identification and error reporting. */
const char* iq_version(void);
int iq_abi_version(void);
const char* iq_status_string(iq_status s);
const char* iq_last_error_detail(void);

/*
 * iq_make_params — build the per-configuration parameters once (host).
 *  d       : vector width.  GPU path: d in {64, 128, 256, 512}.
 *            (Any d >= 1 is accepted when device < 0, for export only.)
 *  bits    : code width b in {1, 2, 3, 4} (the paper uses 2..4).
 *  variant : iq_variant.
 *  seed    : 64-bit seed of the counter-based parameter generator [R12]:
 *            SplitMix64 -> 53-bit uniforms -> Box-Muller; each quaternion is
 *            a normalised N(0, I_4) draw ("Gaussian-normalize sampling on
 *            S^3"); 2D angles theta = 2*pi*U.
 *  device  : CUDA device ordinal that will run the kernels, or -1 for a
 *            host-only handle (parameter export, no device memory).
 *  out     : receives the handle; release with iq_free_params.
 * The codebook is the Gaussian Lloyd-Max quantizer scaled by 1/sqrt(d) [R1],
 * exactly symmetric [R2], rounded to fp32; thresholds are fp32 midpoints of
 * adjacent fp32 centroids.  Cost: O(d) host work + one small H2D copy.
 * Errors: INVALID_ARGUMENT, UNSUPPORTED, CUDA, OUT_OF_MEMORY.
 */
iq_status iq_make_params(int d, int bits, int variant, uint64_t seed, int device,
                         iq_params** out);

/*
 * iq_make_params_sets — n_sets independent rotation sets in one handle
 * (per-(layer, head) parameters; R31): set s
 * is what iq_make_params builds from seed + s; the codebook is shared.  Rows
 * are laid out set-major: row r of any call uses set (r / set_rows) %
 * n_sets (a KV cache [layers, heads, tokens, d] with set_rows = tokens gives
 * one set per (layer, head)); iq_attention_scores uses set h % n_sets for
 * head h, iq_append_kv set r % n_sets for cache slot r.  set_rows >= 1;
 * the batch kernels (iq_quantize / iq_dequantize / iq_roundtrip / the host
 * pipeline) switch sets per tile and need set_rows to be a multiple of 256
 * (else UNSUPPORTED); iq_append_kv and iq_attention_scores take any set_rows
 * (sets finer than 256 rows, e.g. one set per (layer, head) with one row per
 * set per decode step).  The stage-2 sketch takes sets through
 * iq_make_params_qjl_sets; the distortion gradient does not (UNSUPPORTED).
 */
iq_status iq_make_params_sets(int d, int bits, int variant, uint64_t seed, int n_sets, int64_t set_rows,
                              int device, iq_params** out);

/* iq_make_params_sets plus the stage-2 sketch S (one S for every set, R20):
 * iq_quantize_qjl then uses set (r / set_rows) % n_sets for row r (set_rows a
 * multiple of 256, else UNSUPPORTED).  At d in {64, 128} the set-switching
 * sketch kernel forms the residual in the input domain (r = x - x^ against
 * S), since the rotated-domain operator S M^T would be per set. */
iq_status iq_make_params_qjl_sets(int d, int bits, int variant, uint64_t seed, int n_sets, int64_t set_rows,
                                  int device, iq_params** out);

/* n_sets and set_rows of a handle (1 and 0 for a single-set handle). */
iq_status iq_params_sets_info(const iq_params* p, int* n_sets, int64_t* set_rows);

/* Rotation parameters of one set (iq_export_params exports set 0). */
iq_status iq_export_params_set(const iq_params* p, int set, double* rot, size_t rot_len);

/* Release a handle (NULL is a no-op).  The caller guarantees no kernel that
 * uses it is still in flight. */
iq_status iq_free_params(iq_params* p);

/* Read back the configuration of a handle (any out pointer may be NULL). */
iq_status iq_params_info(const iq_params* p, int* d, int* bits, int* variant,
                         int* device);

/* Packed code bytes per row: ceil(d * bits / 8) (d padded to the block width
 * is d itself on the GPU path). */
size_t iq_code_bytes_per_vector(int d, int bits);

/* Number of fp64 rotation parameters iq_export_params writes: Full 8*ceil(d/4),
 * Fast 4*ceil(d/4), 2D 2*ceil(d/2) — the Params column of Table 1 and the
 * formulas of P:333. */
size_t iq_rotation_param_count(int d, int variant);

/*
 * iq_export_params — copy the canonical parameters to host buffers.
 *  rot        : fp64, Full [g][8] = (q_L w,x,y,z, q_R w,x,y,z) per block,
 *               Fast [g][4] = q_L, 2D [g2][2] = (cos theta, sin theta).
 *  centroids  : fp32 [2^bits] ascending.
 *  thresholds : fp32 [2^bits - 1] ascending.
 * Any pointer may be NULL to skip that output; lengths are element counts.
 * Errors: INVALID_ARGUMENT, BUFFER_TOO_SMALL.
 */
iq_status iq_export_params(const iq_params* p, double* rot, size_t rot_len,
                           float* centroids, size_t centroids_len,
                           float* thresholds, size_t thresholds_len);

/* The fp32 per-block operator the kernels apply (4-D variants: [g][16]
 * row-major M with y = M v, inverse y' = M^T v; 2D: [g2][4] = (c, -s, s, c)).
 * M = L(q_L) R(conj q_R) is formed in fp64 from the canonical quaternions
 * and rounded once to fp32. */
iq_status iq_export_block_matrices(const iq_params* p, float* m, size_t m_len);

/*
 * iq_quantize — encoder (Alg. 1 lines 1-14): x[n,d] -> codes[n, bytes], norms[n].
 * One kernel: 128-bit loads, fp32 norm via warp shuffles, forward block
 * rotation, nearest-centroid code, shuffle bit-packing, stores.
 */
iq_status iq_quantize(const iq_params* p, int dtype, int64_t n, const void* x,
                      uint8_t* codes, float* norms, void* cuda_stream);

/*
 * iq_dequantize — decoder (Alg. 1 lines 15-18): codes, norms -> y[n,d] of dtype.
 * y = rho * T^-1(C[codes]), rounded to dtype (round-to-nearest-even).
 */
iq_status iq_dequantize(const iq_params* p, int dtype, int64_t n,
                        const uint8_t* codes, const float* norms, void* y,
                        void* cuda_stream);

/*
 * iq_roundtrip — fused quantize->dequantize (the path Table 2 times,
 * P:369): x -> y = D(Q(E(x))) without materialising codes.  If codes and
 * norms are both non-NULL the kernel additionally writes them (same values
 * iq_quantize would); pass both NULL for the pure roundtrip.  y may alias x
 * (in place) — each 16-byte chunk is read before it is written by the same
 * thread.
 */
iq_status iq_roundtrip(const iq_params* p, int dtype, int64_t n, const void* x,
                       void* y, uint8_t* codes, float* norms, void* cuda_stream);

/* ------------------------------------------------------------------------
 * Stage 2: residual sketch (QJL-style correction, PAPER.md section
 * "Compatibility with Residual Correction"; R20-R24).
 * The paper fixes only r = x - x^_mse and "project the residual with a
 * quantized Johnson-Lindenstrauss transform"; the rest is our reading:
 *  - S is m x d with m = d, S[i][k] = fp16_rn(N_(i*d+k)), N_j the j-th
 *    standard normal of the [R12] generator keyed with seed ^
 *    0x514A4C534B455443.  The fp16-rounded values are the sketch.
 *  - r = x - x^ with x^ = rho T^-1(C[code]) evaluated in fp32 (before any
 *    rounding to dtype); gamma = ||r||_2 (fp32).
 *  - q_i = +1 if (S r)_i >= 0 else -1; stored LSB-first, bit i of a row set
 *    iff q_i = +1.  Rows of qjl are iq_qjl_bytes_per_vector(d) = d/8 bytes.
 *  - Estimators a consumer builds from (codes, norms, qjl, rnorms):
 *      <y, x> ~= <y, x^> + sqrt(pi/2)/m * gamma * <S y, q>,
 *      x~ = x^ + sqrt(pi/2)/m * gamma * S^T q  (unbiased over S).
 * ------------------------------------------------------------------------ */

/* iq_make_params plus the stage-2 sketch S (m = d).  The GPU sketch path
 * supports d in {64, 128, 256, 512} -- the paper's head widths
 * (UNSUPPORTED otherwise when device >= 0). */
iq_status iq_make_params_qjl(int d, int bits, int variant, uint64_t seed, int device,
                             iq_params** out);

/* Sketch bytes per row: ceil(m / 8) with m = d. */
size_t iq_qjl_bytes_per_vector(int d);

/* Copy S (row-major [m][d], the fp16 values widened to float) to a host
 * buffer of len >= m*d floats.  INVALID_ARGUMENT if the handle has no
 * sketch, BUFFER_TOO_SMALL if len is short. */
iq_status iq_export_qjl_matrix(const iq_params* p, float* S, size_t len);

/*
 * iq_quantize_qjl — stage 1 + stage 2: x[n,d] -> codes, norms (bit-identical
 * to iq_quantize), qjl[n, d/8] sign bits of S r and rnorms[n] = ||r||.
 * d in {64, 128}: one persistent kernel -- TMA ring for x, the stage-1
 * encoder in CUDA cores, r split into fp16 hi + lo tiles in shared memory,
 * z = S (r_hi + r_lo) on the tensor cores (tcgen05.mma, fp32 accumulators in
 * TMEM), sign packing from TMEM.  d in {256, 512} (S no longer fits shared
 * memory): two launches on the stream -- the iq_quantize kernel, then a
 * sketch kernel that reads x, the codes and the norms back, rebuilds r
 * K-chunk by K-chunk and streams S from L2 through shared memory (same
 * arithmetic, same readings).  x 16-byte aligned; codes, norms, rnorms
 * 4-byte and qjl 8-byte aligned.
 */
iq_status iq_quantize_qjl(const iq_params* p, int dtype, int64_t n, const void* x,
                          uint8_t* codes, float* norms, uint8_t* qjl, float* rnorms,
                          void* cuda_stream);

/*
 * iq_attention_scores — fused KV-cache decode consumer (
 * DESIGN.md R25-R27): attention logits straight from the packed cache,
 *   scores[h][j][k] = <q_hj, x^_hk> = rho_hk <T q_hj, C[code_hk]>
 *                   (+ sqrt(pi/2)/m * gamma_hk * <S q_hj, sign_hk> if qjl != NULL)
 * for `heads` independent heads sharing the handle, n_keys keys and n_q
 * queries (1..16) per head.  No key is inverse-rotated: queries are rotated
 * once per head, keys are only decoded; the dot products run on the tensor
 * cores (tcgen05, fp16 operands, fp32 accumulation).
 *  codes  : [heads, n_keys, code bytes]   norms  : [heads, n_keys] float
 *  qjl    : [heads, n_keys, d/8] or NULL  rnorms : [heads, n_keys] or NULL
 *           (both set: the stage-2 estimate; needs iq_make_params_qjl)
 *  q      : [heads, n_q, d] of q_dtype      scores : [heads, n_q, n_keys] float
 * Precision: fp16 centroids and queries (per-query power-of-two scaling):
 * |error| <= ~1e-3 * rho_hk * ||q_hj|| (stage 1), see DESIGN.md.  d in
 * {64, 128, 256, 512} (d > 128: the key tile's operand is built and
 * accumulated in 128-coordinate chunks); the stage-2 term needs d in
 * {64, 128}, or d = 256 at bits <= 3 (UNSUPPORTED otherwise: the sketch
 * operands of wider key tiles do not fit shared memory).  Head h uses
 * parameter set h % n_sets.
 * codes, norms, qjl, rnorms 16-byte aligned; with heads > 1,
 * n_keys % 4 == 0 (else MISALIGNED).
 */
iq_status iq_attention_scores(const iq_params* p, int q_dtype, int heads, int64_t n_keys,
                              const uint8_t* codes, const float* norms, const uint8_t* qjl,
                              const float* rnorms, int n_q, const void* q, float* scores,
                              void* cuda_stream);

/* ------------------------------------------------------------------------
 * Learning the rotations (PAPER.md "Parameterization and Learning",
 * q = u / ||u|| with free u; R29, R30).  Objective:
 * the stage-1 distortion on normalised rows L = sum_rows ||T xbar - Q(T xbar)||^2,
 * whose gradient is exact almost everywhere (Q is piecewise constant).  A
 * training step: iq_distortion_grad (GPU, dL/dM per block) ->
 * iq_rot_grad_from_operator_grad (host, chain rule to the parameters) ->
 * rot <- rot - lr * grad_rot -> iq_make_params_explicit (renormalises).
 * ------------------------------------------------------------------------ */

/*
 * iq_append_kv — quantize-on-append into a KV cache during autoregressive
 * decoding (PAPER.md:460 / P:477, "fused KV-cache compression during
 * autoregressive decoding").  One new row per cache
 * slot: slot r (r = layer * heads + head for a [layers, heads, tokens, .]
 * cache) appends row x[r] at token position pos_r:
 *     codes bytes  [(r * cap_tokens + pos_r) * code_bytes, + code_bytes)
 *     norms        [r * cap_tokens + pos_r]
 *   pos_r = positions ? positions[r] : position.
 * The layout is exactly what iq_quantize writes for the whole cache viewed
 * as n_rows * cap_tokens rows, and row r uses parameter set r % n_sets
 * (iq_make_params_sets; one set per (layer, head) with n_sets = n_rows), so
 * appending tokens one at a time produces, bit for bit, the codes and norms
 * of iq_quantize over the full cache with set_rows = cap_tokens.
 *  dtype      : I/O dtype of x.
 *  n_rows     : slots appended this call (n_rows = 0 is a no-op).
 *  x          : DEVICE [n_rows, d] of dtype, 16-byte aligned.
 *  codes      : DEVICE cache base, n_rows * cap_tokens rows of
 *               iq_code_bytes_per_vector(d, bits) bytes, 4-byte aligned.
 *  norms      : DEVICE fp32 cache base [n_rows * cap_tokens], 4-byte aligned.
 *  cap_tokens : token capacity per slot (the cache's token stride), >= 1.
 *  positions  : DEVICE int64 [n_rows] (nullable, 8-byte aligned): per-slot
 *               positions (ragged decode batches); a position outside
 *               [0, cap_tokens) writes nothing for that slot.
 *  position   : the position of every slot when positions is NULL; must be
 *               in [0, cap_tokens) (else INVALID_ARGUMENT).
 * One kernel launch on `cuda_stream`; nothing else in the cache is touched.
 * Errors: INVALID_ARGUMENT, MISALIGNED, UNSUPPORTED, DEVICE_MISMATCH, CUDA.
 */
iq_status iq_append_kv(const iq_params* p, int dtype, int64_t n_rows, const void* x, uint8_t* codes,
                       float* norms, int64_t cap_tokens, const int64_t* positions, int64_t position,
                       void* cuda_stream);

/* Parameters from explicit rotations in the iq_export_params layout (Full
 * [g][8] = q_L, q_R; Fast [g][4]; 2D [g2][2] = (cos, sin)); each quaternion /
 * pair is normalised on input.  No stage-2 sketch. */
iq_status iq_make_params_explicit(int d, int bits, int variant, const double* rot, size_t rot_len,
                                  int device, iq_params** out);

/* GPU: grad[b][i][j] += dL/dM_b[i][j] = 2 sum_rows e_i xbar_j with e = T xbar
 * - Q(T xbar), per block operator (DEVICE buffer of block_matrix_count doubles:
 * 16 per 4-D block, 4 per 2-D pair; caller zeroes it); loss (nullable DEVICE
 * double) += L.  One kernel; fp32 per-row math, fp64 accumulation across
 * CTAs. */
iq_status iq_distortion_grad(const iq_params* p, int dtype, int64_t n, const void* x, double* grad,
                             double* loss, void* cuda_stream);

/* Host: chain rule from dL/dM (host copy of the iq_distortion_grad output)
 * to the rotation parameters (iq_export_params layout), each unit vector's
 * gradient projected on its tangent space (the gradient w.r.t. u at
 * ||u|| = 1). */
iq_status iq_rot_grad_from_operator_grad(const iq_params* p, const double* G, size_t G_len,
                                         double* grad_rot, size_t rot_len);

/*
 * iq_error_sums — reconstruction statistics on the device (not part of the
 * timed path): sums[0] += sum_{i,j} (x_ij - y_ij)^2, sums[1] += sum x_ij^2,
 * accumulated in fp64 with atomics into the DEVICE buffer sums[2] (caller
 * zeroes it).  MSE = sums[0] / (n*d) [R17].
 */
iq_status iq_error_sums(const iq_params* p, int dtype, int64_t n, const void* x,
                        const void* y, double* sums, void* cuda_stream);

/*
 * Host-buffer pipeline (the end-to-end user call): x and y live in HOST
 * memory; the library streams them through device staging buffers in chunks
 * of chunk_vectors rows, overlapping H2D copy, the fused kernel and D2H copy
 * on its own streams.  Host buffers should be page-locked (cudaHostAlloc or
 * cudaHostRegister) for the copies to overlap; pageable memory works but is
 * slower.  iq_host_pipeline_create allocates the staging buffers (the only
 * allocation the library makes outside iq_make_params).
 */
typedef struct iq_host_pipeline iq_host_pipeline;

iq_status iq_host_pipeline_create(const iq_params* p, int dtype,
                                  int64_t chunk_vectors, iq_host_pipeline** out);
iq_status iq_host_pipeline_destroy(iq_host_pipeline* pl);

/* Synchronous: returns when y (and codes/norms if non-NULL) are in host
 * memory.  codes/norms are HOST pointers here (both NULL or both set). */
iq_status iq_host_roundtrip(iq_host_pipeline* pl, int64_t n, const void* x_host,
                            void* y_host, uint8_t* codes_host, float* norms_host);

#ifdef __cplusplus
}
#endif
#endif /* ISOQUANT_H_ */
