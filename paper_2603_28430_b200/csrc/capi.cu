// C ABI of libisoquant (include/isoquant.h): validation, parameter handles,
// dispatch to the template instances, reconstruction statistics and the
// host-buffer streaming pipeline.  No exception crosses this boundary.
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstring>
#include <new>
#include <string>

#include "iq_internal.h"
#include "kernels.cuh"

namespace iq {
int launch_full_f32(Kernel, int, int, const LaunchArgs&);
int launch_full_f16(Kernel, int, int, const LaunchArgs&);
int launch_fast_f32(Kernel, int, int, const LaunchArgs&);
int launch_fast_f16(Kernel, int, int, const LaunchArgs&);
int launch_planar2d_f32(Kernel, int, int, const LaunchArgs&);
int launch_planar2d_f16(Kernel, int, int, const LaunchArgs&);
int launch_full_bf16(Kernel, int, int, const LaunchArgs&);
int launch_fast_bf16(Kernel, int, int, const LaunchArgs&);
int launch_planar2d_bf16(Kernel, int, int, const LaunchArgs&);

bool attn_supported(int d) { return d == 64 || d == 128 || d == 256 || d == 512; }

bool gpu_supported(int d, int bits, int variant) {
  const bool dok = d == 64 || d == 128 || d == 256 || d == 512;
  return dok && bits >= 1 && bits <= kMaxBits && variant >= 0 && variant <= 2;
}

int launch(Kernel k, int variant, int dtype, int d, int bits, const LaunchArgs& a) {
  using Fn = int (*)(Kernel, int, int, const LaunchArgs&);
  static const Fn table[3][3] = {{launch_full_f32, launch_full_f16, launch_full_bf16},
                                 {launch_fast_f32, launch_fast_f16, launch_fast_bf16},
                                 {launch_planar2d_f32, launch_planar2d_f16, launch_planar2d_bf16}};
  if (variant < 0 || variant > 2 || dtype < 0 || dtype > 2) return -1;
  return table[variant][dtype](k, d, bits, a);
}
}  // namespace iq

struct iq_params {
  iq::HostParams hp;
  int device = -1;
  float* d_mat = nullptr;
  uint8_t* d_qjl = nullptr;   // UMMA image of the stage-2 sketch S (iq_make_params_qjl)
  uint8_t* d_qjl_a = nullptr; // the same S as a 128-row A operand (attention consumer)
  uint8_t* d_qjl_rot = nullptr; // S' = S M^T as fp16 hi + lo B images (16-bit sketch kernel)
};

namespace {

thread_local std::string g_detail;

iq_status fail(iq_status s, const std::string& why) {
  g_detail = why;
  return s;
}

iq_status cuda_fail(cudaError_t e, const char* what) {
  g_detail = std::string(what) + ": " + cudaGetErrorName(e) + " (" + cudaGetErrorString(e) + ")";
  return e == cudaErrorMemoryAllocation ? IQ_ERR_OUT_OF_MEMORY : IQ_ERR_CUDA;
}

bool aligned(const void* p, uintptr_t a) { return (reinterpret_cast<uintptr_t>(p) % a) == 0; }

size_t dtype_size(int dt) { return dt == IQ_DTYPE_F32 ? 4 : 2; }

// Common validation of a compute call.  Returns IQ_OK or the error.
iq_status check_call(const iq_params* p, int dtype, int64_t n) {
  if (!p) return fail(IQ_ERR_INVALID_ARGUMENT, "params handle is NULL");
  if (dtype != IQ_DTYPE_F32 && dtype != IQ_DTYPE_F16 && dtype != IQ_DTYPE_BF16)
    return fail(IQ_ERR_INVALID_ARGUMENT, "dtype must be 0 (f32), 1 (f16) or 2 (bf16)");
  if (n < 0) return fail(IQ_ERR_INVALID_ARGUMENT, "n must be >= 0");
  if (p->device < 0 || !p->d_mat)
    return fail(IQ_ERR_DEVICE_MISMATCH, "params handle is host-only (device = -1)");
  if (!iq::gpu_supported(p->hp.d, p->hp.bits, p->hp.variant))
    return fail(IQ_ERR_UNSUPPORTED, "d must be one of 64, 128, 256, 512 on the GPU path");
  int cur = -1;
  cudaError_t e = cudaGetDevice(&cur);
  if (e != cudaSuccess) return cuda_fail(e, "cudaGetDevice");
  if (cur != p->device)
    return fail(IQ_ERR_DEVICE_MISMATCH, "current CUDA device " + std::to_string(cur) +
                                            " != params device " + std::to_string(p->device));
  return IQ_OK;
}

// The batch stage-1 kernels switch sets per tile: tiles (<= 256 rows, every
// tile size divides 256) must not straddle sets.
iq_status check_batch_sets(const iq_params* p) {
  if (p->hp.n_sets > 1 && p->hp.set_rows % 256 != 0)
    return fail(IQ_ERR_UNSUPPORTED, "batch kernels with parameter sets need set_rows to be a multiple of 256 "
                                    "(finer sets: iq_append_kv and iq_attention_scores)");
  return IQ_OK;
}

iq::LaunchArgs base_args(const iq_params* p, int64_t n, void* stream) {
  iq::LaunchArgs a{};
  a.mat = p->d_mat;
  a.cb = p->hp.kcb;
  a.n = n;
  a.stream = stream;
  return a;
}

iq_status run(iq::Kernel k, const iq_params* p, int dtype, const iq::LaunchArgs& a) {
  const int r = iq::launch(k, p->hp.variant, dtype, p->hp.d, p->hp.bits, a);
  if (r == -1) return fail(IQ_ERR_UNSUPPORTED, "no kernel instance for this configuration");
  if (r != 0) return cuda_fail(static_cast<cudaError_t>(r), "kernel launch");
  return IQ_OK;
}

}  // namespace

extern "C" {

const char* iq_version(void) { return "isoquant-b200 0.2.0 (sm_100a)"; }
int iq_abi_version(void) { return IQ_ABI_VERSION; }

const char* iq_status_string(iq_status s) {
  switch (s) {
    case IQ_OK: return "IQ_OK";
    case IQ_ERR_INVALID_ARGUMENT: return "IQ_ERR_INVALID_ARGUMENT";
    case IQ_ERR_UNSUPPORTED: return "IQ_ERR_UNSUPPORTED";
    case IQ_ERR_MISALIGNED: return "IQ_ERR_MISALIGNED";
    case IQ_ERR_DEVICE_MISMATCH: return "IQ_ERR_DEVICE_MISMATCH";
    case IQ_ERR_CUDA: return "IQ_ERR_CUDA";
    case IQ_ERR_OUT_OF_MEMORY: return "IQ_ERR_OUT_OF_MEMORY";
    case IQ_ERR_BUFFER_TOO_SMALL: return "IQ_ERR_BUFFER_TOO_SMALL";
  }
  return "IQ_ERR_UNKNOWN";
}

const char* iq_last_error_detail(void) { return g_detail.c_str(); }

static iq_status make_params_impl(int d, int bits, int variant, uint64_t seed, int device, bool qjl,
                                  iq_params** out, const double* rot_in = nullptr, int n_sets = 1,
                                  int64_t set_rows = 0) {
  if (!out) return fail(IQ_ERR_INVALID_ARGUMENT, "out is NULL");
  *out = nullptr;
  if (device < -1) return fail(IQ_ERR_INVALID_ARGUMENT, "device must be >= -1");
  iq_params* p = new (std::nothrow) iq_params();
  if (!p) return fail(IQ_ERR_OUT_OF_MEMORY, "host allocation failed");
  std::string err;
  if (!iq::build_host_params(d, bits, variant, seed, &p->hp, &err, rot_in) ||
      (qjl && !iq::build_qjl(&p->hp, &err)) || (n_sets > 1 && !iq::add_param_sets(&p->hp, n_sets, set_rows, &err))) {
    delete p;
    return fail(IQ_ERR_INVALID_ARGUMENT, err);
  }
  if (qjl && device >= 0 && !iq::qjl_supported(d)) {
    delete p;
    return fail(IQ_ERR_UNSUPPORTED, "the stage-2 sketch kernels support d in {64, 128, 256, 512}");
  }
  p->device = device;
  if (device >= 0) {
    if (!iq::gpu_supported(d, bits, variant)) {
      delete p;
      return fail(IQ_ERR_UNSUPPORTED, "d must be one of 64, 128, 256, 512 on the GPU path");
    }
    int prev = -1;
    cudaError_t e = cudaGetDevice(&prev);
    if (e == cudaSuccess && prev != device) e = cudaSetDevice(device);
    if (e == cudaSuccess) e = cudaMalloc(&p->d_mat, p->hp.mat.size() * sizeof(float));
    if (e == cudaSuccess)
      e = cudaMemcpy(p->d_mat, p->hp.mat.data(), p->hp.mat.size() * sizeof(float),
                     cudaMemcpyHostToDevice);
    if (e == cudaSuccess && qjl) e = cudaMalloc(&p->d_qjl, p->hp.qjl_img.size());
    if (e == cudaSuccess && qjl)
      e = cudaMemcpy(p->d_qjl, p->hp.qjl_img.data(), p->hp.qjl_img.size(), cudaMemcpyHostToDevice);
    // the rotated-domain and attention images exist for the fused d <= 128 kernels only
    const bool rot = qjl && !p->hp.qjl_img_rot.empty(), aimg = qjl && !p->hp.qjl_img_a.empty();
    if (e == cudaSuccess && rot) e = cudaMalloc(&p->d_qjl_rot, p->hp.qjl_img_rot.size());
    if (e == cudaSuccess && rot)
      e = cudaMemcpy(p->d_qjl_rot, p->hp.qjl_img_rot.data(), p->hp.qjl_img_rot.size(), cudaMemcpyHostToDevice);
    if (e == cudaSuccess && aimg) e = cudaMalloc(&p->d_qjl_a, p->hp.qjl_img_a.size());
    if (e == cudaSuccess && aimg)
      e = cudaMemcpy(p->d_qjl_a, p->hp.qjl_img_a.data(), p->hp.qjl_img_a.size(), cudaMemcpyHostToDevice);
    if (prev >= 0 && prev != device) cudaSetDevice(prev);
    if (e != cudaSuccess) {
      if (p->d_mat) cudaFree(p->d_mat);
      if (p->d_qjl) cudaFree(p->d_qjl);
      if (p->d_qjl_a) cudaFree(p->d_qjl_a);
      if (p->d_qjl_rot) cudaFree(p->d_qjl_rot);
      delete p;
      return cuda_fail(e, "iq_make_params device upload");
    }
  }
  *out = p;
  return IQ_OK;
}

iq_status iq_make_params(int d, int bits, int variant, uint64_t seed, int device, iq_params** out) {
  return make_params_impl(d, bits, variant, seed, device, false, out);
}

iq_status iq_make_params_qjl(int d, int bits, int variant, uint64_t seed, int device, iq_params** out) {
  return make_params_impl(d, bits, variant, seed, device, true, out);
}

iq_status iq_make_params_sets(int d, int bits, int variant, uint64_t seed, int n_sets, int64_t set_rows, int device,
                              iq_params** out) {
  if (n_sets < 1) return fail(IQ_ERR_INVALID_ARGUMENT, "n_sets must be >= 1");
  if (n_sets > 1 && set_rows < 1) return fail(IQ_ERR_INVALID_ARGUMENT, "set_rows must be >= 1");
  return make_params_impl(d, bits, variant, seed, device, false, out, nullptr, n_sets, set_rows);
}

iq_status iq_make_params_qjl_sets(int d, int bits, int variant, uint64_t seed, int n_sets, int64_t set_rows,
                                  int device, iq_params** out) {
  if (n_sets < 1) return fail(IQ_ERR_INVALID_ARGUMENT, "n_sets must be >= 1");
  if (n_sets > 1 && set_rows < 1) return fail(IQ_ERR_INVALID_ARGUMENT, "set_rows must be >= 1");
  return make_params_impl(d, bits, variant, seed, device, true, out, nullptr, n_sets, set_rows);
}

iq_status iq_params_sets_info(const iq_params* p, int* n_sets, int64_t* set_rows) {
  if (!p) return fail(IQ_ERR_INVALID_ARGUMENT, "params handle is NULL");
  if (n_sets) *n_sets = p->hp.n_sets;
  if (set_rows) *set_rows = p->hp.set_rows;
  return IQ_OK;
}

iq_status iq_export_params_set(const iq_params* p, int set, double* rot, size_t rot_len) {
  if (!p || !rot) return fail(IQ_ERR_INVALID_ARGUMENT, "NULL argument");
  if (set < 0 || set >= p->hp.n_sets) return fail(IQ_ERR_INVALID_ARGUMENT, "set out of range");
  const size_t nr = iq::rotation_param_count(p->hp.d, p->hp.variant);
  if (rot_len < nr) return fail(IQ_ERR_BUFFER_TOO_SMALL, "rot buffer too small");
  std::memcpy(rot, p->hp.rot.data() + (size_t)set * nr, nr * sizeof(double));
  return IQ_OK;
}

iq_status iq_make_params_explicit(int d, int bits, int variant, const double* rot, size_t rot_len, int device,
                                  iq_params** out) {
  if (!rot) return fail(IQ_ERR_INVALID_ARGUMENT, "rot is NULL");
  if (d < 1 || rot_len < iq::rotation_param_count(d, variant))
    return fail(IQ_ERR_BUFFER_TOO_SMALL, "rot shorter than iq_rotation_param_count(d, variant)");
  return make_params_impl(d, bits, variant, 0, device, false, out, rot);
}

iq_status iq_rot_grad_from_operator_grad(const iq_params* p, const double* G, size_t G_len, double* grad_rot,
                                         size_t rot_len) {
  if (!p || !G || !grad_rot) return fail(IQ_ERR_INVALID_ARGUMENT, "NULL argument");
  if (p->hp.n_sets > 1) return fail(IQ_ERR_UNSUPPORTED, "single-set handles only");
  if (G_len < p->hp.mat.size()) return fail(IQ_ERR_BUFFER_TOO_SMALL, "G shorter than the block operators");
  if (rot_len < p->hp.rot.size()) return fail(IQ_ERR_BUFFER_TOO_SMALL, "grad_rot shorter than the rotation params");
  iq::operator_grad_to_rot(p->hp, G, grad_rot);
  return IQ_OK;
}

iq_status iq_free_params(iq_params* p) {
  if (!p) return IQ_OK;
  if (p->d_mat) {
    int prev = -1;
    cudaGetDevice(&prev);
    if (prev != p->device) cudaSetDevice(p->device);
    cudaFree(p->d_mat);
    if (p->d_qjl) cudaFree(p->d_qjl);
    if (p->d_qjl_a) cudaFree(p->d_qjl_a);
    if (p->d_qjl_rot) cudaFree(p->d_qjl_rot);
    if (prev >= 0 && prev != p->device) cudaSetDevice(prev);
  }
  delete p;
  return IQ_OK;
}

iq_status iq_params_info(const iq_params* p, int* d, int* bits, int* variant, int* device) {
  if (!p) return fail(IQ_ERR_INVALID_ARGUMENT, "params handle is NULL");
  if (d) *d = p->hp.d;
  if (bits) *bits = p->hp.bits;
  if (variant) *variant = p->hp.variant;
  if (device) *device = p->device;
  return IQ_OK;
}

size_t iq_code_bytes_per_vector(int d, int bits) {
  if (d <= 0 || bits <= 0) return 0;
  return (static_cast<size_t>(d) * bits + 7) / 8;
}

size_t iq_rotation_param_count(int d, int variant) {
  if (d <= 0) return 0;
  return iq::rotation_param_count(d, variant);
}

iq_status iq_export_params(const iq_params* p, double* rot, size_t rot_len, float* centroids,
                           size_t centroids_len, float* thresholds, size_t thresholds_len) {
  if (!p) return fail(IQ_ERR_INVALID_ARGUMENT, "params handle is NULL");
  const auto& hp = p->hp;
  if (rot) {                                  // set 0 (iq_export_params_set for the others)
    const size_t nr = iq::rotation_param_count(hp.d, hp.variant);
    if (rot_len < nr) return fail(IQ_ERR_BUFFER_TOO_SMALL, "rot buffer too small");
    std::memcpy(rot, hp.rot.data(), nr * sizeof(double));
  }
  if (centroids) {
    if (centroids_len < hp.centroids.size())
      return fail(IQ_ERR_BUFFER_TOO_SMALL, "centroids buffer too small");
    std::memcpy(centroids, hp.centroids.data(), hp.centroids.size() * sizeof(float));
  }
  if (thresholds) {
    if (thresholds_len < hp.thresholds.size())
      return fail(IQ_ERR_BUFFER_TOO_SMALL, "thresholds buffer too small");
    std::memcpy(thresholds, hp.thresholds.data(), hp.thresholds.size() * sizeof(float));
  }
  return IQ_OK;
}

iq_status iq_export_block_matrices(const iq_params* p, float* m, size_t m_len) {
  if (!p || !m) return fail(IQ_ERR_INVALID_ARGUMENT, "NULL argument");
  const size_t nm = iq::block_matrix_count(p->hp.d, p->hp.variant);   // set 0
  if (m_len < nm) return fail(IQ_ERR_BUFFER_TOO_SMALL, "matrix buffer too small");
  std::memcpy(m, p->hp.mat.data(), nm * sizeof(float));
  return IQ_OK;
}

size_t iq_qjl_bytes_per_vector(int d) {
  if (d <= 0) return 0;
  return (static_cast<size_t>(d) + 7) / 8;
}

iq_status iq_export_qjl_matrix(const iq_params* p, float* S, size_t len) {
  if (!p || !S) return fail(IQ_ERR_INVALID_ARGUMENT, "NULL argument");
  if (!p->hp.has_qjl) return fail(IQ_ERR_INVALID_ARGUMENT, "handle has no stage-2 sketch (use iq_make_params_qjl)");
  const size_t need = p->hp.qjl_half.size();
  if (len < need) return fail(IQ_ERR_BUFFER_TOO_SMALL, "S buffer too small (m * d floats)");
  for (size_t i = 0; i < need; ++i) {
    __half_raw r;
    r.x = p->hp.qjl_half[i];
    S[i] = __half2float(__half(r));
  }
  return IQ_OK;
}

iq_status iq_quantize_qjl(const iq_params* p, int dtype, int64_t n, const void* x, uint8_t* codes,
                          float* norms, uint8_t* qjl, float* rnorms, void* stream) {
  iq_status s = check_call(p, dtype, n);
  if (s != IQ_OK) return s;
  if (!p->hp.has_qjl || !p->d_qjl)
    return fail(IQ_ERR_INVALID_ARGUMENT, "handle has no stage-2 sketch (use iq_make_params_qjl)");
  s = check_batch_sets(p);
  if (s != IQ_OK) return s;
  if (n == 0) return IQ_OK;
  if (!x || !codes || !norms || !qjl || !rnorms)
    return fail(IQ_ERR_INVALID_ARGUMENT, "x, codes, norms, qjl and rnorms are required");
  if (!aligned(x, 16)) return fail(IQ_ERR_MISALIGNED, "x must be 16-byte aligned");
  if (!aligned(codes, 4) || !aligned(norms, 4) || !aligned(rnorms, 4) || !aligned(qjl, 8))
    return fail(IQ_ERR_MISALIGNED, "codes, norms, rnorms must be 4-byte and qjl 8-byte aligned");
  iq::LaunchArgs a = base_args(p, n, stream);
  a.x = x;
  a.codes = codes;
  a.norms = norms;
  a.qjl_img = p->d_qjl;
  a.qjl_img_rot = p->d_qjl_rot;
  a.qjl = qjl;
  a.rnorms = rnorms;
  if (iq::qjl_fused(p->hp.d)) return run(iq::Kernel::kQuantizeQjl, p, dtype, a);
  // d in {256, 512}: the stage-1 quantizer, then the sketch kernel reading
  // back x, the codes and the norms (two launches on the caller's stream)
  s = run(iq::Kernel::kQuantize, p, dtype, a);
  if (s != IQ_OK) return s;
  return run(iq::Kernel::kQjlSketch, p, dtype, a);
}

iq_status iq_attention_scores(const iq_params* p, int q_dtype, int heads, int64_t n_keys,
                              const uint8_t* codes, const float* norms, const uint8_t* qjl,
                              const float* rnorms, int n_q, const void* q, float* scores, void* stream) {
  iq_status s = check_call(p, q_dtype, n_keys);
  if (s != IQ_OK) return s;
  if (!iq::attn_supported(p->hp.d))
    return fail(IQ_ERR_UNSUPPORTED, "the attention consumer supports d in {64, 128, 256, 512}");
  if (heads < 1) return fail(IQ_ERR_INVALID_ARGUMENT, "heads must be >= 1");
  if (n_q < 1 || n_q > 16) return fail(IQ_ERR_INVALID_ARGUMENT, "n_q must be in [1, 16]");
  if ((qjl == nullptr) != (rnorms == nullptr))
    return fail(IQ_ERR_INVALID_ARGUMENT, "qjl and rnorms must be both NULL or both set");
  if (qjl && !(p->hp.d <= 128 || (p->hp.d == 256 && p->hp.bits <= 3)))
    return fail(IQ_ERR_UNSUPPORTED, "the stage-2 term of the consumer supports d in {64, 128}, and 256 at bits <= 3");
  if (qjl && (!p->hp.has_qjl || !p->d_qjl_a))
    return fail(IQ_ERR_INVALID_ARGUMENT, "stage-2 scores need a handle with the sketch (iq_make_params_qjl)");
  if (n_keys == 0) return IQ_OK;
  if (!codes || !norms || !q || !scores)
    return fail(IQ_ERR_INVALID_ARGUMENT, "codes, norms, q and scores are required");
  if (!aligned(codes, 16) || !aligned(norms, 16) || (qjl && (!aligned(qjl, 16) || !aligned(rnorms, 16))) ||
      !aligned(scores, 4) || !aligned(q, 4))
    return fail(IQ_ERR_MISALIGNED, "codes, norms, qjl, rnorms must be 16-byte aligned (TMA), q and scores 4-byte");
  if (heads > 1 && n_keys % 4 != 0)
    return fail(IQ_ERR_MISALIGNED, "with heads > 1, n_keys must be a multiple of 4 (16-byte head strides)");
  iq::LaunchArgs a = base_args(p, n_keys, stream);
  a.heads = heads;
  a.n_q = n_q;
  a.q = q;
  a.scores = scores;
  a.codes_in = codes;
  a.norms_in = norms;
  a.qjl_in = qjl;
  a.rnorms_in = rnorms;
  a.qjl_img_a = p->d_qjl_a;
  return run(iq::Kernel::kAttnScores, p, q_dtype, a);
}

iq_status iq_append_kv(const iq_params* p, int dtype, int64_t n_rows, const void* x, uint8_t* codes,
                       float* norms, int64_t cap_tokens, const int64_t* positions, int64_t position,
                       void* stream) {
  iq_status s = check_call(p, dtype, n_rows);
  if (s != IQ_OK) return s;
  if (cap_tokens < 1) return fail(IQ_ERR_INVALID_ARGUMENT, "cap_tokens must be >= 1");
  if (!positions && (position < 0 || position >= cap_tokens))
    return fail(IQ_ERR_INVALID_ARGUMENT, "position must be in [0, cap_tokens)");
  if (n_rows == 0) return IQ_OK;
  if (!x || !codes || !norms) return fail(IQ_ERR_INVALID_ARGUMENT, "x, codes and norms are required");
  if (!aligned(x, 16)) return fail(IQ_ERR_MISALIGNED, "x must be 16-byte aligned");
  if (!aligned(codes, 4) || !aligned(norms, 4) || (positions && !aligned(positions, 8)))
    return fail(IQ_ERR_MISALIGNED, "codes and norms must be 4-byte, positions 8-byte aligned");
  iq::LaunchArgs a = base_args(p, n_rows, stream);
  a.x = x;
  a.codes = codes;
  a.norms = norms;
  a.cap = cap_tokens;
  a.positions = positions;
  a.position = position;
  return run(iq::Kernel::kAppend, p, dtype, a);
}

iq_status iq_distortion_grad(const iq_params* p, int dtype, int64_t n, const void* x, double* grad, double* loss,
                             void* stream) {
  iq_status s = check_call(p, dtype, n);
  if (s != IQ_OK) return s;
  if (p->hp.n_sets > 1) return fail(IQ_ERR_UNSUPPORTED, "the distortion gradient takes a single-set handle");
  if (n == 0) return IQ_OK;
  if (!x || !grad) return fail(IQ_ERR_INVALID_ARGUMENT, "x and grad are required");
  if (!aligned(x, 16) || !aligned(grad, 8) || (loss && !aligned(loss, 8)))
    return fail(IQ_ERR_MISALIGNED, "x must be 16-byte, grad and loss 8-byte aligned");
  iq::LaunchArgs a = base_args(p, n, stream);
  a.x = x;
  a.grad = grad;
  a.loss = loss;
  return run(iq::Kernel::kDistortionGrad, p, dtype, a);
}

iq_status iq_quantize(const iq_params* p, int dtype, int64_t n, const void* x, uint8_t* codes,
                      float* norms, void* stream) {
  iq_status s = check_call(p, dtype, n);
  if (s != IQ_OK) return s;
  if ((s = check_batch_sets(p)) != IQ_OK) return s;
  if (n == 0) return IQ_OK;
  if (!x || !codes || !norms) return fail(IQ_ERR_INVALID_ARGUMENT, "x, codes and norms are required");
  if (!aligned(x, 16)) return fail(IQ_ERR_MISALIGNED, "x must be 16-byte aligned");
  if (!aligned(codes, 4) || !aligned(norms, 4))
    return fail(IQ_ERR_MISALIGNED, "codes and norms must be 4-byte aligned");
  iq::LaunchArgs a = base_args(p, n, stream);
  a.x = x;
  a.codes = codes;
  a.norms = norms;
  return run(iq::Kernel::kQuantize, p, dtype, a);
}

iq_status iq_dequantize(const iq_params* p, int dtype, int64_t n, const uint8_t* codes,
                        const float* norms, void* y, void* stream) {
  iq_status s = check_call(p, dtype, n);
  if (s != IQ_OK) return s;
  if ((s = check_batch_sets(p)) != IQ_OK) return s;
  if (n == 0) return IQ_OK;
  if (!y || !codes || !norms) return fail(IQ_ERR_INVALID_ARGUMENT, "codes, norms and y are required");
  if (!aligned(y, 16) || !aligned(codes, 16) || !aligned(norms, 16))
    return fail(IQ_ERR_MISALIGNED, "y, codes and norms must be 16-byte aligned (TMA bulk loads)");
  iq::LaunchArgs a = base_args(p, n, stream);
  a.codes_in = codes;
  a.norms_in = norms;
  a.y = y;
  return run(iq::Kernel::kDequantize, p, dtype, a);
}

iq_status iq_roundtrip(const iq_params* p, int dtype, int64_t n, const void* x, void* y,
                       uint8_t* codes, float* norms, void* stream) {
  iq_status s = check_call(p, dtype, n);
  if (s != IQ_OK) return s;
  if ((s = check_batch_sets(p)) != IQ_OK) return s;
  if (n == 0) return IQ_OK;
  if (!x || !y) return fail(IQ_ERR_INVALID_ARGUMENT, "x and y are required");
  if ((codes == nullptr) != (norms == nullptr))
    return fail(IQ_ERR_INVALID_ARGUMENT, "codes and norms must be both NULL or both set");
  if (!aligned(x, 16) || !aligned(y, 16)) return fail(IQ_ERR_MISALIGNED, "x and y must be 16-byte aligned");
  if (codes && (!aligned(codes, 4) || !aligned(norms, 4)))
    return fail(IQ_ERR_MISALIGNED, "codes and norms must be 4-byte aligned");
  iq::LaunchArgs a = base_args(p, n, stream);
  a.x = x;
  a.y = y;
  a.codes = codes;
  a.norms = norms;
  return run(iq::Kernel::kRoundtrip, p, dtype, a);
}

iq_status iq_error_sums(const iq_params* p, int dtype, int64_t n, const void* x, const void* y,
                        double* sums, void* stream) {
  iq_status s = check_call(p, dtype, n);
  if (s != IQ_OK) return s;
  if (n == 0) return IQ_OK;
  if (!x || !y || !sums) return fail(IQ_ERR_INVALID_ARGUMENT, "x, y and sums are required");
  if (!aligned(x, 16) || !aligned(y, 16) || !aligned(sums, 8))
    return fail(IQ_ERR_MISALIGNED, "x, y must be 16-byte and sums 8-byte aligned");
  const int epc = dtype == IQ_DTYPE_F32 ? 4 : 8;
  const int64_t nchunks = n * p->hp.d / epc;
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, p->device);
  int64_t grid = std::min<int64_t>((nchunks + iq::kThreads - 1) / iq::kThreads, (int64_t)sms * 8);
  if (grid < 1) grid = 1;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (dtype == IQ_DTYPE_F16)
    iq::k_error_sums<__half><<<(int)grid, iq::kThreads, 0, st>>>(
        nchunks, static_cast<const __half*>(x), static_cast<const __half*>(y), sums);
  else if (dtype == IQ_DTYPE_BF16)
    iq::k_error_sums<__nv_bfloat16><<<(int)grid, iq::kThreads, 0, st>>>(
        nchunks, static_cast<const __nv_bfloat16*>(x), static_cast<const __nv_bfloat16*>(y), sums);
  else
    iq::k_error_sums<float><<<(int)grid, iq::kThreads, 0, st>>>(
        nchunks, static_cast<const float*>(x), static_cast<const float*>(y), sums);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return cuda_fail(e, "k_error_sums launch");
  return IQ_OK;
}

}  // extern "C"

// ------------------------------------------------------------ host pipeline
struct iq_host_pipeline {
  const iq_params* p = nullptr;
  int dtype = 0;
  int64_t chunk = 0;
  static constexpr int kSlots = 3;
  cudaStream_t st[kSlots] = {};
  void* dx[kSlots] = {};
  void* dy[kSlots] = {};
  uint8_t* dcodes[kSlots] = {};
  float* dnorms[kSlots] = {};
};

extern "C" {

iq_status iq_host_pipeline_destroy(iq_host_pipeline* pl) {
  if (!pl) return IQ_OK;
  for (int i = 0; i < iq_host_pipeline::kSlots; ++i) {
    if (pl->st[i]) { cudaStreamSynchronize(pl->st[i]); cudaStreamDestroy(pl->st[i]); }
    cudaFree(pl->dx[i]);
    cudaFree(pl->dy[i]);
    cudaFree(pl->dcodes[i]);
    cudaFree(pl->dnorms[i]);
  }
  delete pl;
  return IQ_OK;
}

iq_status iq_host_pipeline_create(const iq_params* p, int dtype, int64_t chunk_vectors,
                                  iq_host_pipeline** out) {
  if (!out) return fail(IQ_ERR_INVALID_ARGUMENT, "out is NULL");
  *out = nullptr;
  iq_status s = check_call(p, dtype, 0);
  if (s != IQ_OK) return s;
  if (chunk_vectors <= 0) return fail(IQ_ERR_INVALID_ARGUMENT, "chunk_vectors must be > 0");
  if ((s = check_batch_sets(p)) != IQ_OK) return s;
  if (p->hp.n_sets > 1 && chunk_vectors % (p->hp.set_rows * p->hp.n_sets) != 0)
    return fail(IQ_ERR_INVALID_ARGUMENT, "with parameter sets, chunk_vectors must be a multiple of set_rows * n_sets");
  iq_host_pipeline* pl = new (std::nothrow) iq_host_pipeline();
  if (!pl) return fail(IQ_ERR_OUT_OF_MEMORY, "host allocation failed");
  pl->p = p;
  pl->dtype = dtype;
  pl->chunk = chunk_vectors;
  const size_t xb = (size_t)chunk_vectors * p->hp.d * dtype_size(dtype);
  const size_t cbytes = (size_t)chunk_vectors * iq_code_bytes_per_vector(p->hp.d, p->hp.bits);
  for (int i = 0; i < iq_host_pipeline::kSlots; ++i) {
    cudaError_t e = cudaStreamCreateWithFlags(&pl->st[i], cudaStreamNonBlocking);
    if (e == cudaSuccess) e = cudaMalloc(&pl->dx[i], xb);
    if (e == cudaSuccess) e = cudaMalloc(&pl->dy[i], xb);
    if (e == cudaSuccess) e = cudaMalloc(reinterpret_cast<void**>(&pl->dcodes[i]), cbytes + 16);
    if (e == cudaSuccess) e = cudaMalloc(reinterpret_cast<void**>(&pl->dnorms[i]), chunk_vectors * 4 + 16);
    if (e != cudaSuccess) {
      iq_host_pipeline_destroy(pl);
      return cuda_fail(e, "iq_host_pipeline_create");
    }
  }
  *out = pl;
  return IQ_OK;
}

iq_status iq_host_roundtrip(iq_host_pipeline* pl, int64_t n, const void* x_host, void* y_host,
                            uint8_t* codes_host, float* norms_host) {
  if (!pl) return fail(IQ_ERR_INVALID_ARGUMENT, "pipeline is NULL");
  iq_status s = check_call(pl->p, pl->dtype, n);
  if (s != IQ_OK) return s;
  if (n == 0) return IQ_OK;
  if (!x_host || !y_host) return fail(IQ_ERR_INVALID_ARGUMENT, "x_host and y_host are required");
  if ((codes_host == nullptr) != (norms_host == nullptr))
    return fail(IQ_ERR_INVALID_ARGUMENT, "codes and norms must be both NULL or both set");
  const size_t row = (size_t)pl->p->hp.d * dtype_size(pl->dtype);
  const size_t crow = iq_code_bytes_per_vector(pl->p->hp.d, pl->p->hp.bits);
  const bool emit = codes_host != nullptr;
  int64_t c = 0;
  for (int64_t r0 = 0; r0 < n; r0 += pl->chunk, ++c) {
    const int slot = (int)(c % iq_host_pipeline::kSlots);
    const int64_t m = std::min<int64_t>(pl->chunk, n - r0);
    cudaStream_t st = pl->st[slot];
    cudaError_t e = cudaMemcpyAsync(pl->dx[slot], static_cast<const char*>(x_host) + r0 * row,
                                    m * row, cudaMemcpyHostToDevice, st);
    if (e != cudaSuccess) return cuda_fail(e, "H2D copy");
    iq::LaunchArgs a = base_args(pl->p, m, st);
    a.x = pl->dx[slot];
    a.y = pl->dy[slot];
    a.codes = emit ? pl->dcodes[slot] : nullptr;
    a.norms = emit ? pl->dnorms[slot] : nullptr;
    s = run(iq::Kernel::kRoundtrip, pl->p, pl->dtype, a);
    if (s != IQ_OK) return s;
    e = cudaMemcpyAsync(static_cast<char*>(y_host) + r0 * row, pl->dy[slot], m * row,
                        cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess && emit)
      e = cudaMemcpyAsync(codes_host + r0 * crow, pl->dcodes[slot], m * crow,
                          cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess && emit)
      e = cudaMemcpyAsync(norms_host + r0, pl->dnorms[slot], m * 4, cudaMemcpyDeviceToHost, st);
    if (e != cudaSuccess) return cuda_fail(e, "D2H copy");
  }
  for (int i = 0; i < iq_host_pipeline::kSlots; ++i) {
    cudaError_t e = cudaStreamSynchronize(pl->st[i]);
    if (e != cudaSuccess) return cuda_fail(e, "pipeline synchronize");
  }
  return IQ_OK;
}

}  // extern "C"
