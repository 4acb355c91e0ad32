// Host-side parameter construction for IsoQuant stage 1 (runs once per
// configuration, off the hot path).
//
//  * Random fixed block rotations: each unit quaternion is
//    a normalised N(0, I_4) draw ("Gaussian-normalize sampling on S^3",
//    P:227); planar angles theta ~ U[0, 2pi) ("uniform angle sampling",
//    P:227).  Generator: counter-based SplitMix64 -> 53-bit uniforms ->
//    Box-Muller, reading [R12].
//  * The per-block operator M = L(q_L) R(conj q_R) (Full) or L(q_L) (Fast),
//    formed column by column as T(e_j) with Hamilton products in fp64 and
//    rounded once to fp32; the inverse map conj(q_L) v q_R is exactly M^T
//    (P:108-110), so the kernels apply M and M^T.
//  * Scalar codebook: Lloyd-Max for N(0,1) ("per-coordinate Lloyd-Max";
//    fit unspecified, reading [R1]), exactly symmetrised [R2], scaled by
//    1/sqrt(d), rounded to fp32; thresholds are fp32 midpoints of adjacent
//    fp32 centroids [R14b].
#include <cuda_fp16.h>

#include <cmath>
#include <cstring>
#include <limits>

#include "iq_internal.h"

namespace iq {
namespace {

constexpr uint64_t kGamma = 0x9E3779B97F4A7C15ull;
constexpr uint64_t kThetaStreamKey = 0x2D358DCCAA6C78A5ull;
constexpr uint64_t kResampleStride = 1ull << 40;

// k-th output of SplitMix64 seeded with s: mix(s + (k+1) * gamma).
inline uint64_t splitmix64_at(uint64_t s, uint64_t k) {
  uint64_t z = s + (k + 1) * kGamma;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

// Uniform in (0, 1].
inline double unit_open0(uint64_t s, uint64_t k) {
  return static_cast<double>((splitmix64_at(s, k) >> 11) + 1) * (1.0 / 9007199254740992.0);
}

// j-th standard normal: Box-Muller on uniforms (2p, 2p+1), p = j/2;
// even j -> cosine branch, odd j -> sine branch.
inline double normal_at(uint64_t s, uint64_t j) {
  const uint64_t p = j / 2;
  const double u1 = unit_open0(s, 2 * p);
  const double u2 = unit_open0(s, 2 * p + 1);
  const double r = std::sqrt(-2.0 * std::log(u1));
  const double t = 2.0 * M_PI * u2;
  return r * ((j % 2 == 0) ? std::cos(t) : std::sin(t));
}

void unit_quaternion(uint64_t s, uint64_t j0, double q[4]) {
  for (uint64_t attempt = 0;; ++attempt) {
    const uint64_t off = j0 + attempt * kResampleStride;
    double u[4];
    for (int c = 0; c < 4; ++c) u[c] = normal_at(s, off + c);
    const double nrm = std::sqrt(u[0] * u[0] + u[1] * u[1] + u[2] * u[2] + u[3] * u[3]);
    if (nrm >= 1e-12) {
      for (int c = 0; c < 4; ++c) q[c] = u[c] / nrm;
      return;
    }
  }
}

// Hamilton product r = a * b, components (w, x, y, z) = w + x i + y j + z k.
inline void hamilton(const double a[4], const double b[4], double r[4]) {
  r[0] = a[0] * b[0] - a[1] * b[1] - a[2] * b[2] - a[3] * b[3];
  r[1] = a[0] * b[1] + a[1] * b[0] + a[2] * b[3] - a[3] * b[2];
  r[2] = a[0] * b[2] - a[1] * b[3] + a[2] * b[0] + a[3] * b[1];
  r[3] = a[0] * b[3] + a[1] * b[2] - a[2] * b[1] + a[3] * b[0];
}

inline double Phi(double x) {
  if (std::isinf(x)) return x > 0 ? 1.0 : 0.0;
  return 0.5 * std::erfc(-x / std::sqrt(2.0));
}
inline double phi(double x) {
  if (std::isinf(x)) return 0.0;
  return std::exp(-0.5 * x * x) / std::sqrt(2.0 * M_PI);
}

// Inverse normal CDF for the Lloyd start point only (any monotone start
// converges to the same fixed point): bisection on Phi, fp64.
double inv_Phi(double p) {
  double lo = -40.0, hi = 40.0;
  for (int i = 0; i < 200; ++i) {
    const double mid = 0.5 * (lo + hi);
    if (Phi(mid) < p) lo = mid; else hi = mid;
  }
  return 0.5 * (lo + hi);
}

// Lloyd-Max levels of a b-bit quantizer for N(0,1), symmetrised exactly.
std::vector<double> lloyd_max_gaussian(int bits) {
  const int L = 1 << bits;
  std::vector<double> c(L), t(L + 1), nc(L);
  for (int k = 0; k < L; ++k) c[k] = inv_Phi((k + 0.5) / L);
  const double inf = std::numeric_limits<double>::infinity();
  for (int it = 0; it < 200000; ++it) {
    t[0] = -inf;
    t[L] = inf;
    for (int k = 0; k + 1 < L; ++k) t[k + 1] = 0.5 * (c[k] + c[k + 1]);
    double delta = 0.0;
    for (int k = 0; k < L; ++k) {
      nc[k] = (phi(t[k]) - phi(t[k + 1])) / (Phi(t[k + 1]) - Phi(t[k]));
      delta = std::fmax(delta, std::fabs(nc[k] - c[k]));
    }
    c.swap(nc);
    if (delta < 1e-15) break;
  }
  const int h = L / 2;
  std::vector<double> pos(h), out(L);
  for (int m = 0; m < h; ++m) pos[m] = 0.5 * (c[h + m] - c[h - 1 - m]);
  for (int m = 0; m < h; ++m) {
    out[h + m] = pos[m];
    out[h - 1 - m] = -pos[m];
  }
  return out;
}

// Uniform-grid decision tables (reading R19, see KCodebook).  S is the
// largest power of two for which the last positive threshold lands in a cell
// below 15 (so NC = cell + 2 <= 16); the cells of the thresholds must then be
// distinct.  The construction is verified exhaustively against the counting
// definition code = #{m : u >= tau_m S} on every threshold, its fp32
// neighbours and every cell boundary.
bool build_grid(KCodebook& kc, int h, std::string* err) {
  const float inf = std::numeric_limits<float>::infinity();
  const float tmax = h > 1 ? kc.tau[h - 1] : 0.0f;
  float S = 1.0f;
  if (h > 1) {
    S = std::ldexp(1.0f, 40);
    while (S > 0.0f && std::floor(tmax * S) > 14.0f) S *= 0.5f;
  }
  int cell[kMaxHalf] = {0};
  for (int m = 1; m < h; ++m) {
    cell[m] = static_cast<int>(std::floor(kc.tau[m] * S));   // tau * S exact (S = 2^k)
    if (m > 1 && cell[m] <= cell[m - 1]) { *err = "grid: two thresholds share a cell"; return false; }
  }
  const int nc = (h > 1 ? cell[h - 1] : -1) + 2;
  if (nc > 16) { *err = "grid: more than 16 cells"; return false; }
  kc.gscale = S;
  kc.gclamp = 0x4B000000u + static_cast<uint32_t>(nc - 1);
  for (int j = 0; j < 16; ++j) {
    float t = inf;
    int mstart = 0;
    for (int m = 1; m < h; ++m) {
      if (cell[m] == j) t = std::nextafter(kc.tau[m] * S, 0.0f);   // nextdown (see grid_index)
      if (cell[m] < j) ++mstart;
    }
    kc.gtab[j] = t;
    kc.gval[j] = kc.cpos[mstart];
    kc.gcode[j] = static_cast<uint32_t>(mstart | h);
    kc.gtab[16 + j] = inf;
    kc.gval[16 + j] = 0.0f;
    kc.gcode[16 + j] = 0u;
  }
  // check the decision at every threshold, its fp32 neighbours and every
  // cell boundary against the counting definition
  std::vector<float> probes = {0.0f, 1e30f};   // (the kernels' u is finite)
  for (int m = 1; m < h; ++m) {
    const float t = kc.tau[m] * S;
    probes.insert(probes.end(), {t, std::nextafter(t, 0.0f), std::nextafter(t, inf)});
  }
  for (int j = 0; j <= 17; ++j) {
    const float b = static_cast<float>(j);
    probes.insert(probes.end(), {b, std::nextafter(b, 0.0f), std::nextafter(b, inf)});
  }
  for (float u : probes) {
    int want = 0;
    for (int m = 1; m < h; ++m) want += (u >= kc.tau[m] * S);
    float fl = std::floor(u);
    uint32_t j = fl >= static_cast<float>(nc - 1) ? static_cast<uint32_t>(nc - 1) : static_cast<uint32_t>(fl);
    const float dlt = kc.gtab[j] - u;                            // the kernel's test
    const uint32_t idx = (j + (std::signbit(dlt) ? 1u : 0u)) & 31u;
    const int got = static_cast<int>(kc.gcode[idx]) - h;
    if (got != want || kc.gval[idx] != kc.cpos[want]) {
      *err = "grid: decision table self-check failed";
      return false;
    }
  }
  return true;
}

}  // namespace

size_t rotation_param_count(int d, int variant) {
  const size_t g4 = (d + 3) / 4, g2 = (d + 1) / 2;
  switch (variant) {
    case IQ_VARIANT_FULL: return 8 * g4;
    case IQ_VARIANT_FAST: return 4 * g4;
    case IQ_VARIANT_PLANAR2D: return 2 * g2;
    default: return 0;
  }
}

size_t block_matrix_count(int d, int variant) {
  if (variant == IQ_VARIANT_PLANAR2D) return 4 * static_cast<size_t>((d + 1) / 2);
  return 16 * static_cast<size_t>((d + 3) / 4);
}

bool build_host_params(int d, int bits, int variant, uint64_t seed, HostParams* hp,
                       std::string* err, const double* rot_in) {
  if (d < 1 || d > (1 << 20)) { *err = "d must be in [1, 2^20]"; return false; }
  if (bits < 1 || bits > kMaxBits) { *err = "bits must be in [1, 4]"; return false; }
  if (variant < IQ_VARIANT_FULL || variant > IQ_VARIANT_PLANAR2D) {
    *err = "variant must be 0 (full), 1 (fast) or 2 (planar2d)";
    return false;
  }
  hp->d = d;
  hp->bits = bits;
  hp->variant = variant;
  hp->seed = seed;
  hp->rot.assign(rotation_param_count(d, variant), 0.0);
  hp->mat.assign(block_matrix_count(d, variant), 0.0f);

  if (variant == IQ_VARIANT_PLANAR2D) {
    const uint64_t s2 = seed ^ kThetaStreamKey;
    const int g2 = (d + 1) / 2;
    for (int j = 0; j < g2; ++j) {
      double c, s;
      if (rot_in) {                                   // explicit (cos, sin), normalised
        const double r = std::hypot(rot_in[2 * j], rot_in[2 * j + 1]);
        if (!(r > 1e-12)) { *err = "explicit 2D parameters must be nonzero pairs"; return false; }
        c = rot_in[2 * j] / r;
        s = rot_in[2 * j + 1] / r;
      } else {
        const double th = 2.0 * M_PI * unit_open0(s2, j);
        c = std::cos(th);
        s = std::sin(th);
      }
      hp->rot[2 * j] = c;
      hp->rot[2 * j + 1] = s;
      // R(theta) = [[c, -s], [s, c]] row-major
      float* m = &hp->mat[4 * j];
      m[0] = static_cast<float>(c);
      m[1] = static_cast<float>(-s);
      m[2] = static_cast<float>(s);
      m[3] = static_cast<float>(c);
    }
  } else {
    const int g = (d + 3) / 4;
    const bool full = variant == IQ_VARIANT_FULL;
    for (int b = 0; b < g; ++b) {
      double qL[4], qR[4] = {1.0, 0.0, 0.0, 0.0};
      const int stride = full ? 8 : 4;
      if (rot_in) {                                   // explicit quaternions u -> u / ||u||
        for (int part = 0; part < (full ? 2 : 1); ++part) {
          const double* u = rot_in + stride * b + 4 * part;
          const double nu = std::sqrt(u[0] * u[0] + u[1] * u[1] + u[2] * u[2] + u[3] * u[3]);
          if (!(nu > 1e-12)) { *err = "explicit quaternions must be nonzero"; return false; }
          double* q = part ? qR : qL;
          for (int c = 0; c < 4; ++c) q[c] = u[c] / nu;
        }
      } else {
        unit_quaternion(seed, 8ull * b, qL);
        if (full) unit_quaternion(seed, 8ull * b + 4, qR);
      }
      for (int c = 0; c < 4; ++c) hp->rot[stride * b + c] = qL[c];
      if (full) for (int c = 0; c < 4; ++c) hp->rot[stride * b + 4 + c] = qR[c];
      // Column j of M is T(e_j): Full q_L e_j conj(q_R), Fast q_L e_j.
      const double qRc[4] = {qR[0], -qR[1], -qR[2], -qR[3]};
      for (int j = 0; j < 4; ++j) {
        double e[4] = {0, 0, 0, 0}, t1[4], t2[4];
        e[j] = 1.0;
        hamilton(qL, e, t1);
        if (full) hamilton(t1, qRc, t2); else std::memcpy(t2, t1, sizeof t2);
        for (int i = 0; i < 4; ++i) hp->mat[16 * b + 4 * i + j] = static_cast<float>(t2[i]);
      }
    }
  }

  // Codebook [R1][R2][R14b]
  const std::vector<double> lv = lloyd_max_gaussian(bits);
  const int L = 1 << bits, h = L / 2;
  hp->centroids.resize(L);
  hp->thresholds.resize(L - 1);
  const double scale = 1.0 / std::sqrt(static_cast<double>(d));
  for (int k = 0; k < L; ++k) hp->centroids[k] = static_cast<float>(lv[k] * scale);
  for (int k = 0; k + 1 < L; ++k)
    hp->thresholds[k] = static_cast<float>(
        (static_cast<double>(hp->centroids[k]) + static_cast<double>(hp->centroids[k + 1])) * 0.5);
  KCodebook& kc = hp->kcb;
  std::memset(&kc, 0, sizeof kc);
  kc.n_sets = 1;
  kc.set_rows = 0;
  kc.set_stride = static_cast<int32_t>(hp->mat.size());
  for (int m = 0; m < h; ++m) kc.cpos[m] = hp->centroids[h + m];
  for (int m = 1; m < h; ++m) kc.tau[m] = hp->thresholds[h - 1 + m];
  for (int m = 0; m < kMaxHalf; ++m) std::memcpy(&kc.tau_bits[m], &kc.tau[m], 4);
  for (int m = h; m < kMaxHalf; ++m) kc.tau_bits[m] = 0xFFFFFFFFu;  // never reached
  for (int k = 0; k < L; ++k) kc.cent[k] = hp->centroids[k];
  // Exact steps: fl(cpos[m-1] + delta) must equal cpos[m] (fp32 add, RN) so
  // that the kernels' indicator-FMA chain reproduces the table value bit for
  // bit; search the fp32 neighbours of the rounded difference.
  for (int m = 1; m < h; ++m) {
    const float a = kc.cpos[m - 1], b = kc.cpos[m];
    float dlt = b - a;
    volatile float probe = a + dlt;
    for (int step = 0; probe != b && step < 64; ++step) {
      dlt = (probe < b) ? std::nextafter(dlt, 1.0f) : std::nextafter(dlt, -1.0f);
      probe = a + dlt;
    }
    if (probe != b) { *err = "no exact fp32 codebook step"; return false; }
    kc.delta[m] = dlt;
  }
  if (!build_grid(kc, h, err)) return false;
  return true;
}

// ------------------------------------------------------------ sets (R31)
bool add_param_sets(HostParams* hp, int n_sets, int64_t set_rows, std::string* err) {
  if (n_sets < 1) { *err = "n_sets must be >= 1"; return false; }
  const size_t nmat = hp->mat.size();
  for (int s = 1; s < n_sets; ++s) {
    HostParams t;
    if (!build_host_params(hp->d, hp->bits, hp->variant, hp->seed + static_cast<uint64_t>(s), &t, err))
      return false;
    hp->rot.insert(hp->rot.end(), t.rot.begin(), t.rot.end());
    hp->mat.insert(hp->mat.end(), t.mat.begin(), t.mat.end());
  }
  hp->n_sets = n_sets;
  hp->set_rows = set_rows;
  hp->kcb.n_sets = n_sets;
  hp->kcb.set_rows = set_rows;
  hp->kcb.set_stride = static_cast<int32_t>(nmat);
  return true;
}

// ------------------------------------------------------- learning (R29, R30)
// dL/dM_b -> dL/d(rot).  Full: M = L(q_L) R(conj q_R), column j of M is
// q_L e_j conj(q_R), so dL/dq_L[k] = sum_ij G_ij (e_k e_j conj(q_R))_i and
// dL/dq_R[k] = sum_ij G_ij (q_L e_j conj(e_k))_i; Fast drops q_R; 2D: M =
// [[c, -s], [s, c]].  Each unit vector's gradient is projected on the tangent
// space (g - (g.q) q), the gradient with respect to u at ||u|| = 1.
void operator_grad_to_rot(const HostParams& hp, const double* G, double* grad_rot) {
  if (hp.variant == IQ_VARIANT_PLANAR2D) {
    const int g2 = (hp.d + 1) / 2;
    for (int j = 0; j < g2; ++j) {
      const double* m = G + 4 * j;
      const double c = hp.rot[2 * j], s = hp.rot[2 * j + 1];
      const double gc = m[0] + m[3], gs = -m[1] + m[2];
      const double dot = gc * c + gs * s;
      grad_rot[2 * j] = gc - dot * c;
      grad_rot[2 * j + 1] = gs - dot * s;
    }
    return;
  }
  const bool full = hp.variant == IQ_VARIANT_FULL;
  const int stride = full ? 8 : 4;
  const int g = (hp.d + 3) / 4;
  for (int b = 0; b < g; ++b) {
    const double* qL = &hp.rot[stride * b];
    const double qR[4] = {full ? hp.rot[stride * b + 4] : 1.0, full ? hp.rot[stride * b + 5] : 0.0,
                          full ? hp.rot[stride * b + 6] : 0.0, full ? hp.rot[stride * b + 7] : 0.0};
    const double qRc[4] = {qR[0], -qR[1], -qR[2], -qR[3]};
    const double* Gb = G + 16 * b;
    double gl[4] = {0, 0, 0, 0}, gr[4] = {0, 0, 0, 0};
    for (int k = 0; k < 4; ++k) {
      double ek[4] = {0, 0, 0, 0};
      ek[k] = 1.0;
      const double ekc[4] = {ek[0], -ek[1], -ek[2], -ek[3]};
      for (int j = 0; j < 4; ++j) {
        double ej[4] = {0, 0, 0, 0}, t1[4], t2[4];
        ej[j] = 1.0;
        hamilton(ek, ej, t1);
        hamilton(t1, qRc, t2);                               // e_k e_j conj(q_R)
        for (int i = 0; i < 4; ++i) gl[k] += Gb[4 * i + j] * t2[i];
        if (full) {
          hamilton(qL, ej, t1);
          hamilton(t1, ekc, t2);                             // q_L e_j conj(e_k)
          for (int i = 0; i < 4; ++i) gr[k] += Gb[4 * i + j] * t2[i];
        }
      }
    }
    for (int part = 0; part < (full ? 2 : 1); ++part) {
      const double* q = part ? qR : qL;
      const double* gq = part ? gr : gl;
      const double dot = gq[0] * q[0] + gq[1] * q[1] + gq[2] * q[2] + gq[3] * q[3];
      for (int c = 0; c < 4; ++c) grad_rot[stride * b + 4 * part + c] = gq[c] - dot * q[c];
    }
  }
}

// ---------------------------------------------------------------- stage 2
// Sketch matrix of the residual correction (R20): S is
// m x d with m = d, S[i][k] = fp16_rn(N_(i*d + k)) where N_j is the j-th
// standard normal of the parameter generator [R12] keyed with
// seed ^ kQjlStreamKey.  The fp16-rounded values ARE the sketch (both the
// kernels and the oracle use them exactly).
namespace {
constexpr uint64_t kQjlStreamKey = 0x514A4C534B455443ull;

// IEEE binary16 bits of x, rounded to nearest even directly from double.
uint16_t half_rn(double x) {
  uint16_t sign = std::signbit(x) ? 0x8000 : 0;
  double a = std::fabs(x);
  if (std::isnan(a)) return 0x7E00;
  if (a >= 65520.0) return sign | 0x7C00;                     // rounds to infinity
  if (a < std::ldexp(1.0, -14)) {                              // subnormal (or zero)
    const double q = std::nearbyint(a * std::ldexp(1.0, 24));  // units of 2^-24
    return sign | static_cast<uint16_t>(q);                    // q == 1024 -> min normal
  }
  int e;
  std::frexp(a, &e);                                           // a = f * 2^e, f in [0.5, 1)
  e -= 1;                                                      // a in [2^e, 2^(e+1))
  double q = std::nearbyint(std::ldexp(a, 10 - e));            // [1024, 2048]
  if (q >= 2048.0) { q = 1024.0; ++e; }
  if (e > 15) return sign | 0x7C00;
  return sign | static_cast<uint16_t>(((e + 15) << 10) | (static_cast<int>(q) - 1024));
}
}  // namespace

bool qjl_fused(int d) { return d == 64 || d == 128; }
bool qjl_supported(int d) { return qjl_fused(d) || d == 256 || d == 512; }

bool build_qjl(HostParams* hp, std::string* err) {
  const int d = hp->d, m = d;
  if (d <= 0 || d % 8 != 0) { *err = "stage-2 sketch needs d % 8 == 0"; return false; }
  const uint64_t s = hp->seed ^ kQjlStreamKey;
  hp->qjl_half.assign(static_cast<size_t>(m) * d, 0);
  for (int i = 0; i < m; ++i)
    for (int k = 0; k < d; ++k)
      hp->qjl_half[static_cast<size_t>(i) * d + k] = half_rn(normal_at(s, static_cast<uint64_t>(i) * d + k));
  hp->qjl_img.clear();
  if (qjl_supported(d)) {
    hp->qjl_img.assign(static_cast<size_t>(m) * d * 2, 0);
    for (int i = 0; i < m; ++i)
      for (int k = 0; k < d; ++k)
        std::memcpy(&hp->qjl_img[umma_sw128_off(i, k, m)], &hp->qjl_half[static_cast<size_t>(i) * d + k], 2);
  }
  // S as the consumer's S q A operand: 128-row tiles (rows >= m zero), tile
  // t holding sketch rows 128 t .. 128 t + 127 (d <= 256: the consumer's
  // stage-2 widths)
  hp->qjl_img_a.clear();
  if (d <= 256) {
    const int mt = (m + 127) / 128;
    const size_t tile = static_cast<size_t>(128) * d * 2;
    hp->qjl_img_a.assign(mt * tile, 0);
    for (int i = 0; i < m; ++i)
      for (int k = 0; k < d; ++k)
        std::memcpy(&hp->qjl_img_a[(i / 128) * tile + umma_sw128_off(i % 128, k, 128)],
                    &hp->qjl_half[static_cast<size_t>(i) * d + k], 2);
  }
  hp->qjl_img_rot.clear();
  if (qjl_fused(d)) {
    const int pw = hp->variant == IQ_VARIANT_PLANAR2D ? 2 : 4;
    const size_t img = static_cast<size_t>(m) * d * 2;
    hp->qjl_img_rot.assign(2 * img, 0);
    for (int i = 0; i < m; ++i)
      for (int b = 0; b < d / pw; ++b)
        for (int j = 0; j < pw; ++j) {
          // S'[i][pw b + j] = sum_c S[i][pw b + c] M_b[j][c]   (S' = S M^T)
          double acc = 0.0;
          for (int c = 0; c < pw; ++c) {
            __half_raw hr;
            hr.x = hp->qjl_half[static_cast<size_t>(i) * d + pw * b + c];
            acc += static_cast<double>(__half2float(__half(hr))) *
                   static_cast<double>(hp->mat[static_cast<size_t>(pw * pw) * b + pw * j + c]);
          }
          const uint16_t hi = half_rn(acc);
          __half_raw hh;
          hh.x = hi;
          const uint16_t lo = half_rn(acc - static_cast<double>(__half2float(__half(hh))));
          const uint32_t off = umma_sw128_off(i, pw * b + j, m);
          std::memcpy(&hp->qjl_img_rot[off], &hi, 2);
          std::memcpy(&hp->qjl_img_rot[img + off], &lo, 2);
        }
  }
  hp->has_qjl = true;
  return true;
}

}  // namespace iq
