// data_io.cpp -- host-side data formats either side of the hot path
// (the `cnmf factorize` / `cnmf project` front end).
//
// These are the reference's host utilities that decide WHICH matrix reaches
// the device and how its compressed views are judged; they are not on the
// device hot path and stay host C++ here too (fp64, sequential, so their
// output is bitwise the reference's on the same libm):
//   cnmf_generate_synthetic    generate_synthetic   data_io.cpp:376-415
//   cnmf_pairwise_distortion   pairwise_distortion  metrics.cpp:123-155
//   cnmf_estimate_cost         estimate_cost        metrics.cpp:20-50
// The random stream is cnmf::Rng (rng.hpp:13-60) on std::mt19937_64, whose
// output sequence the C++ standard fixes.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <random>
#include <string>
#include <vector>

#include "../../include/cnmf_b200.h"

namespace {

// cnmf::Rng draws: uniform = top 53 bits * 2^-53; uniform_positive rejects 0;
// normal = Box-Muller on (uniform_positive, uniform), the sine half cached
// for the next call; index = rejection below the largest multiple of n.
class Stream {
 public:
  explicit Stream(uint64_t seed) : e_(seed) {}
  double uniform() { return static_cast<double>(e_() >> 11) * 0x1.0p-53; }
  double uniform_positive() {
    double v = uniform();
    while (v == 0.0) v = uniform();
    return v;
  }
  double normal() {
    if (cached_) {
      cached_ = false;
      return cache_;
    }
    const double u1 = uniform_positive();
    const double u2 = uniform();
    const double rad = std::sqrt(-2.0 * std::log(u1));
    const double theta = 2.0 * 3.141592653589793238462643383279502884 * u2;
    cache_ = rad * std::sin(theta);
    cached_ = true;
    return rad * std::cos(theta);
  }
  uint64_t index(uint64_t n) {
    const uint64_t limit = ~uint64_t(0) / n * n;
    uint64_t x = e_();
    while (x >= limit) x = e_();
    return x % n;
  }

 private:
  std::mt19937_64 e_;
  double cache_ = 0.0;
  bool cached_ = false;
};

void set_msg(char* msg, size_t cap, const std::string& m) {
  if (msg && cap) std::snprintf(msg, cap, "%s", m.c_str());
}

// Orthonormal factor Q (rows x cols, row-major) of a tall matrix by
// Householder reflections: the reflector for column j maps w(j:, j) to
// alpha e_1 with alpha = -sign(w_jj) |w(j:, j)|; columns whose remaining norm
// is below 1e-12 |M|_F are treated as dependent (no reflection, zero R
// diagonal).  Q = H_0 ... H_{c-1} applied to the leading identity columns,
// last reflector first.  Same arithmetic order as qr.cpp:10-76 (every
// sum runs over increasing row index), hence the same bits.
std::vector<double> householder_q(std::vector<double> w, size_t rows, size_t cols) {
  double fro = 0.0;
  for (double v : w) fro += v * v;
  const double floor_norm = 1e-12 * std::sqrt(fro);
  std::vector<std::vector<double>> refl(cols);
  std::vector<double> col(rows);
  for (size_t j = 0; j < cols; ++j) {
    double ss = 0.0;
    for (size_t i = j; i < rows; ++i) ss += w[i * cols + j] * w[i * cols + j];
    const double nrm = std::sqrt(ss);
    if (nrm < floor_norm) {
      for (size_t i = j; i < rows; ++i) w[i * cols + j] = 0.0;
      continue;
    }
    const double alpha = w[j * cols + j] >= 0.0 ? -nrm : nrm;
    std::vector<double>& v = refl[j];
    v.resize(rows - j);
    for (size_t i = j; i < rows; ++i) v[i - j] = w[i * cols + j];
    v[0] -= alpha;
    double vv = 0.0;
    for (double t : v) vv += t * t;
    const double vn = std::sqrt(vv);
    for (double& t : v) t /= vn;
    for (size_t c = j; c < cols; ++c) {
      double p = 0.0;
      for (size_t i = j; i < rows; ++i) p += v[i - j] * w[i * cols + c];
      p *= 2.0;
      for (size_t i = j; i < rows; ++i) w[i * cols + c] -= p * v[i - j];
    }
    w[j * cols + j] = alpha;
    for (size_t i = j + 1; i < rows; ++i) w[i * cols + j] = 0.0;
  }
  std::vector<double> q(rows * cols, 0.0);
  for (size_t j = 0; j < cols; ++j) q[j * cols + j] = 1.0;
  for (size_t jj = cols; jj-- > 0;) {
    const std::vector<double>& v = refl[jj];
    if (v.empty()) continue;
    for (size_t c = 0; c < cols; ++c) {
      double p = 0.0;
      for (size_t i = jj; i < rows; ++i) p += v[i - jj] * q[i * cols + c];
      p *= 2.0;
      for (size_t i = jj; i < rows; ++i) q[i * cols + c] -= p * v[i - jj];
    }
  }
  return q;
}

bool is_rp(int a) { return a == CNMF_MU_RP || a == CNMF_HALS_RP || a == CNMF_FASTHALS_RP; }

}  // namespace

extern "C" {

cnmf_status cnmf_generate_synthetic(uint64_t d, uint64_t n, uint64_t true_rank, double decay_p,
                                    double noise_level, uint64_t seed, double* out, char* msg,
                                    size_t msg_cap) {
  if (d == 0 || n == 0) {
    set_msg(msg, msg_cap, "synthetic dimensions must be positive");
    return CNMF_ERR_CONFIG;
  }
  if (true_rank == 0 || true_rank > std::min(d, n)) {
    set_msg(msg, msg_cap, "true_rank must satisfy 1 <= true_rank <= min(d, n)");
    return CNMF_ERR_CONFIG;
  }
  if (!(decay_p >= 0.0) || !(noise_level >= 0.0)) {
    set_msg(msg, msg_cap, "decay_p and noise_level must be non-negative");
    return CNMF_ERR_CONFIG;
  }
  const size_t r = true_rank;
  Stream rng(seed);
  std::vector<double> u(d * r), v(n * r);
  for (double& t : u) t = rng.normal();
  for (double& t : v) t = rng.normal();
  u = householder_q(std::move(u), d, r);
  v = householder_q(std::move(v), n, r);
  // spectrum j^(-decay_p) folded into U's columns, X = (U S) V^T
  for (size_t j = 0; j < r; ++j) {
    const double s = std::pow(static_cast<double>(j + 1), -decay_p);
    for (size_t i = 0; i < d; ++i) u[i * r + j] *= s;
  }
  for (size_t i = 0; i < d; ++i) {
    const double* ui = &u[i * r];
    for (size_t j = 0; j < n; ++j) {
      const double* vj = &v[j * r];
      double s = 0.0;
      for (size_t l = 0; l < r; ++l) s += ui[l] * vj[l];
      out[i * n + j] = s;
    }
  }
  const size_t total = d * n;
  if (noise_level > 0.0) {
    for (size_t e = 0; e < total; ++e) out[e] += noise_level * rng.normal();
  } else {
    // shift by the minimum so the final clamp removes nothing
    const double lo = *std::min_element(out, out + total);
    if (lo < 0.0)
      for (size_t e = 0; e < total; ++e) out[e] -= lo;
  }
  for (size_t e = 0; e < total; ++e) out[e] = out[e] > 0.0 ? out[e] : 0.0;
  return CNMF_OK;
}

cnmf_status cnmf_pairwise_distortion(const double* x, uint64_t d, uint64_t n, const float* xhat,
                                     uint64_t q, uint64_t sample_pairs, uint64_t seed,
                                     double* max_relative, double* mean_relative, char* msg,
                                     size_t msg_cap) {
  if (n < 2) {
    set_msg(msg, msg_cap, "pairwise_distortion: need at least two columns");
    return CNMF_ERR_INPUT;
  }
  if (sample_pairs == 0) {
    set_msg(msg, msg_cap, "pairwise_distortion: sample_pairs must be positive");
    return CNMF_ERR_INPUT;
  }
  Stream rng(seed);
  double mx = 0.0, sum = 0.0;
  for (uint64_t s = 0; s < sample_pairs; ++s) {
    const uint64_t i = rng.index(n);
    uint64_t j = rng.index(n);
    while (j == i) j = rng.index(n);
    double a = 0.0, b = 0.0;
    for (uint64_t r = 0; r < d; ++r) {
      const double t = x[r * n + i] - x[r * n + j];
      a += t * t;
    }
    for (uint64_t r = 0; r < q; ++r) {
      const double t = static_cast<double>(xhat[r * n + i]) - static_cast<double>(xhat[r * n + j]);
      b += t * t;
    }
    const double orig = std::sqrt(a), comp = std::sqrt(b);
    const double rel = orig == 0.0 ? 0.0 : std::abs(comp - orig) / orig;
    mx = std::max(mx, rel);
    sum += rel;
  }
  *max_relative = mx;
  *mean_relative = sum / static_cast<double>(sample_pairs);
  return CNMF_OK;
}

cnmf_status cnmf_estimate_cost(int algorithm, uint64_t d, uint64_t n, uint64_t k, uint64_t q,
                               cnmf_cost_estimate* out, char* msg, size_t msg_cap) {
  if (algorithm < CNMF_MU || algorithm > CNMF_FASTHALS_RP) {
    set_msg(msg, msg_cap, "estimate_cost: unknown algorithm");
    return CNMF_ERR_CONFIG;
  }
  if (d == 0 || n == 0 || k == 0) {
    set_msg(msg, msg_cap, "estimate_cost: d, n, k must all be positive");
    return CNMF_ERR_CONFIG;
  }
  if (is_rp(algorithm) && q == 0) {
    set_msg(msg, msg_cap, "estimate_cost: compressed algorithms require q > 0");
    return CNMF_ERR_CONFIG;
  }
  if (!is_rp(algorithm) && q != 0) {
    set_msg(msg, msg_cap, "estimate_cost: q applies to compressed algorithms only");
    return CNMF_ERR_CONFIG;
  }
  const double dd = (double)d, dn = (double)n, dk = (double)k, dq = (double)q;
  double f = 0.0;
  switch (algorithm) {
    case CNMF_MU:
    case CNMF_HALS: f = 8.0 * dd * dn * dk; break;
    case CNMF_FASTHALS: f = 4.0 * dd * dn * dk; break;
    case CNMF_MU_RP: f = 4.0 * dd * dk * dq; break;
    case CNMF_HALS_RP: f = 4.0 * dd * dn * dk * dq; break;
    default: f = 2.0 * dd * dk * dq; break;
  }
  out->algorithm = algorithm;
  out->d = d;
  out->n = n;
  out->k = k;
  out->q = q;
  out->flops_per_iteration = f;
  out->memory_floats = is_rp(algorithm) ? (2.0 * dq + dk) * (dd + dn) : dd * dn + dd * dk + dn * dk;
  return CNMF_OK;
}

}  // extern "C"
