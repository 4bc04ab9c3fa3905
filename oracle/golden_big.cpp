// golden_big.cpp -- full-size reference trajectories for the BASELINE configs.
//
// TEST INFRASTRUCTURE ONLY (golden generator).  oracle/Makefile links this
// file with the reference's own, unmodified sources (where they lie under
// /root/reference/proj/src) and the oracle's synthetic generator
// (cnmf_oracle.c, orc_synth_x_block) into oracle/_ref/golden_big.  Run by
// tests/golden/make_golden_big.py here, where /root/reference exists; the
// fixtures it writes are committed, the binary is not.
//
// It restates run_impl (solvers.cpp:189-294) step by step through the
// reference's PUBLIC functions so that it can also record what run() keeps
// private:
//   * the number of raw mt19937_64 draws each fasthals_rp_step consumed from
//     the run Rng (its dead-component redraws, solvers.cpp:28-31,424-452);
//   * per-step seconds.
// Everything that decides the trajectory is the reference's own code:
// Rng (rng.hpp), the A-then-B uniform_positive fill (solvers.cpp:206-211),
// build_projectors / compress_* (compression.cpp:44-96) and
// fasthals_rp_step (solvers.cpp:414-456).  The objective is the reference's
// reconstruction_error (metrics.cpp:61-77) evaluated on row blocks in
// parallel threads and summed in block order: the same terms as the serial
// loop, grouped differently (a few ulp in the fp64 sum), so an error
// evaluation at 50000 x 100000 takes ~1 min instead of ~6.
//
// X is built in place as the reference's fp64 DenseMatrix from the fp32
// synthetic values (no second copy: C4 is 40 GB in fp64).
#include <atomic>
#include <chrono>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include "cnmf/compression.hpp"
#include "cnmf/metrics.hpp"
#include "cnmf/qr.hpp"
#include "cnmf/rng.hpp"
#include "cnmf/solvers.hpp"

extern "C" void orc_synth_x_block(size_t d, size_t n, size_t rank, int factor_kind,
                                  int noise_kind, double sigma, uint64_t seed, size_t row_lo,
                                  size_t row_hi, size_t col_lo, size_t col_hi, size_t ldx,
                                  float* xf, double* xd);

using namespace cnmf;
using clk = std::chrono::steady_clock;

namespace {

int g_threads = 8;

double secs(clk::time_point a) { return std::chrono::duration<double>(clk::now() - a).count(); }

template <typename F>
void parallel_blocks(std::size_t rows, std::size_t block, F&& f) {
  const std::size_t nb = (rows + block - 1) / block;
  std::atomic<std::size_t> next{0};
  std::vector<std::thread> th;
  for (int t = 0; t < g_threads; ++t)
    th.emplace_back([&] {
      for (std::size_t b; (b = next.fetch_add(1)) < nb;)
        f(b, b * block, std::min(rows, (b + 1) * block));
    });
  for (auto& t : th) t.join();
}

// reconstruction_error (metrics.cpp:61-77) over row blocks, summed in order.
double par_error(const DenseMatrix& x, const FactorPair& f) {
  const std::size_t block = 500;
  const std::size_t nb = (x.rows + block - 1) / block;
  std::vector<double> part(nb, 0.0);
  parallel_blocks(x.rows, block, [&](std::size_t b, std::size_t r0, std::size_t r1) {
    DenseMatrix xb(r1 - r0, x.cols);
    std::memcpy(xb.values.data(), x.row(r0), sizeof(double) * (r1 - r0) * x.cols);
    FactorPair fb;
    fb.a = DenseMatrix(r1 - r0, f.a.cols);
    std::memcpy(fb.a.values.data(), f.a.row(r0), sizeof(double) * (r1 - r0) * f.a.cols);
    fb.b = f.b;
    part[b] = reconstruction_error(xb, fb);
  });
  double s = 0.0;
  for (double p : part) s += p;
  return s;
}


// ---- sensitivity experiments (tools/c3_sensitivity.sh; never used for the
// committed goldens).  GOLDEN_RF_PERTURB=eps rebuilds the projectors with
// the reference's own gaussian_sketch and thin_qr but multithreaded fp64
// contractions, and multiplies every range-finder product (the sketch and each
// power-iteration product, before its thin_qr) by (1 + eps u), u uniform in
// [-1, 1): a stand-in for the device contraction's rounding.  The compressed
// views are then formed exactly (fp64).
std::uint64_t g_lcg = 0x9E3779B97F4A7C15ull;
void perturb(DenseMatrix& m, double eps) {
  if (eps == 0.0) return;
  for (double& v : m.values) {
    g_lcg = g_lcg * 6364136223846793005ull + 1442695040888963407ull;
    v *= 1.0 + eps * (static_cast<double>(g_lcg >> 11) * 0x1.0p-53 * 2.0 - 1.0);
  }
}
// x (d x n) * s (n x l), rows in parallel
DenseMatrix par_xs(const DenseMatrix& x, const DenseMatrix& s) {
  DenseMatrix y(x.rows, s.cols);
  parallel_blocks(x.rows, 64, [&](std::size_t, std::size_t r0, std::size_t r1) {
    for (std::size_t i = r0; i < r1; ++i)
      for (std::size_t j = 0; j < x.cols; ++j) {
        const double xv = x(i, j);
        const double* sr = s.row(j);
        double* yr = y.row(i);
        for (std::size_t c = 0; c < s.cols; ++c) yr[c] += xv * sr[c];
      }
  });
  return y;
}
// x^T (n x d) * t (d x l), output rows (columns of x) in parallel
DenseMatrix par_xts(const DenseMatrix& x, const DenseMatrix& t) {
  DenseMatrix z(x.cols, t.cols);
  parallel_blocks(x.cols, 256, [&](std::size_t, std::size_t c0, std::size_t c1) {
    for (std::size_t i = 0; i < x.rows; ++i) {
      const double* xr = x.row(i);
      const double* tr = t.row(i);
      for (std::size_t j = c0; j < c1; ++j) {
        double* zr = z.row(j);
        const double xv = xr[j];
        for (std::size_t c = 0; c < t.cols; ++c) zr[c] += xv * tr[c];
      }
    }
  });
  return z;
}
DenseMatrix rf_perturbed(const DenseMatrix& x, bool tr, std::size_t q, std::size_t w,
                         std::uint64_t seed, double eps) {
  const std::size_t op_cols = tr ? x.rows : x.cols;
  DenseMatrix omega = gaussian_sketch(op_cols, q, seed);
  DenseMatrix y = tr ? par_xts(x, omega) : par_xs(x, omega);
  perturb(y, eps);
  DenseMatrix basis = thin_qr(y).q;
  for (std::size_t it = 0; it < w; ++it) {
    DenseMatrix z0 = tr ? par_xs(x, basis) : par_xts(x, basis);
    perturb(z0, eps);
    DenseMatrix z = thin_qr(z0).q;
    DenseMatrix b0 = tr ? par_xts(x, z) : par_xs(x, z);
    perturb(b0, eps);
    basis = thin_qr(b0).q;
  }
  return basis;
}

void put(const std::string& dir, const std::string& name, const void* p, std::size_t bytes) {
  const std::string path = dir + "/" + name;
  FILE* fp = std::fopen(path.c_str(), "wb");
  if (!fp || std::fwrite(p, 1, bytes, fp) != bytes) {
    std::perror(path.c_str());
    std::exit(3);
  }
  std::fclose(fp);
}

}  // namespace

int main(int argc, char** argv) {
  if (argc < 16) {
    std::fprintf(stderr,
                 "usage: golden_big OUTDIR d n rank factor_kind noise_kind sigma data_seed "
                 "k q w iterations error_interval seed threads\n");
    return 2;
  }
  const std::string out = argv[1];
  const std::size_t d = std::strtoull(argv[2], nullptr, 10);
  const std::size_t n = std::strtoull(argv[3], nullptr, 10);
  const std::size_t rank = std::strtoull(argv[4], nullptr, 10);
  const int fkind = std::atoi(argv[5]), nkind = std::atoi(argv[6]);
  const double sigma = std::strtod(argv[7], nullptr);
  const std::uint64_t dseed = std::strtoull(argv[8], nullptr, 10);
  const std::size_t k = std::strtoull(argv[9], nullptr, 10);
  const std::size_t q = std::strtoull(argv[10], nullptr, 10);
  const std::size_t w = std::strtoull(argv[11], nullptr, 10);
  const std::size_t iters = std::strtoull(argv[12], nullptr, 10);
  const std::size_t interval = std::strtoull(argv[13], nullptr, 10);
  const std::uint64_t seed = std::strtoull(argv[14], nullptr, 10);
  g_threads = std::atoi(argv[15]);

  FILE* log = std::fopen((out + "/meta.txt").c_str(), "w");
  if (!log) {
    std::perror("meta.txt");
    return 3;
  }
  auto meta = [&](const char* key, double v) {
    std::fprintf(log, "%s=%.17g\n", key, v);
    std::fflush(log);
    std::fprintf(stderr, "%s=%.17g\n", key, v);
  };

  // X in place, fp64 holding the fp32 synthetic values.
  auto t = clk::now();
  DenseMatrix x(d, n);
  parallel_blocks(d, 256, [&](std::size_t, std::size_t r0, std::size_t r1) {
    orc_synth_x_block(d, n, rank, fkind, nkind, sigma, dseed, r0, r1, 0, n, n, nullptr,
                      x.row(r0));
  });
  meta("synth_seconds", secs(t));
  // Checksum of the fp32 bit patterns per 1000-row block (the GPU tests
  // compare their device-generated X against these).
  {
    const std::size_t hb = 1000, nb = (d + hb - 1) / hb;
    std::vector<std::uint64_t> hash(nb, 0);
    std::vector<double> sums(2 * nb, 0.0);
    parallel_blocks(d, hb, [&](std::size_t b, std::size_t r0, std::size_t r1) {
      std::uint64_t h = 0;
      double s = 0.0, s2 = 0.0;
      for (std::size_t i = r0; i < r1; ++i)
        for (std::size_t j = 0; j < n; ++j) {
          const float f = static_cast<float>(x(i, j));
          std::uint32_t u;
          std::memcpy(&u, &f, 4);
          h += u;
          s += f;
          s2 += static_cast<double>(f) * f;
        }
      hash[b] = h;
      sums[2 * b] = s;
      sums[2 * b + 1] = s2;
    });
    put(out, "x_hash.u64", hash.data(), nb * 8);
    put(out, "x_sums.f64", sums.data(), sums.size() * 8);
  }

  SolverConfig cfg;
  cfg.algorithm = Algorithm::fasthals_rp;
  cfg.k = k;
  cfg.sketch.q = q;
  cfg.sketch.power_iterations = w;
  cfg.sketch.seed = seed;
  cfg.max_iterations = iters;
  cfg.error_interval = interval;
  cfg.rel_tolerance = 1e-300;
  cfg.seed = seed;
  cfg.validate(d, n);

  // run_impl steps 4-5 (solvers.cpp:204-221).
  Rng rng(cfg.seed);
  FactorPair f;
  f.a = DenseMatrix(d, k);
  for (double& v : f.a.values) v = rng.uniform_positive();
  f.b = DenseMatrix(n, k);
  for (double& v : f.b.values) v = rng.uniform_positive();
  t = clk::now();
  const char* rfp = std::getenv("GOLDEN_RF_PERTURB");
  ProjectorPair p;
  if (rfp) {
    const double eps = std::strtod(rfp, nullptr);
    p.left = rf_perturbed(x, false, q, w, seed * 2, eps);
    p.right = transpose(rf_perturbed(x, true, q, w, seed * 2 + 1, eps));
    meta("rf_perturbed", eps);
  } else {
    p = build_projectors(x, cfg.sketch);
  }
  meta("build_projectors_seconds", secs(t));
  DenseMatrix xhat = rfp ? transpose(par_xts(x, p.left)) : compress_left(x, p);
  DenseMatrix xcheck = rfp ? par_xs(x, transpose(p.right)) : compress_right(x, p);
  // Sensitivity experiments only (tools/c3_sensitivity.sh; never set for the
  // committed goldens): GOLDEN_VIEWS_F32=1 rounds the projectors and the
  // compressed views to fp32 (the device path's storage precision);
  // GOLDEN_VIEWS_PERTURB=eps multiplies every entry by (1 + eps u), u uniform
  // in [-1, 1) from a fixed LCG (a stand-in for contraction rounding).
  if (std::getenv("GOLDEN_VIEWS_F32") || std::getenv("GOLDEN_VIEWS_PERTURB")) {
    ProjectorPair& pm = p;
    const double eps = std::getenv("GOLDEN_VIEWS_PERTURB")
                           ? std::strtod(std::getenv("GOLDEN_VIEWS_PERTURB"), nullptr)
                           : 0.0;
    std::uint64_t st = 0x9E3779B97F4A7C15ull;
    for (DenseMatrix* m : {&pm.left, &pm.right, &xhat, &xcheck})
      for (double& v : m->values) {
        if (eps != 0.0) {
          st = st * 6364136223846793005ull + 1442695040888963407ull;
          const double u = static_cast<double>(st >> 11) * 0x1.0p-53 * 2.0 - 1.0;
          v *= 1.0 + eps * u;
        }
        if (std::getenv("GOLDEN_VIEWS_F32")) v = static_cast<double>(static_cast<float>(v));
      }
    meta("views_perturbed", eps);
  }
  DenseMatrix a_hat = compress_factor_a(f.a, p);
  DenseMatrix b_check = compress_factor_b(f.b, p);
  meta("compress_seconds", secs(t));

  std::vector<double> rec_iter, rec_err, rec_elapsed, step_draws, step_secs;
  double update = 0.0;
  t = clk::now();
  rec_iter.push_back(0);
  rec_err.push_back(par_error(x, f));
  rec_elapsed.push_back(0.0);
  meta("error_seconds", secs(t));

  for (std::size_t it = 1; it <= iters; ++it) {
    Rng before = rng;
    const auto s0 = clk::now();
    fasthals_rp_step(xhat, xcheck, f, a_hat, b_check, p, cfg.normalize_a, cfg.alpha, cfg.beta,
                     rng);
    const double dt = secs(s0);
    update += dt;
    step_secs.push_back(dt);
    // Raw engine draws this step consumed (engine_ is Rng's first member).
    std::uint64_t draws = 0;
    while (std::memcmp(&before, &rng, sizeof(std::mt19937_64)) != 0) {
      before.next_u64();
      if (++draws > (std::uint64_t{1} << 34)) {
        std::fprintf(stderr, "draw count runaway\n");
        return 4;
      }
    }
    step_draws.push_back(static_cast<double>(draws));
    if (it % interval == 0 || it == iters) {
      rec_iter.push_back(static_cast<double>(it));
      rec_err.push_back(par_error(x, f));
      rec_elapsed.push_back(update);
      std::fprintf(stderr, "iter %zu err %.17g draws %llu update %.3f\n", it, rec_err.back(),
                   static_cast<unsigned long long>(draws), update);
    }
  }
  meta("update_seconds", update);
  double g = 0.0;
  try {
    g = gini(f.b);
  } catch (...) {
    g = -1.0;
  }
  meta("gini_b", g);
  put(out, "rec_iter.f64", rec_iter.data(), rec_iter.size() * 8);
  put(out, "rec_err.f64", rec_err.data(), rec_err.size() * 8);
  put(out, "rec_elapsed.f64", rec_elapsed.data(), rec_elapsed.size() * 8);
  put(out, "step_draws.f64", step_draws.data(), step_draws.size() * 8);
  put(out, "step_secs.f64", step_secs.data(), step_secs.size() * 8);
  put(out, "a.f64", f.a.values.data(), f.a.values.size() * 8);
  put(out, "b.f64", f.b.values.data(), f.b.values.size() * 8);
  meta("done", 1);
  std::fclose(log);
  return 0;
}
