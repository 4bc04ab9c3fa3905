// ref_driver.cpp -- C-ABI shim over the UNMODIFIED reference library.
//
// TEST / BASELINE INFRASTRUCTURE ONLY.  oracle/Makefile compiles this file
// together with the reference's own sources, where they lie under
// /root/reference/proj/src (nothing is copied into this repo), into
// oracle/_ref/libcnmf_ref.so.  tests/ use it to pin oracle/cnmf_oracle.c bit
// for bit and to make the golden fixtures; bench.py --impl reference times
// the reference's own cnmf::run through it.
#include <chrono>
#include <cstdint>
#include <cstring>
#include <exception>
#include <string>

#include "cnmf/compression.hpp"
#include "cnmf/data_io.hpp"
#include "cnmf/errors.hpp"
#include "cnmf/metrics.hpp"
#include "cnmf/qr.hpp"
#include "cnmf/rng.hpp"
#include "cnmf/solvers.hpp"

using namespace cnmf;

namespace {

std::string g_msg;

DenseMatrix wrap(const double* v, std::size_t r, std::size_t c) {
  DenseMatrix m(r, c);
  std::memcpy(m.values.data(), v, sizeof(double) * r * c);
  return m;
}

void unwrap(const DenseMatrix& m, double* out) {
  std::memcpy(out, m.values.data(), sizeof(double) * m.values.size());
}

template <typename F>
int guarded(F&& f) {
  try {
    f();
    return 0;
  } catch (const ConfigError& e) {
    g_msg = e.what();
    return 1;
  } catch (const DimensionError& e) {
    g_msg = e.what();
    return 2;
  } catch (const InputError& e) {
    g_msg = e.what();
    return 3;
  } catch (const std::exception& e) {
    g_msg = e.what();
    return 9;
  }
}

}  // namespace

extern "C" {

const char* ref_last_message() { return g_msg.c_str(); }

// Rng draws: kind 0 next_u64 (as double bits), 1 uniform, 2 uniform_positive, 3 normal.
void ref_rng_draws(std::uint64_t seed, int kind, std::size_t count, double* out) {
  Rng rng(seed);
  for (std::size_t i = 0; i < count; ++i) {
    switch (kind) {
      case 0: {
        const std::uint64_t v = rng.next_u64();
        std::memcpy(out + i, &v, 8);
        break;
      }
      case 1: out[i] = rng.uniform(); break;
      case 2: out[i] = rng.uniform_positive(); break;
      default: out[i] = rng.normal(); break;
    }
  }
}

void ref_gaussian_sketch(std::size_t rows, std::size_t cols, std::uint64_t seed, double* out) {
  unwrap(gaussian_sketch(rows, cols, seed), out);
}

void ref_initialize(std::size_t d, std::size_t n, std::size_t k, std::uint64_t seed, double* a,
                    double* b) {
  const FactorPair f = initialize(d, n, k, seed);
  unwrap(f.a, a);
  unwrap(f.b, b);
}

int ref_matmul(const double* m, std::size_t mr, std::size_t mc, const double* n, std::size_t nr,
               std::size_t nc, int tl, int tr, double* c) {
  return guarded([&] { unwrap(matmul(wrap(m, mr, mc), wrap(n, nr, nc), tl, tr), c); });
}

int ref_thin_qr(const double* m, std::size_t rows, std::size_t cols, double* q, double* r) {
  return guarded([&] {
    const QrResult res = thin_qr(wrap(m, rows, cols));
    unwrap(res.q, q);
    if (r) unwrap(res.r, r);
  });
}

int ref_powered_range_finder(const double* x, std::size_t d, std::size_t n, std::size_t q,
                             std::size_t w, std::uint64_t seed, double* basis) {
  return guarded([&] {
    SketchConfig sk;
    sk.q = q;
    sk.power_iterations = w;
    sk.seed = seed;
    unwrap(powered_range_finder(wrap(x, d, n), sk), basis);
  });
}

int ref_build_projectors(const double* x, std::size_t d, std::size_t n, std::size_t q,
                         std::size_t w, std::uint64_t seed, double* left, double* right) {
  return guarded([&] {
    SketchConfig sk;
    sk.q = q;
    sk.power_iterations = w;
    sk.seed = seed;
    const ProjectorPair p = build_projectors(wrap(x, d, n), sk);
    unwrap(p.left, left);
    unwrap(p.right, right);
  });
}

// Times build_projectors + compress_left + compress_right on the given X
// (the reference's compression half; it is untimed inside cnmf::run).
int ref_compress(const double* x, std::size_t d, std::size_t n, std::size_t q, std::size_t w,
                 std::uint64_t seed, double* left, double* right, double* xhat, double* xcheck,
                 double* seconds) {
  return guarded([&] {
    const DenseMatrix xm = wrap(x, d, n);
    SketchConfig sk;
    sk.q = q;
    sk.power_iterations = w;
    sk.seed = seed;
    const auto t0 = std::chrono::steady_clock::now();
    const ProjectorPair p = build_projectors(xm, sk);
    const DenseMatrix xh = compress_left(xm, p);
    const DenseMatrix xc = compress_right(xm, p);
    *seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    if (left) unwrap(p.left, left);
    if (right) unwrap(p.right, right);
    if (xhat) unwrap(xh, xhat);
    if (xcheck) unwrap(xc, xcheck);
  });
}

// `steps` FastHALS-RP sweeps from the given state with Rng(rng_seed); state
// arrays are updated in place.
int ref_fasthals_rp_steps(const double* xhat, const double* xcheck, const double* left,
                          const double* right, std::size_t d, std::size_t n, std::size_t q,
                          std::size_t k, double* a, double* b, double* a_hat, double* b_check,
                          int normalize_a, double alpha, double beta, std::uint64_t rng_seed,
                          std::size_t steps, double* seconds) {
  return guarded([&] {
    const DenseMatrix xh = wrap(xhat, q, n), xc = wrap(xcheck, d, q);
    ProjectorPair p{wrap(left, d, q), wrap(right, q, n)};
    FactorPair f{wrap(a, d, k), wrap(b, n, k)};
    DenseMatrix ah = wrap(a_hat, q, k), bc = wrap(b_check, q, k);
    Rng rng(rng_seed);
    const auto t0 = std::chrono::steady_clock::now();
    for (std::size_t s = 0; s < steps; ++s)
      fasthals_rp_step(xh, xc, f, ah, bc, p, normalize_a != 0, alpha, beta, rng);
    if (seconds)
      *seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    unwrap(f.a, a);
    unwrap(f.b, b);
    unwrap(ah, a_hat);
    unwrap(bc, b_check);
  });
}

int ref_fasthals_steps(const double* x, std::size_t d, std::size_t n, std::size_t k, double* a,
                       double* b, int normalize_a, std::uint64_t rng_seed, std::size_t steps) {
  return guarded([&] {
    const DenseMatrix xm = wrap(x, d, n);
    FactorPair f{wrap(a, d, k), wrap(b, n, k)};
    Rng rng(rng_seed);
    for (std::size_t s = 0; s < steps; ++s) fasthals_step(xm, f, normalize_a != 0, rng);
    unwrap(f.a, a);
    unwrap(f.b, b);
  });
}

double ref_reconstruction_error(const double* x, std::size_t d, std::size_t n, const double* a,
                                const double* b, std::size_t k) {
  FactorPair f{wrap(a, d, k), wrap(b, n, k)};
  return reconstruction_error(wrap(x, d, n), f);
}

namespace {
SparseMatrix g_csr;  // the CSR input of the next ref_run with x == nullptr
}

// run(SparseMatrix) input: stored here, consumed by ref_run(x = nullptr, ...).
int ref_set_csr(std::size_t d, std::size_t n, const std::size_t* row_offsets,
                const std::size_t* col_indices, const double* values) {
  return guarded([&] {
    g_csr = SparseMatrix{};
    g_csr.rows = d;
    g_csr.cols = n;
    g_csr.row_offsets.assign(row_offsets, row_offsets + d + 1);
    g_csr.col_indices.assign(col_indices, col_indices + row_offsets[d]);
    g_csr.values.assign(values, values + row_offsets[d]);
    g_csr.validate();
  });
}

int ref_run(const double* x, std::size_t d, std::size_t n, int algorithm, std::size_t k,
            std::size_t q, std::size_t w, std::uint64_t sketch_seed, double alpha, double beta,
            std::size_t max_iterations, double rel_tolerance, std::size_t error_interval,
            std::uint64_t seed, int normalize_a, double* a_out, double* b_out,
            std::size_t* rec_iter, double* rec_err, double* rec_elapsed, std::size_t rec_cap,
            std::size_t* rec_count, double* update_seconds, double* gini_b, int* status,
            std::size_t* iterations_run, char* message, std::size_t message_cap) {
  return guarded([&] {
    SolverConfig cfg;
    cfg.algorithm = static_cast<Algorithm>(algorithm);
    cfg.k = k;
    cfg.sketch.q = q;
    cfg.sketch.power_iterations = w;
    cfg.sketch.seed = sketch_seed;
    cfg.alpha = alpha;
    cfg.beta = beta;
    cfg.max_iterations = max_iterations;
    cfg.rel_tolerance = rel_tolerance;
    cfg.error_interval = error_interval;
    cfg.seed = seed;
    cfg.normalize_a = normalize_a != 0;
    const RunResult r = x ? run(wrap(x, d, n), cfg) : run(g_csr, cfg);
    unwrap(r.factors.a, a_out);
    unwrap(r.factors.b, b_out);
    *rec_count = r.trace.records.size();
    for (std::size_t i = 0; i < r.trace.records.size() && i < rec_cap; ++i) {
      rec_iter[i] = r.trace.records[i].iteration;
      rec_err[i] = r.trace.records[i].error;
      rec_elapsed[i] = r.trace.records[i].elapsed_seconds;
    }
    *update_seconds = r.trace.update_seconds;
    *gini_b = r.trace.gini_b;
    *status = static_cast<int>(r.trace.status);
    *iterations_run = r.trace.iterations_run;
    std::snprintf(message, message_cap, "%s", r.trace.message.c_str());
  });
}

// generate_synthetic (data_io.cpp:383-415): d x n, row-major.
int ref_generate_synthetic(std::size_t d, std::size_t n, std::size_t rank, double decay,
                           double noise, std::uint64_t seed, double* out) {
  return guarded([&] {
    SyntheticSpec spec;
    spec.d = d;
    spec.n = n;
    spec.true_rank = rank;
    spec.decay_p = decay;
    spec.noise_level = noise;
    spec.seed = seed;
    unwrap(generate_synthetic(spec), out);
  });
}

// pairwise_distortion (metrics.cpp:123-155): left is d x q row-major.
int ref_pairwise_distortion(const double* x, std::size_t d, std::size_t n, const double* left,
                            std::size_t q, std::size_t pairs, std::uint64_t seed,
                            double* max_relative, double* mean_relative) {
  return guarded([&] {
    const DistortionStats s = pairwise_distortion(wrap(x, d, n), wrap(left, d, q), pairs, seed);
    *max_relative = s.max_relative;
    *mean_relative = s.mean_relative;
  });
}

}  // extern "C"
