// shim_cnmf_b200.cpp -- the reference-side binding: cnmf::run on a B200
// through the C ABI of libcnmf_b200.so (include/cnmf_b200.h).
//
// A maintainer of the reference library adds this file to its build in place
// of the dense `run` and `SolverConfig::validate` definitions in
// proj/src/solvers.cpp (solvers.cpp:298-312, 511-513; declared in
// proj/include/cnmf/solvers.hpp:28, 104) and links -lcnmf_b200.  Signatures,
// exception classes (proj/include/cnmf/errors.hpp:10-28) and the RunResult
// contents (solvers.hpp:94-97, metrics.hpp:54-84) are the reference's.
//
// tests/test_integration_shim.py compiles this file against the reference's
// own headers (/root/reference/proj/include) and links it with the built
// library: without a GPU a valid run throws std::runtime_error and an invalid
// configuration throws ConfigError with the reference's message; on a B200
// the run matches the reference's trajectory.
#include <cnmf/errors.hpp>
#include <cnmf/solvers.hpp>

#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "cnmf_b200.h"

namespace cnmf {
namespace {

struct Ctx {
  cnmf_context* c = nullptr;
  Ctx() {
    if (cnmf_context_create(0, &c) != CNMF_OK) {
      const std::string why = c ? cnmf_context_last_error(c) : "no context";
      cnmf_context_destroy(c);
      throw std::runtime_error("cnmf_b200: no usable CUDA device (" + why + ")");
    }
  }
  ~Ctx() { cnmf_context_destroy(c); }
  Ctx(const Ctx&) = delete;
  Ctx& operator=(const Ctx&) = delete;
};

// run() is reentrant in the reference (cli.cpp:229-247 runs it from a thread
// pool); one context per calling thread keeps that (a context serialises its
// own calls on its stream).
cnmf_context* context() {
  thread_local std::unique_ptr<Ctx> ctx;
  if (!ctx) ctx = std::make_unique<Ctx>();
  return ctx->c;
}

[[noreturn]] void rethrow(cnmf_status s, const std::string& msg) {
  switch (s) {
    case CNMF_ERR_CONFIG: throw ConfigError(msg);
    case CNMF_ERR_DIMENSION: throw DimensionError(msg);
    case CNMF_ERR_INPUT: throw InputError(msg);
    default: throw std::runtime_error("cnmf_b200: " + msg);  // CUDA / NCCL / UNSUPPORTED
  }
}

cnmf_solver_config to_c(const SolverConfig& s) {
  cnmf_solver_config c;
  cnmf_solver_config_init(&c);
  c.algorithm = static_cast<int32_t>(s.algorithm);  // enum order of solvers.hpp:8-11
  c.k = s.k;
  c.sketch_q = s.sketch.q;
  c.sketch_power_iterations = s.sketch.power_iterations;
  c.sketch_seed = s.sketch.seed;
  c.alpha = s.alpha;
  c.beta = s.beta;
  c.max_iterations = s.max_iterations;
  c.rel_tolerance = s.rel_tolerance;
  c.error_interval = s.error_interval;
  c.seed = s.seed;
  c.normalize_a = s.normalize_a ? 1 : 0;
  return c;
}

}  // namespace

// solvers.cpp:298-312: the same checks and messages, evaluated by the
// library (no device needed).
void SolverConfig::validate(std::size_t d, std::size_t n) const {
  const cnmf_solver_config c = to_c(*this);
  char msg[256] = {0};
  const cnmf_status s = cnmf_solver_config_validate(&c, d, n, msg, sizeof msg);
  if (s != CNMF_OK) rethrow(s, msg);
}

// solvers.cpp:189-294 via 511-513.
RunResult run(const DenseMatrix& x, const SolverConfig& config) {
  config.validate(x.rows, x.cols);  // run_impl validates before touching the device
  cnmf_context* c = context();
  const cnmf_solver_config cfg = to_c(config);
  // The path computes on fp32 X (exact for data that was fp32 to begin with).
  std::vector<float> xf(x.values.begin(), x.values.end());
  std::vector<float> af(x.rows * config.k), bf(x.cols * config.k);
  std::vector<cnmf_run_record> recs(config.max_iterations / config.error_interval + 2);
  cnmf_run_trace tr{};
  tr.records = recs.data();
  tr.records_capacity = recs.size();
  const cnmf_status s =
      cnmf_run(c, xf.data(), x.rows, x.cols, x.cols, &cfg, af.data(), bf.data(), &tr);
  if (s != CNMF_OK) rethrow(s, cnmf_context_last_error(c));

  RunResult r;
  r.factors.a = DenseMatrix(x.rows, config.k);
  r.factors.b = DenseMatrix(x.cols, config.k);
  std::copy(af.begin(), af.end(), r.factors.a.values.begin());  // row-major, like DenseMatrix
  std::copy(bf.begin(), bf.end(), r.factors.b.values.begin());
  RunTrace& t = r.trace;
  for (uint64_t i = 0; i < tr.records_count && i < tr.records_capacity; ++i)
    t.records.push_back({recs[i].iteration, recs[i].error, recs[i].elapsed_seconds});
  t.update_seconds = tr.update_seconds;  // (tr.compress_seconds has no RunTrace field)
  t.estimate = CostEstimate{config.algorithm, x.rows, x.cols, config.k, config.sketch.q,
                            tr.estimate_flops_per_iteration, tr.estimate_memory_floats};
  t.iterations_run = tr.iterations_run;
  t.status = static_cast<RunStatus>(tr.status);  // converged / reached_max_iterations / aborted
  t.message = tr.message;
  t.gini_b = tr.gini_b;
  t.power_iterations = tr.power_iterations;
  t.alpha = tr.alpha;
  t.beta = tr.beta;
  t.seed = tr.seed;
  return r;
}

}  // namespace cnmf
