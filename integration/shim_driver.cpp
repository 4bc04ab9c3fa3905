// shim_driver.cpp -- TEST DRIVER for integration/shim_cnmf_b200.cpp: calls the
// reference's public API (cnmf::run, SolverConfig::validate; reference
// headers only) as a reference user would, with the shim linked in.  Used by
// tests/test_integration_shim.py.
//
//   shim_driver config                 invalid configurations -> one line each:
//                                      "<ExceptionClass>|<what()>"
//   shim_driver run X.f32 d n k q w iters every seed
//                                      fasthals-rp run on a d x n fp32 matrix
//                                      file; prints "rec <it> <error>" lines,
//                                      "status <s> <iterations_run>", or the
//                                      exception as above
#include <cnmf/errors.hpp>
#include <cnmf/solvers.hpp>

#include <cstdio>
#include <cstdlib>
#include <exception>
#include <functional>
#include <string>
#include <vector>

using namespace cnmf;

static void report(const std::function<void()>& f) {
  try {
    f();
    std::printf("ok|\n");
  } catch (const ConfigError& e) {
    std::printf("ConfigError|%s\n", e.what());
  } catch (const DimensionError& e) {
    std::printf("DimensionError|%s\n", e.what());
  } catch (const InputError& e) {
    std::printf("InputError|%s\n", e.what());
  } catch (const std::runtime_error& e) {
    std::printf("runtime_error|%s\n", e.what());
  }
}

int main(int argc, char** argv) {
  if (argc >= 2 && std::string(argv[1]) == "config") {
    DenseMatrix x(6, 5);
    for (double& v : x.values) v = 1.0;
    SolverConfig c;
    c.algorithm = Algorithm::fasthals_rp;
    c.sketch.q = 4;
    c.k = 0;
    report([&] { run(x, c); });  // k out of range
    c.k = 4;
    report([&] { run(x, c); });  // q <= k
    c.k = 2;
    c.alpha = -1.0;
    report([&] { run(x, c); });  // negative penalty
    c.alpha = 0.0;
    c.error_interval = 0;
    report([&] { run(x, c); });
    c.error_interval = 5;
    c.rel_tolerance = 0.0;
    report([&] { run(x, c); });
    c.rel_tolerance = 1e-9;
    c.algorithm = Algorithm::mu;
    c.beta = 0.5;
    report([&] { run(x, c); });  // penalty on an unconstrained algorithm
    c.algorithm = Algorithm::fasthals_rp;
    c.beta = 0.0;
    report([&] { run(x, c); });  // valid: runs (GPU) or runtime_error (no GPU)
    return 0;
  }
  if (argc >= 11 && std::string(argv[1]) == "run") {
    const std::size_t d = std::strtoull(argv[3], nullptr, 10), n = std::strtoull(argv[4], nullptr, 10);
    std::vector<float> xf(d * n);
    FILE* f = std::fopen(argv[2], "rb");
    if (!f || std::fread(xf.data(), 4, xf.size(), f) != xf.size()) return 3;
    std::fclose(f);
    DenseMatrix x(d, n);
    for (std::size_t i = 0; i < xf.size(); ++i) x.values[i] = xf[i];
    SolverConfig c;
    c.algorithm = Algorithm::fasthals_rp;
    c.k = std::strtoull(argv[5], nullptr, 10);
    c.sketch.q = std::strtoull(argv[6], nullptr, 10);
    c.sketch.power_iterations = std::strtoull(argv[7], nullptr, 10);
    c.max_iterations = std::strtoull(argv[8], nullptr, 10);
    c.error_interval = std::strtoull(argv[9], nullptr, 10);
    c.seed = c.sketch.seed = std::strtoull(argv[10], nullptr, 10);
    c.rel_tolerance = 1e-300;
    try {
      const RunResult r = run(x, c);
      for (const RunRecord& rec : r.trace.records)
        std::printf("rec %zu %.17g\n", rec.iteration, rec.error);
      std::printf("status %d %zu\n", static_cast<int>(r.trace.status), r.trace.iterations_run);
      std::printf("a00 %.9g b00 %.9g\n", r.factors.a.values[0], r.factors.b.values[0]);
    } catch (const std::runtime_error& e) {
      std::printf("runtime_error|%s\n", e.what());
    } catch (const std::invalid_argument& e) {
      std::printf("invalid_argument|%s\n", e.what());
    }
    return 0;
  }
  std::fprintf(stderr, "usage: shim_driver config | run X.f32 d n k q w iters every seed\n");
  return 2;
}
