/*
 * cnmf_b200.h -- C ABI of the B200-native compressed-NMF hot path.
 *
 * Drop-in boundary for the reference's solver API (/root/reference/proj):
 *   RunResult cnmf::run(const DenseMatrix&, const SolverConfig&)   solvers.hpp:104
 * plus the step-level entry points the reference exposes for the same path
 * (compression.hpp:28-51, solvers.hpp:33-71, metrics.hpp:35).  Every
 * function takes plain pointers and sizes; matrices are row-major fp32
 * (A is d x k, B is n x k = H^T, as FactorPair, matrix.hpp:57-62) unless a
 * comment says otherwise.  The library computes on the device in fp32 with
 * fp64 reductions and never falls back to a CPU path: without a usable CUDA
 * device every compute entry returns CNMF_ERR_CUDA.
 *
 * Errors mirror the reference's exception classes (errors.hpp:10-28):
 * CNMF_ERR_CONFIG <-> ConfigError, CNMF_ERR_DIMENSION <-> DimensionError,
 * CNMF_ERR_INPUT <-> InputError; the message is available from
 * cnmf_context_last_error().  A non-finite objective is not an error but
 * trace->status == CNMF_ABORTED, as in run_impl (solvers.cpp:223-229,265-269).
 *
 * Threading: a context owns one CUDA stream and serializes its calls; use
 * one context per concurrent caller (the reference's run() is reentrant,
 * solvers.hpp:100-105, cli.cpp:231-247).
 *
 * Streams: the context's stream does not synchronise with other streams.
 * Entry points taking device pointers read their inputs when called: the
 * caller completes the work producing them first (the Python binding
 * synchronises torch's current stream before every call).  Every entry point
 * returns with its own work complete.
 */
#ifndef CNMF_B200_H_
#define CNMF_B200_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define CNMF_B200_ABI_VERSION 3

typedef enum cnmf_status {
  CNMF_OK = 0,
  CNMF_ERR_CONFIG = 1,      /* cnmf::ConfigError     */
  CNMF_ERR_DIMENSION = 2,   /* cnmf::DimensionError  */
  CNMF_ERR_INPUT = 3,       /* cnmf::InputError      */
  CNMF_ERR_CUDA = 4,        /* device / driver failure, or no device */
  CNMF_ERR_NCCL = 5,        /* collective failure (sharded runs)     */
  CNMF_ERR_UNSUPPORTED = 6  /* valid for the reference, not built here: k or q above 128
                               (rows of A past 1536 per SM in the streaming HALS kernel) */
} cnmf_status;

/* cnmf::Algorithm, algorithm.hpp:8-15 (same order). */
typedef enum cnmf_algorithm {
  CNMF_MU = 0,
  CNMF_MU_RP = 1,
  CNMF_HALS = 2,
  CNMF_HALS_RP = 3,
  CNMF_FASTHALS = 4,
  CNMF_FASTHALS_RP = 5
} cnmf_algorithm;

/* cnmf::RunStatus, metrics.hpp:62-66. */
typedef enum cnmf_run_status {
  CNMF_CONVERGED = 0,
  CNMF_REACHED_MAX_ITERATIONS = 1,
  CNMF_ABORTED = 2
} cnmf_run_status;

/* cnmf::SolverConfig (solvers.hpp:13-29) with its SketchConfig
 * (compression.hpp:13-17) flattened.  cnmf_solver_config_init() sets the
 * reference defaults. */
typedef struct cnmf_solver_config {
  int32_t algorithm;             /* cnmf_algorithm; this build runs CNMF_FASTHALS_RP */
  uint64_t k;
  uint64_t sketch_q;             /* SketchConfig::q (l = k + oversampling)      */
  uint64_t sketch_power_iterations; /* SketchConfig::power_iterations (w)      */
  uint64_t sketch_seed;          /* SketchConfig::seed                          */
  double alpha;                  /* L1 penalty on b_j                           */
  double beta;                   /* L2 penalty on b_j                           */
  uint64_t max_iterations;
  double rel_tolerance;
  uint64_t error_interval;
  uint64_t seed;                 /* init + redraw stream                        */
  int32_t normalize_a;
} cnmf_solver_config;

/* cnmf::RunRecord, metrics.hpp:56-60, plus the run Rng's position. */
typedef struct cnmf_run_record {
  uint64_t iteration;
  double error;            /* 1/2 ||X - A B^T||_F^2 */
  double elapsed_seconds;  /* cumulative update time at this record */
  uint64_t rng_draws;      /* raw mt19937_64 draws the dead-component redraws
                              (reinit_column, solvers.cpp:28-31) took from the
                              run Rng up to this record (initialize()'s excluded) */
} cnmf_run_record;

/* cnmf::RunTrace (metrics.hpp:70-84) plus device timing.  `records` is
 * caller-owned storage for up to records_capacity entries; records_count is
 * the number the run produced (may exceed the capacity). */
typedef struct cnmf_run_trace {
  cnmf_run_record* records;
  uint64_t records_capacity;
  uint64_t records_count;
  double update_seconds;      /* device time of the update steps (CUDA events around each
                                 iteration range, redraw servicing included) */
  double compress_seconds;    /* device time of build_projectors + compress_* (RNG included) */
  double error_seconds;       /* device time of objective evaluations */
  double gini_b;
  int32_t status;             /* cnmf_run_status */
  uint64_t iterations_run;
  uint64_t power_iterations;
  double alpha;
  double beta;
  uint64_t seed;
  double estimate_flops_per_iteration; /* estimate_cost, metrics.cpp:20-50 */
  double estimate_memory_floats;
  double x_norm_sq;           /* ||X||_F^2 (for relative errors)   */
  uint64_t redraws;           /* dead-component redraws (served on the device from the
                                 run Rng's stream) */
  uint64_t x_passes;          /* X-streaming contractions performed */
  char message[256];
  double sketch_kappa;        /* condition estimate of X Omega that chose the range finder's
                                 arithmetic (0: not estimated) */
  int32_t range_finder_fp64;  /* 1: the range finder ran in fp64 (engine.cpp rf_mode) */
} cnmf_run_trace;

typedef struct cnmf_context cnmf_context;

int cnmf_abi_version(void);
/* Creates a context bound to CUDA device `device` (one stream). */
cnmf_status cnmf_context_create(int device, cnmf_context** out);
void cnmf_context_destroy(cnmf_context* ctx);
const char* cnmf_context_last_error(const cnmf_context* ctx);
/* Synchronizes the context's stream; returns its CUDA stream handle. */
void* cnmf_context_stream(cnmf_context* ctx);

/* SolverConfig{} defaults (solvers.hpp:13-23, compression.hpp:13-17). */
void cnmf_solver_config_init(cnmf_solver_config* cfg);
/* SolverConfig::validate (solvers.cpp:298-312); message optional. */
cnmf_status cnmf_solver_config_validate(const cnmf_solver_config* cfg, uint64_t d, uint64_t n,
                                        char* message, size_t message_capacity);

/* cnmf::run(x, config) (solvers.cpp:189-294, 511-513) with X in HOST memory
 * (d x n, leading dimension ldx >= n); a_out d x k and b_out n x k in host
 * memory.  Copies X to the device, runs everything there, copies A and B
 * back. */
cnmf_status cnmf_run(cnmf_context* ctx, const float* x, uint64_t d, uint64_t n, uint64_t ldx,
                     const cnmf_solver_config* cfg, float* a_out, float* b_out,
                     cnmf_run_trace* trace);
/* Same with X, A and B already in device memory (X resident in HBM). */
cnmf_status cnmf_run_device(cnmf_context* ctx, const float* x_dev, uint64_t d, uint64_t n,
                            uint64_t ldx, const cnmf_solver_config* cfg, float* a_dev,
                            float* b_dev, cnmf_run_trace* trace);

/* ---- column-sharded multi-GPU run (one process per GPU, NCCL) ---------
 * cnmf::run (solvers.hpp:104) with X column-sharded over `world` ranks:
 * rank g holds columns [cnmf_shard_begin(n, g, world), cnmf_shard_begin(n,
 * g + 1, world)).  Rank 0 calls cnmf_nccl_unique_id, the caller broadcasts
 * the 128 bytes (e.g. over torch.distributed), every rank then creates its
 * context.  All ranks must call cnmf_run_sharded_device collectively with
 * the same d, n and config; each gets the full A (d x k) and its own rows of
 * B (n_local x k).  Collectives: NCCL sum all-reduces of d x l sketch
 * partials and l x l Gram partials in the compression, one (l + 1) x k
 * all-reduce per HALS iteration (B-check partial + zero-column flags), an
 * all-gather of B for the final Gini. */
uint64_t cnmf_shard_begin(uint64_t n, int rank, int world);
cnmf_status cnmf_nccl_unique_id(unsigned char id[128]);
cnmf_status cnmf_context_create_sharded(int device, int rank, int world,
                                        const unsigned char id[128], cnmf_context** out);
/* Host-staged collectives: a sharded context whose cross-rank combines go
 * through the caller instead of NCCL (device buffer -> host, callback, host
 * -> device; synchronous).  A test / debugging transport: it lets world-size
 * > 1 runs share one GPU (NCCL refuses two ranks on one device), e.g. with
 * torch.distributed gloo behind the callbacks.  Callbacks return 0 on
 * success.  dtype: 0 fp32, 1 fp64; op: 0 sum, 1 max. */
typedef struct cnmf_host_collectives {
  int (*allreduce)(void* buf, uint64_t count, int dtype, int op, void* user);
  /* `bytes` from every rank, concatenated in rank order into recv */
  int (*allgather)(const void* send, void* recv, uint64_t bytes, void* user);
  void* user;
} cnmf_host_collectives;
cnmf_status cnmf_context_create_hosted(int device, int rank, int world,
                                       const cnmf_host_collectives* coll, cnmf_context** out);
cnmf_status cnmf_run_sharded_device(cnmf_context* ctx, const float* x_shard_dev, uint64_t d,
                                    uint64_t n, uint64_t col_begin, uint64_t n_local,
                                    uint64_t ldx, const cnmf_solver_config* cfg, float* a_dev,
                                    float* b_local_dev, cnmf_run_trace* trace);

/* ---- step-level entry points (all pointers are DEVICE pointers) ------- */

/* gaussian_sketch(rows, cols, seed), compression.cpp:11-16; fp32 rounding
 * of the reference's fp64 normals, row-major rows x cols. */
cnmf_status cnmf_gaussian_sketch(cnmf_context* ctx, uint64_t rows, uint64_t cols, uint64_t seed,
                                 float* out);
/* initialize(d, n, k, seed), solvers.cpp:314-325. */
cnmf_status cnmf_initialize(cnmf_context* ctx, uint64_t d, uint64_t n, uint64_t k, uint64_t seed,
                            float* a, float* b);
/* powered_range_finder (compression.cpp:23-42, 57-63): basis of X (transpose
 * = 0, d x q) or of X^T (transpose = 1, n x q, the row basis R^T). */
cnmf_status cnmf_powered_range_finder(cnmf_context* ctx, const float* x, uint64_t d, uint64_t n,
                                      uint64_t ldx, uint64_t q, uint64_t power_iterations,
                                      uint64_t seed, int transpose, float* basis);
/* build_projectors (compression.cpp:44-53): left d x q, right q x n.
 * Bases handed out by cnmf_powered_range_finder, cnmf_build_projectors and
 * cnmf_thin_qr carry the reference's Householder column signs (qr.cpp:35);
 * cnmf_run skips that pass (FastHALS-RP uses L, R only through
 * sign-invariant products). */
cnmf_status cnmf_build_projectors(cnmf_context* ctx, const float* x, uint64_t d, uint64_t n,
                                  uint64_t ldx, uint64_t q, uint64_t power_iterations,
                                  uint64_t seed, float* left, float* right);
/* compress_left / compress_right (compression.cpp:73-84): xhat q x n, xcheck d x q. */
cnmf_status cnmf_compress(cnmf_context* ctx, const float* x, uint64_t d, uint64_t n,
                          uint64_t ldx, const float* left, const float* right, uint64_t q,
                          float* xhat, float* xcheck);
/* compress_factor_a / compress_factor_b (compression.cpp:90-96): fp64 q x k. */
cnmf_status cnmf_compress_factors(cnmf_context* ctx, const float* a, const float* b,
                                  const float* left, const float* right, uint64_t d, uint64_t n,
                                  uint64_t q, uint64_t k, double* a_hat, double* b_check);
/* `steps` calls of fasthals_rp_step (solvers.cpp:414-456) with a fresh
 * Rng(rng_seed) for the redraw path; a, b, a_hat, b_check updated in place. */
cnmf_status cnmf_fasthals_rp_steps(cnmf_context* ctx, const float* xhat, const float* xcheck,
                                   const float* left, const float* right, uint64_t d,
                                   uint64_t n, uint64_t q, uint64_t k, float* a, float* b,
                                   double* a_hat, double* b_check, int normalize_a, double alpha,
                                   double beta, uint64_t rng_seed, uint64_t steps,
                                   uint64_t* redraws);
/* reconstruction_error (metrics.cpp:61-77) -> *out (host pointer). */
cnmf_status cnmf_reconstruction_error(cnmf_context* ctx, const float* x, uint64_t d, uint64_t n,
                                      uint64_t ldx, const float* a, const float* b, uint64_t k,
                                      double* out);
/* thin_qr (qr.cpp:10-75) up to basis: q_out spans y (rows x l), orthonormal. */
cnmf_status cnmf_thin_qr(cnmf_context* ctx, const float* y, uint64_t rows, uint64_t l,
                         float* q_out);
/* The raw X-stream contractions (matrix.cpp:105-116 NN, 129-140 TN):
 * y = X s (s: n x l, y: d x l) and z = X^T t (t: d x l, z: n x l). */
cnmf_status cnmf_xs_nn(cnmf_context* ctx, const float* x, uint64_t d, uint64_t n, uint64_t ldx,
                       const float* s, uint64_t l, float* y);
cnmf_status cnmf_xs_tn(cnmf_context* ctx, const float* x, uint64_t d, uint64_t n, uint64_t ldx,
                       const float* t, uint64_t l, float* z);
/* The range finder's fp64-grade contractions (matrix.cpp:105-140 with fp32 X,
 * fp64 accumulation): out (fp64, d x l for NN, n x l for TN) = X s or X^T s,
 * s fp32 (widened exactly), l a multiple of 16.  use_dmma = 0: the exact
 * int8-sliced tensor-core kernel; 1: the FP64 tensor-core kernel; 2: the
 * int8-sliced kernel's configuration for an X of integers below 8192 (the
 * caller vouches for that: exact X digits, 40 bits of s). */
cnmf_status cnmf_xs_exact(cnmf_context* ctx, const float* x, uint64_t d, uint64_t n, uint64_t ldx,
                          const float* s, uint64_t l, int transpose, int use_dmma, double* out);
/* Seconds per exact-accumulation contraction (cnmf_xs_exact's int8-sliced
 * kernel on a seeded Gaussian operand, S slicing and every column chunk
 * included; the per-X preprocessing once, outside), and the reads of X it makes. */
cnmf_status cnmf_time_xs_exact(cnmf_context* ctx, const float* x, uint64_t d, uint64_t n,
                               uint64_t ldx, uint64_t l, int transpose, int iters,
                               double* seconds_per_launch, int* x_passes);

/* Instrumentation (bench harness). */
/* Total device kernels this library has launched in this process. */
uint64_t cnmf_launch_count(void);
/* Average device time of ONE X-stream contraction launch (NN: transpose = 0,
 * TN: transpose = 1) over `iters` back-to-back launches on the context
 * stream, bracketed by CUDA events (the kernel of the compression half). */
cnmf_status cnmf_time_xstream(cnmf_context* ctx, const float* x, uint64_t d, uint64_t n,
                              uint64_t ldx, uint64_t l, int transpose, int iters,
                              double* seconds_per_launch);

/* Synthetic X for the BASELINE.json configs (bench harness, not the solver
 * path): columns [col_lo, col_hi) of the global d x n matrix into x (ld ldx).
 * factor_kind 0 Uniform, 1 Exponential, 2 Gamma(0.3); noise_kind 0 none,
 * 1 sigma|N(0,1)|, 2 Poisson(W0 H0). */
cnmf_status cnmf_synth_x(cnmf_context* ctx, uint64_t d, uint64_t n, uint64_t rank,
                         int factor_kind, int noise_kind, double sigma, uint64_t seed,
                         uint64_t col_lo, uint64_t col_hi, uint64_t ldx, float* x);

/* run(const SparseMatrix&, const SolverConfig&) (solvers.hpp:105,
 * solvers.cpp:515-517): X given in CSR on the host (SparseMatrix layout,
 * matrix.hpp:34-44 -- d + 1 row offsets, column indices strictly increasing
 * within a row, fp32 values).  Every algorithm of cnmf_run; the X
 * contractions, check_data and the objective (metrics.cpp:79-102) run on the
 * stored entries only.  Structure errors raise CNMF_ERR_DIMENSION with the
 * messages of SparseMatrix::validate (matrix.cpp:37-56). */
cnmf_status cnmf_run_csr(cnmf_context* ctx, const uint64_t* row_offsets,
                         const uint64_t* col_indices, const float* values, uint64_t d, uint64_t n,
                         const cnmf_solver_config* cfg, float* a_out, float* b_out,
                         cnmf_run_trace* trace);

/* ---- host-side data formats around the path (no device, no context) ----
 * The front end's inputs and reports; fp64 host code,
 * bitwise the reference's results.  `msg` (may be NULL) receives the error
 * text of a failing call. */

/* cnmf::CostEstimate, metrics.hpp:20-28. */
typedef struct cnmf_cost_estimate {
  int32_t algorithm;
  uint64_t d, n, k, q;
  double flops_per_iteration;
  double memory_floats;
} cnmf_cost_estimate;

/* estimate_cost(algorithm, d, n, k, q), metrics.cpp:20-50. */
cnmf_status cnmf_estimate_cost(int algorithm, uint64_t d, uint64_t n, uint64_t k, uint64_t q,
                               cnmf_cost_estimate* out, char* msg, size_t msg_cap);
/* generate_synthetic(SyntheticSpec), data_io.cpp:383-415: d x n row-major
 * fp64 into out (caller-owned, d * n doubles). */
cnmf_status cnmf_generate_synthetic(uint64_t d, uint64_t n, uint64_t true_rank, double decay_p,
                                    double noise_level, uint64_t seed, double* out, char* msg,
                                    size_t msg_cap);
/* pairwise_distortion(x, left, sample_pairs, seed), metrics.cpp:123-155,
 * with the projected columns L^T X given as xhat (q x n fp32, the output of
 * cnmf_compress): host x is d x n row-major fp64. */
cnmf_status cnmf_pairwise_distortion(const double* x, uint64_t d, uint64_t n, const float* xhat,
                                     uint64_t q, uint64_t sample_pairs, uint64_t seed,
                                     double* max_relative, double* mean_relative, char* msg,
                                     size_t msg_cap);

#ifdef __cplusplus
}
#endif

#endif /* CNMF_B200_H_ */
