// kernels.h -- host-side launchers for the cnmf-b200 device kernels.
// Internal to the library (the public C ABI is include/cnmf_b200.h).
#pragma once

#include <cuda_runtime.h>

#include <functional>
#include <vector>
#ifndef __CUDACC__
#ifndef __host__
#define __host__
#define __device__
#endif
#endif
#include <stdint.h>

#include <algorithm>

namespace cnmf {

// Widths of every "l-wide" operand (sketches, bases, compressed views) are
// padded to a multiple of 16 columns; padding columns hold zeros.
__host__ __device__ inline int pad16(int l) { return (l + 15) & ~15; }

// Number of device kernels launched by this library (all launchers count).
void note_launches(int n);
uint64_t launch_count();

// ---- rng.cu -------------------------------------------------------------
struct MtJob {
  uint64_t seed;
  uint64_t nwords;
  uint64_t* out;
};
struct MtJobs {
  MtJob job[4];
};
void launch_mt_streams(const MtJobs& jobs, int njobs, cudaStream_t s);
// Jump-ahead generation (rng.cu + mt_jump.cpp): the same stream as one engine,
// in K parallel segments of J outputs.
bool mt_jump_available();
bool mt_jump_polys(uint64_t J, int K, std::vector<uint64_t>& out);
void launch_mt_jump(uint64_t seed, uint64_t nwords, uint64_t J, int K, const uint64_t* polys,
                    uint64_t* ws, uint64_t* out, cudaStream_t s);
size_t mt_jump_ws_words(int K);
void launch_normal_map(const uint64_t* words, uint64_t count, int cols, int ld, float* out,
                       int* flag, int nsm, cudaStream_t s);
void launch_normal_exact(const uint64_t* words, uint64_t nwords, uint64_t count, int cols, int ld,
                         float* out, int* flag, cudaStream_t s);
void launch_uniform_init(const uint64_t* words, uint64_t d, uint64_t n, int k, double* a_cm,
                         double* b_cm, int* flag, int nsm, cudaStream_t s);
void launch_uniform_init_exact(const uint64_t* words, uint64_t nwords, uint64_t d, uint64_t n,
                               int k, double* a_cm, double* b_cm, int* flag, uint64_t* consumed,
                               cudaStream_t s);
// reinit_column (solvers.cpp:28-31) served on the device: rows_total draws
// uniform_positive() * 1e-3 from words[*pos ...] (the run stream), entries
// [off, off + count) into col; advances *pos past the draws (rejections of
// exact zeros included).  flag: scratch, 0 on entry; 2 after = out of words.
void launch_redraw_fill(const uint64_t* words, uint64_t nwords, uint64_t* pos, uint64_t rows_total,
                        uint64_t off, uint64_t count, double* col, int* flag, int nsm,
                        cudaStream_t s);

// ---- xstream.cu: the X-streaming contractions ----------------------------
// Y (m x lp, ld lp) = X (m x n, ld ldx) * S (n x lp, ld lp)          ["NN"]
// Z (n x lp, ld lp) = X^T * T (m x lp, ld lp)                         ["TN"]
// lp is a multiple of 16 in [16, 128].  `ws` is scratch for split-K partials
// (xstream_ws_floats() floats).  Deterministic: fixed-order split reduction.
size_t xstream_ws_floats(int64_t m, int64_t n, int lp, int nsm);
// rexp (optional, from launch_x_rowexp over this X): per-row exponents that
// select the tensor-core kernel's fp16 hi/lo path.
// x_exact: every element of X is exactly a tf32 value (launch_x_tf32_exact /
// check_data): the tensor-core kernel's two-product mode (kX1), bitwise the
// same result.
void launch_xs_nn(const float* x, int64_t ldx, int64_t m, int64_t n, const float* s, int lp,
                  float* y, float* ws, int nsm, cudaStream_t st, const int8_t* rexp = nullptr,
                  bool x_exact = false);
void launch_xs_tn(const float* x, int64_t ldx, int64_t m, int64_t n, const float* t, int lp,
                  float* z, float* ws, int nsm, cudaStream_t st, const int8_t* rexp = nullptr,
                  bool x_exact = false);

// xstream_tc.cu: the same contractions on tcgen05 tensor cores (3xTF32,
// TMA-staged operands, TMEM accumulators).  Returns false (nothing launched)
// when the shape is outside its envelope (lp > 128, misaligned X).
size_t xstream_tc_ws_floats(int64_t m, int64_t n, int lp, int nsm);
void xstream_tc_set_debug(float* dbg);  // tools/tc_debug.cu only
bool launch_xs_tc(bool tn, const float* x, int64_t ldx, int64_t m, int64_t n, const float* s,
                  int lp, float* out, float* ws, int nsm, cudaStream_t st,
                  const int8_t* rexp = nullptr, bool x_exact = false);
// flag |= 1 unless every element of X (d x n, ld ldx, 16 B aligned rows) is
// exactly representable in tf32 (low 13 mantissa bits zero).
void launch_x_tf32_exact(const float* x, int64_t ldx, int64_t d, int64_t n, int* flag, int nsm,
                         cudaStream_t st);
// Per-row exponents of X (d rows, xs_rexp_bytes(d) bytes, zero padded) and a
// flag set when some row's dynamic range exceeds 2^30 (keep 3xTF32 then).
size_t xs_rexp_bytes(int64_t rows);
void launch_x_rowexp(const float* x, int64_t ldx, int64_t d, int64_t n, int8_t* rexp, int* wide,
                     int nsm, cudaStream_t st);

// ---- qr.cu: orthonormal basis with the span of Y --------------------------
// CholeskyQR2 with fp64 Grams; Householder (reference qr.cpp semantics, fp64)
// when the Cholesky factor is numerically singular.  Y and Q are rows x lp
// (ld lp); columns >= l are zero on output.  q must not alias y.
size_t qr_ws_bytes(int64_t rows, int lp, int nsm);
void launch_thin_qr_dist(const float* y, int64_t rows, int l, int lp, float* q, void* ws, int nsm,
                         cudaStream_t st, const std::function<void(double*, size_t)>& allreduce_g,
                         int** flag_out, int passes = 2);
// passes = 2: CholeskyQR2 (the bases handed on); passes = 1: one Cholesky
// pass, for the intermediate re-orthonormalisations of the range finder,
// which only carry a span into the next X pass (span and nested flag are
// the same; the final QR restores full orthogonality).
void launch_thin_qr(const float* y, int64_t rows, int l, int lp, float* q, void* ws, int nsm,
                    cudaStream_t st, int passes = 2);
// fp64 in and out (the range finder's fp64 path); ws: qr64_ws_bytes.
size_t qr64_ws_bytes(int64_t rows, int lp, int nsm);
void launch_thin_qr64(const double* y, int64_t rows, int l, int lp, double* q, void* ws, int nsm,
                      cudaStream_t st, int passes = 2);
void launch_f64_to_f32(const double* a, int64_t total, float* b, int nsm, cudaStream_t st);
double qr_kappa_estimate(const void* ws, int64_t rows, int l, int lp, int nsm, cudaStream_t st);
void launch_thin_qr64_dist(const double* y, int64_t rows, int l, int lp, double* q, void* ws,
                           int nsm, cudaStream_t st,
                           const std::function<void(double*, size_t)>& allreduce_g,
                           int** flag_out, int passes = 2);
void launch_f32_to_f64(const float* a, int64_t total, double* b, int nsm, cudaStream_t st);
// Flip the columns of an orthonormal q (rows x lp, l used) to the reference's
// Householder signs (qr.cpp:35); sgn: l floats of device scratch.  Only the
// step-level entry points that return bases need it: FastHALS-RP uses L, R
// only through sign-invariant products.
void launch_householder_signs(float* q, int64_t rows, int l, int lp, float* sgn, int nsm,
                              cudaStream_t st);

// ---- metrics.cu ------------------------------------------------------------
// check_data: flags[0] |= negative/non-finite; *norm_sq = ||X||_F^2 (fp64).
size_t metrics_ws_bytes(int64_t d, int64_t n, int nsm);
void launch_check_data(const float* x, int64_t ldx, int64_t d, int64_t n, int* flag,
                       double* norm_sq, void* ws, int nsm, cudaStream_t st, int8_t* rexp = nullptr,
                       int* wide = nullptr, int* inexact = nullptr, int* nonint = nullptr);
// 1/2 ||X - A B^T||^2 with column-major A_cm (k x d), B_cm (k x n).
// The same objective on the tensor cores (recon_tc.cu): dense X (ldx % 4 ==
// 0, 16-byte aligned), k <= 128; returns false when those do not hold.
size_t recon_tc_ws_bytes(int64_t d, int64_t n, int k, int nsm);
bool launch_recon_tc(const float* x, int64_t ldx, int64_t d, int64_t n, const double* a_cm,
                     const double* b_cm, int k, double* out, void* ws, int nsm, cudaStream_t st);
void launch_recon_error(const float* x, int64_t ldx, int64_t d, int64_t n, const double* a_cm,
                        const double* b_cm, int k, double* out, void* ws, int nsm,
                        cudaStream_t st);
size_t gini_ws_bytes(int64_t count);
void launch_gini(const double* b_cm, int64_t count, double* out, void* ws, size_t ws_bytes,
                 cudaStream_t st);
// fp64 column-major (k x rows) <-> fp32 row-major (rows x k)
void launch_cm_to_rm(const double* cm, int64_t rows, int k, float* rm, cudaStream_t st);
void launch_rm_to_cm(const float* rm, int64_t rows, int k, double* cm, cudaStream_t st);
// Copy an unpadded row-major (rows x l) matrix into an lp-padded one and back.
void launch_pad_cols(const float* src, int64_t rows, int l, float* dst, int lp, cudaStream_t st);
void launch_unpad_cols(const float* src, int64_t rows, int lp, float* dst, int l,
                       cudaStream_t st);
void launch_transpose(const float* src, int64_t rows, int64_t cols, int64_t lds, float* dst,
                      int64_t ldd, cudaStream_t st);

// ---- hals.cu: FastHALS-RP iterations ---------------------------------------
struct HaltInfo {
  int halted;  // 0 = ran to it_end
  int iter;    // iteration (1-based) in which the event happened
  int half;    // 0 = A half-sweep, 1 = B half-sweep
  int column;
  int kind;    // 1 dead B column (g_jj), 2 zero A column, 3 dead A column (w_jj), 4 zero B column,
               // 5 sharded: B half done on this rank (column = first dead-A column or k)
  int pad;
  unsigned long long last_epoch;  // exchange epoch reached (next launch starts above it)
  unsigned long long last_nr;     // norm all-reduces done so far (next launch's HalsState::nr0)
};
enum { kEvDeadB = 1, kEvZeroA = 2, kEvDeadA = 3, kEvZeroB = 4, kEvShard = 5 };

struct HalsState {
  int64_t d, n;
  int l, lp, k;
  const float* xc;   // X-check = X R^T, d x lp
  const float* xht;  // X-hat^T = X^T L, n x lp
  const float* lm;   // L, d x lp
  const float* rt;   // R^T, n x lp
  double* a;         // A, column-major k x d (fp64 state)
  double* b;         // B, column-major k x n
  double* bold;      // second B buffer (double-buffered B half), k x n
  double* h;         // X-check B-check, column-major k x d
  double* ahat;      // A-hat = L^T A, lp x k
  double* bchk;      // B-check = R B, lp x k
  double* p;         // X-hat^T A-hat, column-major k x n
  double* gsc;       // [grid][k*k] per-CTA copy of g = B-check^T B-check (fp64)
  double* wsc;       // [grid][k*k] per-CTA copy of w = A-hat^T A-hat (fp64)
  double* part;      // [grid][lp*k] partial sums
  int part_ctas;     // CTAs' worth of partial slots in `part` (the run's HALS grid)
  // The run Rng's raw mt19937_64 words (RunStream, engine.cpp), so that the
  // streaming kernel serves an emptied A column itself (reinit_column,
  // solvers.cpp:28-31,435) instead of halting to the host: pos[0] is the next
  // unused word, pos[1] counts the redraws served in-kernel.  words == null:
  // every event halts (resident kernel, dense and sharded runs).
  const unsigned long long* words;
  unsigned long long nwords;
  unsigned long long* pos;
  double* npart;     // [2][grid] column-norm partials (by exchange parity)
  unsigned* zpart;   // [grid][4] non-zero-column bitmasks, then [4] the CTA-OR (sharded halt)
  unsigned* bar;     // monotonic grid-barrier arrival counter (reset per run)
  HaltInfo* halt;
  long long* prof;   // optional per-phase clock64 sums (CTA 0), or null
  // Uncompressed FastHALS / HALS (dense = 1, streaming kernel only): each
  // launch runs ONE half-sweep of one iteration against host-prepared
  // products -- hd = X B (d x lp fp64 row-major) and gd = B^T B (k x k) for
  // the A half, pd = X^T A (n x lp) and wd = A^T A for the B half -- with no
  // compressed factors; a launch finding the halt record set returns at once
  // (launches queued behind a halt are no-ops).
  int dense;
  const double* hd;
  const double* pd;
  const double* gd;
  const double* wd;
  unsigned long long nr0;  // norm all-reduces (allreduce_fused) of earlier launches of this run:
                           // picks the slot buffer and its freshness tag (HaltInfo::last_nr)
  int sharded;       // 1: X column-sharded across ranks: after each B half the kernel halts
                     // (kEvShard) with this rank's B-check partial in bchk, its non-zero
                     // column mask in zpart[4 grid ..], the new B in b (resident kernel:
                     // the old B in bold); the host all-reduces and runs the zero check
};
size_t hals_part_doubles(int grid, int lp, int k);
int hals_grid(const HalsState& st, int nsm);
// Runs iterations [it_begin, it_end) starting at (start_half, start_col).
// Returns the cooperative-launch error, if any.
// it_begin/it_end are 0-based; HaltInfo::iter reports the 1-based iteration.
// epoch0 must exceed every epoch of earlier launches (HaltInfo::last_epoch).
// products_valid: resuming after an emptied column (ZeroA / ZeroB), the halted
// launch's products for the resumed half are reused (dense and sharded runs: 0).
cudaError_t launch_hals(const HalsState& st, int normalize_a, double alpha, double beta,
                        int it_begin, int it_end, int start_half, int start_col, int skip_dead,
                        unsigned long long epoch0, int grid, cudaStream_t s,
                        int products_valid = 0);
// Shared-memory-resident variant (hals_resident.cu): same contract; grid 0
// means the configuration does not fit and the streaming kernel is used.
int hals_resident_grid(const HalsState& st, int nsm);
cudaError_t launch_hals_resident(const HalsState& st, int normalize_a, double alpha, double beta,
                                 int it_begin, int it_end, int start_half, int start_col,
                                 int skip_dead, unsigned long long epoch0, int grid,
                                 cudaStream_t s);
// A-hat = L^T A and B-check = R B (all columns, or only column j >= 0).
void launch_compress_factors(const HalsState& st, int which /*0 A-hat, 1 B-check*/, int column,
                             cudaStream_t s);
// a_j <- a_j / ||a_j|| (no-op on a zero column), fixed-order fp64 norm.
void launch_normalize_column(double* a_cm, int64_t d, int j, cudaStream_t s);

// ---- dense.cu: the uncompressed solvers (fp64 CUDA-core contractions) ----
// out (rows x lp fp64, row-major) = X S (NN, rows = m) or X^T T (TN, rows = n);
// s: K x lp fp64 row-major (lp a multiple of 16, <= 128); ws: xs64_ws_doubles.
size_t xs64_ws_doubles(int64_t m, int64_t n, int lp, int nsm);
// ---- xstream_i8.cu: the same contractions (fp32 X, fp64 S and output) with
// exact int32 accumulation on the integer tensor cores (Ozaki-style int8
// digit slices).  sx: launch_xs_i8_prepare_x's row / column scale exponents
// of X (xs_i8_sx_ints ints).  launch_xs_i8 returns false outside its envelope
// (lp a multiple of 16, <= 128; 16-byte aligned rows).  small_int: X holds only integers below
// 8192 and sx is zero (exact two-digit X, six digits of S).
bool xs_i8_supported(int lp);
void xs_i8_set_debug(unsigned long long* dbg);  // tools/i8_trace.cu only (I8_TRACE builds)
size_t xs_i8_sx_ints(int64_t d, int64_t n);
int xs_i8_x_passes(int lp, bool small_int);
size_t xs_i8_ws_bytes(int64_t m, int64_t n, int lp, int nsm);
void launch_xs_i8_prepare_x(const float* x, int64_t ldx, int64_t d, int64_t n, int* sx, int nsm,
                            cudaStream_t st);
bool launch_xs_i8(bool tn, const float* x, int64_t ldx, int64_t m, int64_t n, const double* s,
                  int lp, double* out, void* ws, const int* sx, int nsm, cudaStream_t st,
                  bool small_int = false);
// halt (nullable): a device flag; when set the launch is a no-op (products
// queued behind a halted dense HALS sweep, engine.cpp run_dense_hals).
void launch_xs64_nn(const float* x, int64_t ldx, int64_t m, int64_t n, const double* s, int lp,
                    double* out, double* ws, int nsm, cudaStream_t st, const int* halt = nullptr);
void launch_xs64_tn(const float* x, int64_t ldx, int64_t m, int64_t n, const double* t, int lp,
                    double* out, double* ws, int nsm, cudaStream_t st, const int* halt = nullptr);
// g (k x k) = F^T F of a column-major k x rows fp64 factor (row_major: a
// rows x k row-major one), fixed-order fp64.
size_t gram_cm_ws_doubles(int64_t rows, int k, int nsm);
void launch_gram_cm(const double* f_cm, int64_t rows, int k, double* g, double* ws, int nsm,
                    cudaStream_t st, bool row_major = false, const int* halt = nullptr);
void launch_cm_to_rm_pad64(const double* f_cm, int64_t rows, int k, int lp, double* out,
                           int nsm, cudaStream_t st, const int* halt = nullptr);
// mu_update_half (semi = 0) / semi_nmf_half (semi = 1) of a column-major
// factor: t_out = t_in .* f(num, t_in g) (solvers.cpp:55-93).
void launch_mu_update(const double* t_in, int64_t rows, int k, const double* num, int ldn,
                      const double* g, int semi, double* t_out, int nsm, cudaStream_t st);
// out (rows x k, ld ldo, fp64) = in (rows x lp fp32, first l columns) m (l x k fp64)
void launch_rows_small64(const float* in, int64_t rows, int l, int lp, const double* m, int k,
                         double* out, int ldo, int nsm, cudaStream_t st);

// ---- sparse.cu: CSR input ------------------------------
// X (d x n) as CSR plus the CSR of X^T (built on the host), device pointers.
struct CsrView {
  int64_t d, n, nnz;
  const int64_t* rp;    // d + 1 row offsets
  const int32_t* ci;    // column indices, ascending within a row
  const float* v;
  const int64_t* t_rp;  // X^T: n + 1 offsets
  const int32_t* t_ci;  // row indices, ascending within a column
  const float* t_v;
};
// out (rows x ldo; columns >= l zero) = X S (transpose = false, rows = d) or
// X^T S (rows = n), S row-major with ld lds; fp64 accumulation.
void launch_csr_spmm_f32(const CsrView& x, bool transpose, const float* s, int lds, int l,
                         float* out, int ldo, int nsm, cudaStream_t st);
void launch_csr_spmm_f64(const CsrView& x, bool transpose, const double* s, int lds, int l,
                         double* out, int ldo, int nsm, cudaStream_t st,
                         const int* halt = nullptr);
size_t csr_metrics_ws_doubles(int nsm);
// check_data (flag |= negative / non-finite value) and ||X||^2
void launch_csr_check(const CsrView& x, int* flag, double* norm_sq, double* ws, int nsm,
                      cudaStream_t st);
// the sparse objective (metrics.cpp:79-102) given ||X||^2, A^T A and B^T B
void launch_csr_objective(const CsrView& x, const double* a_cm, const double* b_cm, int k,
                          const double* xnorm, const double* ata, const double* btb, double* out,
                          double* ws, int nsm, cudaStream_t st);

// ---- synth.cu: synthetic data (bench harness, BASELINE.json configs) ------
void launch_synth_x(int64_t d, int64_t n, int rank, int factor_kind, int noise_kind, double sigma,
                    uint64_t seed, int64_t col_lo, int64_t col_hi, int64_t ldx, float* x,
                    double* scratch, cudaStream_t s);
size_t synth_scratch_doubles(int64_t d, int64_t ncols, int rank);

}  // namespace cnmf
