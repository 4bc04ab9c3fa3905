/*
 * cnmf_oracle.c -- CPU restatement of the reference's compressed-NMF hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  This file is the parity checker for the CUDA
 * product in paper_1712_02248_b200/.  Only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline / --impl reference legs may load it.  Nothing
 * in the product links against it, and the product never falls back to it.
 *
 * Every function restates the algorithm of the reference C++ library
 * (/root/reference/proj, cited below as file:line) in plain C, with the same
 * loop nests and the same floating-point operation order, so that compiled
 * with the reference's Release flags (no FMA contraction on x86-64) it
 * reproduces the reference bit for bit.  That identity is pinned in
 * tests/test_oracle.py against oracle/_ref (the reference compiled from its
 * own sources by oracle/Makefile) and against tests/golden/ fixtures.
 *
 * Storage: every matrix is a row-major double array, as DenseMatrix
 * (proj/include/cnmf/matrix.hpp:11-28).  B is stored n x k (= H^T).
 */
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <time.h>

/* ---- status codes (mirror proj/include/cnmf/errors.hpp:10-28) ---------- */
enum {
  ORC_OK = 0,
  ORC_CONFIG_ERROR = 1,    /* ConfigError    */
  ORC_DIMENSION_ERROR = 2, /* DimensionError */
  ORC_INPUT_ERROR = 3,     /* InputError     */
};

static char g_msg[256];
const char* orc_last_message(void) { return g_msg; }
static int fail(int code, const char* msg) {
  snprintf(g_msg, sizeof g_msg, "%s", msg);
  return code;
}

/* ======================================================================
 * Rng: std::mt19937_64 + the reference's fixed variate mappings.
 * proj/include/cnmf/rng.hpp:13-60.
 * ==================================================================== */
#define MT_N 312
#define MT_M 156
typedef struct {
  uint64_t mt[MT_N];
  int idx;
  double spare;
  int has_spare;
} orc_rng;

size_t orc_rng_sizeof(void) { return sizeof(orc_rng); }

void orc_rng_init(orc_rng* r, uint64_t seed) {
  /* std::mersenne_twister_engine::seed(value), f = 6364136223846793005 */
  r->mt[0] = seed;
  for (int i = 1; i < MT_N; ++i)
    r->mt[i] = 6364136223846793005ULL * (r->mt[i - 1] ^ (r->mt[i - 1] >> 62)) + (uint64_t)i;
  r->idx = MT_N;
  r->spare = 0.0;
  r->has_spare = 0;
}

static void mt_twist(uint64_t* mt) {
  const uint64_t UM = 0xFFFFFFFF80000000ULL, LM = 0x7FFFFFFFULL;
  const uint64_t A = 0xB5026F5AA96619E9ULL;
  int i;
  for (i = 0; i < MT_N - MT_M; ++i) {
    uint64_t y = (mt[i] & UM) | (mt[i + 1] & LM);
    mt[i] = mt[i + MT_M] ^ (y >> 1) ^ ((y & 1ULL) ? A : 0ULL);
  }
  for (; i < MT_N - 1; ++i) {
    uint64_t y = (mt[i] & UM) | (mt[i + 1] & LM);
    mt[i] = mt[i + (MT_M - MT_N)] ^ (y >> 1) ^ ((y & 1ULL) ? A : 0ULL);
  }
  uint64_t y = (mt[MT_N - 1] & UM) | (mt[0] & LM);
  mt[MT_N - 1] = mt[MT_M - 1] ^ (y >> 1) ^ ((y & 1ULL) ? A : 0ULL);
}

uint64_t orc_rng_next(orc_rng* r) { /* rng.hpp:17 */
  if (r->idx >= MT_N) {
    mt_twist(r->mt);
    r->idx = 0;
  }
  uint64_t z = r->mt[r->idx++];
  z ^= (z >> 29) & 0x5555555555555555ULL;
  z ^= (z << 17) & 0x71D67FFFEDA60000ULL;
  z ^= (z << 37) & 0xFFF7EEE000000000ULL;
  z ^= z >> 43;
  return z;
}

double orc_rng_uniform(orc_rng* r) { /* rng.hpp:20-22 */
  return (double)(orc_rng_next(r) >> 11) * 0x1.0p-53;
}

double orc_rng_uniform_positive(orc_rng* r) { /* rng.hpp:25-29 */
  double v = orc_rng_uniform(r);
  while (v == 0.0) v = orc_rng_uniform(r);
  return v;
}

double orc_rng_normal(orc_rng* r) { /* rng.hpp:32-44, cos first, sin cached */
  if (r->has_spare) {
    r->has_spare = 0;
    return r->spare;
  }
  const double u1 = orc_rng_uniform_positive(r);
  const double u2 = orc_rng_uniform(r);
  const double radius = sqrt(-2.0 * log(u1));
  const double angle = 2.0 * 3.141592653589793238462643383279502884 * u2;
  r->spare = radius * sin(angle);
  r->has_spare = 1;
  return radius * cos(angle);
}

/* ======================================================================
 * Dense linear algebra.  proj/src/matrix.cpp
 * ==================================================================== */

/* C = op(M) op(N); c must hold out_rows*out_cols and is overwritten.
 * matrix.cpp:94-154, the four loop nests kept verbatim in order. */
int orc_matmul(const double* m, size_t mr, size_t mc, const double* nn, size_t nr,
               size_t nc, int tl, int tr, double* c) {
  const size_t out_rows = tl ? mc : mr;
  const size_t inner_l = tl ? mr : mc;
  const size_t inner_r = tr ? nc : nr;
  const size_t out_cols = tr ? nr : nc;
  if (inner_l != inner_r) return fail(ORC_DIMENSION_ERROR, "matmul: inner dimensions differ");
  memset(c, 0, sizeof(double) * out_rows * out_cols);
  if (!tl && !tr) { /* 105-116 */
    for (size_t i = 0; i < out_rows; ++i) {
      double* ci = c + i * out_cols;
      const double* mi = m + i * mc;
      for (size_t l = 0; l < inner_l; ++l) {
        const double a = mi[l];
        if (a == 0.0) continue;
        const double* nl = nn + l * nc;
        for (size_t j = 0; j < out_cols; ++j) ci[j] += a * nl[j];
      }
    }
  } else if (!tl && tr) { /* 117-128 */
    for (size_t i = 0; i < out_rows; ++i) {
      double* ci = c + i * out_cols;
      const double* mi = m + i * mc;
      for (size_t j = 0; j < out_cols; ++j) {
        const double* nj = nn + j * nc;
        double s = 0.0;
        for (size_t l = 0; l < inner_l; ++l) s += mi[l] * nj[l];
        ci[j] = s;
      }
    }
  } else if (tl && !tr) { /* 129-140 */
    for (size_t l = 0; l < inner_l; ++l) {
      const double* ml = m + l * mc;
      const double* nl = nn + l * nc;
      for (size_t i = 0; i < out_rows; ++i) {
        const double a = ml[i];
        if (a == 0.0) continue;
        double* ci = c + i * out_cols;
        for (size_t j = 0; j < out_cols; ++j) ci[j] += a * nl[j];
      }
    }
  } else { /* 141-152 */
    for (size_t j = 0; j < out_cols; ++j) {
      const double* nj = nn + j * nc;
      for (size_t l = 0; l < inner_l; ++l) {
        const double b = nj[l];
        if (b == 0.0) continue;
        const double* ml = m + l * mc;
        for (size_t i = 0; i < out_rows; ++i) c[i * out_cols + j] += ml[i] * b;
      }
    }
  }
  return ORC_OK;
}

static double* dalloc(size_t count) {
  double* p = (double*)calloc(count ? count : 1, sizeof(double));
  if (!p) {
    fprintf(stderr, "oracle: out of memory\n");
    abort();
  }
  return p;
}

/* y = op(M) v.  matrix.cpp:191-214 */
static void matvec(const double* m, size_t rows, size_t cols, const double* v, int transpose,
                   double* y) {
  if (!transpose) {
    for (size_t i = 0; i < rows; ++i) {
      const double* mi = m + i * cols;
      double s = 0.0;
      for (size_t j = 0; j < cols; ++j) s += mi[j] * v[j];
      y[i] = s;
    }
    return;
  }
  for (size_t j = 0; j < cols; ++j) y[j] = 0.0;
  for (size_t i = 0; i < rows; ++i) {
    const double a = v[i];
    if (a == 0.0) continue;
    const double* mi = m + i * cols;
    for (size_t j = 0; j < cols; ++j) y[j] += a * mi[j];
  }
}

double orc_frobenius_norm_sq(const double* m, size_t count) { /* matrix.cpp:233-237 */
  double s = 0.0;
  for (size_t i = 0; i < count; ++i) s += m[i] * m[i];
  return s;
}

static void transpose(const double* m, size_t rows, size_t cols, double* t) {
  for (size_t i = 0; i < rows; ++i)
    for (size_t j = 0; j < cols; ++j) t[j * rows + i] = m[i * cols + j];
}

/* Householder thin QR, Q only (R optional).  proj/src/qr.cpp:10-75 */
int orc_thin_qr(const double* m, size_t rows, size_t cols, double* q, double* r_out) {
  if (rows < cols)
    return fail(ORC_DIMENSION_ERROR, "thin_qr: input must have at least as many rows as columns");
  const double deficiency_floor = 1e-12 * sqrt(orc_frobenius_norm_sq(m, rows * cols)); /* 16 */
  double* w = dalloc(rows * cols);
  memcpy(w, m, sizeof(double) * rows * cols);
  double** refl = (double**)calloc(cols ? cols : 1, sizeof(double*));
  for (size_t j = 0; j < cols; ++j) {
    double normx_sq = 0.0;
    for (size_t i = j; i < rows; ++i) normx_sq += w[i * cols + j] * w[i * cols + j];
    const double normx = sqrt(normx_sq);
    if (normx < deficiency_floor) { /* 28-33: dependent column */
      for (size_t i = j; i < rows; ++i) w[i * cols + j] = 0.0;
      continue;
    }
    const double alpha = w[j * cols + j] >= 0.0 ? -normx : normx;
    double* v = dalloc(rows - j);
    for (size_t i = j; i < rows; ++i) v[i - j] = w[i * cols + j];
    v[0] -= alpha;
    double vnorm = 0.0;
    for (size_t i = 0; i < rows - j; ++i) vnorm += v[i] * v[i];
    vnorm = sqrt(vnorm);
    for (size_t i = 0; i < rows - j; ++i) v[i] /= vnorm;
    for (size_t c = j; c < cols; ++c) {
      double proj = 0.0;
      for (size_t i = j; i < rows; ++i) proj += v[i - j] * w[i * cols + c];
      proj *= 2.0;
      for (size_t i = j; i < rows; ++i) w[i * cols + c] -= proj * v[i - j];
    }
    w[j * cols + j] = alpha;
    for (size_t i = j + 1; i < rows; ++i) w[i * cols + j] = 0.0;
    refl[j] = v;
  }
  if (r_out) {
    memset(r_out, 0, sizeof(double) * cols * cols);
    for (size_t i = 0; i < cols; ++i)
      for (size_t j = i; j < cols; ++j) r_out[i * cols + j] = w[i * cols + j];
  }
  /* 61-72: Q = H_0 ... H_{cols-1} applied to the identity slice, reversed */
  memset(q, 0, sizeof(double) * rows * cols);
  for (size_t j = 0; j < cols; ++j) q[j * cols + j] = 1.0;
  for (size_t jj = cols; jj-- > 0;) {
    const double* v = refl[jj];
    if (!v) continue;
    for (size_t c = 0; c < cols; ++c) {
      double proj = 0.0;
      for (size_t i = jj; i < rows; ++i) proj += v[i - jj] * q[i * cols + c];
      proj *= 2.0;
      for (size_t i = jj; i < rows; ++i) q[i * cols + c] -= proj * v[i - jj];
    }
  }
  for (size_t j = 0; j < cols; ++j) free(refl[j]);
  free(refl);
  free(w);
  return ORC_OK;
}

/* ======================================================================
 * Compression.  proj/src/compression.cpp
 * ==================================================================== */

/* compression.cpp:11-16: row-major fill from a fresh Rng(seed). */
void orc_gaussian_sketch(size_t rows, size_t cols, uint64_t seed, double* out) {
  orc_rng r;
  orc_rng_init(&r, seed);
  for (size_t i = 0; i < rows * cols; ++i) out[i] = orc_rng_normal(&r);
}

/* compression.cpp:23-42.  basis_out is op_rows x q. */
int orc_range_finder(const double* x, size_t d, size_t n, int use_transpose, size_t q,
                     size_t power_iterations, uint64_t seed, double* basis_out) {
  const size_t op_rows = use_transpose ? n : d;
  const size_t op_cols = use_transpose ? d : n;
  const size_t mn = op_rows < op_cols ? op_rows : op_cols;
  if (q == 0 || q > mn)
    return fail(ORC_CONFIG_ERROR,
                "powered_range_finder: q must satisfy 1 <= q <= min(rows, cols)");
  double* omega = dalloc(op_cols * q);
  orc_gaussian_sketch(op_cols, q, seed, omega);
  double* y = dalloc(op_rows * q);
  if (use_transpose)
    orc_matmul(x, d, n, omega, op_cols, q, 1, 0, y); /* X^T Omega (TN) */
  else
    orc_matmul(x, d, n, omega, op_cols, q, 0, 0, y); /* X Omega (NN) */
  orc_thin_qr(y, op_rows, q, basis_out, NULL);
  double* zin = dalloc(op_cols * q);
  double* z = dalloc(op_cols * q);
  for (size_t it = 0; it < power_iterations; ++it) {
    if (use_transpose)
      orc_matmul(x, d, n, basis_out, n, q, 0, 0, zin); /* X basis */
    else
      orc_matmul(x, d, n, basis_out, d, q, 1, 0, zin); /* X^T basis */
    orc_thin_qr(zin, op_cols, q, z, NULL);
    if (use_transpose)
      orc_matmul(x, d, n, z, d, q, 1, 0, y);
    else
      orc_matmul(x, d, n, z, n, q, 0, 0, y);
    orc_thin_qr(y, op_rows, q, basis_out, NULL);
  }
  free(omega);
  free(y);
  free(zin);
  free(z);
  return ORC_OK;
}

/* compression.cpp:44-53: L from seed 2s, R = (row basis from seed 2s+1)^T.
 * left is d x q, right is q x n. */
int orc_build_projectors(const double* x, size_t d, size_t n, size_t q, size_t w,
                         uint64_t seed, double* left, double* right) {
  int st = orc_range_finder(x, d, n, 0, q, w, seed * 2, left);
  if (st) return st;
  double* row_basis = dalloc(n * q);
  st = orc_range_finder(x, d, n, 1, q, w, seed * 2 + 1, row_basis);
  if (!st) transpose(row_basis, n, q, right);
  free(row_basis);
  return st;
}

/* compression.cpp:73-96 */
void orc_compress_left(const double* x, size_t d, size_t n, const double* left, size_t q,
                       double* xhat) {
  orc_matmul(left, d, q, x, d, n, 1, 0, xhat); /* q x n */
}
void orc_compress_right(const double* x, size_t d, size_t n, const double* right, size_t q,
                        double* xcheck) {
  orc_matmul(x, d, n, right, q, n, 0, 1, xcheck); /* d x q */
}
void orc_compress_factor_a(const double* a, size_t d, size_t k, const double* left, size_t q,
                           double* a_hat) {
  orc_matmul(left, d, q, a, d, k, 1, 0, a_hat); /* q x k */
}
void orc_compress_factor_b(const double* b, size_t n, size_t k, const double* right, size_t q,
                           double* b_check) {
  orc_matmul(right, q, n, b, n, k, 0, 0, b_check); /* q x k */
}

/* ======================================================================
 * Solvers.  proj/src/solvers.cpp
 * ==================================================================== */
#define K_DEAD 1e-12   /* solvers.cpp:19 */
#define K_REINIT 1e-3  /* solvers.cpp:22 */

static void reinit_column(double* m, size_t rows, size_t cols, size_t j, orc_rng* rng) {
  for (size_t i = 0; i < rows; ++i) m[i * cols + j] = orc_rng_uniform_positive(rng) * K_REINIT;
}
static int column_all_zero(const double* m, size_t rows, size_t cols, size_t j) {
  for (size_t i = 0; i < rows; ++i)
    if (m[i * cols + j] != 0.0) return 0;
  return 1;
}
static void normalize_column(double* m, size_t rows, size_t cols, size_t j) { /* 39-45 */
  double norm_sq = 0.0;
  for (size_t i = 0; i < rows; ++i) norm_sq += m[i * cols + j] * m[i * cols + j];
  const double norm = sqrt(norm_sq);
  if (norm == 0.0) return;
  for (size_t i = 0; i < rows; ++i) m[i * cols + j] /= norm;
}
static void get_column(const double* m, size_t rows, size_t cols, size_t j, double* v) {
  for (size_t i = 0; i < rows; ++i) v[i] = m[i * cols + j];
}
static void set_column(double* m, size_t rows, size_t cols, size_t j, const double* v) {
  for (size_t i = 0; i < rows; ++i) m[i * cols + j] = v[i];
}
static double clamp0(double x) { return x > 0.0 ? x : 0.0; } /* matrix.cpp:258-266 */

void orc_initialize(size_t d, size_t n, size_t k, uint64_t seed, double* a, double* b) {
  orc_rng r; /* solvers.cpp:314-325 */
  orc_rng_init(&r, seed);
  for (size_t i = 0; i < d * k; ++i) a[i] = orc_rng_uniform_positive(&r);
  for (size_t i = 0; i < n * k; ++i) b[i] = orc_rng_uniform_positive(&r);
}

/* refresh_cross_products, solvers.cpp:133-144: data is rows x cols used as
 * op(data) (transposed when data_transposed), factor is f_rows x k. */
static void refresh_cross_products(const double* data, size_t rows, size_t cols,
                                   const double* factor, size_t f_rows, size_t k, double* p,
                                   size_t p_rows, double* g, size_t j, int data_transposed) {
  double* fj = dalloc(f_rows);
  double* pj = dalloc(p_rows);
  double* gj = dalloc(k);
  get_column(factor, f_rows, k, j, fj);
  matvec(data, rows, cols, fj, data_transposed, pj);
  set_column(p, p_rows, k, j, pj);
  matvec(factor, f_rows, k, fj, 1, gj);
  for (size_t l = 0; l < k; ++l) {
    g[l * k + j] = gj[l];
    g[j * k + l] = gj[l];
  }
  free(fj);
  free(pj);
  free(gj);
}

/* solvers.cpp:480-509: column j of the B update (unconstrained at a=b=0). */
static void b_update_fasthals_rp(const double* b, size_t n, size_t k, const double* p,
                                 const double* w, size_t j, double alpha, double beta,
                                 double* out) {
  double* wj = dalloc(k);
  double* bw = dalloc(n);
  get_column(w, k, k, j, wj);
  matvec(b, n, k, wj, 0, bw);
  if (alpha == 0.0 && beta == 0.0) { /* 480-490 */
    const double den = w[j * k + j];
    for (size_t i = 0; i < n; ++i) out[i] = clamp0(b[i * k + j] + (p[i * k + j] - bw[i]) / den);
  } else { /* 502-508 */
    const double wjj = w[j * k + j];
    const double den = wjj + beta;
    for (size_t i = 0; i < n; ++i)
      out[i] = clamp0((b[i * k + j] * wjj + p[i * k + j] - bw[i] - alpha) / den);
  }
  free(wj);
  free(bw);
}

/* exported for the closed-form tests (solvers.cpp:480-509) */
void orc_b_update_fasthals_rp(const double* b, size_t n, size_t k, const double* p,
                              const double* w, size_t j, double alpha, double beta,
                              double* out) {
  b_update_fasthals_rp(b, n, k, p, w, j, alpha, beta, out);
}

/* fasthals_rp_step, solvers.cpp:414-456.  xhat is q x n, xcheck d x q,
 * left d x q, right q x n, a d x k, b n x k, a_hat q x k, b_check q x k. */
int orc_fasthals_rp_step(const double* xhat, const double* xcheck, size_t d, size_t n,
                         size_t q, size_t k, double* a, double* b, double* a_hat,
                         double* b_check, const double* left, const double* right,
                         int normalize_a, double alpha, double beta, orc_rng* rng) {
  {
    double* h = dalloc(d * k);
    double* g = dalloc(k * k);
    double* gj = dalloc(k);
    double* ag = dalloc(d);
    double* aj = dalloc(d);
    double* bj = dalloc(n);
    double* bcj = dalloc(q);
    orc_matmul(xcheck, d, q, b_check, q, k, 0, 0, h);     /* 421 */
    orc_matmul(b_check, q, k, b_check, q, k, 1, 0, g);    /* 422 */
    for (size_t j = 0; j < k; ++j) {
      if (g[j * k + j] < K_DEAD) { /* 424-428 */
        reinit_column(b, n, k, j, rng);
        get_column(b, n, k, j, bj);
        matvec(right, q, n, bj, 0, bcj);
        set_column(b_check, q, k, j, bcj);
        refresh_cross_products(xcheck, d, q, b_check, q, k, h, d, g, j, 0);
      }
      const double den = g[j * k + j];
      get_column(g, k, k, j, gj);
      matvec(a, d, k, gj, 0, ag); /* 430 */
      for (size_t i = 0; i < d; ++i) aj[i] = a[i * k + j] + (h[i * k + j] - ag[i]) / den;
      for (size_t i = 0; i < d; ++i) aj[i] = clamp0(aj[i]);
      set_column(a, d, k, j, aj);
      if (column_all_zero(a, d, k, j)) reinit_column(a, d, k, j, rng); /* 435 */
      if (normalize_a) normalize_column(a, d, k, j);                   /* 436 */
    }
    orc_compress_factor_a(a, d, k, left, q, a_hat); /* 438 */
    free(h); free(g); free(gj); free(ag); free(aj); free(bj); free(bcj);
  }
  {
    double* p = dalloc(n * k);
    double* w = dalloc(k * k);
    double* aj = dalloc(d);
    double* ahj = dalloc(q);
    double* out = dalloc(n);
    orc_matmul(xhat, q, n, a_hat, q, k, 1, 0, p);   /* 442 */
    orc_matmul(a_hat, q, k, a_hat, q, k, 1, 0, w);  /* 443 */
    for (size_t j = 0; j < k; ++j) {
      if (w[j * k + j] < K_DEAD) { /* 445-449 */
        reinit_column(a, d, k, j, rng);
        get_column(a, d, k, j, aj);
        matvec(left, d, q, aj, 1, ahj);
        set_column(a_hat, q, k, j, ahj);
        refresh_cross_products(xhat, q, n, a_hat, q, k, p, n, w, j, 1);
      }
      b_update_fasthals_rp(b, n, k, p, w, j, alpha, beta, out); /* 450-451 */
      set_column(b, n, k, j, out);
      if (column_all_zero(b, n, k, j)) reinit_column(b, n, k, j, rng); /* 452 */
    }
    orc_compress_factor_b(b, n, k, right, q, b_check); /* 454 */
    free(p); free(w); free(aj); free(ahj); free(out);
  }
  return ORC_OK;
}

/* fasthals_step_impl (dense), solvers.cpp:146-187 -- used by the
 * square-sketch reduction tests (test_solvers.cpp:356-370). */
int orc_fasthals_step(const double* x, size_t d, size_t n, size_t k, double* a, double* b,
                      int normalize_a, orc_rng* rng) {
  {
    double* p = dalloc(d * k);
    double* g = dalloc(k * k);
    double* gj = dalloc(k);
    double* ag = dalloc(d);
    double* aj = dalloc(d);
    orc_matmul(x, d, n, b, n, k, 0, 0, p);
    orc_matmul(b, n, k, b, n, k, 1, 0, g);
    for (size_t j = 0; j < k; ++j) {
      if (g[j * k + j] < K_DEAD) {
        reinit_column(b, n, k, j, rng);
        refresh_cross_products(x, d, n, b, n, k, p, d, g, j, 0);
      }
      const double den = g[j * k + j];
      get_column(g, k, k, j, gj);
      matvec(a, d, k, gj, 0, ag);
      for (size_t i = 0; i < d; ++i) aj[i] = clamp0(a[i * k + j] + (p[i * k + j] - ag[i]) / den);
      set_column(a, d, k, j, aj);
      if (column_all_zero(a, d, k, j)) reinit_column(a, d, k, j, rng);
      if (normalize_a) normalize_column(a, d, k, j);
    }
    free(p); free(g); free(gj); free(ag); free(aj);
  }
  {
    double* p = dalloc(n * k);
    double* g = dalloc(k * k);
    double* gj = dalloc(k);
    double* bg = dalloc(n);
    double* bj = dalloc(n);
    orc_matmul(x, d, n, a, d, k, 1, 0, p);
    orc_matmul(a, d, k, a, d, k, 1, 0, g);
    for (size_t j = 0; j < k; ++j) {
      if (g[j * k + j] < K_DEAD) {
        reinit_column(a, d, k, j, rng);
        refresh_cross_products(x, d, n, a, d, k, p, n, g, j, 1);
      }
      const double den = g[j * k + j];
      get_column(g, k, k, j, gj);
      matvec(b, n, k, gj, 0, bg);
      for (size_t i = 0; i < n; ++i) bj[i] = clamp0(b[i * k + j] + (p[i * k + j] - bg[i]) / den);
      set_column(b, n, k, j, bj);
      if (column_all_zero(b, n, k, j)) reinit_column(b, n, k, j, rng);
    }
    free(p); free(g); free(gj); free(bg); free(bj);
  }
  return ORC_OK;
}

/* ======================================================================
 * Metrics.  proj/src/metrics.cpp
 * ==================================================================== */

/* metrics.cpp:61-77: 1/2 ||X - A B^T||^2, direct residual form. */
double orc_reconstruction_error(const double* x, size_t d, size_t n, const double* a,
                                const double* b, size_t k) {
  double sum = 0.0;
  for (size_t i = 0; i < d; ++i) {
    const double* ai = a + i * k;
    const double* xi = x + i * n;
    for (size_t j = 0; j < n; ++j) {
      const double* bj = b + j * k;
      double pred = 0.0;
      for (size_t l = 0; l < k; ++l) pred += ai[l] * bj[l];
      const double diff = xi[j] - pred;
      sum += diff * diff;
    }
  }
  return 0.5 * sum;
}

static int cmp_double(const void* pa, const void* pb) {
  const double a = *(const double*)pa, b = *(const double*)pb;
  return (a > b) - (a < b);
}

/* metrics.cpp:104-121.  Returns NaN where the reference throws InputError
 * (empty, negative/non-finite, all-zero); run() maps that to NaN too. */
double orc_gini(const double* v, size_t count) {
  if (count == 0) return NAN;
  double total = 0.0;
  for (size_t i = 0; i < count; ++i) {
    if (v[i] < 0.0 || !isfinite(v[i])) return NAN;
    total += v[i];
  }
  if (total == 0.0) return NAN;
  double* s = dalloc(count);
  memcpy(s, v, sizeof(double) * count);
  qsort(s, count, sizeof(double), cmp_double); /* equal keys are equal values */
  const double m = (double)count;
  double acc = 0.0;
  for (size_t i = 0; i < count; ++i) acc += (2.0 * (double)(i + 1) - m - 1.0) * s[i];
  free(s);
  return acc / (m * total);
}

/* ======================================================================
 * Driver.  run_impl, solvers.cpp:189-312
 * ==================================================================== */
enum { ORC_ALGO_FASTHALS = 4, ORC_ALGO_FASTHALS_RP = 5 }; /* algorithm.hpp:8-15 */
enum { ORC_CONVERGED = 0, ORC_REACHED_MAX = 1, ORC_ABORTED = 2 }; /* metrics.hpp:62-66 */

typedef struct {
  int algorithm;
  size_t k;
  size_t q;
  size_t power_iterations;
  uint64_t sketch_seed;
  double alpha;
  double beta;
  size_t max_iterations;
  double rel_tolerance;
  size_t error_interval;
  uint64_t seed;
  int normalize_a;
} orc_config;

typedef struct {
  size_t* rec_iter;
  double* rec_error;
  double* rec_elapsed;
  size_t rec_capacity;
  size_t rec_count;
  double update_seconds;
  double compress_seconds; /* build_projectors + compress_*; not in the reference trace */
  double gini_b;
  int status;
  size_t iterations_run;
  char message[256];
} orc_trace;

static double now_s(void) {
  struct timespec ts;
  clock_gettime(CLOCK_MONOTONIC, &ts);
  return (double)ts.tv_sec + 1e-9 * (double)ts.tv_nsec;
}

/* SolverConfig::validate, solvers.cpp:298-312 */
int orc_validate(const orc_config* c, size_t d, size_t n) {
  const size_t mn = d < n ? d : n;
  const int rp = c->algorithm == ORC_ALGO_FASTHALS_RP;
  if (c->k == 0 || c->k > mn) return fail(ORC_CONFIG_ERROR, "k must satisfy 1 <= k <= min(d, n)");
  if (rp && (c->q <= c->k || c->q > mn))
    return fail(ORC_CONFIG_ERROR, "compressed algorithms require k < q <= min(d, n)");
  if (!(c->alpha >= 0.0) || !isfinite(c->alpha) || !(c->beta >= 0.0) || !isfinite(c->beta))
    return fail(ORC_CONFIG_ERROR, "alpha and beta must be finite and non-negative");
  if ((c->alpha != 0.0 || c->beta != 0.0) && !rp)
    return fail(ORC_CONFIG_ERROR, "penalties are supported by hals-rp and fasthals-rp only");
  if (c->error_interval == 0) return fail(ORC_CONFIG_ERROR, "error_interval must be positive");
  if (!(c->rel_tolerance > 0.0) || !isfinite(c->rel_tolerance))
    return fail(ORC_CONFIG_ERROR, "rel_tolerance must be positive and finite");
  if (c->algorithm != ORC_ALGO_FASTHALS && c->algorithm != ORC_ALGO_FASTHALS_RP)
    return fail(ORC_CONFIG_ERROR, "oracle restates fasthals and fasthals-rp only");
  return ORC_OK;
}

static void push_record(orc_trace* t, size_t it, double err, double el) {
  if (t->rec_count < t->rec_capacity) {
    t->rec_iter[t->rec_count] = it;
    t->rec_error[t->rec_count] = err;
    t->rec_elapsed[t->rec_count] = el;
  }
  t->rec_count++;
}

/* run(x, config) for fasthals / fasthals-rp.  a_out d x k, b_out n x k. */
int orc_run(const double* x, size_t d, size_t n, const orc_config* c, double* a_out,
            double* b_out, orc_trace* t) {
  int st = orc_validate(c, d, n);
  if (st) return st;
  for (size_t i = 0; i < d * n; ++i) /* check_data, solvers.cpp:47-52 */
    if (!(x[i] >= 0.0) || !isfinite(x[i]))
      return fail(ORC_INPUT_ERROR, "solver input must be entrywise non-negative and finite");
  const int rp = c->algorithm == ORC_ALGO_FASTHALS_RP;
  const size_t k = c->k, q = c->q;
  t->rec_count = 0;
  t->update_seconds = 0.0;
  t->compress_seconds = 0.0;
  t->status = ORC_REACHED_MAX;
  t->message[0] = 0;
  t->iterations_run = 0;

  orc_rng rng;
  orc_rng_init(&rng, c->seed); /* 206-211: A then B */
  double* a = a_out;
  double* b = b_out;
  for (size_t i = 0; i < d * k; ++i) a[i] = orc_rng_uniform_positive(&rng);
  for (size_t i = 0; i < n * k; ++i) b[i] = orc_rng_uniform_positive(&rng);

  double *left = NULL, *right = NULL, *xhat = NULL, *xcheck = NULL, *a_hat = NULL,
         *b_check = NULL;
  if (rp) { /* 213-221 */
    const double t0 = now_s();
    left = dalloc(d * q);
    right = dalloc(q * n);
    xhat = dalloc(q * n);
    xcheck = dalloc(d * q);
    a_hat = dalloc(q * k);
    b_check = dalloc(q * k);
    orc_build_projectors(x, d, n, q, c->power_iterations, c->sketch_seed, left, right);
    orc_compress_left(x, d, n, left, q, xhat);
    orc_compress_right(x, d, n, right, q, xcheck);
    t->compress_seconds = now_s() - t0;
    orc_compress_factor_a(a, d, k, left, q, a_hat);
    orc_compress_factor_b(b, n, k, right, q, b_check);
  }

  double previous = orc_reconstruction_error(x, d, n, a, b, k); /* 223-229 */
  if (!isfinite(previous)) {
    t->status = ORC_ABORTED;
    snprintf(t->message, sizeof t->message, "non-finite objective at iteration 0");
  } else {
    push_record(t, 0, previous, 0.0);
  }
  for (size_t iter = 1; t->status != ORC_ABORTED && iter <= c->max_iterations; ++iter) {
    const double t0 = now_s();
    if (rp)
      orc_fasthals_rp_step(xhat, xcheck, d, n, q, k, a, b, a_hat, b_check, left, right,
                           c->normalize_a, c->alpha, c->beta, &rng);
    else
      orc_fasthals_step(x, d, n, k, a, b, c->normalize_a, &rng);
    t->update_seconds += now_s() - t0;
    t->iterations_run = iter;
    if (iter % c->error_interval == 0 || iter == c->max_iterations) { /* 262-283 */
      const double err = orc_reconstruction_error(x, d, n, a, b, k);
      if (!isfinite(err)) {
        t->status = ORC_ABORTED;
        snprintf(t->message, sizeof t->message, "non-finite objective at iteration %zu", iter);
        break;
      }
      push_record(t, iter, err, t->update_seconds);
      const int converged = previous == 0.0 ? err == 0.0
                                            : fabs(previous - err) / previous < c->rel_tolerance;
      if (converged) {
        t->status = ORC_CONVERGED;
        snprintf(t->message, sizeof t->message,
                 "relative error decrease below tolerance at iteration %zu", iter);
        break;
      }
      previous = err;
    }
  }
  t->gini_b = orc_gini(b, n * k); /* 286-291 */
  free(left); free(right); free(xhat); free(xcheck); free(a_hat); free(b_check);
  return ORC_OK;
}

/* ======================================================================
 * Synthetic data for the BASELINE.json configs.  Not part of the reference
 * (its own generator, data_io.cpp:383-415, is a different model).  The
 * product's device generator (csrc/synth.cu) implements the same counter
 * streams; tests feed the bytes produced here to both sides, so the two need
 * not agree bitwise (transcendentals may differ by an ulp).
 *
 *   u(stream, i)  = (splitmix64(key(seed, stream) + i) >> 11) * 2^-53
 *   W0 (d x r)    stream 1, H0 (r x n) stream 2, noise stream 3 (pairs 2i, 2i+1),
 *   Gamma draws   stream 4/5 (64 sub-draws per entry), Poisson stream 6.
 *   X = round_fp32( sum_r W0[i,r] * H0[r,j]  (fp64, r ascending, no FMA)
 *                   + sigma * |N(0,1)| )      or Poisson(lambda = W0 H0)
 * ==================================================================== */
static uint64_t splitmix64(uint64_t z) {
  z += 0x9E3779B97F4A7C15ULL;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}
static uint64_t synth_key(uint64_t seed, uint64_t stream) {
  return splitmix64(seed ^ splitmix64(stream * 0xD1B54A32D192ED03ULL));
}
static double synth_u(uint64_t key, uint64_t index) {
  return (double)(splitmix64(key + index) >> 11) * 0x1.0p-53;
}
static double synth_normal(uint64_t key, uint64_t pair) {
  const double u1 = 1.0 - synth_u(key, 2 * pair); /* (0, 1] */
  const double u2 = synth_u(key, 2 * pair + 1);
  return sqrt(-2.0 * log(u1)) * cos(6.283185307179586 * u2);
}
/* Marsaglia-Tsang with the shape<1 boost: G(a) = G(a+1) * U^(1/a). */
static double synth_gamma(uint64_t key, uint64_t index, double shape) {
  const double a = shape < 1.0 ? shape + 1.0 : shape;
  const double dd = a - 1.0 / 3.0, cc = 1.0 / sqrt(9.0 * dd);
  const uint64_t base = index * 64;
  double g = dd;
  for (uint64_t t = 0; t < 20; ++t) {
    const double z = synth_normal(key, base + 3 * t);
    const double v0 = 1.0 + cc * z;
    if (v0 <= 0.0) continue;
    const double v = v0 * v0 * v0;
    const double u = 1.0 - synth_u(key, 2 * (base + 3 * t + 1));
    if (log(u) < 0.5 * z * z + dd - dd * v + dd * log(v)) {
      g = dd * v;
      break;
    }
  }
  if (shape < 1.0) g *= pow(1.0 - synth_u(key, 2 * (base + 63)), 1.0 / shape);
  return g;
}
/* Poisson(lambda): Knuth product below 30, PTRS (Hormann 1993) above. */
static double synth_poisson(uint64_t key, uint64_t index, double lam) {
  const uint64_t base = index * 256;
  if (lam <= 0.0) return 0.0;
  if (lam < 30.0) {
    const double lim = exp(-lam);
    double p = 1.0;
    uint64_t k = 0;
    for (;;) {
      p *= 1.0 - synth_u(key, base + k);
      if (p <= lim || k >= 255) break;
      ++k;
    }
    return (double)k;
  }
  const double slam = sqrt(lam), loglam = log(lam);
  const double b = 0.931 + 2.53 * slam, a = -0.059 + 0.02483 * b;
  const double invalpha = 1.1239 + 1.1328 / (b - 3.4), vr = 0.9277 - 3.6224 / (b - 2);
  for (uint64_t t = 0; t < 127; ++t) {
    const double u = synth_u(key, base + 2 * t) - 0.5;
    const double v = 1.0 - synth_u(key, base + 2 * t + 1);
    const double us = 0.5 - fabs(u);
    const double kk = floor((2 * a / us + b) * u + lam + 0.43);
    if (us >= 0.07 && v <= vr) return kk;
    if (kk < 0 || (us < 0.013 && v > us)) continue;
    if (log(v) + log(invalpha) - log(a / (us * us) + b) <= -lam + kk * loglam - lgamma(kk + 1))
      return kk;
  }
  return floor(lam + 0.5);
}

/* factor_kind: 0 Uniform[0,1), 1 Exponential(1), 2 Gamma(0.3, 1). */
double orc_synth_factor_entry(uint64_t seed, uint64_t stream, uint64_t index, int kind) {
  const uint64_t key = synth_key(seed, stream);
  if (kind == 0) return synth_u(key, index);
  if (kind == 1) return -log(1.0 - synth_u(key, index));
  return synth_gamma(synth_key(seed, stream + 3), index, 0.3);
}

/* Rows [row_lo, row_hi) and columns [col_lo, col_hi) of the global d x n
 * matrix into xf (fp32, ld ldx, zero in the padding columns) or, when xf is
 * NULL, into xd (fp64 holding the same fp32-rounded values).  Entries depend
 * only on their global (i, j), so any blocking gives the same bytes.
 * noise_kind 0: none, 1: sigma|N|, 2: Poisson(W0 H0). */
void orc_synth_x_block(size_t d, size_t n, size_t rank, int factor_kind, int noise_kind,
                       double sigma, uint64_t seed, size_t row_lo, size_t row_hi,
                       size_t col_lo, size_t col_hi, size_t ldx, float* xf, double* xd) {
  const size_t nc = col_hi - col_lo;
  double* w0 = dalloc((row_hi - row_lo) * rank);
  double* h0 = dalloc(rank * nc);
  (void)d;
  for (size_t i = row_lo; i < row_hi; ++i)
    for (size_t r = 0; r < rank; ++r)
      w0[(i - row_lo) * rank + r] = orc_synth_factor_entry(seed, 1, i * rank + r, factor_kind);
  for (size_t r = 0; r < rank; ++r)
    for (size_t j = 0; j < nc; ++j)
      h0[r * nc + j] = orc_synth_factor_entry(seed, 2, r * n + col_lo + j, factor_kind);
  const uint64_t knoise = synth_key(seed, 3), kpois = synth_key(seed, 6);
  double* acc = dalloc(nc);
  for (size_t i = row_lo; i < row_hi; ++i) {
    for (size_t j = 0; j < nc; ++j) acc[j] = 0.0;
    for (size_t r = 0; r < rank; ++r) {
      const double w = w0[(i - row_lo) * rank + r];
      const double* hr = h0 + r * nc;
      for (size_t j = 0; j < nc; ++j) acc[j] = acc[j] + w * hr[j];
    }
    const size_t o = (i - row_lo) * ldx;
    for (size_t j = 0; j < nc; ++j) {
      const uint64_t gidx = (uint64_t)i * n + col_lo + j;
      double v = acc[j];
      if (noise_kind == 1) v = v + sigma * fabs(synth_normal(knoise, gidx));
      if (noise_kind == 2) v = synth_poisson(kpois, gidx, v);
      if (xf) xf[o + j] = (float)v;
      else xd[o + j] = (double)(float)v;
    }
    for (size_t j = nc; j < ldx; ++j) {
      if (xf) xf[o + j] = 0.0f;
      else xd[o + j] = 0.0;
    }
  }
  free(acc);
  free(w0);
  free(h0);
}

/* Fills x (d x ldx fp32, columns [col_lo, col_hi) of the global d x n
 * matrix), zero in the padding columns. */
void orc_synth_x(size_t d, size_t n, size_t rank, int factor_kind, int noise_kind,
                 double sigma, uint64_t seed, size_t col_lo, size_t col_hi, size_t ldx,
                 float* x) {
  orc_synth_x_block(d, n, rank, factor_kind, noise_kind, sigma, seed, 0, d, col_lo, col_hi,
                    ldx, x, NULL);
}
