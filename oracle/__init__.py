"""ctypes bindings for the CPU oracle (TEST INFRASTRUCTURE ONLY).

`Oracle` wraps oracle/build/liboracle.so, the plain-C restatement of the
reference hot path (oracle/cnmf_oracle.c).  `Reference` wraps
oracle/_ref/libcnmf_ref.so, the reference library itself compiled from its
own sources by oracle/Makefile.  Only tests/, __graft_entry__.smoke() and
bench.py's CPU-baseline legs import this package; the product never does.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass, field

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "build", "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libcnmf_ref.so")

_dp = C.POINTER(C.c_double)
_fp = C.POINTER(C.c_float)
_sz = C.c_size_t
_u64 = C.c_uint64


def _d(a: np.ndarray):
    assert a.dtype == np.float64 and a.flags.c_contiguous
    return a.ctypes.data_as(_dp)


def build(ref: bool = False) -> None:
    """Build the oracle (and, when /root/reference exists, oracle/_ref)."""
    subprocess.run(["make", "-s", "-C", HERE], check=True)
    if ref and os.path.isdir("/root/reference/proj"):
        subprocess.run(["make", "-s", "-C", HERE, "ref"], check=True)


class OracleError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"[{code}] {msg}")
        self.code = code


@dataclass
class Trace:
    iterations: list = field(default_factory=list)
    errors: list = field(default_factory=list)
    elapsed: list = field(default_factory=list)
    update_seconds: float = 0.0
    compress_seconds: float = 0.0
    gini_b: float = float("nan")
    status: int = 1
    iterations_run: int = 0
    message: str = ""


class _OrcConfig(C.Structure):
    _fields_ = [("algorithm", C.c_int), ("k", _sz), ("q", _sz), ("power_iterations", _sz),
                ("sketch_seed", _u64), ("alpha", C.c_double), ("beta", C.c_double),
                ("max_iterations", _sz), ("rel_tolerance", C.c_double),
                ("error_interval", _sz), ("seed", _u64), ("normalize_a", C.c_int)]


class _OrcTrace(C.Structure):
    _fields_ = [("rec_iter", C.POINTER(_sz)), ("rec_error", _dp), ("rec_elapsed", _dp),
                ("rec_capacity", _sz), ("rec_count", _sz), ("update_seconds", C.c_double),
                ("compress_seconds", C.c_double), ("gini_b", C.c_double), ("status", C.c_int),
                ("iterations_run", _sz), ("message", C.c_char * 256)]


FASTHALS = 4
FASTHALS_RP = 5


class Oracle:
    """The C restatement (oracle/cnmf_oracle.c)."""

    def __init__(self, path: str = ORACLE_SO):
        if not os.path.exists(path):
            build()
        self.lib = L = C.CDLL(path)
        L.orc_last_message.restype = C.c_char_p
        L.orc_rng_sizeof.restype = _sz
        L.orc_rng_next.restype = _u64
        for f in ("orc_rng_uniform", "orc_rng_uniform_positive", "orc_rng_normal",
                  "orc_reconstruction_error", "orc_gini", "orc_frobenius_norm_sq",
                  "orc_synth_factor_entry"):
            getattr(L, f).restype = C.c_double
        L.orc_reconstruction_error.argtypes = [_dp, _sz, _sz, _dp, _dp, _sz]
        L.orc_gini.argtypes = [_dp, _sz]
        L.orc_synth_factor_entry.argtypes = [_u64, _u64, _u64, C.c_int]
        L.orc_synth_x.argtypes = [_sz, _sz, _sz, C.c_int, C.c_int, C.c_double, _u64, _sz, _sz,
                                  _sz, _fp]
        L.orc_gaussian_sketch.argtypes = [_sz, _sz, _u64, _dp]
        L.orc_initialize.argtypes = [_sz, _sz, _sz, _u64, _dp, _dp]
        L.orc_matmul.argtypes = [_dp, _sz, _sz, _dp, _sz, _sz, C.c_int, C.c_int, _dp]
        L.orc_thin_qr.argtypes = [_dp, _sz, _sz, _dp, _dp]
        L.orc_range_finder.argtypes = [_dp, _sz, _sz, C.c_int, _sz, _sz, _u64, _dp]
        L.orc_build_projectors.argtypes = [_dp, _sz, _sz, _sz, _sz, _u64, _dp, _dp]
        L.orc_compress_left.argtypes = [_dp, _sz, _sz, _dp, _sz, _dp]
        L.orc_compress_right.argtypes = [_dp, _sz, _sz, _dp, _sz, _dp]
        L.orc_compress_factor_a.argtypes = [_dp, _sz, _sz, _dp, _sz, _dp]
        L.orc_compress_factor_b.argtypes = [_dp, _sz, _sz, _dp, _sz, _dp]
        L.orc_fasthals_rp_step.argtypes = [_dp, _dp, _sz, _sz, _sz, _sz, _dp, _dp, _dp, _dp,
                                           _dp, _dp, C.c_int, C.c_double, C.c_double,
                                           C.c_void_p]
        L.orc_fasthals_step.argtypes = [_dp, _sz, _sz, _sz, _dp, _dp, C.c_int, C.c_void_p]
        L.orc_b_update_fasthals_rp.argtypes = [_dp, _sz, _sz, _dp, _dp, _sz, C.c_double,
                                               C.c_double, _dp]
        L.orc_run.argtypes = [_dp, _sz, _sz, C.POINTER(_OrcConfig), _dp, _dp,
                              C.POINTER(_OrcTrace)]
        L.orc_validate.argtypes = [C.POINTER(_OrcConfig), _sz, _sz]

    # -- rng -------------------------------------------------------------
    def rng(self, seed: int):
        buf = C.create_string_buffer(self.lib.orc_rng_sizeof())
        self.lib.orc_rng_init(buf, _u64(seed))
        return buf

    def draws(self, seed: int, kind: int, count: int) -> np.ndarray:
        r = self.rng(seed)
        f = [self.lib.orc_rng_next, self.lib.orc_rng_uniform, self.lib.orc_rng_uniform_positive,
             self.lib.orc_rng_normal][kind]
        if kind == 0:
            return np.array([f(r) for _ in range(count)], dtype=np.uint64)
        return np.array([f(r) for _ in range(count)], dtype=np.float64)

    def _check(self, st: int):
        if st:
            raise OracleError(st, self.lib.orc_last_message().decode())

    # -- linalg / compression -------------------------------------------
    def gaussian_sketch(self, rows, cols, seed):
        out = np.empty((rows, cols))
        self.lib.orc_gaussian_sketch(rows, cols, _u64(seed), _d(out))
        return out

    def initialize(self, d, n, k, seed):
        a, b = np.empty((d, k)), np.empty((n, k))
        self.lib.orc_initialize(d, n, k, _u64(seed), _d(a), _d(b))
        return a, b

    def matmul(self, m, n, tl=False, tr=False):
        m = np.ascontiguousarray(m, dtype=np.float64)
        n = np.ascontiguousarray(n, dtype=np.float64)
        r = m.shape[1] if tl else m.shape[0]
        c = n.shape[0] if tr else n.shape[1]
        out = np.empty((r, c))
        self._check(self.lib.orc_matmul(_d(m), m.shape[0], m.shape[1], _d(n), n.shape[0],
                                        n.shape[1], int(tl), int(tr), _d(out)))
        return out

    def thin_qr(self, m):
        m = np.ascontiguousarray(m, dtype=np.float64)
        q, r = np.empty_like(m), np.empty((m.shape[1], m.shape[1]))
        self._check(self.lib.orc_thin_qr(_d(m), m.shape[0], m.shape[1], _d(q), _d(r)))
        return q, r

    def range_finder(self, x, q, w, seed, transpose=False):
        x = np.ascontiguousarray(x, dtype=np.float64)
        out = np.empty((x.shape[1] if transpose else x.shape[0], q))
        self._check(self.lib.orc_range_finder(_d(x), x.shape[0], x.shape[1], int(transpose), q,
                                              w, _u64(seed), _d(out)))
        return out

    def build_projectors(self, x, q, w, seed):
        x = np.ascontiguousarray(x, dtype=np.float64)
        d, n = x.shape
        left, right = np.empty((d, q)), np.empty((q, n))
        self._check(self.lib.orc_build_projectors(_d(x), d, n, q, w, _u64(seed), _d(left),
                                                  _d(right)))
        return left, right

    def compress(self, x, left, right):
        x = np.ascontiguousarray(x, dtype=np.float64)
        d, n = x.shape
        q = left.shape[1]
        xhat, xcheck = np.empty((q, n)), np.empty((d, q))
        self.lib.orc_compress_left(_d(x), d, n, _d(left), q, _d(xhat))
        self.lib.orc_compress_right(_d(x), d, n, _d(right), q, _d(xcheck))
        return xhat, xcheck

    def compress_factors(self, a, b, left, right):
        q = left.shape[1]
        ah, bc = np.empty((q, a.shape[1])), np.empty((q, b.shape[1]))
        self.lib.orc_compress_factor_a(_d(a), a.shape[0], a.shape[1], _d(left), q, _d(ah))
        self.lib.orc_compress_factor_b(_d(b), b.shape[0], b.shape[1], _d(right), q, _d(bc))
        return ah, bc

    def fasthals_rp_step(self, xhat, xcheck, a, b, a_hat, b_check, left, right,
                         normalize_a=True, alpha=0.0, beta=0.0, rng=None):
        d, k = a.shape
        n = b.shape[0]
        q = left.shape[1]
        self.lib.orc_fasthals_rp_step(_d(xhat), _d(xcheck), d, n, q, k, _d(a), _d(b),
                                      _d(a_hat), _d(b_check), _d(left), _d(right),
                                      int(normalize_a), alpha, beta, rng)

    def fasthals_step(self, x, a, b, normalize_a=True, rng=None):
        x = np.ascontiguousarray(x, dtype=np.float64)
        self.lib.orc_fasthals_step(_d(x), x.shape[0], x.shape[1], a.shape[1], _d(a), _d(b),
                                   int(normalize_a), rng)

    def b_update(self, b, p, w, j, alpha, beta):
        out = np.empty(b.shape[0])
        self.lib.orc_b_update_fasthals_rp(_d(b), b.shape[0], b.shape[1], _d(p), _d(w), j,
                                          alpha, beta, _d(out))
        return out

    def reconstruction_error(self, x, a, b):
        x = np.ascontiguousarray(x, dtype=np.float64)
        return self.lib.orc_reconstruction_error(_d(x), x.shape[0], x.shape[1], _d(a), _d(b),
                                                 a.shape[1])

    def gini(self, v):
        v = np.ascontiguousarray(v, dtype=np.float64).ravel()
        return self.lib.orc_gini(_d(v), v.size)

    # -- driver ---------------------------------------------------------
    def run(self, x, k, q=0, w=4, sketch_seed=1, alpha=0.0, beta=0.0, max_iterations=200,
            rel_tolerance=1e-9, error_interval=5, seed=1, normalize_a=True,
            algorithm=FASTHALS_RP):
        x = np.ascontiguousarray(x, dtype=np.float64)
        d, n = x.shape
        cfg = _OrcConfig(algorithm, k, q, w, sketch_seed, alpha, beta, max_iterations,
                         rel_tolerance, error_interval, seed, int(normalize_a))
        cap = max_iterations + 2
        it = (_sz * cap)()
        er, el = np.zeros(cap), np.zeros(cap)
        tr = _OrcTrace(it, _d(er), _d(el), cap, 0, 0.0, 0.0, 0.0, 1, 0, b"")
        a, b = np.empty((d, k)), np.empty((n, k))
        self._check(self.lib.orc_run(_d(x), d, n, C.byref(cfg), _d(a), _d(b), C.byref(tr)))
        c = tr.rec_count
        t = Trace(list(it[:c]), er[:c].tolist(), el[:c].tolist(), tr.update_seconds,
                  tr.compress_seconds, tr.gini_b, tr.status, tr.iterations_run,
                  tr.message.decode())
        return a, b, t

    # -- synthetic data ---------------------------------------------------
    def synth_x(self, d, n, rank, factor_kind, noise_kind, sigma, seed, col_lo=0, col_hi=None,
                ldx=None):
        col_hi = n if col_hi is None else col_hi
        ldx = (col_hi - col_lo) if ldx is None else ldx
        x = np.empty((d, ldx), dtype=np.float32)
        self.lib.orc_synth_x(d, n, rank, factor_kind, noise_kind, sigma, _u64(seed), col_lo,
                             col_hi, ldx, x.ctypes.data_as(_fp))
        return x


class Reference:
    """The reference library itself (oracle/_ref/libcnmf_ref.so)."""

    def __init__(self, path: str = REF_SO):
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} missing: run `make -C oracle ref` where "
                                    "/root/reference is mounted")
        self.lib = L = C.CDLL(path)
        L.ref_last_message.restype = C.c_char_p
        L.ref_reconstruction_error.restype = C.c_double
        L.ref_reconstruction_error.argtypes = [_dp, _sz, _sz, _dp, _dp, _sz]
        L.ref_rng_draws.argtypes = [_u64, C.c_int, _sz, _dp]
        L.ref_gaussian_sketch.argtypes = [_sz, _sz, _u64, _dp]
        L.ref_initialize.argtypes = [_sz, _sz, _sz, _u64, _dp, _dp]
        L.ref_matmul.argtypes = [_dp, _sz, _sz, _dp, _sz, _sz, C.c_int, C.c_int, _dp]
        L.ref_thin_qr.argtypes = [_dp, _sz, _sz, _dp, _dp]
        L.ref_set_csr.argtypes = [_sz, _sz, C.c_void_p, C.c_void_p, _dp]
        L.ref_pairwise_distortion.argtypes = [_dp, _sz, _sz, _dp, _sz, _sz, _u64, _dp, _dp]
        L.ref_generate_synthetic.argtypes = [_sz, _sz, _sz, C.c_double, C.c_double, _u64, _dp]
        L.ref_powered_range_finder.argtypes = [_dp, _sz, _sz, _sz, _sz, _u64, _dp]
        L.ref_build_projectors.argtypes = [_dp, _sz, _sz, _sz, _sz, _u64, _dp, _dp]
        L.ref_compress.argtypes = [_dp, _sz, _sz, _sz, _sz, _u64, _dp, _dp, _dp, _dp, _dp]
        L.ref_fasthals_rp_steps.argtypes = [_dp, _dp, _dp, _dp, _sz, _sz, _sz, _sz, _dp, _dp,
                                            _dp, _dp, C.c_int, C.c_double, C.c_double, _u64,
                                            _sz, _dp]
        L.ref_fasthals_steps.argtypes = [_dp, _sz, _sz, _sz, _dp, _dp, C.c_int, _u64, _sz]
        L.ref_run.argtypes = [_dp, _sz, _sz, C.c_int, _sz, _sz, _sz, _u64, C.c_double,
                              C.c_double, _sz, C.c_double, _sz, _u64, C.c_int, _dp, _dp,
                              C.POINTER(_sz), _dp, _dp, _sz, C.POINTER(_sz), _dp, _dp,
                              C.POINTER(C.c_int), C.POINTER(_sz), C.c_char_p, _sz]

    def _check(self, st: int):
        if st:
            raise OracleError(st, self.lib.ref_last_message().decode())

    def draws(self, seed, kind, count):
        out = np.empty(count)
        self.lib.ref_rng_draws(_u64(seed), kind, count, _d(out))
        return out.view(np.uint64) if kind == 0 else out

    def gaussian_sketch(self, rows, cols, seed):
        out = np.empty((rows, cols))
        self.lib.ref_gaussian_sketch(rows, cols, _u64(seed), _d(out))
        return out

    def pairwise_distortion(self, x, left, pairs, seed):
        x = np.ascontiguousarray(x, dtype=np.float64)
        left = np.ascontiguousarray(left, dtype=np.float64)
        mx, mean = np.zeros(1), np.zeros(1)
        self._check(self.lib.ref_pairwise_distortion(_d(x), x.shape[0], x.shape[1], _d(left),
                                                     left.shape[1], pairs, _u64(seed), _d(mx),
                                                     _d(mean)))
        return float(mx[0]), float(mean[0])

    def generate_synthetic(self, d, n, rank, decay, noise, seed):
        out = np.empty((d, n))
        self._check(self.lib.ref_generate_synthetic(d, n, rank, decay, noise, _u64(seed), _d(out)))
        return out

    def initialize(self, d, n, k, seed):
        a, b = np.empty((d, k)), np.empty((n, k))
        self.lib.ref_initialize(d, n, k, _u64(seed), _d(a), _d(b))
        return a, b

    def matmul(self, m, n, tl=False, tr=False):
        m = np.ascontiguousarray(m, dtype=np.float64)
        n = np.ascontiguousarray(n, dtype=np.float64)
        out = np.empty((m.shape[1] if tl else m.shape[0], n.shape[0] if tr else n.shape[1]))
        self._check(self.lib.ref_matmul(_d(m), m.shape[0], m.shape[1], _d(n), n.shape[0],
                                        n.shape[1], int(tl), int(tr), _d(out)))
        return out

    def thin_qr(self, m):
        m = np.ascontiguousarray(m, dtype=np.float64)
        q, r = np.empty_like(m), np.empty((m.shape[1], m.shape[1]))
        self._check(self.lib.ref_thin_qr(_d(m), m.shape[0], m.shape[1], _d(q), _d(r)))
        return q, r

    def powered_range_finder(self, x, q, w, seed):
        x = np.ascontiguousarray(x, dtype=np.float64)
        out = np.empty((x.shape[0], q))
        self._check(self.lib.ref_powered_range_finder(_d(x), x.shape[0], x.shape[1], q, w,
                                                      _u64(seed), _d(out)))
        return out

    def build_projectors(self, x, q, w, seed):
        x = np.ascontiguousarray(x, dtype=np.float64)
        d, n = x.shape
        left, right = np.empty((d, q)), np.empty((q, n))
        self._check(self.lib.ref_build_projectors(_d(x), d, n, q, w, _u64(seed), _d(left),
                                                  _d(right)))
        return left, right

    def compress(self, x, q, w, seed):
        """(left, right, xhat, xcheck, seconds) via build_projectors + compress_*."""
        x = np.ascontiguousarray(x, dtype=np.float64)
        d, n = x.shape
        left, right = np.empty((d, q)), np.empty((q, n))
        xhat, xcheck = np.empty((q, n)), np.empty((d, q))
        sec = C.c_double()
        self._check(self.lib.ref_compress(_d(x), d, n, q, w, _u64(seed), _d(left), _d(right),
                                          _d(xhat), _d(xcheck), C.byref(sec)))
        return left, right, xhat, xcheck, sec.value

    def fasthals_rp_steps(self, xhat, xcheck, left, right, a, b, a_hat, b_check, rng_seed,
                          steps, normalize_a=True, alpha=0.0, beta=0.0):
        d, k = a.shape
        n = b.shape[0]
        q = left.shape[1]
        sec = C.c_double()
        self._check(self.lib.ref_fasthals_rp_steps(_d(xhat), _d(xcheck), _d(left), _d(right), d,
                                                   n, q, k, _d(a), _d(b), _d(a_hat),
                                                   _d(b_check), int(normalize_a), alpha, beta,
                                                   _u64(rng_seed), steps, C.byref(sec)))
        return sec.value

    def fasthals_steps(self, x, a, b, rng_seed, steps, normalize_a=True):
        x = np.ascontiguousarray(x, dtype=np.float64)
        self._check(self.lib.ref_fasthals_steps(_d(x), x.shape[0], x.shape[1], a.shape[1],
                                                _d(a), _d(b), int(normalize_a), _u64(rng_seed),
                                                steps))

    def reconstruction_error(self, x, a, b):
        x = np.ascontiguousarray(x, dtype=np.float64)
        return self.lib.ref_reconstruction_error(_d(x), x.shape[0], x.shape[1], _d(a), _d(b),
                                                 a.shape[1])

    def run(self, x, k, q=0, w=4, sketch_seed=1, alpha=0.0, beta=0.0, max_iterations=200,
            rel_tolerance=1e-9, error_interval=5, seed=1, normalize_a=True,
            algorithm=FASTHALS_RP):
        xp = None
        if hasattr(x, "tocsr"):  # run(const SparseMatrix&, ...) (solvers.cpp:515-517)
            csr = x.tocsr()
            csr.sort_indices()
            d, n = csr.shape
            rp = np.ascontiguousarray(csr.indptr, dtype=np.uint64)
            ci = np.ascontiguousarray(csr.indices, dtype=np.uint64)
            vals = np.ascontiguousarray(csr.data, dtype=np.float64)
            self._check(self.lib.ref_set_csr(d, n, rp.ctypes.data, ci.ctypes.data, _d(vals)))
        else:
            x = np.ascontiguousarray(x, dtype=np.float64)
            d, n = x.shape
            xp = _d(x)
        cap = max_iterations + 2
        it = (_sz * cap)()
        er, el = np.zeros(cap), np.zeros(cap)
        cnt, iters = _sz(), _sz()
        upd, gini = C.c_double(), C.c_double()
        status = C.c_int()
        msg = C.create_string_buffer(256)
        a, b = np.empty((d, k)), np.empty((n, k))
        self._check(self.lib.ref_run(xp, d, n, algorithm, k, q, w, _u64(sketch_seed), alpha,
                                     beta, max_iterations, rel_tolerance, error_interval,
                                     _u64(seed), int(normalize_a), _d(a), _d(b), it, _d(er),
                                     _d(el), cap, C.byref(cnt), C.byref(upd), C.byref(gini),
                                     C.byref(status), C.byref(iters), msg, 256))
        c = cnt.value
        t = Trace(list(it[:c]), er[:c].tolist(), el[:c].tolist(), upd.value, 0.0, gini.value,
                  status.value, iters.value, msg.value.decode())
        return a, b, t
