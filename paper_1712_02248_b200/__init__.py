"""B200-native compressed NMF (FastHALS-RP) -- Python mirror of the reference API.

The product is the C-ABI library ``lib/libcnmf_b200.so`` (include/cnmf_b200.h):
CUDA kernels for sm_100a plus a C++ host.  This module binds it with ctypes
and mirrors the reference's interface for this path
(/root/reference/proj/include/cnmf/solvers.hpp, compression.hpp, metrics.hpp):

  SolverConfig, SketchConfig   <- cnmf::SolverConfig / SketchConfig
  run(x, config) -> RunResult  <- cnmf::run (solvers.hpp:104)
  ConfigError / DimensionError / InputError  <- errors.hpp:10-28

plus the step-level entry points (build_projectors, compress, ...) used by the
parity tests.  There is no CPU fallback: without the CUDA library or a GPU,
every compute call raises CudaError.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass, field
from typing import List, Optional

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "lib", "libcnmf_b200.so")
HEADER = os.path.join(os.path.dirname(HERE), "include", "cnmf_b200.h")

# cnmf::Algorithm (algorithm.hpp:8-15)
MU, MU_RP, HALS, HALS_RP, FASTHALS, FASTHALS_RP = range(6)
ALGORITHM_NAMES = {"mu": MU, "mu-rp": MU_RP, "hals": HALS, "hals-rp": HALS_RP,
                   "fasthals": FASTHALS, "fasthals-rp": FASTHALS_RP}
# cnmf::RunStatus (metrics.hpp:62-66)
CONVERGED, REACHED_MAX_ITERATIONS, ABORTED = range(3)
STATUS_NAMES = {CONVERGED: "converged", REACHED_MAX_ITERATIONS: "reached_max_iterations",
                ABORTED: "aborted"}


class CnmfError(Exception):
    pass


class ConfigError(CnmfError, ValueError):
    """cnmf::ConfigError (std::invalid_argument)."""


class DimensionError(CnmfError, ValueError):
    """cnmf::DimensionError (std::invalid_argument)."""


class InputError(CnmfError, ValueError):
    """cnmf::InputError (std::invalid_argument)."""


class IoError(CnmfError, RuntimeError):
    """cnmf::IoError (std::runtime_error): files that cannot be read or written."""


class ParseError(IoError):
    """cnmf::ParseError (an IoError): malformed input files."""


class CudaError(CnmfError, RuntimeError):
    """Device failure or no usable CUDA device (the product never falls back to the CPU)."""


class NcclError(CnmfError, RuntimeError):
    pass


class UnsupportedError(CnmfError, NotImplementedError):
    """Valid for the reference, outside this build's hot path."""


_ERRORS = {1: ConfigError, 2: DimensionError, 3: InputError, 4: CudaError, 5: NcclError,
           6: UnsupportedError}


class _Config(C.Structure):
    _fields_ = [("algorithm", C.c_int32), ("k", C.c_uint64), ("sketch_q", C.c_uint64),
                ("sketch_power_iterations", C.c_uint64), ("sketch_seed", C.c_uint64),
                ("alpha", C.c_double), ("beta", C.c_double), ("max_iterations", C.c_uint64),
                ("rel_tolerance", C.c_double), ("error_interval", C.c_uint64),
                ("seed", C.c_uint64), ("normalize_a", C.c_int32)]


class _Cost(C.Structure):
    _fields_ = [("algorithm", C.c_int32), ("d", C.c_uint64), ("n", C.c_uint64),
                ("k", C.c_uint64), ("q", C.c_uint64), ("flops_per_iteration", C.c_double),
                ("memory_floats", C.c_double)]


class _Record(C.Structure):
    _fields_ = [("iteration", C.c_uint64), ("error", C.c_double),
                ("elapsed_seconds", C.c_double), ("rng_draws", C.c_uint64)]


class _Trace(C.Structure):
    _fields_ = [("records", C.POINTER(_Record)), ("records_capacity", C.c_uint64),
                ("records_count", C.c_uint64), ("update_seconds", C.c_double),
                ("compress_seconds", C.c_double), ("error_seconds", C.c_double),
                ("gini_b", C.c_double), ("status", C.c_int32), ("iterations_run", C.c_uint64),
                ("power_iterations", C.c_uint64), ("alpha", C.c_double), ("beta", C.c_double),
                ("seed", C.c_uint64), ("estimate_flops_per_iteration", C.c_double),
                ("estimate_memory_floats", C.c_double), ("x_norm_sq", C.c_double),
                ("redraws", C.c_uint64), ("x_passes", C.c_uint64), ("message", C.c_char * 256),
                ("sketch_kappa", C.c_double), ("range_finder_fp64", C.c_int32)]


# Every exported symbol of include/cnmf_b200.h (checked by tests/test_abi.py).
EXPORTS = [
    "cnmf_abi_version", "cnmf_context_create", "cnmf_context_destroy",
    "cnmf_context_last_error", "cnmf_context_stream", "cnmf_solver_config_init",
    "cnmf_solver_config_validate", "cnmf_run", "cnmf_run_device", "cnmf_gaussian_sketch",
    "cnmf_initialize", "cnmf_powered_range_finder", "cnmf_build_projectors", "cnmf_compress",
    "cnmf_compress_factors", "cnmf_fasthals_rp_steps", "cnmf_reconstruction_error",
    "cnmf_thin_qr", "cnmf_xs_nn", "cnmf_xs_tn", "cnmf_xs_exact", "cnmf_synth_x", "cnmf_launch_count",
    "cnmf_time_xstream", "cnmf_time_xs_exact", "cnmf_shard_begin", "cnmf_nccl_unique_id", "cnmf_context_create_sharded",
    "cnmf_run_sharded_device", "cnmf_estimate_cost", "cnmf_generate_synthetic",
    "cnmf_pairwise_distortion", "cnmf_run_csr", "cnmf_context_create_hosted",
]


def build(force: bool = False) -> str:
    """Compile lib/libcnmf_b200.so for sm_100a (nvcc, no GPU needed)."""
    cmd = ["make", "-s", "-C", os.path.join(HERE, "csrc")]
    if force:
        subprocess.run(cmd + ["clean"], check=True)
    subprocess.run(cmd + ["-j8"], check=True)
    return LIB_PATH


_lib = None


def load_library(path: str = LIB_PATH):
    """Load the C-ABI library; raises CudaError when it is missing.
    CNMF_LIB overrides the path (kernel-variant experiments only)."""
    global _lib
    if _lib is not None:
        return _lib
    path = os.environ.get("CNMF_LIB", path)
    if not os.path.exists(path):
        raise CudaError(f"{path} is missing: build it with paper_1712_02248_b200.build()")
    L = C.CDLL(path)
    u64, vp, dp, fp = C.c_uint64, C.c_void_p, C.POINTER(C.c_double), C.c_void_p
    L.cnmf_abi_version.restype = C.c_int
    L.cnmf_context_create.argtypes = [C.c_int, C.POINTER(vp)]
    L.cnmf_context_destroy.argtypes = [vp]
    L.cnmf_context_destroy.restype = None
    L.cnmf_context_last_error.argtypes = [vp]
    L.cnmf_context_last_error.restype = C.c_char_p
    L.cnmf_context_stream.argtypes = [vp]
    L.cnmf_context_stream.restype = vp
    L.cnmf_solver_config_init.argtypes = [C.POINTER(_Config)]
    L.cnmf_solver_config_init.restype = None
    L.cnmf_solver_config_validate.argtypes = [C.POINTER(_Config), u64, u64, C.c_char_p,
                                              C.c_size_t]
    L.cnmf_run.argtypes = [vp, fp, u64, u64, u64, C.POINTER(_Config), fp, fp, C.POINTER(_Trace)]
    L.cnmf_run_device.argtypes = L.cnmf_run.argtypes
    L.cnmf_gaussian_sketch.argtypes = [vp, u64, u64, u64, fp]
    L.cnmf_initialize.argtypes = [vp, u64, u64, u64, u64, fp, fp]
    L.cnmf_powered_range_finder.argtypes = [vp, fp, u64, u64, u64, u64, u64, u64, C.c_int, fp]
    L.cnmf_build_projectors.argtypes = [vp, fp, u64, u64, u64, u64, u64, u64, fp, fp]
    L.cnmf_compress.argtypes = [vp, fp, u64, u64, u64, fp, fp, u64, fp, fp]
    L.cnmf_compress_factors.argtypes = [vp, fp, fp, fp, fp, u64, u64, u64, u64, vp, vp]
    L.cnmf_fasthals_rp_steps.argtypes = [vp, fp, fp, fp, fp, u64, u64, u64, u64, fp, fp, vp, vp,
                                         C.c_int, C.c_double, C.c_double, u64, u64,
                                         C.POINTER(u64)]
    L.cnmf_reconstruction_error.argtypes = [vp, fp, u64, u64, u64, fp, fp, u64, dp]
    L.cnmf_thin_qr.argtypes = [vp, fp, u64, u64, fp]
    L.cnmf_xs_nn.argtypes = [vp, fp, u64, u64, u64, fp, u64, fp]
    L.cnmf_xs_tn.argtypes = [vp, fp, u64, u64, u64, fp, u64, fp]
    L.cnmf_xs_exact.argtypes = [vp, fp, u64, u64, u64, fp, u64, C.c_int, C.c_int, vp]
    L.cnmf_synth_x.argtypes = [vp, u64, u64, u64, C.c_int, C.c_int, C.c_double, u64, u64, u64,
                               u64, fp]
    L.cnmf_launch_count.restype = u64
    L.cnmf_time_xstream.argtypes = [vp, fp, u64, u64, u64, u64, C.c_int, C.c_int, dp]
    L.cnmf_time_xs_exact.argtypes = [vp, fp, u64, u64, u64, u64, C.c_int, C.c_int, dp, C.POINTER(C.c_int)]
    L.cnmf_shard_begin.argtypes = [u64, C.c_int, C.c_int]
    L.cnmf_shard_begin.restype = u64
    L.cnmf_nccl_unique_id.argtypes = [C.c_char_p]
    L.cnmf_context_create_sharded.argtypes = [C.c_int, C.c_int, C.c_int, C.c_char_p, C.POINTER(vp)]
    L.cnmf_context_create_hosted.argtypes = [C.c_int, C.c_int, C.c_int, C.POINTER(_HostColl),
                                             C.POINTER(vp)]
    L.cnmf_run_sharded_device.argtypes = [vp, fp, u64, u64, u64, u64, u64, C.POINTER(_Config), fp,
                                          fp, C.POINTER(_Trace)]
    L.cnmf_run_csr.argtypes = [vp, vp, vp, vp, u64, u64, C.POINTER(_Config), fp, fp,
                               C.POINTER(_Trace)]
    L.cnmf_estimate_cost.argtypes = [C.c_int, u64, u64, u64, u64, C.POINTER(_Cost), C.c_char_p,
                                     C.c_size_t]
    L.cnmf_generate_synthetic.argtypes = [u64, u64, u64, C.c_double, C.c_double, u64, vp,
                                          C.c_char_p, C.c_size_t]
    L.cnmf_pairwise_distortion.argtypes = [vp, u64, u64, vp, u64, u64, u64, dp, dp, C.c_char_p,
                                           C.c_size_t]
    if L.cnmf_abi_version() != 3:
        raise CudaError("libcnmf_b200.so ABI version mismatch")
    _lib = L
    return L


@dataclass
class SketchConfig:
    """cnmf::SketchConfig (compression.hpp:13-17)."""
    q: int = 0
    power_iterations: int = 4
    seed: int = 1


@dataclass
class SolverConfig:
    """cnmf::SolverConfig (solvers.hpp:13-29); defaults as the reference."""
    algorithm: int = FASTHALS
    k: int = 2
    sketch: SketchConfig = field(default_factory=SketchConfig)
    alpha: float = 0.0
    beta: float = 0.0
    max_iterations: int = 200
    rel_tolerance: float = 1e-9
    error_interval: int = 5
    seed: int = 1
    normalize_a: bool = True

    def _c(self) -> _Config:
        algo = ALGORITHM_NAMES[self.algorithm] if isinstance(self.algorithm, str) else self.algorithm
        return _Config(int(algo), self.k, self.sketch.q, self.sketch.power_iterations,
                       self.sketch.seed, self.alpha, self.beta, self.max_iterations,
                       self.rel_tolerance, self.error_interval, self.seed,
                       int(bool(self.normalize_a)))

    def validate(self, d: int, n: int) -> None:
        """SolverConfig::validate (solvers.cpp:298-312); pure host logic."""
        L = load_library()
        msg = C.create_string_buffer(256)
        cfg = self._c()
        st = L.cnmf_solver_config_validate(C.byref(cfg), d, n, msg, 256)
        if st:
            raise _ERRORS.get(st, CnmfError)(msg.value.decode())


@dataclass
class RunRecord:
    iteration: int
    error: float
    elapsed_seconds: float
    rng_draws: int = 0  # raw draws the redraws took from the run Rng so far


@dataclass
class RunTrace:
    """cnmf::RunTrace (metrics.hpp:70-84) plus device timing."""
    records: List[RunRecord]
    update_seconds: float
    compress_seconds: float
    error_seconds: float
    gini_b: float
    status: int
    iterations_run: int
    power_iterations: int
    alpha: float
    beta: float
    seed: int
    estimate_flops_per_iteration: float
    estimate_memory_floats: float
    x_norm_sq: float
    redraws: int
    x_passes: int
    message: str
    sketch_kappa: float = 0.0       # condition estimate that chose the range finder's arithmetic
    range_finder_fp64: int = 0      # 1: the range finder ran in fp64

    @property
    def status_name(self) -> str:
        return STATUS_NAMES[self.status]


@dataclass
class RunResult:
    """cnmf::RunResult (solvers.hpp:94-97): factors (A d x k, B n x k) + trace."""
    a: np.ndarray
    b: np.ndarray
    trace: RunTrace


def _ptr(t) -> int:
    """Raw pointer of a numpy array or a torch tensor (device pointers for CUDA tensors)."""
    if isinstance(t, np.ndarray):
        return t.ctypes.data
    return t.data_ptr()


def _check_device_operands(x, a, b, d, n, k):
    """X (d x n) and the factor outputs A (d x k), B (n x k) as the C ABI reads
    them: fp32 CUDA tensors, unit column stride, contiguous factors.  Also
    orders the library's stream after torch's current stream: X or the
    outputs may have been produced by torch work still in flight."""
    import torch
    for name, t, shape in (("x", x, (d, n)), ("a_out", a, (d, k)), ("b_out", b, (n, k))):
        if not (isinstance(t, torch.Tensor) and t.is_cuda and t.dtype == torch.float32):
            raise DimensionError(f"{name} must be a float32 CUDA tensor")
        if tuple(t.shape) != shape or (t.dim() == 2 and shape[1] > 1 and t.stride(1) != 1):
            raise DimensionError(f"{name} must be {shape[0]} x {shape[1]} with unit column stride")
        if t.device != x.device:
            raise DimensionError(f"{name} is on {t.device}, X on {x.device}")
    if not (a.is_contiguous() and b.is_contiguous()):
        raise DimensionError("a_out and b_out must be contiguous")
    if x.stride(0) < n:
        raise DimensionError("x row stride is shorter than its width")
    torch.cuda.current_stream(x.device).synchronize()


def _torch_ready():
    """The library computes on its own (non-blocking) stream: inputs produced by
    torch on its current stream must be complete before a device-pointer call
    reads them (include/cnmf_b200.h, "Streams")."""
    import torch
    if torch.cuda.is_available():
        torch.cuda.current_stream().synchronize()


class Context:
    """One CUDA device + stream (cnmf_context)."""

    def __init__(self, device: int = 0):
        self.L = load_library()
        h = C.c_void_p()
        st = self.L.cnmf_context_create(device, C.byref(h))
        if st:
            raise _ERRORS.get(st, CnmfError)(f"cannot create a context on CUDA device {device}")
        self.h = h

    def close(self):
        if getattr(self, "h", None):
            self.L.cnmf_context_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _check(self, st: int):
        if st:
            raise _ERRORS.get(st, CnmfError)(self.L.cnmf_context_last_error(self.h).decode())

    def stream(self) -> int:
        return self.L.cnmf_context_stream(self.h)

    # ---- run() -------------------------------------------------------------
    def _trace(self, cap: int):
        recs = (_Record * cap)()
        tr = _Trace()
        tr.records = C.cast(recs, C.POINTER(_Record))
        tr.records_capacity = cap
        return recs, tr

    @staticmethod
    def _result_trace(recs, tr) -> RunTrace:
        n = min(tr.records_count, tr.records_capacity)
        return RunTrace([RunRecord(recs[i].iteration, recs[i].error, recs[i].elapsed_seconds,
                                   recs[i].rng_draws)
                         for i in range(n)], tr.update_seconds, tr.compress_seconds,
                        tr.error_seconds, tr.gini_b, tr.status, tr.iterations_run,
                        tr.power_iterations, tr.alpha, tr.beta, tr.seed,
                        tr.estimate_flops_per_iteration, tr.estimate_memory_floats,
                        tr.x_norm_sq, tr.redraws, tr.x_passes, tr.message.decode(),
                        tr.sketch_kappa, tr.range_finder_fp64)

    def run(self, x, config: SolverConfig) -> RunResult:
        """cnmf::run with X in host memory (numpy, float32, row-major)."""
        x = np.ascontiguousarray(x, dtype=np.float32)
        d, n = x.shape
        cfg = config._c()
        recs, tr = self._trace(config.max_iterations + 2)
        a = np.empty((d, config.k), dtype=np.float32)
        b = np.empty((n, config.k), dtype=np.float32)
        self._check(self.L.cnmf_run(self.h, _ptr(x), d, n, n, C.byref(cfg), _ptr(a), _ptr(b),
                                    C.byref(tr)))
        return RunResult(a, b, self._result_trace(recs, tr))

    def run_sparse(self, x, config: SolverConfig) -> RunResult:
        """cnmf::run(const SparseMatrix&, ...) with X in host CSR form: a
        scipy.sparse matrix or a (indptr, indices, data, (d, n)) tuple."""
        if isinstance(x, tuple):
            indptr, indices, data, (d, n) = x
        else:
            csr = x.tocsr()
            csr.sort_indices()
            indptr, indices, data = csr.indptr, csr.indices, csr.data
            d, n = csr.shape
        indptr = np.ascontiguousarray(indptr, dtype=np.uint64)
        indices = np.ascontiguousarray(indices, dtype=np.uint64)
        data = np.ascontiguousarray(data, dtype=np.float32)
        if indptr.shape[0] != d + 1:
            raise DimensionError("sparse matrix: row_offsets size must be rows + 1")
        if indptr[-1] != data.shape[0] or indices.shape[0] != data.shape[0]:
            raise DimensionError("sparse matrix: index/value arrays disagree")
        cfg = config._c()
        recs, tr = self._trace(config.max_iterations + 2)
        a = np.empty((d, config.k), dtype=np.float32)
        b = np.empty((n, config.k), dtype=np.float32)
        self._check(self.L.cnmf_run_csr(self.h, _ptr(indptr), _ptr(indices), _ptr(data), d, n,
                                        C.byref(cfg), _ptr(a), _ptr(b), C.byref(tr)))
        return RunResult(a, b, self._result_trace(recs, tr))

    def run_device(self, x, config: SolverConfig, a_out=None, b_out=None):
        """cnmf::run with X already resident on the device (torch CUDA tensor)."""
        import torch
        d, n = x.shape
        ldx = x.stride(0)
        a = a_out if a_out is not None else torch.empty((d, config.k), device=x.device)
        b = b_out if b_out is not None else torch.empty((n, config.k), device=x.device)
        _check_device_operands(x, a, b, d, n, config.k)
        cfg = config._c()
        recs, tr = self._trace(config.max_iterations + 2)
        self._check(self.L.cnmf_run_device(self.h, _ptr(x), d, n, ldx, C.byref(cfg), _ptr(a),
                                           _ptr(b), C.byref(tr)))
        return a, b, self._result_trace(recs, tr)

    # ---- step level (torch CUDA tensors) -------------------------------------
    def gaussian_sketch(self, rows, cols, seed, out):
        _torch_ready()
        self._check(self.L.cnmf_gaussian_sketch(self.h, rows, cols, seed, _ptr(out)))
        return out

    def initialize(self, d, n, k, seed, a, b):
        _torch_ready()
        self._check(self.L.cnmf_initialize(self.h, d, n, k, seed, _ptr(a), _ptr(b)))
        return a, b

    def powered_range_finder(self, x, q, w, seed, transpose, out):
        _torch_ready()
        d, n = x.shape
        self._check(self.L.cnmf_powered_range_finder(self.h, _ptr(x), d, n, x.stride(0), q, w,
                                                     seed, int(transpose), _ptr(out)))
        return out

    def build_projectors(self, x, q, w, seed, left, right):
        _torch_ready()
        d, n = x.shape
        self._check(self.L.cnmf_build_projectors(self.h, _ptr(x), d, n, x.stride(0), q, w, seed,
                                                 _ptr(left), _ptr(right)))
        return left, right

    def compress(self, x, left, right, xhat, xcheck):
        _torch_ready()
        d, n = x.shape
        q = left.shape[1]
        self._check(self.L.cnmf_compress(self.h, _ptr(x), d, n, x.stride(0), _ptr(left),
                                         _ptr(right), q, _ptr(xhat), _ptr(xcheck)))
        return xhat, xcheck

    def compress_factors(self, a, b, left, right, a_hat, b_check):
        _torch_ready()
        d, k = a.shape
        n = b.shape[0]
        q = left.shape[1]
        self._check(self.L.cnmf_compress_factors(self.h, _ptr(a), _ptr(b), _ptr(left),
                                                 _ptr(right), d, n, q, k, _ptr(a_hat),
                                                 _ptr(b_check)))
        return a_hat, b_check

    def fasthals_rp_steps(self, xhat, xcheck, left, right, a, b, a_hat, b_check,
                          normalize_a=True, alpha=0.0, beta=0.0, rng_seed=1, steps=1) -> int:
        _torch_ready()
        d, k = a.shape
        n = b.shape[0]
        q = left.shape[1]
        red = C.c_uint64()
        self._check(self.L.cnmf_fasthals_rp_steps(self.h, _ptr(xhat), _ptr(xcheck), _ptr(left),
                                                  _ptr(right), d, n, q, k, _ptr(a), _ptr(b),
                                                  _ptr(a_hat), _ptr(b_check), int(normalize_a),
                                                  alpha, beta, rng_seed, steps, C.byref(red)))
        return red.value

    def reconstruction_error(self, x, a, b) -> float:
        _torch_ready()
        d, n = x.shape
        out = C.c_double()
        self._check(self.L.cnmf_reconstruction_error(self.h, _ptr(x), d, n, x.stride(0), _ptr(a),
                                                     _ptr(b), a.shape[1], C.byref(out)))
        return out.value

    def thin_qr(self, y, out):
        _torch_ready()
        self._check(self.L.cnmf_thin_qr(self.h, _ptr(y), y.shape[0], y.shape[1], _ptr(out)))
        return out

    def xs_nn(self, x, s, out):
        _torch_ready()
        d, n = x.shape
        self._check(self.L.cnmf_xs_nn(self.h, _ptr(x), d, n, x.stride(0), _ptr(s), s.shape[1],
                                      _ptr(out)))
        return out

    def xs_tn(self, x, t, out):
        _torch_ready()
        d, n = x.shape
        self._check(self.L.cnmf_xs_tn(self.h, _ptr(x), d, n, x.stride(0), _ptr(t), t.shape[1],
                                      _ptr(out)))
        return out

    def xs_exact(self, x, s, out, transpose=False, dmma=False, small_int=False):
        """out (float64) = X s or X^T s with fp64-grade accumulation: the int8-sliced
        tensor-core kernel (small_int: its configuration for an X of integers below
        8192), or the FP64 tensor-core kernel (dmma=True)."""
        _torch_ready()
        d, n = x.shape
        self._check(self.L.cnmf_xs_exact(self.h, _ptr(x), d, n, x.stride(0), _ptr(s), s.shape[1],
                                         int(transpose), 1 if dmma else (2 if small_int else 0),
                                         _ptr(out)))
        return out

    def time_xstream(self, x, l, transpose, iters=10) -> float:
        _torch_ready()
        d, n = x.shape
        out = C.c_double()
        self._check(self.L.cnmf_time_xstream(self.h, _ptr(x), d, n, x.stride(0), l,
                                             int(transpose), iters, C.byref(out)))
        return out.value

    def time_xs_exact(self, x, l, transpose, iters=5):
        """(seconds per exact-accumulation contraction, reads of X it makes)."""
        _torch_ready()
        d, n = x.shape
        out, passes = C.c_double(), C.c_int()
        self._check(self.L.cnmf_time_xs_exact(self.h, _ptr(x), d, n, x.stride(0), l, int(transpose),
                                              iters, C.byref(out), C.byref(passes)))
        return out.value, passes.value

    def synth_x(self, d, n, rank, factor_kind, noise_kind, sigma, seed, out, col_lo=0,
                col_hi=None):
        _torch_ready()
        col_hi = n if col_hi is None else col_hi
        self._check(self.L.cnmf_synth_x(self.h, d, n, rank, factor_kind, noise_kind, sigma, seed,
                                        col_lo, col_hi, out.stride(0), _ptr(out)))
        return out


_default_ctx: Optional[Context] = None



def shard_begin(n: int, rank: int, world: int) -> int:
    """First column of rank's shard: floor(n * rank / world) (host-only, no GPU)."""
    return int(load_library().cnmf_shard_begin(n, rank, world))


def shard_range(n: int, rank: int, world: int):
    return shard_begin(n, rank, world), shard_begin(n, rank + 1, world)


class ShardedContext(Context):
    """cnmf_context of one rank of a column-sharded run (NCCL communicator).

    from_process_group() builds it on every rank of an initialised
    torch.distributed group: rank 0 draws the NCCL unique id and broadcasts it.
    """

    def __init__(self, device: int, rank: int, world: int, unique_id: bytes):
        self.L = load_library()
        h = C.c_void_p()
        st = self.L.cnmf_context_create_sharded(device, rank, world, bytes(unique_id), C.byref(h))
        if st:
            raise _ERRORS.get(st, CnmfError)(f"cannot create sharded context (rank {rank}/{world})")
        self.h = h
        self.rank, self.world = rank, world

    @staticmethod
    def unique_id() -> bytes:
        buf = C.create_string_buffer(128)
        st = load_library().cnmf_nccl_unique_id(buf)
        if st:
            raise _ERRORS.get(st, CnmfError)("ncclGetUniqueId failed")
        return buf.raw

    @classmethod
    def from_process_group(cls, device: int):
        import torch.distributed as dist
        rank, world = dist.get_rank(), dist.get_world_size()
        obj = [cls.unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        return cls(device, rank, world, obj[0])

    def run_sharded(self, x_shard, n: int, config: SolverConfig, a_out=None, b_out=None):
        """Collective cnmf::run on this rank's columns of a d x n X (torch CUDA
        tensor d x n_local, the columns [shard_begin(n, rank), shard_begin(n, rank+1)))."""
        import torch
        d, nloc = x_shard.shape
        lo = shard_begin(n, self.rank, self.world)
        a = a_out if a_out is not None else torch.empty((d, config.k), device=x_shard.device)
        b = b_out if b_out is not None else torch.empty((nloc, config.k), device=x_shard.device)
        _check_device_operands(x_shard, a, b, d, nloc, config.k)
        cfg = config._c()
        recs, tr = self._trace(config.max_iterations + 2)
        self._check(self.L.cnmf_run_sharded_device(self.h, _ptr(x_shard), d, n, lo, nloc,
                                                   x_shard.stride(0), C.byref(cfg), _ptr(a), _ptr(b),
                                                   C.byref(tr)))
        return a, b, self._result_trace(recs, tr)

_AllreduceFn = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_uint64, C.c_int, C.c_int, C.c_void_p)
_AllgatherFn = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_void_p, C.c_uint64, C.c_void_p)


class _HostColl(C.Structure):
    _fields_ = [("allreduce", _AllreduceFn), ("allgather", _AllgatherFn), ("user", C.c_void_p)]


class HostedShardedContext(ShardedContext):
    """A rank of a column-sharded run whose collectives are host-staged
    through torch.distributed (cnmf_context_create_hosted) instead of NCCL --
    e.g. a gloo group of two processes sharing ONE GPU, where NCCL cannot run
    (tests).  Same kernels, same run_sharded_impl as the NCCL context."""

    def __init__(self, device: int, group=None):
        import torch
        import torch.distributed as dist
        self.L = load_library()
        rank, world = dist.get_rank(group), dist.get_world_size(group)

        def allreduce(buf, count, dtype, op, _user):
            try:
                ct = C.c_double if dtype == 1 else C.c_float
                arr = np.ctypeslib.as_array(C.cast(buf, C.POINTER(ct)), shape=(count,))
                t = torch.from_numpy(arr)
                dist.all_reduce(t, op=dist.ReduceOp.MAX if op else dist.ReduceOp.SUM,
                                group=group)
                return 0
            except Exception:  # noqa: BLE001 -- reported to the library as a failure
                return 1

        def allgather(send, recv, nbytes, _user):
            try:
                src = torch.from_numpy(np.ctypeslib.as_array(
                    C.cast(send, C.POINTER(C.c_uint8)), shape=(nbytes,)).copy())
                parts = [torch.empty(nbytes, dtype=torch.uint8) for _ in range(world)]
                dist.all_gather(parts, src, group=group)
                dst = np.ctypeslib.as_array(C.cast(recv, C.POINTER(C.c_uint8)),
                                            shape=(nbytes * world,))
                for g, part in enumerate(parts):
                    dst[g * nbytes:(g + 1) * nbytes] = part.numpy()
                return 0
            except Exception:  # noqa: BLE001
                return 1

        self._cb = _HostColl(_AllreduceFn(allreduce), _AllgatherFn(allgather), None)
        h = C.c_void_p()
        st = self.L.cnmf_context_create_hosted(device, rank, world, C.byref(self._cb), C.byref(h))
        if st:
            raise _ERRORS.get(st, CnmfError)(f"cannot create hosted context (rank {rank}/{world})")
        self.h = h
        self.rank, self.world = rank, world


# ---- host-side data formats around the path (no device) --------------------
def _host_check(st: int, msg) -> None:
    if st:
        raise _ERRORS.get(st, CnmfError)(msg.value.decode())


@dataclass
class CostEstimate:
    """cnmf::CostEstimate (metrics.hpp:15-23)."""
    algorithm: int
    d: int
    n: int
    k: int
    q: int
    flops_per_iteration: float
    memory_floats: float


def estimate_cost(algorithm, d: int, n: int, k: int, q: int) -> CostEstimate:
    """cnmf::estimate_cost (metrics.cpp:20-50)."""
    algo = ALGORITHM_NAMES[algorithm] if isinstance(algorithm, str) else int(algorithm)
    out, msg = _Cost(), C.create_string_buffer(256)
    _host_check(load_library().cnmf_estimate_cost(algo, d, n, k, q, C.byref(out), msg, 256), msg)
    return CostEstimate(out.algorithm, out.d, out.n, out.k, out.q, out.flops_per_iteration,
                        out.memory_floats)


def generate_synthetic(d: int, n: int, true_rank: int = 1, decay_p: float = 0.0,
                       noise_level: float = 0.0, seed: int = 1) -> np.ndarray:
    """cnmf::generate_synthetic (data_io.cpp:383-415): d x n float64, bitwise the reference's."""
    d, n = int(d), int(n)
    out = np.empty((max(d, 0), max(n, 0)), dtype=np.float64)
    msg = C.create_string_buffer(256)
    _host_check(load_library().cnmf_generate_synthetic(d, n, true_rank, decay_p, noise_level,
                                                       seed, out.ctypes.data, msg, 256), msg)
    return out


def pairwise_distortion(x: np.ndarray, xhat: np.ndarray, sample_pairs: int, seed: int):
    """cnmf::pairwise_distortion (metrics.cpp:123-155) with the projected
    columns L^T X given as xhat (q x n, the cnmf_compress output).
    Returns (max_relative, mean_relative)."""
    x = np.ascontiguousarray(x, dtype=np.float64)
    xhat = np.ascontiguousarray(xhat, dtype=np.float32)
    d, n = x.shape
    if xhat.shape[1] != n:
        raise DimensionError("pairwise_distortion: projector rows must match data rows")
    mx, mean = C.c_double(), C.c_double()
    msg = C.create_string_buffer(256)
    _host_check(load_library().cnmf_pairwise_distortion(
        x.ctypes.data, d, n, xhat.ctypes.data, xhat.shape[0], sample_pairs, seed, C.byref(mx),
        C.byref(mean), msg, 256), msg)
    return mx.value, mean.value


def launch_count() -> int:
    """Device kernels launched by the library so far (this process)."""
    return int(load_library().cnmf_launch_count())


def default_context() -> Context:
    global _default_ctx
    if _default_ctx is None:
        _default_ctx = Context(0)
    return _default_ctx


def run(x, config: SolverConfig) -> RunResult:
    """cnmf::run(x, config) (solvers.hpp:104) on the default CUDA device."""
    return default_context().run(x, config)


# BASELINE.json configurations (synthetic stand-ins).
CONFIGS = {
    "c1": dict(d=1000, n=1000, rank=20, factor_kind=0, noise_kind=1, sigma=0.01, k=20, q=30,
               w=2, iters=100),
    "c2": dict(d=10000, n=5000, rank=16, factor_kind=1, noise_kind=1, sigma=0.05, k=16, q=36,
               w=2, iters=200),
    "c3": dict(d=100000, n=20000, rank=50, factor_kind=0, noise_kind=1, sigma=0.01, k=50, q=70,
               w=2, iters=100),
    "c4": dict(d=50000, n=100000, rank=100, factor_kind=2, noise_kind=2, sigma=0.0, k=100,
               q=120, w=1, iters=100),
    "c5": dict(d=200000, n=500000, rank=64, factor_kind=0, noise_kind=1, sigma=0.01, k=64, q=84,
               w=1, iters=50),
}
