"""CPU tests of the C-ABI library: it loads, exports every symbol that
include/cnmf_b200.h declares, validates configurations like
SolverConfig::validate, and fails loudly (no CPU fallback) without a GPU."""
import ctypes as C
import os
import re

import pytest

import paper_1712_02248_b200 as cb


@pytest.fixture(scope="module")
def lib():
    if not os.path.exists(cb.LIB_PATH):
        cb.build()
    return cb.load_library()


def header_symbols():
    text = open(cb.HEADER).read()
    return sorted(set(re.findall(r"\b(cnmf_[a-z_0-9]+)\s*\(", text)))


def test_exports_every_header_symbol(lib):
    syms = header_symbols()
    assert len(syms) >= 20
    assert sorted(cb.EXPORTS) == syms
    for s in syms:
        assert hasattr(lib, s), s
    assert lib.cnmf_abi_version() == 3


def test_config_defaults_match_reference(lib):
    cfg = cb._Config()
    lib.cnmf_solver_config_init(C.byref(cfg))
    # solvers.hpp:13-23, compression.hpp:13-17
    assert cfg.algorithm == cb.FASTHALS and cfg.k == 2 and cfg.max_iterations == 200
    assert cfg.rel_tolerance == 1e-9 and cfg.error_interval == 5 and cfg.seed == 1
    assert cfg.normalize_a == 1 and cfg.sketch_power_iterations == 4 and cfg.sketch_seed == 1
    d = cb.SolverConfig()
    assert (d.k, d.max_iterations, d.error_interval, d.sketch.power_iterations) == (2, 200, 5, 4)


def test_validation_mirrors_reference(lib):
    """test_solvers.cpp:76-115."""
    c = cb.SolverConfig(k=3)
    c.validate(10, 8)
    for k in (0, 9):
        with pytest.raises(cb.ConfigError):
            cb.SolverConfig(k=k).validate(10, 8)
    c = cb.SolverConfig(algorithm=cb.HALS_RP, k=3, sketch=cb.SketchConfig(q=3))
    with pytest.raises(cb.ConfigError):
        c.validate(10, 8)
    c.sketch.q = 9
    with pytest.raises(cb.ConfigError):
        c.validate(10, 8)
    c.sketch.q = 6
    c.validate(10, 8)
    c.alpha = -0.5
    with pytest.raises(cb.ConfigError):
        c.validate(10, 8)
    c.alpha = float("inf")
    with pytest.raises(cb.ConfigError):
        c.validate(10, 8)
    c.alpha = 0.1
    c.validate(10, 8)
    c.algorithm = cb.FASTHALS
    with pytest.raises(cb.ConfigError, match="penalties"):
        c.validate(10, 8)
    c.alpha, c.beta = 0.0, 0.2
    with pytest.raises(cb.ConfigError):
        c.validate(10, 8)
    c.beta = 0.0
    c.error_interval = 0
    with pytest.raises(cb.ConfigError, match="error_interval"):
        c.validate(10, 8)
    c.error_interval = 5
    c.rel_tolerance = 0.0
    with pytest.raises(cb.ConfigError, match="rel_tolerance"):
        c.validate(10, 8)


def test_no_cpu_fallback_without_gpu(lib):
    try:
        import torch
        has_gpu = torch.cuda.is_available()
    except Exception:
        has_gpu = False
    if has_gpu:
        pytest.skip("a GPU is present")
    with pytest.raises(cb.CudaError):
        cb.Context(0)
