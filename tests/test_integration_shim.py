"""The reference-side binding (integration/shim_cnmf_b200.cpp) compiled against
the reference's OWN public headers (/root/reference/proj/include) and linked
with libcnmf_b200.so, exercised through the reference's API (cnmf::run,
SolverConfig::validate) by integration/shim_driver.cpp.

CPU: every invalid configuration throws cnmf::ConfigError with the message of
SolverConfig::validate (solvers.cpp:298-312), before any device work; a valid
run on a machine without a GPU throws std::runtime_error (no CPU fallback).
GPU: a fasthals-rp run through the shim matches the compiled reference's own
run (per-record relative error within 1e-4).

The driver is built by `make -C integration` (from __graft_entry__.build()
where /root/reference exists) and travels to the GPU box prebuilt.
"""
import os
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
DRIVER = os.path.join(ROOT, "integration", "build", "shim_driver")
REF_SOLVERS = "/root/reference/proj/src/solvers.cpp"

# solvers.cpp:298-312, in the order shim_driver.cpp triggers them
MESSAGES = [
    "k must satisfy 1 <= k <= min(d, n)",
    "compressed algorithms require k < q <= min(d, n)",
    "alpha and beta must be finite and non-negative",
    "error_interval must be positive",
    "rel_tolerance must be positive and finite",
    "penalties are supported by hals-rp and fasthals-rp only",
]


@pytest.fixture(scope="module")
def driver():
    if os.path.isdir("/root/reference/proj/include"):
        subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "integration")], check=True)
    if not os.path.exists(DRIVER):
        pytest.skip("integration/build/shim_driver not built (needs the reference headers)")
    return DRIVER


def _has_gpu():
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


def test_messages_are_the_references():
    if not os.path.exists(REF_SOLVERS):
        pytest.skip("reference sources not present")
    text = open(REF_SOLVERS).read()
    for m in MESSAGES:
        assert f'throw ConfigError("{m}")' in text, m


def test_shim_config_errors_and_no_cpu_fallback(driver):
    out = subprocess.run([driver, "config"], capture_output=True, text=True, timeout=120,
                         check=True).stdout.strip().splitlines()
    assert len(out) == len(MESSAGES) + 1, out
    for line, m in zip(out, MESSAGES):
        assert line == f"ConfigError|{m}", line
    if _has_gpu():
        assert out[-1] == "ok|", out[-1]
    else:
        assert out[-1].startswith("runtime_error|cnmf_b200:"), out[-1]


@pytest.mark.gpu
def test_shim_run_matches_reference(driver, oracle, tmp_path):
    d, n, k, q, w, iters, every, seed = 300, 200, 6, 12, 1, 30, 5, 1
    x = oracle.synth_x(d, n, k, 0, 1, 0.01, 5).astype(np.float32)
    path = tmp_path / "x.f32"
    x.tofile(path)
    out = subprocess.run([driver, "run", str(path), str(d), str(n), str(k), str(q), str(w),
                          str(iters), str(every), str(seed)],
                         capture_output=True, text=True, timeout=300, check=True).stdout
    lines = out.strip().splitlines()
    assert not lines[0].startswith(("runtime_error", "invalid_argument")), lines[0]
    recs = [(int(l.split()[1]), float(l.split()[2])) for l in lines if l.startswith("rec ")]
    _, _, t = oracle.run(x.astype(np.float64), k, q=q, w=w, sketch_seed=seed, max_iterations=iters,
                         error_interval=every, rel_tolerance=1e-300)
    xn = float(np.sum(x.astype(np.float64) ** 2))
    assert [r[0] for r in recs] == list(range(0, iters + 1, every))
    got = np.sqrt(2.0 * np.array([r[1] for r in recs]) / xn)
    want = np.sqrt(2.0 * np.array(t.errors) / xn)
    assert np.max(np.abs(got - want) / want) < 1e-4
    status = [l for l in lines if l.startswith("status ")][0].split()
    assert int(status[1]) == 1 and int(status[2]) == iters  # reached_max_iterations
