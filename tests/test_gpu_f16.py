"""The X-stream kernel's opt-in fp16 hi/lo path (csrc/xstream_tc.cu,
kind::f16 MMAs with exact power-of-two row / column scalings, CNMF_XS=f16).
Same bars as tests/test_gpu_parity.py: contractions within 1e-5 relative
Frobenius of fp64, the C1 trajectory within 1e-4 relative of the oracle's.
(The C2 trajectory lands 4.6e-4 from the reference's golden one with this
path -- outside the bar -- which is why production keeps 3xTF32; see
DESIGN.md section 3.1.)"""
import os

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

TRAJ_RTOL = 1e-4
FACTOR_RTOL = 1e-3


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.float32)).cuda()


def host(t):
    return t.detach().cpu().numpy().astype(np.float64)


def rel_fro(a, b):
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


def rel_err(err, xnorm):
    return np.sqrt(2.0 * np.asarray(err, dtype=np.float64) / xnorm)


@pytest.fixture
def f16(monkeypatch):
    monkeypatch.setenv("CNMF_XS", "f16")


@pytest.mark.parametrize("d,n,l", [(1000, 1000, 30), (333, 517, 17), (64, 4096, 128),
                                   (5000, 37, 8), (3000, 2000, 70)])
def test_f16_contractions(ctx, f16, d, n, l):
    rng = np.random.default_rng(d * 7 + n)
    x = rng.random((d, n), dtype=np.float32)
    s = rng.standard_normal((n, l)).astype(np.float32)
    y = torch.empty((d, l), device="cuda")
    ctx.xs_nn(dev(x), dev(s), y)
    assert rel_fro(host(y), x.astype(np.float64) @ s.astype(np.float64)) < 1e-5


def test_f16_rows_of_very_different_magnitude(ctx, f16):
    """Per-row scaling: rows 1e-12 .. 1e12 apart keep fp32-grade relative
    accuracy row by row (a global scale would flush the small rows)."""
    rng = np.random.default_rng(3)
    x = rng.random((512, 700), dtype=np.float32)
    x *= np.float32(10.0) ** rng.integers(-12, 13, size=(512, 1)).astype(np.float32)
    s = rng.standard_normal((700, 40)).astype(np.float32)
    y = torch.empty((512, 40), device="cuda")
    ctx.xs_nn(dev(x), dev(s), y)
    ref = x.astype(np.float64) @ s.astype(np.float64)
    got = host(y)
    rows = np.linalg.norm(got - ref, axis=1) / np.linalg.norm(ref, axis=1)
    assert rows.max() < 1e-5


def test_f16_run_c1_trajectory(ctx, oracle, f16):
    import paper_1712_02248_b200 as cb
    x = oracle.synth_x(1000, 1000, 20, 0, 1, 0.01, 1)
    cfg = cb.SolverConfig(algorithm=cb.FASTHALS_RP, k=20, sketch=cb.SketchConfig(30, 2, 1),
                          max_iterations=100, error_interval=1, rel_tolerance=1e-300, seed=1)
    res = ctx.run(x, cfg)
    ra, rb, rt = oracle.run(x.astype(np.float64), 20, q=30, w=2, sketch_seed=1, max_iterations=100,
                            error_interval=1, rel_tolerance=1e-300, seed=1)
    xn = float(np.sum(x.astype(np.float64) ** 2))
    got = rel_err([r.error for r in res.trace.records], xn)
    want = rel_err(rt.errors, xn)
    assert np.max(np.abs(got - want) / want) < TRAJ_RTOL
    assert rel_fro(res.a, ra) < FACTOR_RTOL and rel_fro(res.b, rb) < FACTOR_RTOL
