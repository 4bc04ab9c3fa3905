"""Parity of the streaming FastHALS-RP kernel (csrc/hals.cu) on the paths the
shared-memory-resident kernel serves at the small parity sizes: forced with
CNMF_HALS=stream, against the CPU oracle (the restatement of
proj/src/solvers.cpp:414-509, pinned to the compiled reference in
tests/test_oracle.py).

  * redraw halts inside a sweep block (k = 12 and k = 40, every column
    emptied): the kernel resumes at unaligned columns and the sweeps start
    from an aligned block with the already-updated columns skipped;
  * k = 100 (several 16-column blocks, 128-wide views);
  * penalised B updates (solvers.cpp:502-508) with k > 8;
  * A heights above 768 rows per SM (d = 120000 on 148 SMs): the 6-rows-per-
    thread instance of the A sweep (BASELINE configs[4] height class).

Tolerances as tests/test_gpu_parity.py: factors within
1e-3 relative Frobenius, trajectories within 1e-4 relative.
"""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

TRAJ_RTOL = 1e-4
FACTOR_RTOL = 1e-3


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.float32)).cuda()


def dev64(a):
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64)).cuda()


def host(t):
    return t.detach().cpu().numpy().astype(np.float64)


def rel_fro(a, b):
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


@pytest.fixture
def stream(monkeypatch):
    monkeypatch.setenv("CNMF_HALS", "stream")


def _fixture(oracle, d, n, k, q, w, data_seed, init_seed, sketch_seed, rank=None):
    x = oracle.synth_x(d, n, rank or min(k, 10), 0, 1, 0.01, data_seed).astype(np.float64)
    left, right = oracle.build_projectors(x, q, w, sketch_seed)
    xhat, xcheck = oracle.compress(x, left, right)
    a, b = oracle.initialize(d, n, k, init_seed)
    ah, bc = oracle.compress_factors(a, b, left, right)
    return x, left, right, xhat, xcheck, a, b, ah, bc


def test_streaming_steps_k20(ctx, oracle, stream):
    """Plain steps with k = 20: three column blocks, the last one partial."""
    _, left, right, xhat, xcheck, a, b, ah, bc = _fixture(oracle, 700, 500, 20, 28, 1, 3, 4, 5)
    ta, tb, tah, tbc = dev(a), dev(b), dev64(ah), dev64(bc)
    ctx.fasthals_rp_steps(dev(xhat), dev(xcheck), dev(left), dev(right), ta, tb, tah, tbc,
                          True, 0.0, 0.0, 31, 6)
    rng = oracle.rng(31)
    for _ in range(6):
        oracle.fasthals_rp_step(xhat, xcheck, a, b, ah, bc, left, right, True, 0.0, 0.0, rng)
    for got, want in ((ta, a), (tb, b), (tah, ah), (tbc, bc)):
        assert rel_fro(host(got), want) < FACTOR_RTOL


def test_streaming_emptied_columns_unaligned_resume(ctx, oracle, stream):
    """Zero compressed views with k = 12: every A and B column empties and is
    redrawn, so the kernel halts and resumes at columns 1..11 (inside the
    sweep blocks) in both halves (solvers.cpp:435, 452)."""
    x = oracle.synth_x(300, 200, 4, 0, 1, 0.01, 8).astype(np.float64)
    left, right = oracle.build_projectors(x, 14, 1, 2)
    xhat, xcheck = np.zeros((14, 200)), np.zeros((300, 14))
    a, b = oracle.initialize(300, 200, 12, 4)
    ah, bc = oracle.compress_factors(a, b, left, right)
    ta, tb, tah, tbc = dev(a), dev(b), dev64(ah), dev64(bc)
    redraws = ctx.fasthals_rp_steps(dev(xhat), dev(xcheck), dev(left), dev(right), ta, tb, tah,
                                    tbc, True, 0.0, 0.0, 77, 2)
    rng = oracle.rng(77)
    for _ in range(2):
        oracle.fasthals_rp_step(xhat, xcheck, a, b, ah, bc, left, right, True, 0.0, 0.0, rng)
    assert redraws >= 24
    for got, want in ((ta, a), (tb, b), (tbc, bc)):
        assert rel_fro(host(got), want) < FACTOR_RTOL


def test_streaming_emptied_columns_many_blocks(ctx, oracle, stream):
    """k = 40 (three 16-column sweep blocks, the last partial) with zero
    views: every column of both halves empties and is redrawn, so the kernel
    resumes at every in-block position of every block."""
    x = oracle.synth_x(500, 400, 6, 0, 1, 0.01, 9).astype(np.float64)
    left, right = oracle.build_projectors(x, 44, 1, 3)
    xhat, xcheck = np.zeros((44, 400)), np.zeros((500, 44))
    a, b = oracle.initialize(500, 400, 40, 6)
    ah, bc = oracle.compress_factors(a, b, left, right)
    ta, tb, tah, tbc = dev(a), dev(b), dev64(ah), dev64(bc)
    redraws = ctx.fasthals_rp_steps(dev(xhat), dev(xcheck), dev(left), dev(right), ta, tb, tah,
                                    tbc, True, 0.0, 0.0, 13, 1)
    rng = oracle.rng(13)
    oracle.fasthals_rp_step(xhat, xcheck, a, b, ah, bc, left, right, True, 0.0, 0.0, rng)
    assert redraws >= 80
    for got, want in ((ta, a), (tb, b), (tbc, bc)):
        assert rel_fro(host(got), want) < FACTOR_RTOL


def test_streaming_steps_k100(ctx, oracle, stream):
    """k = 100, l = 110 (the C4 class: seven 16-column blocks, 128-wide
    views) -- plain steps against the oracle."""
    _, left, right, xhat, xcheck, a, b, ah, bc = _fixture(oracle, 900, 700, 100, 110, 1, 2, 3, 4,
                                                          rank=20)
    ta, tb, tah, tbc = dev(a), dev(b), dev64(ah), dev64(bc)
    ctx.fasthals_rp_steps(dev(xhat), dev(xcheck), dev(left), dev(right), ta, tb, tah, tbc,
                          True, 0.0, 0.0, 8, 3)
    rng = oracle.rng(8)
    for _ in range(3):
        oracle.fasthals_rp_step(xhat, xcheck, a, b, ah, bc, left, right, True, 0.0, 0.0, rng)
    for got, want in ((ta, a), (tb, b), (tah, ah), (tbc, bc)):
        assert rel_fro(host(got), want) < FACTOR_RTOL


@pytest.mark.parametrize("alpha,beta", [(0.2, 0.7), (1e6, 0.0)])
def test_streaming_penalized_steps(ctx, oracle, stream, alpha, beta):
    """alpha / beta B updates with k = 10; alpha = 1e6 clamps every b_j to zero
    each sweep (the B-half rollback and redraw path)."""
    _, left, right, xhat, xcheck, a, b, ah, bc = _fixture(oracle, 400, 300, 10, 16, 1, 6, 7, 8)
    ta, tb, tah, tbc = dev(a), dev(b), dev64(ah), dev64(bc)
    ctx.fasthals_rp_steps(dev(xhat), dev(xcheck), dev(left), dev(right), ta, tb, tah, tbc,
                          True, alpha, beta, 5, 3)
    rng = oracle.rng(5)
    for _ in range(3):
        oracle.fasthals_rp_step(xhat, xcheck, a, b, ah, bc, left, right, True, alpha, beta, rng)
    assert rel_fro(host(ta), a) < FACTOR_RTOL
    assert rel_fro(host(tb), b) < FACTOR_RTOL


def test_tall_a_six_rows_per_thread(ctx, oracle):
    """d = 120000 (811 A rows per SM on 148 SMs, > 3 x 256): the 6-rows-per-
    thread A sweep, through the full run, against the oracle's run."""
    import paper_1712_02248_b200 as cb
    d, n, k, q = 120000, 48, 6, 10
    x = oracle.synth_x(d, n, 5, 0, 1, 0.01, 12)
    cfg = cb.SolverConfig(algorithm=cb.FASTHALS_RP, k=k, sketch=cb.SketchConfig(q, 1, 1),
                          max_iterations=6, error_interval=1, rel_tolerance=1e-300, seed=1)
    res = ctx.run(x, cfg)
    ra, rb, rt = oracle.run(x.astype(np.float64), k, q=q, w=1, sketch_seed=1, max_iterations=6,
                            error_interval=1, rel_tolerance=1e-300, seed=1)
    xn = float(np.sum(x.astype(np.float64) ** 2))
    got = np.sqrt(2.0 * np.array([r.error for r in res.trace.records]) / xn)
    want = np.sqrt(2.0 * np.array(rt.errors) / xn)
    assert got.shape == want.shape
    assert np.max(np.abs(got - want) / want) < TRAJ_RTOL
    assert rel_fro(res.a, ra) < FACTOR_RTOL and rel_fro(res.b, rb) < FACTOR_RTOL
