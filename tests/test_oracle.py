"""CPU tests: pin the oracle (oracle/cnmf_oracle.c) before trusting it.

1. Against the committed golden fixtures (tests/golden/, generated from the
   reference itself by tests/golden/make_golden.py) -- runs anywhere.
2. Bit for bit against oracle/_ref (the reference compiled from its own
   sources) where that library has been built.
3. The reference's own property tests for this path, restated on the oracle
   (test_compression.cpp, test_solvers.cpp, acceptance.cpp checks 5/10).
"""
import os

import numpy as np
import pytest

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def load(name):
    return np.load(os.path.join(GOLDEN, name))


def x_summary(x):
    x = x.astype(np.float64)
    return np.array([x.sum(), (x * x).sum(), x[0, 0], x[-1, -1], x.max()])


# ------------------------------------------------------------ golden pins --
def test_streams_match_golden(oracle):
    g = load("streams.npz")
    for seed in (1, 2, 3, 5489):
        assert np.array_equal(oracle.draws(seed, 0, 64), g[f"u64_{seed}"])
    assert np.array_equal(oracle.draws(7, 1, 64), g["uniform_7"])
    assert np.array_equal(oracle.draws(1, 2, 64), g["uniform_positive_1"])
    assert np.array_equal(oracle.draws(2, 3, 65), g["normal_2"])
    assert np.array_equal(oracle.gaussian_sketch(7, 5, 11), g["sketch_7x5_11"])
    a, b = oracle.initialize(4, 3, 2, 99)
    assert np.array_equal(a, g["init_a_4x2_99"]) and np.array_equal(b, g["init_b_3x2_99"])


def test_mt19937_64_reference_value(oracle):
    # the C++ standard fixes the 10000th output of default-seeded mt19937_64
    r = oracle.rng(5489)
    for _ in range(9999):
        oracle.lib.orc_rng_next(r)
    assert oracle.lib.orc_rng_next(r) == 9981545732273789042


def test_small_cases_match_golden_bitwise(oracle):
    g = load("small.npz")
    x = oracle.synth_x(60, 45, 5, 0, 1, 0.01, 3).astype(np.float64)
    assert np.array_equal(x_summary(x), g["x_summary"])
    left, right = oracle.build_projectors(x, 10, 2, 4)
    assert np.array_equal(left, g["left"]) and np.array_equal(right, g["right"])
    q, r = oracle.thin_qr(x[:, :12])
    assert np.array_equal(q, g["qr_q"]) and np.array_equal(r, g["qr_r"])
    cases = {"rp": dict(k=4, q=10, w=2, max_iterations=50, error_interval=1,
                        rel_tolerance=1e-300, sketch_seed=4, seed=2),
             "rp_pen": dict(k=3, q=8, w=1, max_iterations=20, error_interval=3,
                            rel_tolerance=1e-300, alpha=0.05, beta=0.2, seed=6),
             "dense": dict(k=4, max_iterations=30, algorithm=4)}
    for tag, kw in cases.items():
        a, b, t = oracle.run(x, **kw)
        assert np.array_equal(a, g[f"{tag}_a"]), tag
        assert np.array_equal(b, g[f"{tag}_b"]), tag
        assert np.array_equal(np.array(t.iterations), g[f"{tag}_iters"]), tag
        assert np.array_equal(np.array(t.errors), g[f"{tag}_errors"]), tag
        assert t.gini_b == g[f"{tag}_gini"][0]
        assert [t.status, t.iterations_run] == list(g[f"{tag}_status"])


def test_zero_start_redraw_matches_golden(oracle):
    g = load("small.npz")
    xs = oracle.draws(9, 1, 144).reshape(12, 12)
    lz, rz = oracle.build_projectors(xs, 12, 0, 5)
    xh, xc = oracle.compress(xs, lz, rz)
    a, b = np.zeros((12, 2)), np.zeros((12, 2))
    ah, bc = oracle.compress_factors(a, b, lz, rz)
    oracle.fasthals_rp_step(xh, xc, a, b, ah, bc, lz, rz, True, 0.0, 0.0, oracle.rng(3))
    assert np.array_equal(a, g["zero_a"]) and np.array_equal(b, g["zero_b"])
    assert np.all(np.isfinite(a)) and np.all(a >= 0)


def test_c1_matches_golden(oracle):
    g = load("c1.npz")
    x = oracle.synth_x(1000, 1000, 20, 0, 1, 0.01, 1)
    assert np.array_equal(x_summary(x), g["x_summary"])
    a, b, t = oracle.run(x.astype(np.float64), 20, q=30, w=2, max_iterations=100,
                         error_interval=1, rel_tolerance=1e-300, sketch_seed=1, seed=1)
    assert np.array_equal(np.array(t.errors), g["errors"])
    assert np.array_equal(a.astype(np.float32), g["a"])
    assert np.array_equal(b.astype(np.float32), g["b"])


# ------------------------------------------------- bitwise vs reference --
def test_oracle_bitwise_vs_reference(oracle, reference):
    rng = np.random.default_rng(0)
    for d, n, q, w in [(30, 20, 5, 0), (40, 50, 8, 2), (17, 23, 17, 1)]:
        x = rng.random((d, n))
        for tl in (0, 1):
            for tr in (0, 1):
                m = rng.standard_normal((7, d) if tl else (d, 7))
                other = rng.standard_normal((9, 7) if tr else (7, 9))
                m[m < -1.0] = 0.0  # exercise the zero-skip branches
                assert np.array_equal(oracle.matmul(m, other, tl, tr),
                                      reference.matmul(m, other, tl, tr))
        lo, ro = oracle.build_projectors(x, q, w, 3)
        lr, rr = reference.build_projectors(x, q, w, 3)
        assert np.array_equal(lo, lr) and np.array_equal(ro, rr)
        a1, b1, t1 = oracle.run(x, 3, q=q, w=w, max_iterations=15, error_interval=2)
        a2, b2, t2 = reference.run(x, 3, q=q, w=w, max_iterations=15, error_interval=2)
        assert np.array_equal(a1, a2) and np.array_equal(b1, b2)
        assert t1.errors == t2.errors and t1.iterations == t2.iterations


# ------------------------------------ reference property tests (restated) --
def random_nonneg(oracle, d, n, seed):
    return oracle.draws(seed, 1, d * n).reshape(d, n)


def test_range_finder_orthonormal(oracle):
    x = random_nonneg(oracle, 20, 15, 3)
    for w in (0, 2):
        b = oracle.range_finder(x, 6, w, 7)
        assert np.abs(b.T @ b - np.eye(6)).max() < 1e-10  # test_compression.cpp:51-63


def test_projectors_orthonormal_and_deterministic(oracle):
    x = random_nonneg(oracle, 18, 14, 21)
    left, right = oracle.build_projectors(x, 5, 4, 4)
    assert np.abs(left.T @ left - np.eye(5)).max() < 1e-10
    assert np.abs(right @ right.T - np.eye(5)).max() < 1e-10
    l2, r2 = oracle.build_projectors(x, 5, 4, 4)
    assert np.array_equal(left, l2) and np.array_equal(right, r2)


def test_q_range_errors(oracle):
    from oracle import OracleError
    x = random_nonneg(oracle, 10, 8, 3)
    for q in (0, 9):
        with pytest.raises(OracleError):
            oracle.range_finder(x, q, 4, 1)
    oracle.range_finder(x, 8, 4, 1)


def test_square_sketch_reduction(oracle):
    """test_solvers.cpp:356-370 / acceptance check 5: q = d = n, w = 0."""
    x = random_nonneg(oracle, 12, 12, 512)
    left, right = oracle.build_projectors(x, 12, 0, 5)
    xhat, xcheck = oracle.compress(x, left, right)
    a, b = oracle.initialize(12, 12, 3, 612)
    pa, pb = a.copy(), b.copy()
    ah, bc = oracle.compress_factors(a, b, left, right)
    r1, r2 = oracle.rng(902), oracle.rng(902)
    for _ in range(5):
        oracle.fasthals_step(x, pa, pb, True, r1)
        oracle.fasthals_rp_step(xhat, xcheck, a, b, ah, bc, left, right, True, 0.0, 0.0, r2)
        assert np.linalg.norm(a - pa) / np.linalg.norm(pa) < 1e-8
        assert np.linalg.norm(b - pb) / np.linalg.norm(pb) < 1e-8


def test_penalized_update_closed_form_and_bitwise_reduction(oracle):
    """test_solvers.cpp:466-494 / acceptance check 10."""
    draws = oracle.draws(71, 1, 16)
    b = draws[:8].reshape(4, 2).copy()
    p = (2.0 * draws[8:16] - 0.5).reshape(4, 2).copy()
    w = np.array([[1.5, 0.3], [0.3, 0.9]])
    got0 = oracle.b_update(b, p, w, 1, 0.0, 0.0)
    plain = np.maximum(0.0, b[:, 1] + (p[:, 1] - b @ w[:, 1]) / w[1, 1])
    assert np.array_equal(got0, plain)
    got = oracle.b_update(b, p, w, 1, 0.2, 0.7)
    want = np.maximum(0.0, (b[:, 1] * w[1, 1] + p[:, 1] - b @ w[:, 1] - 0.2) / (w[1, 1] + 0.7))
    assert np.allclose(got, want, rtol=1e-14, atol=0)


def test_run_cadence_and_zero_iterations(oracle):
    x = random_nonneg(oracle, 10, 8, 7)
    _, _, t = oracle.run(x, 2, q=4, w=1, max_iterations=23, error_interval=5,
                         rel_tolerance=1e-300)
    assert t.iterations == [0, 5, 10, 15, 20, 23] and t.iterations_run == 23
    a, b, t = oracle.run(x, 2, q=4, w=1, max_iterations=0)
    a0, b0 = oracle.initialize(10, 8, 2, 1)
    assert t.iterations == [0] and np.array_equal(a, a0) and np.array_equal(b, b0)


def test_validation_rules(oracle):
    from oracle import OracleError
    x = random_nonneg(oracle, 10, 8, 7)
    for kw in [dict(k=0, q=4), dict(k=9, q=10), dict(k=3, q=3), dict(k=3, q=9),
               dict(k=2, q=4, alpha=-0.5), dict(k=2, q=4, beta=float("inf")),
               dict(k=2, q=4, error_interval=0), dict(k=2, q=4, rel_tolerance=0.0)]:
        with pytest.raises(OracleError) as e:
            oracle.run(x, **kw)
        assert e.value.code == 1
    bad = x.copy()
    bad[2, 2] = -0.1
    with pytest.raises(OracleError) as e:
        oracle.run(bad, 2, q=4)
    assert e.value.code == 3


def test_gini_closed_forms(oracle):
    """acceptance check 9 / test_metrics.cpp:99-114."""
    assert oracle.gini(np.ones(8)) == 0.0
    assert abs(oracle.gini(np.array([0.0, 0.0, 0.0, 1.0])) - 0.75) < 1e-12
    assert abs(oracle.gini(np.array([1.0, 2.0, 3.0, 4.0])) - 0.25) < 1e-12


def test_reconstruction_error_small(oracle):
    x = np.array([[1.0, 2.0], [3.0, 4.0]])
    assert oracle.reconstruction_error(x, np.zeros((2, 1)), np.zeros((2, 1))) == 15.0
    # test_metrics.cpp:56-62: half the squared Frobenius residual (value 7)
    a = np.array([[1.0], [1.0]])
    b = np.array([[1.0], [1.0]])
    assert oracle.reconstruction_error(x, a, b) == 0.5 * (0 + 1 + 4 + 9)


def test_synth_generators(oracle):
    x = oracle.synth_x(50, 40, 5, 0, 1, 0.01, 1)
    assert x.dtype == np.float32 and np.all(x >= 0)
    xs = oracle.synth_x(50, 40, 5, 0, 1, 0.01, 1, col_lo=10, col_hi=30)
    assert np.array_equal(xs, x[:, 10:30])  # shard-local generation is exact
    xe = oracle.synth_x(40, 30, 4, 1, 1, 0.05, 2)
    assert np.all(xe >= 0)
    xp = oracle.synth_x(60, 80, 10, 2, 2, 0.0, 3)
    assert np.all(xp == np.round(xp)) and xp.mean() > 0.5
