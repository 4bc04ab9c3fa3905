"""GPU parity at the FULL BASELINE sizes against the reference's own runs.

tests/golden/<cfg>_full.npz holds what the unmodified reference library
(oracle/_ref, driven step by step through its public functions by
oracle/golden_big.cpp) produced on this repo's seeded synthetic X:

  C2  10000 x 5000,   k 16,  l 36,  w 2, 200 iterations, error every iteration
  C3  100000 x 20000, k 50,  l 70,  w 2, 100 iterations, error every 5
  C4  50000 x 100000, k 100, l 120, w 1, 100 iterations, error every 5

Here X is generated on the device (cnmf_synth_x) and first checked against
the golden's per-1000-row checksums of the fp32 bits (bit-identical input),
then cnmf_run_device runs the whole job and every record is compared:

  * per-iteration relative error sqrt(2 err / ||X||^2) within 1e-4 relative
    (north_star);
  * the run Rng's position at every record -- the raw draws the dead-component
    redraws took (reinit_column, solvers.cpp:28-31) -- EQUAL to the
    reference's, i.e. the same redraw events of the same lengths;
  * the final A and B: relative Frobenius <= 1e-3 and max |delta| <= 1e-3
    max |ref| per factor -- over ALL rows for C2 and C3;
    C4's fixture keeps every 2nd row of A and every 4th of B (16 MB instead
    of 42) plus fp64 column sums and sums of squares over all rows, which are
    checked too;
  * Gini of B within 1e-4.
"""
import os

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")
TRAJ_RTOL = 1e-4
FACTOR_RTOL = 1e-3


def _golden(name):
    path = os.path.join(GOLDEN, f"{name}_full.npz")
    if not os.path.exists(path):
        pytest.skip(f"{path} not generated (tests/golden/make_golden_big.py)")
    return np.load(path)


def _x_block_hash(x, block=1000):
    out = []
    for r0 in range(0, x.shape[0], block):
        out.append(int(x[r0:r0 + block].contiguous().view(torch.int32).sum(dtype=torch.int64)))
    return np.array(out, dtype=np.uint64)


def _check_factor(got, ref, g=None, name=None):
    got = got.double().cpu().numpy()
    ref = ref.astype(np.float64)
    if g is not None and f"{name}_row_stride" in g.files:
        # the fixture keeps every stride-th row plus fp64 column sums and sums
        # of squares over ALL rows (make_golden_big.py ROW_STRIDE)
        for stat, mine in ((f"{name}_colsum", got.sum(axis=0)), (f"{name}_colsumsq", (got * got).sum(axis=0))):
            want = g[stat]
            assert np.max(np.abs(mine - want)) <= FACTOR_RTOL * np.max(np.abs(want)), stat
        got = got[::int(g[f"{name}_row_stride"][0])]
    rel = np.linalg.norm(got - ref) / np.linalg.norm(ref)
    mx = np.abs(got - ref).max() / np.abs(ref).max()
    assert rel <= FACTOR_RTOL and mx <= FACTOR_RTOL, (rel, mx)
    return rel, mx


@pytest.mark.parametrize("name", ["c2", "c3", "c4"])
def test_fullsize_run_matches_reference(ctx, name):
    import paper_1712_02248_b200 as cb
    g = _golden(name)
    d, n, rank, fk, nk, dseed, k, q, w, iters, every = (int(v) for v in g["config"])
    sigma = float(g["sigma"][0])
    xb = torch.empty((d, (n + 3) // 4 * 4), dtype=torch.float32, device="cuda")
    ctx.synth_x(d, n, rank, fk, nk, sigma, dseed, xb)
    x = xb[:, :n]
    assert np.array_equal(_x_block_hash(x), g["x_hash"]), "device X differs from the golden's X"

    cfg = cb.SolverConfig(algorithm=cb.FASTHALS_RP, k=k, sketch=cb.SketchConfig(q, w, 1),
                          max_iterations=iters, error_interval=every, rel_tolerance=1e-300,
                          seed=1)
    a, b, tr = ctx.run_device(x, cfg)
    xn = float(g["x_norm_sq"][0])
    assert abs(tr.x_norm_sq - xn) <= 1e-6 * xn
    assert [r.iteration for r in tr.records] == list(g["iters"])
    got = np.sqrt(2.0 * np.array([r.error for r in tr.records]) / xn)
    want = np.sqrt(2.0 * g["errors"] / xn)
    dev = np.abs(got - want) / want
    print(name, "trajectory deviation per record:", " ".join(f"{v:.1e}" for v in dev))
    assert dev.max() < TRAJ_RTOL, (dev.max(), int(dev.argmax()), dev)
    draws = np.concatenate([[0], np.cumsum(g["step_draws"])])
    assert [r.rng_draws for r in tr.records] == [int(draws[i]) for i in g["iters"]]
    _check_factor(a, g["a"], g, "a")
    _check_factor(b, g["b"], g, "b")
    assert abs(tr.gini_b - float(g["gini"][0])) < 1e-4
    assert tr.status == cb.REACHED_MAX_ITERATIONS and tr.iterations_run == iters
