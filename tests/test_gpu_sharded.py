"""GPU: the column-sharded run path (cnmf_run_sharded_device, NCCL) on the one
GPU a test box has -- world size 1, so every collective is a single-rank NCCL
call -- against the single-GPU run and the oracle trajectory.  The sharded
path differs from the single-GPU one in its structure (one kernel launch per
iteration halting after the B half, host-side zero-column decision on the
all-reduced flags, CholeskyQR2 with all-reduced Grams for the n-side bases),
not in its arithmetic, so the two must agree to fp64 rounding.  The N > 1
decomposition itself is covered on CPU by tests/test_sharded_decomposition.py.
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(autouse=True)
def _tc_range_finder(monkeypatch):
    """Sharded runs build their projectors with the tensor-core range finder
    (csrc/sharded.inc); the single-GPU runs they are compared with take the
    same arithmetic (CNMF_RF=tc, engine.cpp rf_mode)."""
    monkeypatch.setenv("CNMF_RF", "tc")


def _cfg(cb, k, q, w, iters, every=1):
    return cb.SolverConfig(algorithm=cb.FASTHALS_RP, k=k, sketch=cb.SketchConfig(q, w, 1),
                           max_iterations=iters, error_interval=every, rel_tolerance=1e-300, seed=1)


def _synth(ctx, d, n, rank, fk, nk, sigma):
    x = torch.empty((d, (n + 3) // 4 * 4), dtype=torch.float32, device="cuda")
    ctx.synth_x(d, n, rank, fk, nk, sigma, 1, x)
    return x[:, :n]


def _compare(t1, t2, a1, a2, b1, b2, traj_rtol, fac_rtol):
    e1 = np.array([r.error for r in t1.records])
    e2 = np.array([r.error for r in t2.records])
    assert [r.iteration for r in t1.records] == [r.iteration for r in t2.records]
    assert np.max(np.abs(e1 - e2) / e1) < traj_rtol
    for u, v in ((a1, a2), (b1, b2)):
        u = u.double().cpu().numpy()
        v = v.double().cpu().numpy()
        assert np.linalg.norm(u - v) / np.linalg.norm(u) < fac_rtol


@pytest.fixture(scope="module")
def sctx():
    import paper_1712_02248_b200 as cb
    return cb.ShardedContext(0, 0, 1, cb.ShardedContext.unique_id())


def test_shard_ranges_partition():
    import paper_1712_02248_b200 as cb
    for n, world in ((1000, 1), (1000, 3), (20000, 8), (7, 7)):
        r = [cb.shard_range(n, g, world) for g in range(world)]
        assert r[0][0] == 0 and r[-1][1] == n
        assert all(r[g][1] == r[g + 1][0] for g in range(world - 1))


def test_sharded_world1_matches_single_c1(ctx, sctx):
    import paper_1712_02248_b200 as cb
    x = _synth(ctx, 1000, 1000, 20, 0, 0, 0.01)
    cfg = _cfg(cb, 20, 30, 2, 100)
    a1, b1, t1 = ctx.run_device(x, cfg)
    a2, b2, t2 = sctx.run_sharded(x, 1000, cfg)
    assert t2.status == t1.status and t2.iterations_run == 100
    assert abs(t2.x_norm_sq - t1.x_norm_sq) <= 1e-12 * t1.x_norm_sq
    assert t2.x_passes == t1.x_passes
    assert abs(t2.gini_b - t1.gini_b) < 1e-9
    _compare(t1, t2, a1, a2, b1, b2, 1e-9, 1e-7)


def test_sharded_world1_redraws(ctx, sctx):
    """k well above the data rank: components die and are redrawn from the
    run's Rng in both paths (same draws, same event order)."""
    import paper_1712_02248_b200 as cb
    x = _synth(ctx, 300, 240, 2, 0, 0, 0.0)
    cfg = _cfg(cb, 8, 12, 1, 60, every=5)
    a1, b1, t1 = ctx.run_device(x, cfg)
    a2, b2, t2 = sctx.run_sharded(x, 240, cfg)
    assert t2.redraws == t1.redraws
    _compare(t1, t2, a1, a2, b1, b2, 1e-9, 1e-7)


def test_sharded_world1_streaming_kernel(ctx, sctx, monkeypatch):
    """Same through the streaming HALS kernel (configurations too large for
    the shared-memory-resident one)."""
    import paper_1712_02248_b200 as cb
    monkeypatch.setenv("CNMF_HALS", "stream")
    x = _synth(ctx, 1200, 900, 10, 1, 1, 0.05)
    cfg = _cfg(cb, 10, 18, 1, 40, every=4)
    a1, b1, t1 = ctx.run_device(x, cfg)
    a2, b2, t2 = sctx.run_sharded(x, 900, cfg)
    _compare(t1, t2, a1, a2, b1, b2, 1e-9, 1e-7)


def test_sharded_rejects_wrong_columns(sctx):
    import paper_1712_02248_b200 as cb
    x = torch.ones((50, 40), device="cuda")
    with pytest.raises(cb.DimensionError):
        sctx.run_sharded(x, 80, _cfg(cb, 4, 8, 1, 3))  # world 1 must hold all 80 columns
