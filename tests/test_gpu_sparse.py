"""GPU parity of the CSR input path (csrc/sparse.cu):
run(SparseMatrix, ...) for every algorithm against the compiled reference's
own sparse run (solvers.cpp:515-517), the sparse objective
(metrics.cpp:79-102), structure validation (matrix.cpp:37-56) and the
`cnmf factorize --format mm` front end.

Tolerances as tests/test_gpu_parity.py: trajectory 1e-4 relative, factors
relative Frobenius 1e-3.
"""
import json
import os

import numpy as np
import pytest

torch = pytest.importorskip("torch")
sparse = pytest.importorskip("scipy.sparse")
pytestmark = pytest.mark.gpu


def _sparse_x(d, n, density, rank, seed):
    """Non-negative low-rank values on a random support (count-like data)."""
    rng = np.random.default_rng(seed)
    w, h = rng.random((d, rank)), rng.random((rank, n))
    mask = sparse.random(d, n, density=density, random_state=seed, format="csr")
    mask.data[:] = 1.0
    x = mask.multiply(w @ h).tocsr()
    x.data = x.data.astype(np.float32).astype(np.float64)
    x.eliminate_zeros()
    return x


def _rel(a, b):
    return float(np.linalg.norm(np.asarray(a, np.float64) - b) / max(np.linalg.norm(b), 1e-300))


@pytest.mark.parametrize("algo,q", [("fasthals-rp", 20), ("hals-rp", 20), ("mu-rp", 20),
                                    ("fasthals", 0), ("hals", 0), ("mu", 0)])
def test_sparse_run_matches_reference(ctx, reference, algo, q):
    import paper_1712_02248_b200 as cb
    x = _sparse_x(500, 400, 0.05, 10, 1)
    a_id = cb.ALGORITHM_NAMES[algo]
    cfg = cb.SolverConfig(algorithm=a_id, k=8, sketch=cb.SketchConfig(q, 2, 1), max_iterations=30,
                          error_interval=1, rel_tolerance=1e-300, seed=1)
    res = ctx.run_sparse(x, cfg)
    ra, rb, rt = reference.run(x, 8, q=q, w=2, sketch_seed=1, max_iterations=30,
                               error_interval=1, rel_tolerance=1e-300, seed=1, algorithm=a_id)
    assert [r.iteration for r in res.trace.records] == list(rt.iterations)
    got = np.array([r.error for r in res.trace.records])
    want = np.array(rt.errors)
    assert np.max(np.abs(got - want) / want) < 1e-4, (got[:4], want[:4])
    assert _rel(res.a, ra) < 1e-3 and _rel(res.b, rb) < 1e-3
    assert res.trace.status == rt.status
    xn = float(np.sum(x.data.astype(np.float64) ** 2))
    assert abs(res.trace.x_norm_sq - xn) <= 1e-12 * xn


def test_sparse_and_dense_runs_agree(ctx):
    """The same X through cnmf_run_csr and cnmf_run: the CSR contractions and
    the expanded objective against the dense kernels."""
    import paper_1712_02248_b200 as cb
    x = _sparse_x(800, 600, 0.08, 12, 2)
    for algo, q in (("fasthals-rp", 24), ("fasthals", 0)):
        cfg = cb.SolverConfig(algorithm=cb.ALGORITHM_NAMES[algo], k=10,
                              sketch=cb.SketchConfig(q, 2, 3), max_iterations=25,
                              error_interval=5, rel_tolerance=1e-300, seed=2)
        rs = ctx.run_sparse(x, cfg)
        rd = ctx.run(x.toarray().astype(np.float32), cfg)
        es = np.array([r.error for r in rs.trace.records])
        ed = np.array([r.error for r in rd.trace.records])
        assert np.max(np.abs(es - ed) / ed) < 1e-4, algo
        assert _rel(rs.a, rd.a) < 1e-3 and _rel(rs.b, rd.b) < 1e-3


def test_sparse_empty_rows_and_columns(ctx, reference):
    """Rows and columns without stored entries (the CSR of X^T has empty
    columns, the SpMM writes zero rows)."""
    import paper_1712_02248_b200 as cb
    x = _sparse_x(300, 200, 0.05, 6, 3).tolil()
    x[10:20, :] = 0
    x[:, 50:60] = 0
    x = x.tocsr()
    x.eliminate_zeros()
    cfg = cb.SolverConfig(algorithm=cb.FASTHALS_RP, k=5, sketch=cb.SketchConfig(12, 1, 4),
                          max_iterations=20, error_interval=2, rel_tolerance=1e-300, seed=4)
    res = ctx.run_sparse(x, cfg)
    ra, rb, rt = reference.run(x, 5, q=12, w=1, sketch_seed=4, max_iterations=20,
                               error_interval=2, rel_tolerance=1e-300, seed=4)
    got = np.array([r.error for r in res.trace.records])
    assert np.max(np.abs(got - np.array(rt.errors)) / np.array(rt.errors)) < 1e-4


def test_sparse_structure_and_data_errors(ctx):
    import paper_1712_02248_b200 as cb
    cfg = cb.SolverConfig(algorithm=cb.MU, k=2)
    rp = np.array([0, 2, 3], np.uint64)
    with pytest.raises(cb.DimensionError, match="strictly increasing"):
        ctx.run_sparse((rp, np.array([1, 1, 0], np.uint64), np.ones(3), (2, 3)), cfg)
    with pytest.raises(cb.DimensionError, match="out of range"):
        ctx.run_sparse((rp, np.array([0, 1, 3], np.uint64), np.ones(3), (2, 3)), cfg)
    with pytest.raises(cb.DimensionError):
        ctx.run_sparse((np.array([0, 2], np.uint64), np.array([0, 1, 2], np.uint64), np.ones(3),
                        (2, 3)), cfg)
    with pytest.raises(cb.InputError):
        ctx.run_sparse((rp, np.array([0, 1, 2], np.uint64), np.array([1.0, -1.0, 1.0]), (2, 3)),
                       cfg)


def test_cli_factorize_matrix_market(tmp_path, reference):
    """cnmf factorize --format mm: the Matrix Market loader feeds the CSR path."""
    import paper_1712_02248_b200 as cb
    from paper_1712_02248_b200 import cli
    x = _sparse_x(120, 90, 0.1, 4, 5)
    p = tmp_path / "x.mtx"
    p.write_text(cli.save_matrix_market_text(x))
    out = str(tmp_path / "run")
    assert cli.run(["factorize", "--format", "mm", "--input", str(p), "--algo", "fasthals-rp",
                    "--k", "3", "--q", "8", "--w", "2", "--iters", "20", "--tol", "1e-300",
                    "--seed", "2", "--out", out]) == 0
    s = json.load(open(os.path.join(out, "summary.json")))
    assert s["iterations_run"] == 20 and s["k"] == 3
    ra, rb, rt = reference.run(cli.load_matrix_market(str(p)), 3, q=8, w=2, sketch_seed=2,
                               max_iterations=20, rel_tolerance=1e-300, seed=2,
                               algorithm=cb.FASTHALS_RP)
    rows = open(os.path.join(out, "trace.csv")).read().splitlines()[1:]
    got = np.array([float(r.split(",")[3]) for r in rows])
    assert np.max(np.abs(got - np.array(rt.errors)) / np.array(rt.errors)) < 1e-4
    a = cli.load_dense_csv(os.path.join(out, "a.csv"))
    assert _rel(a, ra) < 1e-3
