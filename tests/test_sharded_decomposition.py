"""CPU, world size 2 (gloo): the column-sharded decomposition of the hot path
(csrc/sharded.inc) reproduces the single-process
reference algorithm (the oracle).

* shard ranges: the C ABI's cnmf_shard_begin equals the mirror's formula and
  partitions the columns;
* compression: the sharded range finders (sketch partials summed across
  ranks, row-sharded bases by CholeskyQR2 with all-reduced Grams) span the
  same subspaces as the oracle's build_projectors;
* FastHALS-RP: A half replicated, B half on each rank's rows, one B-check
  all-reduce per step -> the oracle's fasthals_rp_step results (A, B,
  A-hat, B-check) to fp64 rounding.
"""
import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")
import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402

WORLD = 2
D, N, RANK, K, Q, W, STEPS = 64, 50, 8, 4, 8, 1, 6  # rank = q: a well-separated sketch span


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, port, out):
    import sys
    sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=WORLD)
    try:
        import sharded_mirror as sm
        from oracle import Oracle
        o = Oracle()
        res = {}
        x = o.synth_x(D, N, RANK, 0, 0, 0.01, 1).astype(np.float64)
        lo, hi = sm.shard(N, rank, WORLD)
        xl = x[:, lo:hi]
        # --- compression spans
        omega_l = o.gaussian_sketch(N, Q, 2)
        omega_r = o.gaussian_sketch(D, Q, 3)
        left_sh = sm.range_finder_sharded(xl, Q, W, omega_l, False, lo, hi)
        rt_local = sm.range_finder_sharded(xl, Q, W, omega_r, True, lo, hi)
        parts = [torch.zeros((sm.shard(N, g, WORLD)[1] - sm.shard(N, g, WORLD)[0], Q),
                             dtype=torch.float64) for g in range(WORLD)]
        dist.all_gather(parts, torch.from_numpy(np.ascontiguousarray(rt_local)))
        rt_full = torch.cat(parts).numpy()
        left, right = o.build_projectors(x, Q, W, 1)
        res["left_span"] = float(np.linalg.norm(left_sh @ left_sh.T - left @ left.T))
        res["right_span"] = float(np.linalg.norm(rt_full @ rt_full.T - right.T @ right))
        # --- FastHALS-RP steps from the oracle's projectors
        xhat, xcheck = o.compress(x, left, right)
        a, b = o.initialize(D, N, K, 1)
        ah, bc = o.compress_factors(a, b, left, right)
        right_local = right[:, lo:hi].T
        xcheck_sh = sm.allreduce(xl @ right_local)                       # X R^T summed
        xhat_local = left.T @ xl                                         # local columns
        bchk0 = sm.allreduce(right_local.T @ b[lo:hi])                   # R B summed
        res["xcheck"] = float(np.max(np.abs(xcheck_sh - xcheck)) / np.max(np.abs(xcheck)))
        res["bchk0"] = float(np.max(np.abs(bchk0 - bc)) / np.max(np.abs(bc)))
        a_sh, b_sh, ah_sh, bc_sh = sm.fasthals_rp_steps_sharded(
            xhat_local, xcheck_sh, a, b[lo:hi], ah, bchk0, left, right_local, STEPS)
        rng = o.rng(1)
        a_r, b_r, ah_r, bc_r = a.copy(), b.copy(), ah.copy(), bc.copy()
        for _ in range(STEPS):
            o.fasthals_rp_step(xhat, xcheck, a_r, b_r, ah_r, bc_r, left, right, True, 0.0, 0.0, rng)
        rel = lambda u, v: float(np.linalg.norm(u - v) / np.linalg.norm(v))
        res["a"] = rel(a_sh, a_r)
        res["b_local"] = rel(b_sh, b_r[lo:hi])
        res["ahat"] = rel(ah_sh, ah_r)
        res["bchk"] = rel(bc_sh, bc_r)
        out.put((rank, res))
    finally:
        dist.destroy_process_group()


@pytest.fixture(scope="module")
def results():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, port, q)) for r in range(WORLD)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=240) for _ in range(WORLD))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    return res


def test_shard_begin_matches_mirror():
    import paper_1712_02248_b200 as cb
    import sharded_mirror as sm
    for n, world in ((N, WORLD), (20000, 8), (13, 4), (100000, 7)):
        for g in range(world):
            assert (cb.shard_begin(n, g, world), cb.shard_begin(n, g + 1, world)) == sm.shard(n, g, world)


def test_sharded_compression_spans(results):
    for r in range(WORLD):
        assert results[r]["left_span"] < 1e-9
        assert results[r]["right_span"] < 1e-9
        assert results[r]["xcheck"] < 1e-12
        assert results[r]["bchk0"] < 1e-12


def test_sharded_fasthals_steps_match_oracle(results):
    for r in range(WORLD):
        for key in ("a", "b_local", "ahat", "bchk"):
            assert results[r][key] < 1e-9, (r, key, results[r][key])
