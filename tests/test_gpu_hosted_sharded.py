"""GPU: the column-sharded run (run_sharded_impl, the product's multi-GPU path)
at world size 2 on the ONE GPU a test box has.

NCCL cannot put two ranks on one device, so the two processes use the
host-staged collective transport (cnmf_context_create_hosted: every
all-reduce / all-gather goes device -> host -> torch.distributed gloo ->
device).  Everything else -- the sharded compression (d x l sketch
all-reduces, CholeskyQR2 with all-reduced Grams for the row-sharded n-side
bases), the per-iteration B-check + zero-flag all-reduce, the host-side zero
/ dead decisions, the redraws from the run stream with each rank keeping its
slice -- is the code a real 2-GPU run executes.  Kernels of the two ranks
never wait on each other (the collectives are between launches), so sharing
the GPU does not change what is computed.

Checked: both ranks hold the same A bit for bit; the gathered B and the
trajectory match the single-GPU run within the parity bar (the shards only
regroup the fp32 sums of the compression and the fp64 ones of B-check) with
the same redraw draws.  (This test found an R-side range-finder scratch
buffer sized for the local n rows but used for d rows at world size > 1.)
"""
import os
import tempfile

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

CASES = {
    # name: (d, n, rank, factor_kind, noise_kind, sigma, k, q, w, iters, every, stream)
    "c1like": (1000, 1001, 20, 0, 1, 0.01, 20, 30, 2, 25, 5, False),
    # (rank 2 + noise with k = 8 instead is chaotic: there the single-GPU run
    # itself leaves the oracle's trajectory by 4e-4 within 6 iterations)
    "redraws": (300, 241, 8, 0, 1, 0.01, 8, 12, 1, 20, 2, False),
    "redraws2": (600, 401, 3, 1, 1, 0.05, 10, 16, 2, 40, 5, False),
    "redraws3": (500, 333, 4, 0, 1, 0.02, 12, 20, 1, 40, 5, True),
    "streaming": (2000, 1503, 10, 1, 1, 0.05, 12, 20, 1, 30, 5, True),
}


def _cfg(cb, k, q, w, iters, every):
    return cb.SolverConfig(algorithm=cb.FASTHALS_RP, k=k, sketch=cb.SketchConfig(q, w, 1),
                           max_iterations=iters, error_interval=every, rel_tolerance=1e-300,
                           seed=1)


def _worker(rank, world, port, case, out_dir):
    import torch.distributed as dist

    import paper_1712_02248_b200 as cb
    spec = CASES[case] if isinstance(case, str) else case
    d, n, r, fk, nk, sigma, k, q, w, iters, every, stream = spec
    if stream:
        os.environ["CNMF_HALS"] = "stream"
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                            world_size=world)
    torch.cuda.set_device(0)
    ctx = cb.HostedShardedContext(0)
    lo, hi = cb.shard_range(n, rank, world)
    xb = torch.empty((d, (hi - lo + 3) // 4 * 4), dtype=torch.float32, device="cuda")
    ctx.synth_x(d, n, r, fk, nk, sigma, 1, xb, lo, hi)
    a, b, tr = ctx.run_sharded(xb[:, :hi - lo], n, _cfg(cb, k, q, w, iters, every))
    np.savez(os.path.join(out_dir, f"rank{rank}.npz"), a=a.cpu().numpy(), b=b.cpu().numpy(),
             err=np.array([x.error for x in tr.records]),
             it=np.array([x.iteration for x in tr.records]),
             draws=np.array([x.rng_draws for x in tr.records]),
             redraws=np.array([tr.redraws]), gini=np.array([tr.gini_b]))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("case", sorted(CASES))
def test_hosted_sharded_world2_matches_single_gpu(ctx, case):
    _run_case(ctx, case)


@pytest.mark.parametrize("case", ["c1like", "streaming"])
def test_hosted_sharded_world2_fp64_range_finder(ctx, case, monkeypatch):
    """The fp64 range finder through the sharded path:
    fp64 sketch all-reduces, row-sharded fp64 CholeskyQR with all-reduced
    fp64 Grams, against the single-GPU fp64 range finder."""
    monkeypatch.setenv("CNMF_RF", "fp64")
    _run_case(ctx, case)


def _run_case(ctx, case):
    import socket

    import torch.multiprocessing as mp

    import paper_1712_02248_b200 as cb
    d, n, r, fk, nk, sigma, k, q, w, iters, every, stream = CASES[case]
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    with tempfile.TemporaryDirectory() as tmp:
        mp.start_processes(_worker, args=(2, port, case, tmp), nprocs=2, join=True,
                           start_method="spawn")
        res = [np.load(os.path.join(tmp, f"rank{g}.npz")) for g in range(2)]
    if stream:
        os.environ["CNMF_HALS"] = "stream"
    try:
        xb = torch.empty((d, (n + 3) // 4 * 4), dtype=torch.float32, device="cuda")
        ctx.synth_x(d, n, r, fk, nk, sigma, 1, xb)
        a1, b1, t1 = ctx.run_device(xb[:, :n], _cfg(cb, k, q, w, iters, every))
    finally:
        os.environ.pop("CNMF_HALS", None)
    assert np.array_equal(res[0]["a"], res[1]["a"]), "replicated A differs across ranks"
    assert np.array_equal(res[0]["err"], res[1]["err"])
    assert list(res[0]["it"]) == [x.iteration for x in t1.records]
    e1 = np.array([x.error for x in t1.records])
    assert np.max(np.abs(res[0]["err"] - e1) / e1) < 1e-4
    assert list(res[0]["draws"]) == [x.rng_draws for x in t1.records]
    assert int(res[0]["redraws"][0]) == t1.redraws
    a = a1.double().cpu().numpy()
    b = b1.double().cpu().numpy()
    bs = np.concatenate([res[0]["b"], res[1]["b"]]).astype(np.float64)
    assert np.linalg.norm(res[0]["a"] - a) / np.linalg.norm(a) < 1e-3
    assert np.linalg.norm(bs - b) / np.linalg.norm(b) < 1e-3
    assert abs(float(res[0]["gini"][0]) - t1.gini_b) < 1e-4
    if case.startswith("redraws") and case != "redraws2":
        assert t1.redraws > 0
