"""Diagnostic: world-size-2 hosted sharded run vs the single-GPU run and the
oracle, per record (tests/test_gpu_hosted_sharded.py cases)."""
import os
import sys
import tempfile

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import test_gpu_hosted_sharded as T  # noqa: E402


def main(case, world=2):
    import socket

    import torch.multiprocessing as mp

    import paper_1712_02248_b200 as cb
    from oracle import Oracle
    d, n, r, fk, nk, sigma, k, q, w, iters, every, stream = T.CASES[case]
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    with tempfile.TemporaryDirectory() as tmp:
        mp.start_processes(T._worker, args=(world, port, case, tmp), nprocs=world, join=True,
                           start_method="spawn")
        res = [np.load(os.path.join(tmp, f"rank{g}.npz")) for g in range(world)]
    ctx = cb.Context(0)
    xb = torch.empty((d, (n + 3) // 4 * 4), dtype=torch.float32, device="cuda")
    ctx.synth_x(d, n, r, fk, nk, sigma, 1, xb)
    cfg = T._cfg(cb, k, q, w, iters, every)
    a1, b1, t1 = ctx.run_device(xb[:, :n], cfg)
    x = xb[:, :n].cpu().numpy().astype(np.float64)
    o = Oracle()
    _, _, ot = o.run(x, k, q=q, w=w, max_iterations=iters, error_interval=every,
                     rel_tolerance=1e-300)
    e0 = np.array(ot.errors)
    e1 = np.array([z.error for z in t1.records])
    e2 = res[0]["err"]
    for i, it in enumerate(res[0]["it"]):
        print(f"{it:4d} single-oracle {abs(e1[i]-e0[i])/e0[i]:.2e} sharded-oracle "
              f"{abs(e2[i]-e0[i])/e0[i]:.2e} sharded-single {abs(e2[i]-e1[i])/e1[i]:.2e}")
    print("redraws", t1.redraws, res[0]["redraws"], "draws", [z.rng_draws for z in t1.records][-1],
          res[0]["draws"][-1])


if __name__ == "__main__":
    world = int(os.environ.get("WORLD", "2"))
    for c in sys.argv[1:] or sorted(T.CASES):
        print("==", c, "world", world)
        main(c, world)
