"""Diagnostic: single-GPU resident vs streaming HALS kernel vs the oracle,
error every iteration (where does a deviation first appear?)."""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import paper_1712_02248_b200 as cb
    from oracle import Oracle
    o = Oracle()
    ctx = cb.Context(0)
    for (d, n, r, fk, nk, sigma, k, q, w, iters) in [(1000, 1001, 20, 0, 1, 0.01, 20, 30, 2, 12),
                                                     (600, 401, 3, 1, 1, 0.05, 10, 16, 2, 12)]:
        xb = torch.empty((d, (n + 3) // 4 * 4), dtype=torch.float32, device="cuda")
        ctx.synth_x(d, n, r, fk, nk, sigma, 1, xb)
        cfg = cb.SolverConfig(algorithm=cb.FASTHALS_RP, k=k, sketch=cb.SketchConfig(q, w, 1),
                              max_iterations=iters, error_interval=1, rel_tolerance=1e-300, seed=1)
        x = xb[:, :n].cpu().numpy().astype(np.float64)
        _, _, ot = o.run(x, k, q=q, w=w, max_iterations=iters, error_interval=1,
                         rel_tolerance=1e-300)
        e0 = np.array(ot.errors)
        res = {}
        for mode in ("resident", "stream"):
            if mode == "stream":
                os.environ["CNMF_HALS"] = "stream"
            a, b, t = ctx.run_device(xb[:, :n], cfg)
            os.environ.pop("CNMF_HALS", None)
            res[mode] = np.array([z.error for z in t.records])
        print(f"== {d}x{n} k{k}")
        for i in range(len(e0)):
            print(f"{i:3d} resident {abs(res['resident'][i]-e0[i])/e0[i]:.2e} "
                  f"stream {abs(res['stream'][i]-e0[i])/e0[i]:.2e}")


main()
