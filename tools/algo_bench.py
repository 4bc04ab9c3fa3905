"""Device time of every solver of run() on a BASELINE.json configuration
(synthetic X resident in HBM; SURVEY.md 8f rows 2-3 and the reference's
acceptance check "compression speeds up fasthals").

    python tools/algo_bench.py [c1|c2|c3] [iters]

Prints one JSON line per algorithm: update seconds per iteration (CUDA
events around the update launches), compression seconds, total run wall.
"""
import json
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1712_02248_b200 as cb  # noqa: E402


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "c2"
    iters = int(sys.argv[2]) if len(sys.argv) > 2 else 50
    c = cb.CONFIGS[name]
    ctx = cb.Context(0)
    x = torch.empty((c["d"], c["n"]), device="cuda")
    ctx.synth_x(c["d"], c["n"], c["rank"], c["factor_kind"], c["noise_kind"], c["sigma"], 1, x)
    torch.cuda.synchronize()
    for algo in ("fasthals-rp", "hals-rp", "mu-rp", "fasthals", "hals", "mu"):
        rp = algo.endswith("-rp")
        cfg = cb.SolverConfig(algorithm=cb.ALGORITHM_NAMES[algo], k=c["k"],
                              sketch=cb.SketchConfig(c["q"] if rp else 0, c["w"], 1),
                              max_iterations=iters, error_interval=iters,
                              rel_tolerance=1e-300, seed=1)
        ctx.run_device(x, cfg)  # warm-up (workspaces, attributes)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        _, _, tr = ctx.run_device(x, cfg)
        torch.cuda.synchronize()
        wall = time.perf_counter() - t0
        print(json.dumps({"config": name, "algorithm": algo, "iterations": tr.iterations_run,
                          "update_ms_per_iter": 1e3 * tr.update_seconds / max(1, tr.iterations_run),
                          "compress_ms": 1e3 * tr.compress_seconds,
                          "run_wall_ms": 1e3 * wall, "final_error": tr.records[-1].error,
                          "redraws": tr.redraws}), flush=True)


if __name__ == "__main__":
    main()
