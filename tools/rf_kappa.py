"""Condition estimate kappa(X Omega) of each BASELINE configuration's first
sketch and the range-finder arithmetic it selects (engine.cpp rf_mode), with
the compression time of both arithmetics.   python tools/rf_kappa.py c1 c2 c3 c4"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1712_02248_b200 as cb  # noqa: E402

ctx = cb.Context(0)
for name in sys.argv[1:]:
    c = cb.CONFIGS[name]
    x = torch.empty((c["d"], c["n"]), device="cuda")
    ctx.synth_x(c["d"], c["n"], c["rank"], c["factor_kind"], c["noise_kind"], c["sigma"], 1, x)
    cfg = cb.SolverConfig(algorithm=cb.FASTHALS_RP, k=c["k"], sketch=cb.SketchConfig(c["q"], c["w"], 1),
                          max_iterations=2, error_interval=2, rel_tolerance=1e-300, seed=1)
    out = []
    for mode in ("auto", "tc", "fp64"):
        os.environ["CNMF_RF"] = mode
        ctx.run_device(x, cfg)  # warm
        _, _, tr = ctx.run_device(x, cfg)
        out.append(f"{mode}: compress {1e3 * tr.compress_seconds:.1f} ms fp64={tr.range_finder_fp64}"
                   + (f" kappa={tr.sketch_kappa:.3g}" if mode == "auto" else ""))
    del os.environ["CNMF_RF"]
    print(name, " | ".join(out), flush=True)
    del x
    torch.cuda.empty_cache()
