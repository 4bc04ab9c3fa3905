"""Per-phase HALS cycle profile (CTA 0, clock64) of a fasthals-rp run on a
BASELINE.json configuration: sets CNMF_PROFILE before the library loads.

    python tools/hals_profile.py [c1|c2|c3|c4] [iters] [--noprof]
"""
import os
import sys

if "--noprof" not in sys.argv:
    os.environ["CNMF_PROFILE"] = "1"
import torch  # noqa: E402

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1712_02248_b200 as cb  # noqa: E402


def main():
    args = [a for a in sys.argv[1:] if a != "--noprof"]
    name = args[0] if args else "c3"
    iters = int(args[1]) if len(args) > 1 else 20
    c = cb.CONFIGS[name]
    ctx = cb.Context(0)
    x = torch.empty((c["d"], c["n"]), device="cuda")
    ctx.synth_x(c["d"], c["n"], c["rank"], c["factor_kind"], c["noise_kind"], c["sigma"], 1, x)
    cfg = cb.SolverConfig(algorithm=cb.FASTHALS_RP, k=c["k"], sketch=cb.SketchConfig(c["q"], c["w"], 1),
                          max_iterations=iters, error_interval=iters, rel_tolerance=1e-300, seed=1)
    _, _, tr = ctx.run_device(x, cfg)
    torch.cuda.synchronize()
    print(f"{name}: {1e3 * tr.update_seconds / tr.iterations_run:.3f} ms/iteration, "
          f"compress {1e3 * tr.compress_seconds:.2f} ms", flush=True)


if __name__ == "__main__":
    main()
