"""Where a bench step's device time goes: run_device on a BASELINE config,
trace fields (compress, update, error seconds) vs the CUDA-event time of the
whole call."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1712_02248_b200 as cb  # noqa: E402


def main():
    for name in sys.argv[1:] or ["c4"]:
        c = cb.CONFIGS[name]
        ctx = cb.Context(0)
        x = torch.empty((c["d"], c["n"]), device="cuda")
        ctx.synth_x(c["d"], c["n"], c["rank"], c["factor_kind"], c["noise_kind"], c["sigma"], 1, x)
        cfg = cb.SolverConfig(algorithm=cb.FASTHALS_RP, k=c["k"],
                              sketch=cb.SketchConfig(c["q"], c["w"], 1), max_iterations=c["iters"],
                              error_interval=c["iters"], rel_tolerance=1e-300, seed=1)
        st = torch.cuda.ExternalStream(ctx.stream())
        for rep in range(3):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            e0.record(st)
            _, _, tr = ctx.run_device(x, cfg)
            e1.record(st)
            e1.synchronize()
            tot = e0.elapsed_time(e1)
            print(f"{name} rep{rep}: call {tot:.2f} ms | compress {1e3 * tr.compress_seconds:.2f} "
                  f"update {1e3 * tr.update_seconds:.2f} errors {1e3 * tr.error_seconds:.2f} "
                  f"(2 evals) other {tot - 1e3 * (tr.compress_seconds + tr.update_seconds + tr.error_seconds):.2f}"
                  f" | redraws {tr.redraws}", flush=True)
        del x
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
