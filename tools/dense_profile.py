"""One short dense-fasthals run on a BASELINE config for kernel launch lists
(ncu --metrics gpu__time_duration.sum).  python tools/dense_profile.py c2 3 [algo]"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1712_02248_b200 as cb  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c2"
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 3
algo = sys.argv[3] if len(sys.argv) > 3 else "fasthals"
c = cb.CONFIGS[name]
ctx = cb.Context(0)
x = torch.empty((c["d"], c["n"]), device="cuda")
ctx.synth_x(c["d"], c["n"], c["rank"], c["factor_kind"], c["noise_kind"], c["sigma"], 1, x)
rp = algo.endswith("-rp")
cfg = cb.SolverConfig(algorithm=cb.ALGORITHM_NAMES[algo], k=c["k"],
                      sketch=cb.SketchConfig(c["q"] if rp else 0, c["w"], 1),
                      max_iterations=iters, error_interval=iters, rel_tolerance=1e-300)
ctx.run_device(x, cfg)
torch.cuda.synchronize()
print("ok")
