"""Diagnostic: objective values of real runs, tensor-core vs SIMT kernel
(same run, CNMF_RECON switch read per process -> two subprocesses)."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

CHILD = r'''
import json, os, sys
import torch
sys.path.insert(0, %r)
import paper_1712_02248_b200 as cb
name, iters, every = sys.argv[1], int(sys.argv[2]), int(sys.argv[3])
c = cb.CONFIGS[name]
ctx = cb.Context(0)
x = torch.empty((c["d"], (c["n"] + 3) // 4 * 4), device="cuda")
ctx.synth_x(c["d"], c["n"], c["rank"], c["factor_kind"], c["noise_kind"], c["sigma"], 1, x)
cfg = cb.SolverConfig(algorithm=cb.FASTHALS_RP, k=c["k"], sketch=cb.SketchConfig(c["q"], c["w"], 1),
                      max_iterations=iters, error_interval=every, rel_tolerance=1e-300, seed=1)
_, _, tr = ctx.run_device(x[:, :c["n"]], cfg)
print(json.dumps([[r.iteration, r.error] for r in tr.records]))
''' % ROOT


def run(name, iters, every, mode):
    env = dict(os.environ)
    if mode == "simt":
        env["CNMF_RECON"] = "simt"
    out = subprocess.run([sys.executable, "-c", CHILD, name, str(iters), str(every)], env=env,
                         capture_output=True, text=True, check=True).stdout
    return json.loads(out.strip().splitlines()[-1])


for spec in sys.argv[1:] or ["c1:100:5", "c2:200:10", "c3:60:5", "c4:30:5"]:
    name, iters, every = spec.split(":")
    a = run(name, int(iters), int(every), "tc")
    b = run(name, int(iters), int(every), "simt")
    worst = max(abs(x[1] - y[1]) / y[1] for x, y in zip(a, b))
    print(name, "records", len(a), "worst |tc - simt| / simt", f"{worst:.2e}",
          " ".join(f"{abs(x[1]-y[1])/y[1]:.1e}" for x, y in zip(a, b)), flush=True)
