"""Time the X-stream contraction (cnmf_time_xstream) on a seeded synthetic X.
usage: python tools/xs_bench.py CONFIG [tn] [iters]   (CONFIG in c1..c4)"""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
import paper_1712_02248_b200 as cb

name = sys.argv[1] if len(sys.argv) > 1 else "c3"
tn = int(sys.argv[2]) if len(sys.argv) > 2 else 0
iters = int(sys.argv[3]) if len(sys.argv) > 3 else 10
l_override = int(sys.argv[4]) if len(sys.argv) > 4 else 0
c = cb.CONFIGS[name]
ctx = cb.Context(0)
d, n, q = c["d"], c["n"], c["q"]
if l_override: q = l_override
ldx = (n + 3) // 4 * 4
x = torch.empty((d, ldx), dtype=torch.float32, device="cuda")
ctx.synth_x(d, n, c["rank"], c["factor_kind"], c["noise_kind"], c["sigma"], 1, x)
xv = x[:, :n]
t = ctx.time_xstream(xv, q, tn, iters=iters)
alg = 4.0 * d * n + 4.0 * (d + n) * q
hbm = 6549.4
print(f"{name} {'TN' if tn else 'NN'} d={d} n={n} l={q}: {t*1e6:.1f} us  {alg/t/1e9:.0f} GB/s  {alg/t/1e9/hbm:.1%} of {hbm} GB/s")
