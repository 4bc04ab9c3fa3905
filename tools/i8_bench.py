"""Time the fp64-grade range-finder contraction (cnmf_xs_exact: int8-sliced kernel or, with
`dmma`, the FP64 tensor-core kernel) on a seeded synthetic X, operand preparation included.
usage: python tools/i8_bench.py CONFIG [tn] [iters] [dmma]"""
import os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
import paper_1712_02248_b200 as cb

name = sys.argv[1] if len(sys.argv) > 1 else "c3"
tn = int(sys.argv[2]) if len(sys.argv) > 2 else 0
iters = int(sys.argv[3]) if len(sys.argv) > 3 else 5
dmma = len(sys.argv) > 4 and sys.argv[4] == "dmma"
c = cb.CONFIGS[name]
ctx = cb.Context(0)
d, n, q = c["d"], c["n"], c["q"]
lp = (q + 15) // 16 * 16
x = torch.empty((d, (n + 3) // 4 * 4), dtype=torch.float32, device="cuda")
ctx.synth_x(d, n, c["rank"], c["factor_kind"], c["noise_kind"], c["sigma"], 1, x)
xv = x[:, :n]
s = torch.randn((d if tn else n, lp), device="cuda")
out = torch.empty((n if tn else d, lp), dtype=torch.float64, device="cuda")
ctx.xs_exact(xv, s, out, transpose=bool(tn), dmma=dmma)
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(iters):
    ctx.xs_exact(xv, s, out, transpose=bool(tn), dmma=dmma)
torch.cuda.synchronize()
t = (time.perf_counter() - t0) / iters
alg = 4.0 * d * n
print(f"{name} {'TN' if tn else 'NN'} lp={lp} {'dmma' if dmma else 'int8'}: {t*1e3:.2f} ms per call incl. exponent passes and S slicing ({alg/t/1e9:.0f} GB/s of X)")
