"""Stress the tcgen05 X-stream kernel against fp64 numpy over shapes, widths
and K-split lengths (CNMF_TC_KCHUNK).  Prints the worst relative error per case."""
import os, subprocess, sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
if len(sys.argv) == 1:
    for chunk in ["", "32", "64", "96", "256", "1024"]:
        env = dict(os.environ)
        if chunk: env["CNMF_TC_KCHUNK"] = chunk
        out = subprocess.run([sys.executable, __file__, "run"], env=env, capture_output=True, text=True)
        print(f"kchunk={chunk or 'plan':>5s}: {out.stdout.strip()} {out.stderr.strip()[-300:]}", flush=True)
    sys.exit(0)
import torch
import paper_1712_02248_b200 as cb
ctx = cb.Context(0)
rng = np.random.default_rng(3)
res = []
for (d, n, l) in [(1024, 20000, 32), (256, 4000, 30), (1000, 3000, 60), (640, 2000, 96), (300, 2500, 120)]:
    x = rng.random((d, n), dtype=np.float32)
    xt = torch.from_numpy(x).cuda()
    for tn in (0, 1):
        kd = d if tn else n
        s = rng.standard_normal((kd, l)).astype(np.float32)
        y = torch.empty((n if tn else d, l), device="cuda")
        (ctx.xs_tn if tn else ctx.xs_nn)(xt, torch.from_numpy(s).cuda(), y)
        ref = (x.astype(np.float64).T if tn else x.astype(np.float64)) @ s.astype(np.float64)
        err = np.linalg.norm(y.cpu().numpy() - ref) / np.linalg.norm(ref)
        res.append(f"{'TN' if tn else 'NN'}{d}x{n}l{l}={err:.1e}")
print(" ".join(res))
