"""Relative error of the X-stream contraction (tensor vs SIMT) vs K-chunk length."""
import os, subprocess, sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
if len(sys.argv) == 1:
    for mode, chunk in [("simt", ""), ("tc", "32"), ("tc", "256"), ("tc", "1024"), ("tc", "4096"), ("tc", "100000")]:
        env = dict(os.environ, CNMF_XS=mode)
        if chunk: env["CNMF_TC_KCHUNK"] = chunk
        out = subprocess.run([sys.executable, __file__, "run"], env=env, capture_output=True, text=True)
        print(f"{mode:5s} kchunk={chunk or '-':>7s}: {out.stdout.strip()} {out.stderr.strip()[-200:]}")
    sys.exit(0)
import torch
import paper_1712_02248_b200 as cb
ctx = cb.Context(0)
rng = np.random.default_rng(1)
for (d, n, l) in [(1024, 20000, 32), (512, 5000, 48)]:
    x = rng.random((d, n), dtype=np.float32)
    s = rng.standard_normal((n, l)).astype(np.float32)
    y = torch.empty((d, l), device="cuda")
    ctx.xs_nn(torch.from_numpy(x).cuda(), torch.from_numpy(s).cuda(), y)
    ref = x.astype(np.float64) @ s.astype(np.float64)
    got = y.cpu().numpy().astype(np.float64)
    err = got - ref
    print(f"NN {d}x{n} l={l}: relF {np.linalg.norm(err)/np.linalg.norm(ref):.2e} bias {err.mean()/np.abs(ref).mean():+.2e}", end="; ")
print()
