"""Relative error of the X-stream NN contraction, fp16 hi/lo path vs 3xTF32,
against fp64, on a BASELINE-shaped synthetic X (CNMF_XS toggled per call).
    python tools/f16_accuracy.py [c2|c3-slice]"""
import os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1712_02248_b200 as cb
from oracle import Oracle

o = Oracle(); ctx = cb.Context(0)
d, n, l = (10000, 5000, 36)
x = o.synth_x(d, n, 16, 1, 1, 0.05, 1)
rng = np.random.default_rng(1)
for name, s in (("gaussian", rng.standard_normal((n, l))), ("orthonormal", np.linalg.qr(rng.standard_normal((n, l)))[0])):
    s = s.astype(np.float32)
    ref = x.astype(np.float64) @ s.astype(np.float64)
    for mode in ("tf32", "f16"):
        os.environ["CNMF_XS"] = mode
        y = torch.empty((d, l), device="cuda")
        ctx.xs_nn(torch.from_numpy(x).cuda(), torch.from_numpy(s).cuda(), y)
        g = y.cpu().numpy().astype(np.float64)
        rf = np.linalg.norm(g - ref) / np.linalg.norm(ref)
        col = np.linalg.norm(g - ref, axis=0) / np.linalg.norm(ref, axis=0)
        bias = np.mean((g - ref) / np.abs(ref).clip(1e-30))
        print(f"{name:12s} {mode:5s} relF {rf:.3e} worst col {col.max():.3e} mean signed rel {bias:.3e}", flush=True)
