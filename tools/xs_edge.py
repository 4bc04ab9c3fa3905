"""Diagnostic: X-stream contractions on small / odd shapes vs fp64 numpy."""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1712_02248_b200 as cb  # noqa: E402

ctx = cb.Context(0)
rng = np.random.default_rng(0)
for d, n, l in [(300, 120, 12), (300, 121, 12), (300, 241, 12), (1000, 500, 30), (1000, 501, 30),
                (300, 60, 12), (300, 33, 12), (300, 17, 12), (64, 120, 16), (5000, 130, 40)]:
    ldx = (n + 3) // 4 * 4
    xb = torch.zeros((d, ldx), device="cuda")
    x = torch.from_numpy(rng.random((d, n)).astype(np.float32)).cuda()
    xb[:, :n] = x
    xv = xb[:, :n]
    s = torch.from_numpy(rng.standard_normal((n, l)).astype(np.float32)).cuda()
    t = torch.from_numpy(rng.standard_normal((d, l)).astype(np.float32)).cuda()
    y = torch.empty((d, l), device="cuda")
    z = torch.empty((n, l), device="cuda")
    ctx.xs_nn(xv, s, y)
    ctx.xs_tn(xv, t, z)
    X = x.double().cpu().numpy()
    yr = X @ s.double().cpu().numpy()
    zr = X.T @ t.double().cpu().numpy()
    e1 = np.linalg.norm(y.double().cpu().numpy() - yr) / np.linalg.norm(yr)
    e2 = np.linalg.norm(z.double().cpu().numpy() - zr) / np.linalg.norm(zr)
    print(f"{d}x{n} l{l}: NN {e1:.2e}  TN {e2:.2e}")
