"""Diagnostic: tensor-core objective on tiny shapes (X = 0 -> 1/2 sum p^2)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1712_02248_b200 as cb  # noqa: E402

ctx = cb.Context(0)
rng = np.random.default_rng(1)
for d, n, k in [(128, 64, 8), (128, 64, 16), (128, 64, 1), (128, 128, 8), (256, 64, 8),
                (128, 64, 24), (128, 64, 32), (128, 64, 40), (128, 64, 104), (200, 100, 12)]:
    for kind in ("zero_x", "ones"):
        a = rng.random((d, k)).astype(np.float32)
        b = rng.random((n, k)).astype(np.float32)
        if kind == "ones":
            a[:] = 1.0
            b[:] = 1.0
        x = np.zeros((d, n), np.float32)
        got = ctx.reconstruction_error(torch.from_numpy(x).cuda(), torch.from_numpy(a).cuda(),
                                       torch.from_numpy(b).cuda())
        p = a.astype(np.float64) @ b.astype(np.float64).T
        want = 0.5 * np.sum(p * p)
        print(f"{d}x{n} k{k} {kind}: got {got:.10g} want {want:.10g} rel {abs(got-want)/want:.2e}",
              flush=True)
