"""Diagnostic: tensor-core objective vs the SIMT one (value and time)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1712_02248_b200 as cb  # noqa: E402

ctx = cb.Context(0)
for d, n, k in [(10000, 5000, 16), (1000, 1001, 20), (10000, 5000, 24), (50000, 100000, 100)]:
    x = torch.rand((d, n), device="cuda")
    a = torch.rand((d, k), device="cuda")
    b = torch.rand((n, k), device="cuda")
    for rep in range(3):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        v = ctx.reconstruction_error(x, a, b)
        e1.record()
        e1.synchronize()
        print(d, n, k, v, f"{e0.elapsed_time(e1):.3f} ms", flush=True)
