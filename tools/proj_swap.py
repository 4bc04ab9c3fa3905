"""Split a full-size trajectory difference between the compression and the
HALS loop: the reference's range finder (Householder QR, fp64 contractions,
the reference's fp64 Gaussian sketches from the oracle) recomputed on the GPU
in torch float64, handed to the device run through CNMF_DIAG_PROJ (projectors
only, then projectors + compressed views), trajectories compared with the
golden.   python tools/proj_swap.py [c3]
"""
import os
import struct
import subprocess
import sys
import tempfile

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1712_02248_b200 as cb  # noqa: E402
from oracle import Oracle  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c3"
g = np.load(os.path.join(ROOT, "tests", "golden", f"{name}_full.npz"))
d, n, rank, fk, nk, dseed, k, q, w, iters, every = (int(v) for v in g["config"])
lp = (q + 15) // 16 * 16  # engine.cpp: pad16(q)
ctx = cb.Context(0)
xb = torch.empty((d, (n + 3) // 4 * 4), device="cuda")
ctx.synth_x(d, n, rank, fk, nk, float(g["sigma"][0]), dseed, xb)
x = xb[:, :n]
x64 = x.double()
o = Oracle()
om_l = torch.from_numpy(o.gaussian_sketch(n, q, 2)).cuda()
om_r = torch.from_numpy(o.gaussian_sketch(d, q, 3)).cuda()


def rf64(om, transpose):  # range_finder_impl, compression.cpp:23-42
    b = torch.linalg.qr(x64.T @ om if transpose else x64 @ om).Q
    for _ in range(w):
        z = torch.linalg.qr(x64 @ b if transpose else x64.T @ b).Q
        b = torch.linalg.qr(x64.T @ z if transpose else x64 @ z).Q
    return b


L = rf64(om_l, False)          # d x q
Rt = rf64(om_r, True)          # n x q (the row basis; R = Rt^T)
xc = x64 @ Rt                  # X-check = X R^T
xht = x64.T @ L                # X-hat^T = X^T L


def pad(m):
    out = torch.zeros((m.shape[0], lp), dtype=torch.float32)
    out[:, :q] = m.float().cpu()
    return out.numpy()


xn = float(g["x_norm_sq"][0])
want = np.sqrt(2.0 * g["errors"] / xn)
cfg = cb.SolverConfig(algorithm=cb.FASTHALS_RP, k=k, sketch=cb.SketchConfig(q, w, 1),
                      max_iterations=iters, error_interval=every, rel_tolerance=1e-300, seed=1)
for views in (0, 1, 2):
    path = os.path.join(tempfile.gettempdir(), f"proj_{views}.bin")
    with open(path, "wb") as f:
        f.write(struct.pack("<4q", d, n, lp, views))
        f.write(pad(L).tobytes())
        f.write(pad(Rt).tobytes())
        if views:
            f.write(pad(xc).tobytes())
            f.write(pad(xht).tobytes())
    if views == 2:  # fp64 views of the DEVICE projectors: isolates the views' contraction
        left = torch.empty((d, q), device="cuda")
        right = torch.empty((q, n), device="cuda")
        ctx.build_projectors(x, q, w, 1, left, right)
        Lg, Rg = left.double(), right.double().T
        with open(path, "wb") as f:
            f.write(struct.pack("<4q", d, n, lp, 1))
            f.write(pad(Lg).tobytes())
            f.write(pad(Rg).tobytes())
            f.write(pad(x64 @ Rg).tobytes())
            f.write(pad(x64.T @ Lg).tobytes())
    os.environ["CNMF_DIAG_PROJ"] = path
    _, _, tr = ctx.run_device(x, cfg)
    del os.environ["CNMF_DIAG_PROJ"]
    got = np.sqrt(2.0 * np.array([r.error for r in tr.records]) / xn)
    dev = np.abs(got - want) / want
    tag = ["fp64 projectors, device views", "fp64 projectors + fp64 views",
           "device projectors + fp64 views"][views]
    print(f"{tag}: max dev {dev.max():.2e} |",
          " ".join(f"{r.iteration}:{v:.1e}" for r, v in zip(tr.records, dev)), flush=True)
