"""Which range-finder steps need which precision (C3)?  The range finder
(compression.cpp:23-42) is rebuilt in torch on the GPU with each contraction
taken either from the device X-stream kernel ('d', fp32 output) or exact
fp64 ('e'), or exact fp64 times (1 + eps u) ('pEPS'), thin_qr in fp64
Householder; the projectors go to the device run through CNMF_DIAG_PROJ
(the device then forms the views itself) and the FastHALS-RP trajectory is
compared with the golden.

    python tools/rf_mix.py c3 dddddd eeeeee eeeeed ...   (one letter per
    contraction in order: sketch, then (z, y) per power iteration; same
    pattern for L and R)
"""
import os
import struct
import sys
import tempfile

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1712_02248_b200 as cb  # noqa: E402
from oracle import Oracle  # noqa: E402

name = sys.argv[1]
g = np.load(os.path.join(ROOT, "tests", "golden", f"{name}_full.npz"))
d, n, rank, fk, nk, dseed, k, q, w, iters, every = (int(v) for v in g["config"])
lp = (q + 15) // 16 * 16
ctx = cb.Context(0)
xb = torch.empty((d, (n + 3) // 4 * 4), device="cuda")
ctx.synth_x(d, n, rank, fk, nk, float(g["sigma"][0]), dseed, xb)
x = xb[:, :n]
x64 = x.double()
o = Oracle()
om_l = torch.from_numpy(o.gaussian_sketch(n, q, 2)).cuda()
om_r = torch.from_numpy(o.gaussian_sketch(d, q, 3)).cuda()
gen = torch.Generator(device="cuda")
gen.manual_seed(7)


def contract(mode, s, tn):
    """X^T s (tn) or X s with the chosen precision."""
    if mode == "d":
        sp = torch.zeros((s.shape[0], lp), device="cuda")
        sp[:, :q] = s.float()
        out = torch.empty((n if tn else d, lp), device="cuda")
        (ctx.xs_tn if tn else ctx.xs_nn)(x, sp, out)
        return out[:, :q].double()
    exact = x64.T @ s if tn else x64 @ s
    if mode.startswith("p"):
        eps = float(mode[1:])
        u = torch.rand(exact.shape, generator=gen, device="cuda", dtype=torch.float64) * 2 - 1
        exact = exact * (1 + eps * u)
    return exact


def rf(om, transpose, modes):
    b = torch.linalg.qr(contract(modes[0], om, transpose)).Q
    for it in range(w):
        z = torch.linalg.qr(contract(modes[1 + 2 * it], b, not transpose)).Q
        b = torch.linalg.qr(contract(modes[2 + 2 * it], z, transpose)).Q
    return b


def pad(m):
    out = torch.zeros((m.shape[0], lp), dtype=torch.float32)
    out[:, :q] = m.float().cpu()
    return out.numpy()


xn = float(g["x_norm_sq"][0])
want = np.sqrt(2.0 * g["errors"] / xn)
cfg = cb.SolverConfig(algorithm=cb.FASTHALS_RP, k=k, sketch=cb.SketchConfig(q, w, 1),
                      max_iterations=iters, error_interval=every, rel_tolerance=1e-300, seed=1)
for pat in sys.argv[2:]:
    modes = pat.split(",") if "," in pat else list(pat)
    L = rf(om_l, False, modes)
    Rt = rf(om_r, True, modes)
    path = os.path.join(tempfile.gettempdir(), "rf_mix.bin")
    with open(path, "wb") as f:
        f.write(struct.pack("<4q", d, n, lp, 0))
        f.write(pad(L).tobytes())
        f.write(pad(Rt).tobytes())
    os.environ["CNMF_DIAG_PROJ"] = path
    _, _, tr = ctx.run_device(x, cfg)
    del os.environ["CNMF_DIAG_PROJ"]
    got = np.sqrt(2.0 * np.array([r.error for r in tr.records]) / xn)
    dev = np.abs(got - want) / want
    print(f"{pat:28s} max dev {dev.max():.2e} | " + " ".join(f"{v:.1e}" for v in dev[::2]), flush=True)
