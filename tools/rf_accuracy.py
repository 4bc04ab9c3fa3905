"""Accuracy of the device range finder at a BASELINE shape against an fp64
restatement on the same GPU (torch float64 matmuls + Householder QR, the
reference's algorithm, same fp32 Gaussian sketch):

  * single X contractions (NN X*Omega, TN X^T*T): relative Frobenius error,
    signed bias sum(err*sign(exact))/sum(|exact|), and the error's share in
    the exact product's trailing (noise) singular directions;
  * the final projectors: principal angles between span(L_device) and
    span(L_fp64) (sin theta, largest and per direction).

    CNMF_XS=tf32|simt|f16 python tools/rf_accuracy.py [c3]
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1712_02248_b200 as cb  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c3"
c = cb.CONFIGS[name]
d, n, k, l, w = c["d"], c["n"], c["k"], c["q"], c["w"]
ctx = cb.Context(0)
x = torch.empty((d, n), device="cuda")
ctx.synth_x(d, n, c["rank"], c["factor_kind"], c["noise_kind"], c["sigma"], 1, x)
x64 = x.double()
print("variant", os.environ.get("CNMF_XS", "default"), name, flush=True)


def report(tag, got, exact, rank):
    e = got.double() - exact
    rel = (e.norm() / exact.norm()).item()
    bias = ((e * torch.sign(exact)).sum() / exact.abs().sum()).item()
    u, s, vh = torch.linalg.svd(exact, full_matrices=False)
    tail = u[:, rank:]
    en = (tail.T @ e).norm().item()
    noise = s[rank:].norm().item()
    print(f"{tag}: rel {rel:.2e} bias {bias:+.2e} | error in trailing dirs {en:.3e} vs their "
          f"signal {noise:.3e} (ratio {en / noise:.2e}); sigma1/sigma_{rank + 1} "
          f"{(s[0] / s[rank]).item():.2e}", flush=True)


om = torch.empty((n, l), device="cuda")
ctx.gaussian_sketch(n, l, 2, om)
y = torch.empty((d, l), device="cuda")
ctx.xs_nn(x, om, y)
y64 = x64 @ om.double()
report("NN X*Omega", y, y64, k)
q64 = torch.linalg.qr(y64).Q
qf = q64.float().contiguous()
z = torch.empty((n, l), device="cuda")
ctx.xs_tn(x, qf, z)
z64 = x64.T @ qf.double()
report("TN X^T*Q", z, z64, k)


def rf64(om64, transpose):
    b = torch.linalg.qr(x64.T @ om64 if transpose else x64 @ om64).Q
    for _ in range(w):
        zz = torch.linalg.qr(x64 @ b if transpose else x64.T @ b).Q
        b = torch.linalg.qr(x64.T @ zz if transpose else x64 @ zz).Q
    return b


L64 = rf64(om.double(), False)
left = torch.empty((d, l), device="cuda")
right = torch.empty((l, n), device="cuda")
try:
    ctx.build_projectors(x, l, w, 1, left, right)
    Lg = left.double()
    s = torch.linalg.svdvals(L64.T @ Lg).clamp(max=1.0)
    sin = torch.sqrt(1 - s ** 2).cpu().numpy()
    print("span(L) vs fp64 range finder: sin(theta) largest", f"{sin.max():.2e}",
          "per direction (ascending):", " ".join(f"{v:.1e}" for v in np.sort(sin)), flush=True)
except Exception as e:  # noqa: BLE001
    print("build_projectors:", e)
