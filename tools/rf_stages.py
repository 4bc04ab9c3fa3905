"""Which part of the device range finder moves the C3 trajectory?  The range
finder (compression.cpp:23-42) is rebuilt in torch on the GPU with one change
at a time from the exact reference algorithm (fp64 Householder, fp64 sketch),
and the device run takes the projectors through CNMF_DIAG_PROJ (it forms the
views itself):
  exact        fp64 everything (the reference's algorithm)
  om32         the Gaussian sketch rounded to fp32 (the device's sketch)
  store32      every range-finder product and basis rounded to fp32
  chol         CholeskyQR (one pass for intermediates, two for the final basis)
  chol32       chol + store32 + om32 (the device's algorithm in fp64 arithmetic)
  device       the device's own projectors (cnmf_build_projectors)
    python tools/rf_stages.py c3 exact om32 store32 chol chol32 device
"""
import os
import struct
import sys
import tempfile
import time

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


def r32(m):
    return m.float().double()


def qr_h(m):
    return torch.linalg.qr(m).Q


def qr_c(m, passes):
    for _ in range(passes):
        rr = torch.linalg.cholesky(m.T @ m, upper=True)
        m = torch.linalg.solve_triangular(rr, m, upper=True, left=False)
    return m


def dev_xs(s, tn):
    """the device X-stream kernel on s (fp64 -> fp32 operand), fp64 result"""
    sp = s.float().contiguous()
    out = torch.empty((n if tn else d, s.shape[1]), device="cuda")
    (ctx.xs_tn if tn else ctx.xs_nn)(x, sp, out)
    return out.double()


def dev_qr(m):
    """the device thin_qr (CholeskyQR2 / Householder fallback) on fp32 m"""
    mf = m.float().contiguous()
    out = torch.empty_like(mf)
    ctx.thin_qr(mf, out)
    return out.double()


first = {}


def rf(om, transpose, opts):
    st = r32 if "store32" in opts else (lambda m: m)
    cnt = [0]
    nlast = 2 * w + 1  # contractions per range finder

    if "devxs" in opts:
        def mm(a_is_t, s):
            cnt[0] += 1
            if "lastexact" in opts and cnt[0] == nlast:
                return x64.T @ s if a_is_t else x64 @ s
            if "firstexact" in opts and cnt[0] < nlast:
                return x64.T @ s if a_is_t else x64 @ s
            ndev = int(next((o[5:] for o in opts if o.startswith("first")
                             and o[5:].isdigit()), "0"))
            if ndev and cnt[0] > ndev:  # the first ndev contractions on the device, the rest exact
                return x64.T @ s if a_is_t else x64 @ s
            out = dev_xs(s, a_is_t)
            if "chk" not in first:
                ex = x64.T @ r32(s) if a_is_t else x64 @ r32(s)
                first["chk"] = ((out - ex).norm() / ex.norm()).item()
                print("  device contraction vs fp64 (same fp32 operand):", f"{first['chk']:.2e}", flush=True)
            return out
    else:
        def mm(a_is_t, s):
            return x64.T @ s if a_is_t else x64 @ s
    if "om32" in opts:
        om = r32(om)
    chol = "chol" in opts
    qr1 = (lambda m: st(qr_c(m, 1))) if chol else (lambda m: st(qr_h(m)))
    qr2 = (lambda m: st(qr_c(m, 2))) if chol else qr1
    if "devqr" in opts:
        qr1 = qr2 = dev_qr
    b = (qr2 if w == 0 else qr1)(st(mm(True, om) if transpose else mm(False, om)))
    for it in range(w):
        z = qr1(st(mm(False, b) if transpose else mm(True, b)))
        b = (qr2 if it + 1 == w else qr1)(st(mm(True, z) if transpose else mm(False, z)))
    return b


def pad(m):
    out = torch.zeros((m.shape[0], lp), dtype=torch.float32)
    out[:, :q] = m.float().cpu()
    return out.numpy()


xn = float(g["x_norm_sq"][0])
want = np.sqrt(2.0 * g["errors"] / xn)
cfg = cb.SolverConfig(algorithm=cb.FASTHALS_RP, k=k, sketch=cb.SketchConfig(q, w, 1),
                      max_iterations=iters, error_interval=every, rel_tolerance=1e-300, seed=1)
for tag in sys.argv[2:]:
    t0 = time.time()
    if tag == "device":
        left = torch.empty((d, q), device="cuda")
        right = torch.empty((q, n), device="cuda")
        ctx.build_projectors(x, q, w, 1, left, right)
        L, Rt = left.double(), right.double().T
    else:
        opts = {"exact": set(), "om32": {"om32"}, "store32": {"store32"}, "chol": {"chol"},
                "chol32": {"chol", "store32", "om32"},
                "devxs": {"chol", "store32", "om32", "devxs"},
                "devqr": {"store32", "om32", "devqr"},
                "devboth": {"store32", "om32", "devqr", "devxs"},
                "lastexact": {"store32", "om32", "devqr", "devxs", "lastexact"},
                "firstexact": {"store32", "om32", "devqr", "devxs", "firstexact"},
                "lastexact_c": {"chol", "store32", "om32", "devxs", "lastexact"},
                "first1": {"store32", "om32", "devqr", "devxs", "first1"},
                "first2": {"store32", "om32", "devqr", "devxs", "first2"},
                "first3": {"store32", "om32", "devqr", "devxs", "first3"}}[tag]
        L = rf(om_l, False, opts)
        Rt = rf(om_r, True, opts)
    torch.cuda.synchronize()
    t1 = time.time()
    path = os.path.join(tempfile.gettempdir(), "rf_stage.bin")
    with open(path, "wb") as f:
        f.write(struct.pack("<4q", d, n, lp, 0))
        f.write(pad(L).tobytes())
        f.write(pad(Rt).tobytes())
    os.environ["CNMF_DIAG_PROJ"] = path
    _, _, tr = ctx.run_device(x, cfg)
    del os.environ["CNMF_DIAG_PROJ"]
    got = np.sqrt(2.0 * np.array([r.error for r in tr.records]) / xn)
    dev = np.abs(got - want) / want
    print(f"{tag:8s} max dev {dev.max():.2e} ({t1 - t0:.1f} s + {time.time() - t1:.1f} s) | "
          + " ".join(f"{v:.1e}" for v in dev[::2]), flush=True)
