"""CPU experiment: how precise must the compression be for 1e-4 trajectory
parity on a C3-class (low-noise) problem?

The reference computes everything in fp64.  This script runs the oracle's
FastHALS-RP loop (fp64) on compressed views that carry modelled GPU errors
and reports the relative-error trajectory deviation from the exact run:

  fp32_views   L, R rounded to fp32, X-hat / X-check from them, rounded to fp32
  xview_1e-6   exact L, R; X-hat / X-check times (1 + 1e-6 N(0,1)) entrywise
  xview_1e-7   the same at 1e-7
  span_1e-7    L, R times (1 + 1e-7 N(0,1)) then re-orthonormalised (fp64)

    python tools/precision_budget.py [d n]
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from oracle import Oracle  # noqa: E402


def rel_err(x, a, b, xn):
    r = x - a @ b.T
    return np.sqrt(np.sum(r * r) / xn)


def trajectory(o, x, xn, left, right, xhat, xcheck, k, iters=100, every=5):
    d, n = x.shape
    a, b = o.initialize(d, n, k, 1)
    ah, bc = o.compress_factors(a, b, left, right)
    rg = o.rng(1)
    for _ in range((d + n) * k):  # the run Rng after initialize()
        o.lib.orc_rng_uniform_positive(rg)
    out = [rel_err(x, a, b, xn)]
    for it in range(1, iters + 1):
        o.fasthals_rp_step(xhat, xcheck, a, b, ah, bc, left, right, True, 0.0, 0.0, rg)
        if it % every == 0:
            out.append(rel_err(x, a, b, xn))
    return np.array(out)


def main():
    d = int(sys.argv[1]) if len(sys.argv) > 1 else 20000
    n = int(sys.argv[2]) if len(sys.argv) > 2 else 10000
    k, q, w = 50, 70, 2
    o = Oracle()
    x = o.synth_x(d, n, 50, 0, 1, 0.01, 1).astype(np.float64)
    xn = float(np.sum(x * x))
    left, right = o.build_projectors(x, q, w, 1)
    xhat, xcheck = o.compress(x, left, right)
    ref = trajectory(o, x, xn, left, right, xhat, xcheck, k)
    print("reference final relative error", ref[-1], flush=True)
    rng = np.random.default_rng(0)

    def orth(m):
        return np.linalg.qr(m)[0]

    variants = {}
    l32, r32 = left.astype(np.float32).astype(np.float64), right.astype(np.float32).astype(np.float64)
    xh32, xc32 = o.compress(x, l32, r32)
    variants["fp32_views"] = (l32, r32, xh32.astype(np.float32).astype(np.float64),
                              xc32.astype(np.float32).astype(np.float64))
    for eps in (1e-6, 1e-7):
        variants[f"xview_{eps:g}"] = (left, right, xhat * (1 + eps * rng.standard_normal(xhat.shape)),
                                      xcheck * (1 + eps * rng.standard_normal(xcheck.shape)))
    lp = orth(left * (1 + 1e-7 * rng.standard_normal(left.shape)))
    rp = orth((right * (1 + 1e-7 * rng.standard_normal(right.shape))).T).T.copy()
    xhp, xcp = o.compress(x, lp, rp)
    variants["span_1e-7"] = (lp, rp, xhp, xcp)
    for name, (l_, r_, xh_, xc_) in variants.items():
        t = trajectory(o, x, xn, np.ascontiguousarray(l_), np.ascontiguousarray(r_),
                       np.ascontiguousarray(xh_), np.ascontiguousarray(xc_), k)
        dev = np.abs(t - ref) / ref
        print(f"{name:12s} max {dev.max():.2e} |", " ".join(f"{v:.1e}" for v in dev), flush=True)


if __name__ == "__main__":
    main()
