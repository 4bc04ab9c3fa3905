"""Diagnostic: apportion the C2 trajectory deviation between the compression
half and the HALS half by crossing GPU and oracle pipelines (20 iterations)."""
import os, sys
import numpy as np
import torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1712_02248_b200 as cb
from oracle import Oracle
o = Oracle(); ctx = cb.Context(0)
g = np.load(os.path.join(ROOT, "tests", "golden", "c2_full.npz"))
d, n, k, q, w, IT = 10000, 5000, 16, 36, 2, 20
x = o.synth_x(d, n, 16, 1, 1, 0.05, 1); x64 = x.astype(np.float64)
xn = float(np.sum(x64 ** 2))
want = np.sqrt(2 * g["errors"][:IT + 1] / xn)
dev = lambda t: torch.from_numpy(np.ascontiguousarray(t, dtype=np.float32)).cuda()
def report(label, errs):
    got = np.sqrt(2 * np.array(errs) / xn)
    dv = np.abs(got - want[1:len(got) + 1]) / want[1:len(got) + 1]
    print("%-40s max dev %.2e at it %d" % (label, dv.max(), dv.argmax() + 1), flush=True)
# GPU compression
xd = dev(x)
Lg = torch.empty((d, q), device="cuda"); Rg = torch.empty((q, n), device="cuda")
ctx.build_projectors(xd, q, w, 1, Lg, Rg)
xhg = torch.empty((q, n), device="cuda"); xcg = torch.empty((d, q), device="cuda")
ctx.compress(xd, Lg, Rg, xhg, xcg)
Lg, Rg, xhg, xcg = [t.cpu().numpy().astype(np.float64) for t in (Lg, Rg, xhg, xcg)]
# oracle compression
Lo, Ro = o.build_projectors(x64, q, w, 1)
xho, xco = o.compress(x64, Lo, Ro)
def oracle_hals(L, R, xh, xc):
    a, b = o.initialize(d, n, k, 1); ah, bc = o.compress_factors(a, b, L, R); rng = o.rng(1)
    errs = []
    for _ in range(IT):
        o.fasthals_rp_step(xh, xc, a, b, ah, bc, L, R, True, 0.0, 0.0, rng)
        errs.append(o.reconstruction_error(x64, a, b))
    return errs
def gpu_hals(L, R, xh, xc):
    a, b = o.initialize(d, n, k, 1); ah, bc = o.compress_factors(a, b, L, R)
    ta, tb = dev(a), dev(b)
    tah = torch.from_numpy(ah).cuda(); tbc = torch.from_numpy(bc).cuda()
    args = [dev(xh), dev(xc), dev(L), dev(R)]
    errs = []
    for i in range(IT):
        ctx.fasthals_rp_steps(*args, ta, tb, tah, tbc, True, 0.0, 0.0, 1, 1)
        errs.append(ctx.reconstruction_error(xd, ta, tb))
    return errs
report("oracle compression + oracle HALS", oracle_hals(Lo, Ro, xho, xco))
report("GPU compression    + oracle HALS", oracle_hals(Lg, Rg, xhg, xcg))
report("oracle compression + GPU HALS", gpu_hals(Lo, Ro, xho, xco))
report("GPU compression    + GPU HALS", gpu_hals(Lg, Rg, xhg, xcg))
