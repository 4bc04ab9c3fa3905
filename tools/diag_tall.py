import sys, os, numpy as np, torch
sys.path.insert(0, os.getcwd())
import paper_1712_02248_b200 as cb
from oracle import Oracle
o = Oracle(); ctx = cb.Context(0)
d, n, k, q = int(sys.argv[2]), int(sys.argv[3]), 6, 10
rank = int(sys.argv[4]) if len(sys.argv) > 4 else 5
x = o.synth_x(d, n, rank, 0, 1, 0.01, 12).astype(np.float64)
mode = sys.argv[1]
if mode == "proj":
    cfg = cb.SolverConfig(algorithm=cb.FASTHALS_RP, k=k, sketch=cb.SketchConfig(q, 1, 1), max_iterations=0, error_interval=1, rel_tolerance=1e-300, seed=1)
    res = ctx.run(x.astype(np.float32), cfg); print("proj+0 iters ok")
else:
    left, right = o.build_projectors(x, q, 1, 2)
    xhat, xcheck = o.compress(x, left, right)
    a, b = o.initialize(d, n, k, 4)
    ah, bc = o.compress_factors(a, b, left, right)
    f32 = lambda z: torch.from_numpy(np.ascontiguousarray(z, dtype=np.float32)).cuda()
    f64 = lambda z: torch.from_numpy(np.ascontiguousarray(z, dtype=np.float64)).cuda()
    ta, tb, tah, tbc = f32(a), f32(b), f64(ah), f64(bc)
    nr = ctx.fasthals_rp_steps(f32(xhat), f32(xcheck), f32(left), f32(right), ta, tb, tah, tbc, True, 0.0, 0.0, 5, 2)
    torch.cuda.synchronize(); print("steps ok, redraws", nr)
