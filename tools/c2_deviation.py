import os, sys, numpy as np
sys.path.insert(0, os.getcwd())
import paper_1712_02248_b200 as cb
from oracle import Oracle
o = Oracle(); ctx = cb.Context(0)
g = np.load("tests/golden/c2_full.npz")
x = o.synth_x(10000, 5000, 16, 1, 1, 0.05, 1)
xn = float(np.sum(x.astype(np.float64) ** 2))
cfg = cb.SolverConfig(algorithm=cb.FASTHALS_RP, k=16, sketch=cb.SketchConfig(36, 2, 1), max_iterations=200, error_interval=1, rel_tolerance=1e-300, seed=1)
for mode in ("tf32", "f16"):
    os.environ["CNMF_XS"] = mode
    res = ctx.run(x, cfg)
    got = np.sqrt(2 * np.array([r.error for r in res.trace.records]) / xn)
    want = np.sqrt(2 * np.array(g["errors"]) / xn)
    dev = np.abs(got - want) / want
    print(mode, "max dev %.3e at it %d; dev at it 10/50/100/200: %s" % (dev.max(), dev.argmax(), [f"{dev[i]:.1e}" for i in (10, 50, 100, 200)]), "redraws", res.trace.redraws)
