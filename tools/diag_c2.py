"""Diagnostic: GPU C2 trajectory vs the committed reference trajectory."""
import os, sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1712_02248_b200 as cb
from oracle import Oracle
o = Oracle()
g = np.load(os.path.join(ROOT, "tests", "golden", "c2_full.npz"))
x = o.synth_x(10000, 5000, 16, 1, 1, 0.05, 1)
xn = float(np.sum(x.astype(np.float64) ** 2))
cfg = cb.SolverConfig(algorithm=cb.FASTHALS_RP, k=16, sketch=cb.SketchConfig(36, 2, 1),
                      max_iterations=200, error_interval=1, rel_tolerance=1e-300, seed=1)
res = cb.Context(0).run(x, cfg)
got = np.sqrt(2 * np.array([r.error for r in res.trace.records]) / xn)
want = np.sqrt(2 * g["errors"] / xn)
dev = np.abs(got - want) / want
print("max dev %.3e at it %d; dev at 1,5,10,15,20,50,100,200:" % (dev.max(), dev.argmax()),
      " ".join("%.1e" % dev[i] for i in (1, 5, 10, 15, 20, 50, 100, 200)))
print("redraws", res.trace.redraws)
