"""Full-size C4 run against tests/golden/c4_full.npz: trajectory deviation per record, redraw
positions and factor errors (diagnostics for the range-finder arithmetic; set CNMF_RF /
CNMF_XS_EXACT / CNMF_RF64 in the environment)."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
import torch
import paper_1712_02248_b200 as cb

name = sys.argv[1] if len(sys.argv) > 1 else "c4"
g = np.load(os.path.join(ROOT, "tests", "golden", f"{name}_full.npz"))
d, n, rank, fk, nk, dseed, k, q, w, iters, every = (int(v) for v in g["config"])
sigma = float(g["sigma"][0])
ctx = cb.Context(0)
xb = torch.empty((d, (n + 3) // 4 * 4), dtype=torch.float32, device="cuda")
ctx.synth_x(d, n, rank, fk, nk, sigma, dseed, xb)
x = xb[:, :n]
cfg = cb.SolverConfig(algorithm=cb.FASTHALS_RP, k=k, sketch=cb.SketchConfig(q, w, 1),
                      max_iterations=iters, error_interval=every, rel_tolerance=1e-300, seed=1)
a, b, tr = ctx.run_device(x, cfg)
xn = float(g["x_norm_sq"][0])
got = np.sqrt(2.0 * np.array([r.error for r in tr.records]) / xn)
want = np.sqrt(2.0 * g["errors"] / xn)
dev = np.abs(got - want) / want
print("env", {e: os.environ.get(e) for e in ("CNMF_RF", "CNMF_RF64", "CNMF_XS_EXACT", "CNMF_XS")})
print("kappa", tr.sketch_kappa, "rf64", tr.range_finder_fp64, "compress ms", 1e3 * tr.compress_seconds)
print("deviation per record:", " ".join(f"{v:.1e}" for v in dev), " max", f"{dev.max():.2e}")
draws = np.concatenate([[0], np.cumsum(g["step_draws"])])
mine = [r.rng_draws for r in tr.records]
ref = [int(draws[i]) for i in g["iters"]]
print("draws equal:", mine == ref, mine[:4], ref[:4])
for nm, gotf, reff in (("A", a, g["a"]), ("B", b, g["b"])):
    gf = gotf.double().cpu().numpy(); rf = reff.astype(np.float64)
    if rf.shape != gf.shape: gf = gf[:: gf.shape[0] // rf.shape[0]]
    print(nm, "relF", np.linalg.norm(gf - rf) / np.linalg.norm(rf), "max", np.abs(gf - rf).max() / np.abs(rf).max())
