"""C3 full-size run on the device against tests/golden/c3_full.npz, printing
the per-record trajectory deviation and the run Rng positions (redraw events)
next to the reference's.  Run once per X-stream variant (CNMF_XS=tf32|simt|f16)
to separate the compression's precision from the HALS path:

    CNMF_XS=simt python tools/c3_gpu_variants.py [c3|c4] [out.npz]
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1712_02248_b200 as cb  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c3"
g = np.load(os.path.join(os.path.dirname(__file__), "..", "tests", "golden", f"{name}_full.npz"))
d, n, rank, fk, nk, dseed, k, q, w, iters, every = (int(v) for v in g["config"])
ctx = cb.Context(0)
xb = torch.empty((d, (n + 3) // 4 * 4), dtype=torch.float32, device="cuda")
ctx.synth_x(d, n, rank, fk, nk, float(g["sigma"][0]), dseed, xb)
x = xb[:, :n]
cfg = cb.SolverConfig(algorithm=cb.FASTHALS_RP, k=k, sketch=cb.SketchConfig(q, w, 1),
                      max_iterations=iters, error_interval=every, rel_tolerance=1e-300, seed=1)
a, b, tr = ctx.run_device(x, cfg)
xn = float(g["x_norm_sq"][0])
got = np.sqrt(2.0 * np.array([r.error for r in tr.records]) / xn)
want = np.sqrt(2.0 * g["errors"] / xn)
draws = np.concatenate([[0], np.cumsum(g["step_draws"])])
print("variant", os.environ.get("CNMF_XS", "default"), name)
for i, r in enumerate(tr.records):
    print(f"it {r.iteration:4d} err {got[i]:.9f} ref {want[i]:.9f} dev {abs(got[i]-want[i])/want[i]:.2e} "
          f"draws {r.rng_draws} ref {int(draws[g['iters'][i]])}")
# the final objective recomputed in fp64 (torch, row chunks) from the run's
# own final factors: separates factor accuracy from objective-evaluation accuracy
a64, b64 = a.double(), b.double()
tot = 0.0
for r0 in range(0, d, 4096):
    rr = x[r0:r0 + 4096].double() - a64[r0:r0 + 4096] @ b64.T
    tot += float((rr * rr).sum())
e64 = np.sqrt(tot / xn)
print(f"final objective: device {got[-1]:.9f}  fp64(torch) {e64:.9f}  reference {want[-1]:.9f}  "
      f"device-vs-fp64 {abs(got[-1] - e64) / e64:.2e}  fp64-vs-ref {abs(e64 - want[-1]) / want[-1]:.2e}")
af = a.double().cpu().numpy(); bf = b.double().cpu().numpy()
for nm, gf, rf in (("A", af, g["a"]), ("B", bf, g["b"])):
    rf = rf.astype(np.float64)
    print(nm, "relF", np.linalg.norm(gf - rf) / np.linalg.norm(rf), "max", np.abs(gf - rf).max() / np.abs(rf).max())
if len(sys.argv) > 2:
    np.savez(sys.argv[2], err=got)
