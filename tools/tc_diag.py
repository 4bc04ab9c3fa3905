"""Locate wrong outputs of the tcgen05 X-stream kernel for one NN case and test
whether the error equals missing / duplicated K-block contributions."""
import os, sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
import paper_1712_02248_b200 as cb
d, n, l = [int(v) for v in sys.argv[1:4]]
ctx = cb.Context(0)
rng = np.random.default_rng(3)
x = rng.random((d, n), dtype=np.float32)
s = rng.standard_normal((n, l)).astype(np.float32)
y = torch.empty((d, l), device="cuda")
ctx.xs_nn(torch.from_numpy(x).cuda(), torch.from_numpy(s).cuda(), y)
got = y.cpu().numpy().astype(np.float64)
ref = x.astype(np.float64) @ s.astype(np.float64)
err = got - ref
rel_row = np.linalg.norm(err, axis=1) / np.linalg.norm(ref, axis=1)
bad = np.where(rel_row > 1e-5)[0]
print("bad rows:", len(bad), "tiles:", sorted(set((bad // 128).tolist()))[:20], "row%128 sample:", sorted(set((bad % 128).tolist()))[:40])
if len(bad):
    r = bad[0]
    kb = n // 32
    contrib = np.stack([x[r, 32 * b:32 * b + 32].astype(np.float64) @ s[32 * b:32 * b + 32].astype(np.float64) for b in range(kb)])
    # find single block b with err[r] ~ +/- contrib[b]
    res = [np.linalg.norm(err[r] - sgn * contrib[b]) / np.linalg.norm(err[r]) for b in range(kb) for sgn in (1, -1)]
    i = int(np.argmin(res))
    print(f"row {r}: |err|={np.linalg.norm(err[r]):.3e} best single-block match block {i // 2} sign {'+-'[i % 2]} resid {res[i]:.3f}")
    print("err row first 8:", np.round(err[r, :8], 4))
    kc = int(os.environ.get("CNMF_TC_KCHUNK", "0"))
    if kc:
        for r in bad[:6]:
            parts = [x[r, a:a + kc].astype(np.float64) @ s[a:a + kc].astype(np.float64) for a in range(0, n, kc)]
            res = [(np.linalg.norm(err[r] - sg * p) / np.linalg.norm(err[r]), i, sg) for i, p in enumerate(parts) for sg in (1, -1)]
            best = min(res)
            # also: difference between two units (one unit's partial written in place of another's)
            print(f"row {r} (tile {r // 128}, lane {r % 32}, warp {(r % 128) // 32}): unit match resid {best[0]:.3f} split {best[1]} sign {best[2]:+d}")
