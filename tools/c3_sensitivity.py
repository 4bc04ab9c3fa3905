"""Compare the sensitivity runs' error trajectories (tools/c3_sensitivity.sh,
stderr logs "iter N err E ...") with tests/golden/c3_full.npz: relative
deviation of sqrt(2 err / ||X||^2) per record."""
import re
import sys

import numpy as np

g = np.load("tests/golden/c3_full.npz")
xn = float(g["x_norm_sq"][0])
want = dict(zip(g["iters"].tolist(), np.sqrt(2 * g["errors"] / xn)))
for path in sys.argv[1:]:
    got = {int(m.group(1)): float(m.group(2)) for m in re.finditer(r"iter (\d+) err (\S+)", open(path).read())}
    dev = [(it, abs(np.sqrt(2 * e / xn) - want[it]) / want[it]) for it, e in sorted(got.items())]
    print(path, " ".join(f"{it}:{d:.1e}" for it, d in dev))
    print("  max", max(d for _, d in dev) if dev else None)
