"""Full-size reference trajectories for BASELINE configs C2, C3 and C4.

Runs oracle/_ref/golden_big -- the unmodified reference library (compiled
from /root/reference/proj/src by `make -C oracle ref`) driven step by step
through its public functions (see oracle/golden_big.cpp) -- on the repo's
seeded synthetic X at the full BASELINE sizes, and packs the result into
tests/golden/<config>_full.npz:

    iters, errors       the RunTrace records (iteration 0 and every
                        `error_interval`-th, error = 1/2 ||X - A B^T||^2)
    step_draws          raw mt19937_64 draws each fasthals_rp_step took from
                        the run Rng (its dead-component redraws)
    a, b                the final factors, fp32 (d x k, n x k); C4 keeps every
                        a_row_stride-th / b_row_stride-th row (2 / 4: a 16 MB
                        fixture instead of 42) together with the fp64 column
                        sums and sums of squares over ALL rows
                        (a_colsum, a_colsumsq, b_colsum, b_colsumsq)
    x_hash, x_sums      per-1000-row-block checksums of X's fp32 bits and its
                        fp64 sum / sum of squares (the GPU tests check their
                        device-generated X against these first)
    seconds             reference timings on this host (1 core per step)

Run here, where /root/reference exists (C3 ~25 min, C4 ~70 min, 44 GB RAM):

    make -C oracle ref && python tests/golden/make_golden_big.py c2 c3 c4
"""
import os
import subprocess
import sys
import tempfile

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
BIN = os.path.join(ROOT, "oracle", "_ref", "golden_big")

# name: (d, n, rank, factor_kind, noise_kind, sigma, data_seed, k, q, w, iterations, interval)
CONFIGS = {
    "c2": (10000, 5000, 16, 1, 1, 0.05, 1, 16, 36, 2, 200, 1),
    "c3": (100000, 20000, 50, 0, 1, 0.01, 1, 50, 70, 2, 100, 5),
    "c4": (50000, 100000, 100, 2, 2, 0.0, 1, 100, 120, 1, 100, 5),
}


# rows of the final factors kept in the fixture (all rows when absent)
ROW_STRIDE = {"c4": {"a": 2, "b": 4}}


def main(names):
    for name in names:
        d, n, rank, fk, nk, sigma, dseed, k, q, w, iters, interval = CONFIGS[name]
        with tempfile.TemporaryDirectory() as tmp:
            cmd = [BIN, tmp] + [str(v) for v in (d, n, rank, fk, nk, sigma, dseed, k, q, w,
                                                  iters, interval, 1, os.cpu_count() or 8)]
            print(" ".join(cmd), flush=True)
            subprocess.run(cmd, check=True)
            meta = dict(l.strip().split("=") for l in open(os.path.join(tmp, "meta.txt")))

            def f64(x):
                return np.fromfile(os.path.join(tmp, x), dtype=np.float64)

            sums = f64("x_sums.f64").reshape(-1, 2)
            out = dict(
                config=np.array([d, n, rank, fk, nk, dseed, k, q, w, iters, interval]),
                sigma=np.array([sigma]),
                iters=f64("rec_iter.f64").astype(np.int64),
                errors=f64("rec_err.f64"),
                step_draws=f64("step_draws.f64").astype(np.int64),
                a=f64("a.f64").reshape(d, k).astype(np.float32),
                b=f64("b.f64").reshape(n, k).astype(np.float32),
                x_hash=np.fromfile(os.path.join(tmp, "x_hash.u64"), dtype=np.uint64),
                x_sums=sums,
                x_norm_sq=np.array([sums[:, 1].sum()]),
                gini=np.array([float(meta["gini_b"])]),
                seconds=np.array([float(meta["build_projectors_seconds"]),
                                  float(meta["compress_seconds"]),
                                  float(meta["update_seconds"])]),
            )
            for nm, stride in ROW_STRIDE.get(name, {}).items():
                f = out[nm].astype(np.float64)
                out[nm + "_colsum"] = f.sum(axis=0)
                out[nm + "_colsumsq"] = (f * f).sum(axis=0)
                out[nm + "_row_stride"] = np.array([stride])
                out[nm] = out[nm][::stride].copy()
            path = os.path.join(HERE, f"{name}_full.npz")
            np.savez_compressed(path, **out)
            print(f"{name}: {len(out['errors'])} records, "
                  f"{int((out['step_draws'] > 0).sum())} steps with redraws, wrote {path}",
                  flush=True)


if __name__ == "__main__":
    main(sys.argv[1:] or ["c2", "c3", "c4"])
