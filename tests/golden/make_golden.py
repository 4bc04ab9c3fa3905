"""Generates tests/golden/*.npz from the REFERENCE itself (oracle/_ref).

The reference ships no golden vectors, so the fixtures
are outputs of the unmodified reference library compiled from its own
sources (oracle/Makefile `ref` target), on inputs this repo can regenerate
anywhere (mt19937_64 streams and the oracle's counter-based synthetic
generator).  Run here, where /root/reference is mounted:

    make -C oracle ref && python tests/golden/make_golden.py

The GPU box has no /root/reference; tests read only these committed files.
"""
import argparse
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from oracle import FASTHALS, FASTHALS_RP, Oracle, Reference  # noqa: E402


def x_summary(x):
    x = x.astype(np.float64)
    return np.array([x.sum(), (x * x).sum(), x[0, 0], x[-1, -1], x.max()])


def main():
    ap = argparse.ArgumentParser()
    ap.parse_args()
    o, r = Oracle(), Reference()

    # 1. variate streams (rng.hpp:17-44) and gaussian_sketch / initialize
    streams = {}
    for seed in (1, 2, 3, 5489):
        streams[f"u64_{seed}"] = r.draws(seed, 0, 64)
    streams["uniform_7"] = r.draws(7, 1, 64)
    streams["uniform_positive_1"] = r.draws(1, 2, 64)
    streams["normal_2"] = r.draws(2, 3, 65)
    streams["sketch_7x5_11"] = r.gaussian_sketch(7, 5, 11)
    a, b = r.initialize(4, 3, 2, 99)
    streams["init_a_4x2_99"], streams["init_b_3x2_99"] = a, b
    np.savez_compressed(os.path.join(HERE, "streams.npz"), **streams)

    # 2. small cases: projectors, one-step state, full runs (bitwise pins)
    small = {}
    x = o.synth_x(60, 45, 5, 0, 1, 0.01, 3).astype(np.float64)
    small["x_summary"] = x_summary(x)
    small["left"], small["right"] = r.build_projectors(x, 10, 2, 4)
    q, rr = r.thin_qr(x[:, :12])
    small["qr_q"], small["qr_r"] = q, rr
    for tag, kw in {"rp": dict(k=4, q=10, w=2, max_iterations=50, error_interval=1,
                               rel_tolerance=1e-300, sketch_seed=4, seed=2),
                    "rp_pen": dict(k=3, q=8, w=1, max_iterations=20, error_interval=3,
                                   rel_tolerance=1e-300, alpha=0.05, beta=0.2, seed=6),
                    "dense": dict(k=4, max_iterations=30, algorithm=FASTHALS)}.items():
        A, B, t = r.run(x, **kw)
        small[f"{tag}_a"], small[f"{tag}_b"] = A, B
        small[f"{tag}_iters"] = np.array(t.iterations)
        small[f"{tag}_errors"] = np.array(t.errors)
        small[f"{tag}_gini"] = np.array([t.gini_b])
        small[f"{tag}_status"] = np.array([t.status, t.iterations_run])
    # all-zero start on a square sketch (test_solvers.cpp:394-413): redraw path
    xs = r.draws(9, 1, 144).reshape(12, 12)
    lz, rz = r.build_projectors(xs, 12, 0, 5)
    xh, xc = o.compress(xs, lz, rz)
    za, zb = np.zeros((12, 2)), np.zeros((12, 2))
    zah, zbc = o.compress_factors(za, zb, lz, rz)
    r.fasthals_rp_steps(xh, xc, lz, rz, za, zb, zah, zbc, 3, 1)
    small["zero_a"], small["zero_b"] = za, zb
    np.savez_compressed(os.path.join(HERE, "small.npz"), **small)

    # 3. C1 (BASELINE configs[0]) full size, error at every iteration
    x1 = o.synth_x(1000, 1000, 20, 0, 1, 0.01, 1)
    A, B, t = r.run(x1.astype(np.float64), 20, q=30, w=2, max_iterations=100, error_interval=1,
                    rel_tolerance=1e-300, sketch_seed=1, seed=1)
    np.savez_compressed(os.path.join(HERE, "c1.npz"), x_summary=x_summary(x1),
                        iters=np.array(t.iterations), errors=np.array(t.errors),
                        a=A.astype(np.float32), b=B.astype(np.float32),
                        gini=np.array([t.gini_b]), update_seconds=np.array([t.update_seconds]))

    # C2, C3 and C4 at full size: tests/golden/make_golden_big.py
    print("golden fixtures written to", HERE)


if __name__ == "__main__":
    main()
