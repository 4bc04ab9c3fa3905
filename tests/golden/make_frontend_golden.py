"""Golden fixtures for the `cnmf` front end (paper_1712_02248_b200/cli.py),
all produced by the reference itself, here where /root/reference is mounted:

* json_dump.txt -- nlohmann::json's rendering of a battery of doubles and of one
  nested object (oracle/json_pin.cpp), the library the reference's cli.cpp
  writes trace.json / summary.json / distortion.json with;
* frontend.npz -- generate_synthetic outputs (data_io.cpp:383-415),
  pairwise_distortion on exactly-projectable inputs (metrics.cpp:123-155), and
  the reference's run / build_projectors / compress on the synthetic matrix of
  the reference's own CLI tests (test_cli.cpp:41-46).

    make -C oracle ref && python tests/golden/make_frontend_golden.py
"""
import os
import struct
import subprocess

import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
BIN = os.path.join(os.path.dirname(os.path.dirname(HERE)), "oracle", "_ref", "json_pin")


def battery():
    vals = [0.0, -0.0, 1.0, -1.0, 0.5, 0.1, 1 / 3, 2 / 3, 12.25, 1e-4, 1e-5, 1.5e-4, 0.00012345,
            1e14, 1e15, 1e16, 1e17, 123456789012345.0, 1234567890123456.0, 9007199254740993.0,
            1e21, 1e22, 1e100, 1e-100, 5e-324, 2.2250738585072014e-308, 1.7976931348623157e308,
            -2.5e-7, 3.0e8, 6.02214076e23, 1e-9, 1e-300, float("nan"), float("inf"),
            -float("inf"), 4.0 * 12 * 10 * 2, (2.0 * 9 + 5) * (100 + 80), 0.001, 0.01]
    rng = np.random.default_rng(1712)
    for e in range(-12, 20):
        vals.extend((rng.random(3) * 10.0 ** e).tolist())
    vals.extend((rng.standard_normal(20) * 1e3).tolist())
    vals.extend(float(np.float32(v)) for v in rng.random(20))
    # random bit patterns over the whole finite range, subnormals included
    bits = rng.integers(0, 0x7FF0000000000000, size=1500, dtype=np.uint64)
    vals.extend(bits.view(np.float64).tolist())
    vals.extend((rng.random(300) * 1e6).astype(np.float32).astype(np.float64).tolist())
    return vals


SYNTH_SPECS = [(12, 10, 2, 0.5, 0.05, 7), (30, 20, 3, 1.0, 0.0, 3), (40, 25, 4, 0.0, 0.2, 9),
               (9, 9, 9, 2.0, 0.0, 1)]
CLI_SPEC = (12, 10, 2, 0.5, 0.05, 7)   # test_cli.cpp:41-46 synth_args()


def frontend(r):
    sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
    from oracle import FASTHALS_RP  # noqa: E402
    HALS_RP = 3                     # cnmf::Algorithm::hals_rp (algorithm.hpp:8-15)
    g = {}
    for i, spec in enumerate(SYNTH_SPECS):
        g[f"synth_spec_{i}"] = np.array(spec, dtype=np.float64)
        g[f"synth_{i}"] = r.generate_synthetic(*spec)
    # distortion on inputs whose projection L^T X is exact in fp32 (L selects rows)
    rng = np.random.default_rng(2248)
    for i, (d, n, q, pairs, seed) in enumerate([(16, 12, 5, 50, 3), (8, 3, 2, 1000, 11),
                                                 (20, 40, 6, 200, 1)]):
        x = rng.integers(0, 64, size=(d, n)).astype(np.float64) / 8.0
        rows = np.sort(rng.choice(d, size=q, replace=False))
        left = np.zeros((d, q))
        left[rows, np.arange(q)] = 1.0
        g[f"dist_x_{i}"], g[f"dist_left_{i}"] = x, left
        g[f"dist_args_{i}"] = np.array([pairs, seed], dtype=np.float64)
        g[f"dist_out_{i}"] = np.array(r.pairwise_distortion(x, left, pairs, seed))
    # the reference's own runs on the CLI test matrix (cli.cpp make_config:
    # the run seed is also the sketch seed)
    x = r.generate_synthetic(*CLI_SPEC)
    for tag, kw in {"fh": dict(algorithm=FASTHALS_RP, k=2, q=6, w=4, seed=3, sketch_seed=3,
                               max_iterations=40, error_interval=5, rel_tolerance=1e-300),
                    "cfg": dict(algorithm=FASTHALS_RP, k=3, q=6, w=4, seed=1, sketch_seed=1,
                                max_iterations=7, error_interval=5, rel_tolerance=1e-300),
                    "hrp": dict(algorithm=HALS_RP, k=2, q=5, w=2, seed=5, sketch_seed=5,
                                max_iterations=30, error_interval=3, rel_tolerance=1e-300,
                                alpha=0.01, beta=0.02),
                    # test_cli.cpp:85-130: the default algorithm, default tolerance
                    "fhd": dict(algorithm=4, k=2, seed=3, sketch_seed=3, max_iterations=40,
                                error_interval=5, rel_tolerance=1e-9, w=0)}.items():
        a, b, t = r.run(x, **kw)
        g[f"run_{tag}_a"], g[f"run_{tag}_b"] = a, b
        g[f"run_{tag}_iter"] = np.array(t.iterations, dtype=np.int64)
        g[f"run_{tag}_err"] = np.array(t.errors)
        g[f"run_{tag}_meta"] = np.array([t.status, t.iterations_run, t.gini_b])
    left, right, xhat, xcheck, _ = r.compress(x, 5, 2, 3)
    g["proj_xhat"], g["proj_xcheck"] = xhat, xcheck
    g["proj_dist"] = np.array(r.pairwise_distortion(x, left, 50, 3))
    np.savez_compressed(os.path.join(HERE, "frontend.npz"), **g)


sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))


def main():
    lines = "".join("%016x\n" % struct.unpack("<Q", struct.pack("<d", v))[0] for v in battery())
    out = subprocess.run([BIN], input=lines, capture_output=True, text=True, check=True).stdout
    with open(os.path.join(HERE, "json_dump.txt"), "w") as f:
        f.write(out)
    from oracle import Reference  # noqa: E402
    frontend(Reference())


if __name__ == "__main__":
    main()
