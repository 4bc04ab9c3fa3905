"""CPU tests of the `cnmf` front end (paper_1712_02248_b200/cli.py) and the
host-side data formats around the path (csrc/data_io.cpp), modelled on the
reference's proj/tests/test_cli.cpp and test_data_io.cpp.  Nothing here
launches a kernel: the factorizations themselves are in tests/test_gpu_cli.py.

Pins, all against outputs of the reference itself (tests/golden/
make_frontend_golden.py): nlohmann::json's number/object rendering,
generate_synthetic bit for bit, pairwise_distortion bit for bit.
"""
import json
import math
import os
import struct

import numpy as np
import pytest

import paper_1712_02248_b200 as cb
from paper_1712_02248_b200 import cli

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
SYNTH = ["--format", "synthetic", "--rows", "12", "--cols", "10", "--rank", "2", "--decay",
         "0.5", "--noise", "0.05", "--data-seed", "7"]   # test_cli.cpp:41-46


@pytest.fixture(scope="module")
def golden():
    return np.load(os.path.join(GOLD, "frontend.npz"))


# ------------------------------------------------------------ JSON writer --
def _json_lines():
    nums, obj, in_obj = [], [], False
    for line in open(os.path.join(GOLD, "json_dump.txt")).read().split("\n"):
        if line == "OBJECT":
            in_obj = True
        elif in_obj:
            obj.append(line)
        elif line:
            bits, text = line.split(" ", 1)
            nums.append((struct.unpack("<d", struct.pack("<Q", int(bits, 16)))[0], text))
    return nums, "\n".join(obj).rstrip("\n")


def test_json_numbers_match_nlohmann():
    nums, _ = _json_lines()
    assert len(nums) > 150
    for v, text in nums:
        assert cli.json_dump(v) == text, (repr(v), text)


def test_json_object_layout_matches_nlohmann():
    _, obj = _json_lines()
    tree = {"zeta": 1, "alpha": 0.5, "nan": float("nan"), "text": 'a"b\\c\n\t\x01 end',
            "empty": [], "flag": False, "size": 18446744073709551615,
            "records": [{"iteration": 0, "error": 12.25, "elapsed_seconds": 1e-7},
                        {"iteration": 5, "error": 3.0, "elapsed_seconds": 0.125}]}
    assert cli.json_dump(tree) == obj


# ------------------------------------------------------ data formats (host) --
def test_generate_synthetic_bitwise(golden):
    for i in range(4):
        d, n, r, decay, noise, seed = golden[f"synth_spec_{i}"].tolist()
        x = cb.generate_synthetic(int(d), int(n), int(r), decay, noise, int(seed))
        assert np.array_equal(x, golden[f"synth_{i}"]), i
        assert (x >= 0).all()


def test_generate_synthetic_validation():
    # data_io.cpp:384-389
    with pytest.raises(cb.ConfigError):
        cb.generate_synthetic(0, 5, 1)
    with pytest.raises(cb.ConfigError):
        cb.generate_synthetic(5, 4, 5)
    with pytest.raises(cb.ConfigError):
        cb.generate_synthetic(5, 5, 2, decay_p=-1.0)
    with pytest.raises(cb.ConfigError):
        cb.generate_synthetic(5, 5, 2, noise_level=float("nan"))


def test_pairwise_distortion_bitwise(golden):
    for i in range(3):
        x, left = golden[f"dist_x_{i}"], golden[f"dist_left_{i}"]
        pairs, seed = (int(v) for v in golden[f"dist_args_{i}"])
        xhat = (left.T @ x).astype(np.float32)      # exact: left selects rows
        got = cb.pairwise_distortion(x, xhat, pairs, seed)
        assert got == tuple(golden[f"dist_out_{i}"].tolist()), i
    with pytest.raises(cb.InputError):
        cb.pairwise_distortion(np.ones((3, 1)), np.ones((2, 1), np.float32), 5, 1)
    with pytest.raises(cb.InputError):
        cb.pairwise_distortion(np.ones((3, 4)), np.ones((2, 4), np.float32), 0, 1)


def test_estimate_cost_model():
    # metrics.cpp:20-50, test_cli.cpp:309-328
    e = cb.estimate_cost("mu", 100, 80, 5, 0)
    assert e.flops_per_iteration == 8.0 * 100 * 80 * 5
    assert e.memory_floats == 100.0 * 80 + 100 * 5 + 80 * 5
    e = cb.estimate_cost("fasthals-rp", 100, 80, 5, 9)
    assert e.flops_per_iteration == 2.0 * 100 * 5 * 9
    assert e.memory_floats == (2.0 * 9 + 5) * (100 + 80)
    assert cb.estimate_cost("hals-rp", 10, 20, 2, 3).flops_per_iteration == 4.0 * 10 * 20 * 2 * 3
    for bad in (("mu", 10, 10, 2, 5), ("mu-rp", 10, 10, 2, 0), ("fasthals", 0, 10, 2, 0)):
        with pytest.raises(cb.ConfigError):
            cb.estimate_cost(*bad)


def test_dense_csv_round_trips_bitwise(tmp_path):
    rng = np.random.default_rng(3)
    m = np.abs(rng.standard_normal((7, 5))) * 10.0 ** rng.integers(-300, 300, (7, 5))
    m[0, 0], m[1, 1] = 0.0, 5e-324
    p = tmp_path / "m.csv"
    p.write_text(cli.dense_csv_text(m))
    assert np.array_equal(cli.load_dense_csv(str(p)), m)


def test_dense_csv_header_blank_lines_and_crlf(tmp_path):
    p = tmp_path / "h.csv"
    p.write_bytes(b"a,b\r\n1,2\r\n\r\n   \n3, 4\n")
    m = cli.load_dense_csv(str(p), True)
    assert m.tolist() == [[1.0, 2.0], [3.0, 4.0]]


def test_dense_csv_failures(tmp_path):
    # test_data_io.cpp:64-84: line numbers, error classes
    ragged = tmp_path / "ragged.csv"
    ragged.write_text("1,2\n3\n")
    with pytest.raises(cb.ParseError, match="line 2"):
        cli.load_dense_csv(str(ragged))
    neg = tmp_path / "neg.csv"
    neg.write_text("1,-2\n")
    with pytest.raises(cb.InputError):
        cli.load_dense_csv(str(neg))
    for text in ("1,abc\n", "1,2x\n", "1,2 \n", "1,\n"):
        bad = tmp_path / "bad.csv"
        bad.write_text(text)
        with pytest.raises(cb.ParseError):
            cli.load_dense_csv(str(bad))
    inf = tmp_path / "inf.csv"
    inf.write_text("1,inf\n")
    with pytest.raises(cb.InputError):
        cli.load_dense_csv(str(inf))
    empty = tmp_path / "empty.csv"
    empty.write_text("\n  \n")
    with pytest.raises(cb.ParseError):
        cli.load_dense_csv(str(empty))
    with pytest.raises(cb.IoError):
        cli.load_dense_csv(str(tmp_path / "missing.csv"))


# ----------------------------------------------------------- options/config --
def test_list_options_and_median():
    vals, given = cli.parse_args("sweep", ["--seeds", "3,1", "--k-grid", "2,3", "--k-grid=4",
                                           "--alpha-grid", "0,0.1"])
    assert vals["seeds"] == [3, 1] and vals["k-grid"] == [2, 3, 4]
    assert vals["alpha-grid"] == [0.0, 0.1] and vals["q-grid"] == []
    assert cli.median([3.0, 1.0, 2.0]) == 2.0 and cli.median([4.0, 1.0]) == 2.5
    with pytest.raises(cb.InputError):
        cli.median([])
    assert cli.sanitize_cell("a,b\nc") == "a;b;c"


def test_read_config_file(tmp_path):
    p = tmp_path / "run.cfg"
    p.write_text("# comment\n; also a comment\n\n k = 3 \niters=7\nk=4\n")
    assert cli.read_config_file(str(p)) == [("k", "3"), ("iters", "7"), ("k", "4")]
    bad = tmp_path / "bad.cfg"
    bad.write_text("k\n")
    with pytest.raises(cb.ParseError, match="line 1"):
        cli.read_config_file(str(bad))
    bad.write_text("=3\n")
    with pytest.raises(cb.ParseError, match="empty key"):
        cli.read_config_file(str(bad))


def test_config_defaults_and_explicit_flags(tmp_path):
    p = tmp_path / "run.cfg"
    p.write_text("k=3\niters=7\nno-normalize=yes\nk=5\n")
    vals, given = cli.parse_args("factorize", SYNTH + ["--config", str(p), "--iters", "9"])
    cli.apply_config("factorize", vals, given)
    assert vals["k"] == 5 and vals["iters"] == 9 and vals["no-normalize"] is True
    assert vals["tol"] == 1e-9 and vals["w"] == 4 and vals["algo"] == "fasthals"
    for text, exc in (("frobnicate=1\n", cb.ConfigError), ("config=x\n", cb.ConfigError),
                      ("no-normalize=maybe\n", cb.ConfigError)):
        p.write_text(text)
        vals, given = cli.parse_args("factorize", ["--config", str(p)])
        with pytest.raises(exc):
            cli.apply_config("factorize", vals, given)


def test_make_config_seeds_sketch_and_init():
    vals, _ = cli.parse_args("factorize", ["--algo", "FastHALS_RP", "--k", "4", "--q", "9",
                                           "--w", "1", "--seed", "17", "--alpha", "0.5",
                                           "--no-normalize", "--error-interval=3"])
    cfg = cli.make_config(vals, vals["seed"])
    assert cfg.algorithm == cb.FASTHALS_RP and cfg.k == 4 and cfg.sketch.q == 9
    assert cfg.sketch.power_iterations == 1 and cfg.sketch.seed == 17 and cfg.seed == 17
    assert cfg.alpha == 0.5 and cfg.normalize_a is False and cfg.error_interval == 3


def test_estimate_prints_cost_model(capsys):
    assert cli.run(["estimate", "--algo", "mu", "--rows", "100", "--cols", "80", "--k",
                    "5"]) == 0
    j = json.loads(capsys.readouterr().out)
    assert j == {"algorithm": "mu", "d": 100, "n": 80, "k": 5, "q": 0,
                 "flops_per_iter": 8.0 * 100 * 80 * 5,
                 "memory_floats": 100.0 * 80 + 100 * 5 + 80 * 5}
    assert cli.run(["estimate", "--algo", "mu-rp", "--rows", "100", "--cols", "80", "--k", "5",
                    "--q", "9"]) == 0
    j = json.loads(capsys.readouterr().out)
    assert j["flops_per_iter"] == 4.0 * 100 * 5 * 9
    assert j["memory_floats"] == (2.0 * 9 + 5) * (100 + 80)


def test_bad_invocations_exit_2_and_write_nothing(tmp_path, capsys):
    # test_cli.cpp:330-351 (the ones decided before any device work)
    out = str(tmp_path / "a")
    assert cli.run(["factorize", "--format", "csv", "--input", str(tmp_path / "missing.csv"),
                    "--out", out]) == 2
    assert not os.path.exists(out)
    out = str(tmp_path / "b")
    assert cli.run(["factorize"] + SYNTH + ["--algo", "mu", "--alpha", "0.5", "--out", out]) == 2
    assert not os.path.exists(out)
    assert cli.run(["factorize", "--format", "bogus", "--out", str(tmp_path / "c")]) == 2
    assert cli.run(["factorize", "--frobnicate"]) == 2
    assert cli.run(["factorize"] + SYNTH) == 2                     # --out missing
    assert cli.run(["estimate", "--algo", "mu", "--rows", "10", "--cols", "10", "--q", "5"]) == 2
    assert cli.run(["estimate", "--rows", "10"]) == 2
    assert cli.run(["factorize", "--k", "-1", "--out", out]) == 2
    assert cli.run(["project"] + SYNTH + ["--out", str(tmp_path / "p")]) == 2   # --q missing
    assert cli.run(["compare"] + SYNTH + ["--seeds", "1,x", "--out", str(tmp_path / "d")]) == 2
    assert cli.run(["factorize", "--format", "mm", "--input", "x.mtx", "--out", out]) == 2
    assert cli.run([]) == 2
    assert cli.run(["--help"]) == 0
    assert not any(os.path.exists(tmp_path / s) for s in "bcdp")
    capsys.readouterr()


def test_artifact_writers_format(tmp_path):
    """trace.csv / trace.json / summary.json from a RunTrace (cli.cpp:176-227)."""
    recs = [cb.RunRecord(0, 12.5, 0.0), cb.RunRecord(5, 1.0 / 3.0, 2.5e-5)]
    t = cb.RunTrace(recs, 1e-3, 0.0, 0.0, float("nan"), cb.REACHED_MAX_ITERATIONS, 5, 4, 0.0,
                    0.0, 3, 480.0, 500.0, 1.0, 0, 0, "")
    cfg = cb.SolverConfig(algorithm=cb.FASTHALS_RP, k=2, seed=3,
                          sketch=cb.SketchConfig(q=6, power_iterations=4, seed=3))
    rows = cli.trace_csv_rows("fasthals-rp", 3, t)
    assert rows == ("fasthals-rp,3,0,12.5,0\n"
                    "fasthals-rp,3,5,0.33333333333333331,2.5000000000000001e-05\n")
    s = cli.summary_json(cfg, t)
    assert sorted(s) == sorted(["algorithm", "k", "q", "w", "alpha", "beta", "final_error",
                                "gini_b", "flops_per_iter", "memory_floats", "iterations_run",
                                "converged"])
    text = cli.json_dump(s)
    j = json.loads(text)
    assert j["gini_b"] is None and j["final_error"] == 1.0 / 3.0 and j["converged"] is False
    assert j["q"] == 6 and j["w"] == 4 and j["k"] == 2 and '"alpha": 0.0' in text
    tj = json.loads(cli.json_dump(cli.trace_json(cfg, t)))
    assert tj["status"] == "reached_max_iterations" and tj["seed"] == 3
    assert tj["records"][1] == {"iteration": 5, "error": 1.0 / 3.0, "elapsed_seconds": 2.5e-5}
    p = tmp_path / "x.txt"
    cli.write_text_atomic(str(p), "abc")
    assert p.read_text() == "abc" and not os.path.exists(str(p) + ".tmp")
    assert math.isnan(cli.summary_json(cfg, cb.RunTrace([], *([0.0] * 3), 0.0, cb.ABORTED, 0, 0,
                                                        0.0, 0.0, 3, 0.0, 0.0, 0.0, 0, 0,
                                                        "x"))["final_error"])


# ------------------------------------------------------------ Matrix Market --
def _mm(tmp_path, text, name="m.mtx"):
    p = tmp_path / name
    p.write_text(text)
    return str(p)


def test_matrix_market_loader_semantics(tmp_path):
    """load_matrix_market (data_io.cpp:228-288) + sparse_from_triplets
    (matrix.cpp:58-92): comments before the size line, 1-based entries,
    duplicates summed, zero sums dropped, rows sorted."""
    text = ("%%MatrixMarket matrix coordinate real general\n% comment\n\n  % indented\n"
            "3 4 6\n3 1 2.5\n1 2 1\n1 2 0.5\n2 4 0\n1 1 7\n3 4 1e-3\n")
    m = cli.load_matrix_market(_mm(tmp_path, text))
    assert m.shape == (3, 4) and m.nnz == 4
    assert m.toarray().tolist() == [[7.0, 1.5, 0.0, 0.0], [0.0, 0.0, 0.0, 0.0],
                                    [2.5, 0.0, 0.0, 1e-3]]
    assert m.indptr.tolist() == [0, 2, 2, 4]
    back = cli.load_matrix_market(_mm(tmp_path, cli.save_matrix_market_text(m), "b.mtx"))
    assert (back != m).nnz == 0
    ints = "%%MatrixMarket matrix coordinate integer general\n2 2 1\n2 2 5\n"
    assert cli.load_matrix_market(_mm(tmp_path, ints, "i.mtx")).toarray()[1, 1] == 5.0


def test_matrix_market_loader_errors(tmp_path):
    bad = {
        "": (cb.ParseError, "missing banner"),
        "%%MatrixMarket matrix array real general\n2 2\n": (cb.ParseError, "banner"),
        "%%MatrixMarket matrix coordinate complex general\n": (cb.ParseError, "banner"),
        "%%MatrixMarket matrix coordinate real symmetric\n": (cb.ParseError, "banner"),
        "%%MatrixMarket matrix coordinate real general\n% only comments\n":
            (cb.ParseError, "missing size line"),
        "%%MatrixMarket matrix coordinate real general\n2 x 1\n": (cb.ParseError, "line 2"),
        "%%MatrixMarket matrix coordinate real general\n0 2 0\n": (cb.ParseError, "zero"),
        "%%MatrixMarket matrix coordinate real general\n2 2 2\n1 1 1\n":
            (cb.ParseError, "after 1 of 2"),
        "%%MatrixMarket matrix coordinate real general\n2 2 1\n3 1 1\n":
            (cb.ParseError, "out of range"),
        "%%MatrixMarket matrix coordinate real general\n2 2 1\n1 1\n": (cb.ParseError, "malformed"),
        "%%MatrixMarket matrix coordinate real general\n2 2 1\n1 1 x\n": (cb.ParseError, "parse"),
        "%%MatrixMarket matrix coordinate real general\n2 2 1\n1 1 -2\n": (cb.InputError, "negative"),
        "%%MatrixMarket matrix coordinate real general\n2 2 1\n1 1 inf\n":
            (cb.InputError, "non-finite"),
    }
    for i, (text, (exc, msg)) in enumerate(bad.items()):
        with pytest.raises(exc, match=msg):
            cli.load_matrix_market(_mm(tmp_path, text, f"b{i}.mtx"))
    with pytest.raises(cb.IoError):
        cli.load_matrix_market(str(tmp_path / "missing.mtx"))
