"""`cnmf` command-line front end over the B200 path.

    python -m paper_1712_02248_b200.cli factorize --format synthetic --rows 12 \\
        --cols 10 --rank 2 --noise 0.05 --algo fasthals-rp --k 2 --q 6 --out run/

Mirrors the reference tool's subcommands that sit on the compressed path
(/root/reference/proj/src/cli.cpp):

  factorize   cmd_factorize  cli.cpp:304-326  a.csv, b.csv, trace.csv,
              trace.json, summary.json
  project     cmd_project    cli.cpp:516-553  xhat.csv, xcheck.csv,
              distortion.json
  estimate    cmd_estimate   cli.cpp:555-570  cost model as JSON on stdout
  compare     cmd_compare    cli.cpp:328-409  runs.csv, runs_summary.csv, table.csv
  sweep       cmd_sweep      cli.cpp:411-514  sweep_runs.csv, sweep.csv

with the same option names and defaults (cli.cpp:43-81, 644-755), the same
`--config` key=value files (cli.cpp:573-634: '#'/';' comment lines, the last
occurrence of a key wins, explicit flags win, no nesting, boolean values for
flags), the same artifact columns and keys, number formats (%.17g cells,
nlohmann-style JSON with sorted keys and NaN -> null), atomic writes
(cli.cpp:156-174) and exit codes (0 ok, 1 aborted run or runtime failure,
2 usage / configuration / input / IO error; cli.cpp:759-799).

The factorization itself is the C-ABI library on the GPU (fp32 storage, see
DESIGN.md); inputs are dense CSV (data_io.cpp:75-106), Matrix Market
coordinate files run through the CSR path (data_io.cpp:228-288, cnmf_run_csr)
or the reference's synthetic generator (bitwise, cnmf_generate_synthetic).
Image directories and text corpora are outside this build (scope)
and are rejected with exit code 2.  Runs of a
compare / sweep plan execute one after another on the device (`--jobs` is
accepted; the reference's output bytes do not depend on it either,
cli.cpp:229-247).
"""
from __future__ import annotations

import math
import os
import struct
import sys
from typing import Dict, List, Optional, Sequence, Tuple

import numpy as np

from . import (ALGORITHM_NAMES, ConfigError, CudaError, DimensionError, InputError, IoError,
               ParseError, SketchConfig, SolverConfig, STATUS_NAMES, ABORTED, CONVERGED,
               UnsupportedError, estimate_cost, generate_synthetic, pairwise_distortion)

TRACE_HEADER = "algorithm,seed,iteration,error,elapsed_seconds\n"  # cli.cpp:36-37
CANONICAL = {v: k for k, v in ALGORITHM_NAMES.items()}          # algorithm.cpp:10-20


class UsageError(Exception):
    """A command line the parser rejects (CLI11's ParseError: exit code 2)."""


# ------------------------------------------------------------- formatting --
def fmt(v: float) -> str:
    """%.17g, as cli.cpp:83-87 and format_value (data_io.cpp:44-48)."""
    return "%.17g" % v


def _cached_power(k: int):
    """(f, e) with f * 2^e = 10^k rounded to a 64-bit significand (the table
    Grisu2 indexes; computed exactly with rationals)."""
    num, den = (10 ** k, 1) if k >= 0 else (1, 10 ** -k)
    e = num.bit_length() - den.bit_length() - 64
    while True:   # normalise to 2^63 <= 10^k / 2^e < 2^64
        n2, d2 = (num, den << e) if e >= 0 else (num << -e, den)
        if n2 >= d2 << 64:
            e += 1
        elif n2 < d2 << 63:
            e -= 1
        else:
            break
    f, r = divmod(n2, d2)
    return f + (2 * r >= d2), e


_POW_CACHE = {}


def _grisu2(v: float):
    """Shortest-in-interval digits of v > 0 and their decimal exponent by
    Grisu2 (Loitsch 2010) with alpha = -60, gamma = -32 and 10^k cached in
    steps of 8 from 10^-300 -- the algorithm nlohmann::json's to_chars uses
    for doubles (not always the shortest or nearest digits, so Python's
    repr cannot stand in for it)."""
    M64 = (1 << 64) - 1
    bits = struct.unpack("<Q", struct.pack("<d", v))[0]
    E, F = bits >> 52, bits & ((1 << 52) - 1)
    f, e = (F, -1074) if E == 0 else (F + (1 << 52), E - 1075)
    closer = F == 0 and E > 1
    mp_f, mp_e = 2 * f + 1, e - 1
    mm_f, mm_e = (4 * f - 1, e - 2) if closer else (2 * f - 1, e - 1)
    sh = 64 - mp_f.bit_length()                       # normalise m+
    mp_f, mp_e = mp_f << sh, mp_e - sh
    mm_f, mm_e = mm_f << (mm_e - mp_e), mp_e          # m- on m+'s exponent
    sh = 64 - f.bit_length()
    w_f, w_e = f << sh, e - sh
    # cached power c = 10^-k with alpha <= e(c * m+) <= gamma
    t = -60 - mp_e - 1
    q = (abs(t) * 78913) >> 18                        # C++ division truncates toward zero
    k = (q if t >= 0 else -q) + (t > 0)
    index = (300 + k + 7) // 8
    dk = -300 + 8 * index
    if dk not in _POW_CACHE:
        _POW_CACHE[dk] = _cached_power(dk)
    c_f, c_e = _POW_CACHE[dk]

    def mul(a):                                       # rounded high half of a 64x64 product
        return (a * c_f + (1 << 63)) >> 64

    W_f, Wm_f, Wp_f, e_all = mul(w_f), mul(mm_f), mul(mp_f), mp_e + c_e + 64
    assert w_e + c_e + 64 == e_all
    Mm, Mp = Wm_f + 1, Wp_f - 1
    dec_exp = -dk
    delta, dist = Mp - Mm, Mp - W_f
    one_e = e_all                                     # one = 2^-e_all
    sh = -one_e
    p1, p2 = Mp >> sh, Mp & ((1 << sh) - 1)
    n = len(str(p1)) if p1 else 1
    pow10 = 10 ** (n - 1)
    digits = []

    def round_last(rest, ten_k):
        while (rest < dist and delta - rest >= ten_k
               and (rest + ten_k < dist or dist - rest > rest + ten_k - dist)):
            digits[-1] -= 1
            rest += ten_k

    while n > 0:
        d, p1 = divmod(p1, pow10)
        digits.append(d)
        n -= 1
        rest = (p1 << sh) + p2
        if rest <= delta:
            dec_exp += n
            round_last(rest, pow10 << sh)
            return "".join(map(str, digits)), dec_exp
        pow10 //= 10
    m = 0
    while True:
        p2 = (p2 * 10) & M64
        digits.append(p2 >> sh)
        p2 &= (1 << sh) - 1
        m += 1
        delta = (delta * 10) & M64
        dist = (dist * 10) & M64
        if p2 <= delta:
            break
    dec_exp -= m
    round_last(p2, 1 << sh)
    return "".join(map(str, digits)), dec_exp


def _json_number(v: float) -> str:
    """nlohmann::json's double output (to_chars): Grisu2 digits, plain
    notation for decimal-point positions in (-4, 15], else d.ddde+XX with at
    least two exponent digits; NaN/inf -> null."""
    if not math.isfinite(v):
        return "null"
    if v == 0.0:
        return "-0.0" if math.copysign(1.0, v) < 0 else "0.0"
    ds, exp = _grisu2(abs(v))
    k = len(ds)
    n = k + exp                           # position of the decimal point
    if k <= n <= 15:
        s = ds + "0" * (n - k) + ".0"
    elif 0 < n <= 15:
        s = ds[:n] + "." + ds[n:]
    elif -4 < n <= 0:
        s = "0." + "0" * (-n) + ds
    else:
        e = n - 1
        mant = ds if k == 1 else ds[0] + "." + ds[1:]
        s = mant + "e" + ("-" if e < 0 else "+") + ("%02d" % abs(e))
    return ("-" if v < 0 else "") + s


def _json_string(s: str) -> str:
    out = ['"']
    esc = {'"': '\\"', "\\": "\\\\", "\b": "\\b", "\f": "\\f", "\n": "\\n", "\r": "\\r",
           "\t": "\\t"}
    for ch in s:
        if ch in esc:
            out.append(esc[ch])
        elif ord(ch) < 0x20:
            out.append("\\u%04x" % ord(ch))
        else:
            out.append(ch)
    out.append('"')
    return "".join(out)


def json_dump(v, indent: int = 2, level: int = 0) -> str:
    """nlohmann::json::dump(indent) of an object tree (keys sorted: the
    reference's json objects are std::map-backed)."""
    pad, inner = " " * (indent * level), " " * (indent * (level + 1))
    if isinstance(v, bool):
        return "true" if v else "false"
    if v is None:
        return "null"
    if isinstance(v, (int, np.integer)):
        return str(int(v))
    if isinstance(v, (float, np.floating)):
        return _json_number(float(v))
    if isinstance(v, str):
        return _json_string(v)
    if isinstance(v, dict):
        if not v:
            return "{}"
        items = [inner + _json_string(k) + ": " + json_dump(v[k], indent, level + 1)
                 for k in sorted(v)]
        return "{\n" + ",\n".join(items) + "\n" + pad + "}"
    if isinstance(v, (list, tuple)):
        if not v:
            return "[]"
        items = [inner + json_dump(e, indent, level + 1) for e in v]
        return "[\n" + ",\n".join(items) + "\n" + pad + "]"
    raise TypeError(f"json_dump: {type(v).__name__}")


# -------------------------------------------------------------- artifacts --
def write_text_atomic(path: str, text: str) -> None:
    """Stage next to the target, then rename (cli.cpp:156-167)."""
    tmp = path + ".tmp"
    try:
        with open(tmp, "w", newline="") as f:
            f.write(text)
    except OSError as e:
        raise IoError(f"cannot open {tmp} for writing: {e.strerror}") from None
    os.replace(tmp, path)


def dense_csv_text(m: np.ndarray) -> str:
    """save_dense_csv (data_io.cpp:108-118): one row per line, %.17g cells."""
    m = np.asarray(m, dtype=np.float64)
    return "".join(",".join(fmt(v) for v in row) + "\n" for row in m.tolist())


def load_dense_csv(path: str, has_header: bool = False) -> np.ndarray:
    """load_dense_csv (data_io.cpp:75-106): optional header line, blank lines
    skipped, CR stripped, every row as wide as the first, cells parsed whole as
    numbers, finite and non-negative."""
    try:
        f = open(path, "r", newline="")
    except OSError:
        raise IoError(f"cannot open {path} for reading") from None
    values: List[float] = []
    rows = cols = 0
    with f:
        lines = f.read().split("\n")
    if lines and lines[-1] == "":
        lines.pop()
    start = 1 if has_header and lines else 0
    for ln in range(start, len(lines)):
        line = lines[ln]
        if line.endswith("\r"):
            line = line[:-1]
        if line.strip(" \t") == "":
            continue
        cells = line.split(",")
        if cols == 0:
            cols = len(cells)
        where = f"{path}: line {ln + 1}"
        if len(cells) != cols:
            raise ParseError(f"{where}: expected {cols} columns, found {len(cells)}")
        for cell in cells:
            v = _strtod_whole(cell, where)
            if not math.isfinite(v):
                raise InputError(f"{where}: non-finite value")
            if v < 0.0:
                raise InputError(f"{where}: negative value {cell}")
            values.append(v)
        rows += 1
    if rows == 0:
        raise ParseError(f"{path}: no data rows")
    return np.array(values, dtype=np.float64).reshape(rows, cols)


def _strtod_whole(token: str, where: str) -> float:
    """parse_value (data_io.cpp:50-57): strtod must consume the whole cell --
    leading whitespace is skipped, anything after the number is an error."""
    t = token.lstrip(" \t\n\v\f\r")
    try:
        if not t or t != t.rstrip() or "_" in t:
            raise ValueError
        body = t.lstrip("+-")
        if body[:2].lower() == "0x":
            v = float.fromhex(t)
        else:
            v = float(t)
        return v
    except ValueError:
        raise ParseError(f"{where}: cannot parse '{token}' as a number") from None


def load_matrix_market(path: str):
    """load_matrix_market (data_io.cpp:228-288) + sparse_from_triplets
    (matrix.cpp:58-92): coordinate real|integer general, 1-based entries,
    duplicates summed, entries summing to zero dropped -> scipy CSR (fp64)."""
    import scipy.sparse as sparse
    try:
        f = open(path, "r", newline="")
    except OSError:
        raise IoError(f"cannot open {path} for reading") from None
    with f:
        lines = f.read().split("\n")
    if lines and lines[-1] == "":
        lines.pop()
    strip = lambda t: t[:-1] if t.endswith("\r") else t  # noqa: E731
    if not lines:
        raise ParseError(f"{path}: line 1: missing banner")
    ban = strip(lines[0]).split()
    if (len(ban) != 5 or ban[0] != "%%MatrixMarket" or ban[1] != "matrix"
            or ban[2] != "coordinate" or ban[3] not in ("real", "integer") or ban[4] != "general"):
        raise ParseError(f"{path}: line 1: expected banner '%%MatrixMarket matrix coordinate "
                         "real general'")
    ln = 1
    while True:
        if ln >= len(lines):
            raise ParseError(f"{path}: missing size line")
        line = strip(lines[ln])
        ln += 1
        t = line.lstrip(" \t")
        if t and t[0] != "%":
            break
    try:
        tok = line.split()
        rows, cols, entries = int(tok[0]), int(tok[1]), int(tok[2])
        if min(rows, cols, entries) < 0:
            raise ValueError
    except (ValueError, IndexError):
        raise ParseError(f"{path}: line {ln}: malformed size line") from None
    if rows == 0 or cols == 0:
        raise ParseError(f"{path}: line {ln}: zero matrix dimension")
    ri, cj, vals = [], [], []
    for e in range(entries):
        if ln >= len(lines):
            raise ParseError(f"{path}: unexpected end of file after {e} of {entries} entries")
        line = strip(lines[ln])
        ln += 1
        where = f"{path}: line {ln}"
        tok = line.split()
        try:
            i, j = int(tok[0]), int(tok[1])
            vt = tok[2]
        except (ValueError, IndexError):
            raise ParseError(f"{where}: malformed entry") from None
        if i < 1 or i > rows or j < 1 or j > cols:
            raise ParseError(f"{where}: index out of range")
        v = _strtod_whole(vt, where)
        if not math.isfinite(v):
            raise InputError(f"{where}: non-finite value")
        if v < 0.0:
            raise InputError(f"{where}: negative value {vt}")
        ri.append(i - 1)
        cj.append(j - 1)
        vals.append(v)
    ri, cj, vals = np.array(ri, np.int64), np.array(cj, np.int64), np.array(vals, np.float64)
    order = np.lexsort((cj, ri))  # by row, then column (stable: duplicates keep file order)
    ri, cj, vals = ri[order], cj[order], vals[order]
    keep_r, keep_c, keep_v = [], [], []
    e = 0
    while e < len(vals):
        f2, tot = e, 0.0
        while f2 < len(vals) and ri[f2] == ri[e] and cj[f2] == cj[e]:
            tot += vals[f2]
            f2 += 1
        if tot != 0.0:
            keep_r.append(ri[e])
            keep_c.append(cj[e])
            keep_v.append(tot)
        e = f2
    return sparse.csr_matrix((np.array(keep_v, np.float64), (np.array(keep_r, np.int64),
                                                             np.array(keep_c, np.int64))),
                             shape=(rows, cols))


def save_matrix_market_text(m) -> str:
    """save_matrix_market (data_io.cpp:290-299)."""
    m = m.tocsr()
    m.sort_indices()
    out = ["%%MatrixMarket matrix coordinate real general\n",
           f"{m.shape[0]} {m.shape[1]} {m.nnz}\n"]
    for i in range(m.shape[0]):
        for p in range(m.indptr[i], m.indptr[i + 1]):
            out.append(f"{i + 1} {m.indices[p] + 1} {fmt(m.data[p])}\n")
    return "".join(out)


# ---------------------------------------------------------------- options --
# name -> (kind, default); kinds: str, uint, float, flag (cli.cpp:43-81)
_DATASET = {"input": ("str", ""), "format": ("str", "csv"), "csv-header": ("flag", False),
            "per-file": ("flag", False), "vocab-size": ("uint", 1000),
            "max-docs": ("uint", 5000), "rows": ("uint", 0), "cols": ("uint", 0),
            "rank": ("uint", 1), "decay": ("float", 0.0), "noise": ("float", 0.0),
            "data-seed": ("uint", 1), "config": ("str", "")}
_SOLVER = {"k": ("uint", 2), "q": ("uint", 0), "w": ("uint", 4), "iters": ("uint", 200),
           "tol": ("float", 1e-9), "error-interval": ("uint", 5),
           "no-normalize": ("flag", False)}
_PENALTIES = {"alpha": ("float", 0.0), "beta": ("float", 0.0)}
_SEEDS = {"seeds": ("uints", [1, 2, 3, 4, 5]), "jobs": ("uint", 1)}
SUBCOMMANDS = {
    "factorize": {**_DATASET, **_SOLVER, **_PENALTIES, "out": ("str", ""),
                  "algo": ("str", "fasthals"), "seed": ("uint", 1)},
    "compare": {**_DATASET, **_SOLVER, "out": ("str", ""), **_SEEDS},
    "sweep": {**_DATASET, **_SOLVER, **_PENALTIES, "out": ("str", ""),
              "algo": ("str", "fasthals"), **_SEEDS, "k-grid": ("uints", []),
              "q-grid": ("uints", []), "w-grid": ("uints", []), "alpha-grid": ("floats", []),
              "beta-grid": ("floats", [])},
    "project": {**_DATASET, "out": ("str", ""), "q": ("uint", 0), "w": ("uint", 4),
                "seed": ("uint", 1), "pairs": ("uint", 200)},
    "estimate": {"algo": ("str", "fasthals"), "rows": ("uint", 0), "cols": ("uint", 0),
                 "k": ("uint", 2), "q": ("uint", 0), "config": ("str", "")},
}


def _convert(name: str, kind: str, value: str):
    try:
        if kind in ("uints", "floats"):   # comma-delimited lists (CLI11 ->delimiter(','))
            one = "uint" if kind == "uints" else "float"
            return [_convert(name, one, v) for v in value.split(",")]
        if kind == "uint":
            v = int(value.strip(), 10)
            if v < 0:
                raise ValueError
            return v
        if kind == "float":
            return float(value)
        return value
    except ValueError:
        raise UsageError(f"--{name}: invalid value '{value}'") from None


def parse_args(sub: str, argv: Sequence[str]) -> Tuple[Dict[str, object], set]:
    """Explicit options of one subcommand -> (values, names given)."""
    spec = SUBCOMMANDS[sub]
    vals: Dict[str, object] = {k: v[1] for k, v in spec.items()}
    given = set()
    i = 0
    while i < len(argv):
        tok = argv[i]
        if tok in ("-h", "--help"):
            raise SystemExit(_usage(sub))
        if not tok.startswith("--"):
            raise UsageError(f"unexpected argument '{tok}'")
        name, eq, inline = tok[2:].partition("=")
        if name not in spec:
            raise UsageError(f"the following argument was not expected: {tok}")
        kind = spec[name][0]
        if kind == "flag":
            if eq:
                raise UsageError(f"--{name} takes no value")
            vals[name] = True
        else:
            if eq:
                raw = inline
            else:
                i += 1
                if i >= len(argv):
                    raise UsageError(f"--{name} requires a value")
                raw = argv[i]
            v = _convert(name, kind, raw)
            if kind in ("uints", "floats") and name in given:
                v = vals[name] + v                 # repeated list options accumulate
            vals[name] = v
        given.add(name)
        i += 1
    return vals, given


def read_config_file(path: str) -> List[Tuple[str, str]]:
    """read_config_file (cli.cpp:573-600)."""
    try:
        with open(path, "r") as f:
            lines = f.read().split("\n")
    except OSError:
        raise IoError(f"cannot open config file {path}") from None
    if lines and lines[-1] == "":
        lines.pop()
    items = []
    for no, line in enumerate(lines, 1):
        t = line.strip(" \t\r")
        if not t or t[0] in "#;":
            continue
        if "=" not in t:
            raise ParseError(f"{path}: line {no}: expected key=value")
        key, _, value = t.partition("=")
        key = key.strip(" \t\r")
        if not key:
            raise ParseError(f"{path}: line {no}: empty key")
        items.append((key, value.strip(" \t\r")))
    return items


def flag_value(key: str, v: str) -> bool:
    """flag_value (cli.cpp:602-607)."""
    s = v.lower()
    if s in ("true", "1", "yes", "on"):
        return True
    if s in ("false", "0", "no", "off"):
        return False
    raise ConfigError(f"config key {key} expects a boolean, got: {s}")


def apply_config(sub: str, vals: Dict[str, object], given: set) -> None:
    """config_extras (cli.cpp:612-634): file keys fill the options the command
    line left unset; the last occurrence of a repeated key wins."""
    path = vals.get("config") or ""
    if not path:
        return
    spec = SUBCOMMANDS[sub]
    items = read_config_file(path)
    last = {k: i for i, (k, _) in enumerate(items)}
    for i, (key, value) in enumerate(items):
        if last[key] != i:
            continue
        if key == "config":
            raise ConfigError("config files cannot nest")
        if key not in spec:
            raise ConfigError(f"unknown config key for {sub}: {key}")
        if key in given:
            continue
        kind = spec[key][0]
        vals[key] = flag_value(key, value) if kind == "flag" else _convert(key, kind, value)


def _usage(sub: Optional[str] = None) -> str:
    subs = [sub] if sub else list(SUBCOMMANDS)
    lines = ["compressed non-negative matrix factorization toolkit (B200)",
             "usage: python -m paper_1712_02248_b200.cli SUBCOMMAND [OPTIONS]"]
    for s in subs:
        opts = " ".join(f"[--{k}]" if v[0] == "flag" else
                        f"[--{k} V,V..]" if v[0] in ("uints", "floats") else f"[--{k} V]"
                        for k, v in SUBCOMMANDS[s].items())
        lines.append(f"  {s} {opts}")
    return "\n".join(lines)


# ---------------------------------------------------------------- commands --
def parse_algorithm(name: str) -> int:
    """parse_algorithm (algorithm.cpp:22-35): case-insensitive, '_' as '-'."""
    s = name.replace("_", "-").lower()
    if s not in ALGORITHM_NAMES:
        raise ConfigError(f"unknown algorithm '{name}' (expected one of mu, mu-rp, hals, "
                          "hals-rp, fasthals, fasthals-rp)")
    return ALGORITHM_NAMES[s]


def load_dataset(o: Dict[str, object]) -> np.ndarray:
    """make_descriptor + load_dataset (cli.cpp:98-111, data_io.cpp:417-445),
    dense formats."""
    fmt_name = o["format"]
    if fmt_name not in ("csv", "mm", "pgm-dir", "corpus", "synthetic"):
        raise ConfigError(f"unknown dataset format: {fmt_name}")
    if fmt_name != "synthetic" and not o["input"]:
        raise ConfigError(f"--input is required for format {fmt_name}")
    if fmt_name == "csv":
        return load_dense_csv(o["input"], bool(o["csv-header"]))
    if fmt_name == "synthetic":
        return generate_synthetic(o["rows"], o["cols"], o["rank"], o["decay"], o["noise"],
                                  o["data-seed"])
    if fmt_name == "mm":
        return load_matrix_market(o["input"])
    raise UnsupportedError(f"dataset format {fmt_name} (image directories and text corpora) "
                           "is not part of this build (csv, mm and synthetic are)")


def make_config(o: Dict[str, object], seed: int) -> SolverConfig:
    """make_config (cli.cpp:120-135): the run seed drives the init and the sketch."""
    return SolverConfig(algorithm=parse_algorithm(o["algo"]), k=o["k"],
                        sketch=SketchConfig(q=o["q"], power_iterations=o["w"], seed=seed),
                        alpha=o.get("alpha", 0.0), beta=o.get("beta", 0.0),
                        max_iterations=o["iters"],
                        rel_tolerance=o["tol"], error_interval=o["error-interval"], seed=seed,
                        normalize_a=not o["no-normalize"])


def _context():
    from . import default_context
    return default_context()


def is_sparse(x) -> bool:
    return hasattr(x, "tocsr")


def solve(x, cfg: SolverConfig):
    """cli.cpp:137-139: the dense or the sparse run (x: fp32 ndarray or CSR)."""
    return _context().run_sparse(x, cfg) if is_sparse(x) else _context().run(x, cfg)


def device_input(x):
    """fp32 dense rows, or the CSR as is (values go to fp32 on upload)."""
    return x if is_sparse(x) else x.astype(np.float32)


def summary_json(cfg: SolverConfig, t) -> dict:
    """summary_json (cli.cpp:196-211)."""
    return {"algorithm": CANONICAL[cfg.algorithm], "k": cfg.k, "q": cfg.sketch.q,
            "w": t.power_iterations, "alpha": float(cfg.alpha), "beta": float(cfg.beta),
            "final_error": t.records[-1].error if t.records else float("nan"),
            "gini_b": t.gini_b, "flops_per_iter": t.estimate_flops_per_iteration,
            "memory_floats": t.estimate_memory_floats, "iterations_run": t.iterations_run,
            "converged": t.status == CONVERGED}


def trace_json(cfg: SolverConfig, t) -> dict:
    """trace_json (cli.cpp:213-227)."""
    return {"algorithm": CANONICAL[cfg.algorithm], "seed": cfg.seed,
            "status": STATUS_NAMES[t.status], "message": t.message,
            "update_seconds": t.update_seconds,
            "records": [{"iteration": r.iteration, "error": r.error,
                         "elapsed_seconds": r.elapsed_seconds} for r in t.records]}


def trace_csv_rows(algo: str, seed: int, t) -> str:
    """append_trace_rows (cli.cpp:176-190)."""
    return "".join(f"{algo},{seed},{r.iteration},{fmt(r.error)},{fmt(r.elapsed_seconds)}\n"
                   for r in t.records)


def cmd_factorize(o: Dict[str, object]) -> int:
    """cmd_factorize (cli.cpp:304-326)."""
    if not o["out"]:
        raise ConfigError("--out is required")
    x = load_dataset(o)
    cfg = make_config(o, o["seed"])
    cfg.validate(*x.shape)
    res = solve(device_input(x), cfg)
    out = o["out"]
    os.makedirs(out, exist_ok=True)
    write_text_atomic(os.path.join(out, "a.csv"), dense_csv_text(res.a))
    write_text_atomic(os.path.join(out, "b.csv"), dense_csv_text(res.b))
    name = CANONICAL[cfg.algorithm]
    write_text_atomic(os.path.join(out, "trace.csv"),
                      TRACE_HEADER + trace_csv_rows(name, cfg.seed, res.trace))
    write_text_atomic(os.path.join(out, "trace.json"), json_dump(trace_json(cfg, res.trace)) + "\n")
    write_text_atomic(os.path.join(out, "summary.json"),
                      json_dump(summary_json(cfg, res.trace)) + "\n")
    if res.trace.status == ABORTED:
        print(f"cnmf: run aborted: {res.trace.message}", file=sys.stderr)
        return 1
    return 0


def cmd_project(o: Dict[str, object]) -> int:
    """cmd_project (cli.cpp:516-553): the QB compression's views of X and the
    pairwise-distance distortion of the left projection."""
    import torch
    if not o["out"]:
        raise ConfigError("--out is required")
    q = o["q"]
    if q == 0:
        raise ConfigError("--q is required")
    x = load_dataset(o)
    if is_sparse(x):
        # the distortion metric walks dense columns anyway (cli.cpp:528-532);
        # the views of the densified matrix are the same products
        x = x.toarray()
    d, n = x.shape
    if q > min(d, n):
        raise ConfigError("powered_range_finder: q must satisfy 1 <= q <= min(rows, cols)")
    ctx = _context()
    xd = torch.from_numpy(x.astype(np.float32)).cuda()
    left = torch.empty((d, q), device="cuda")
    right = torch.empty((q, n), device="cuda")
    ctx.build_projectors(xd, q, o["w"], o["seed"], left, right)
    xhat = torch.empty((q, n), device="cuda")
    xcheck = torch.empty((d, q), device="cuda")
    ctx.compress(xd, left, right, xhat, xcheck)
    xhat_h, xcheck_h = xhat.cpu().numpy(), xcheck.cpu().numpy()
    mx, mean = pairwise_distortion(x, xhat_h, o["pairs"], o["seed"])
    report = {"q": q, "w": o["w"], "seed": o["seed"], "sample_pairs": o["pairs"],
              "max_relative": mx, "mean_relative": mean, "xhat_rows": q, "xhat_cols": n,
              "xcheck_rows": d, "xcheck_cols": q}
    out = o["out"]
    os.makedirs(out, exist_ok=True)
    write_text_atomic(os.path.join(out, "xhat.csv"), dense_csv_text(xhat_h))
    write_text_atomic(os.path.join(out, "xcheck.csv"), dense_csv_text(xcheck_h))
    write_text_atomic(os.path.join(out, "distortion.json"), json_dump(report) + "\n")
    return 0


def cmd_estimate(o: Dict[str, object]) -> int:
    """cmd_estimate (cli.cpp:555-570)."""
    if o["rows"] == 0 or o["cols"] == 0:
        raise ConfigError("--rows and --cols are required")
    e = estimate_cost(parse_algorithm(o["algo"]), o["rows"], o["cols"], o["k"], o["q"])
    print(json_dump({"algorithm": CANONICAL[e.algorithm], "d": e.d, "n": e.n, "k": e.k,
                     "q": e.q, "flops_per_iter": e.flops_per_iteration,
                     "memory_floats": e.memory_floats}))
    return 0


def median(values: List[float]) -> float:
    """median (metrics.cpp:157-162)."""
    if not values:
        raise InputError("median: empty input")
    v = sorted(values)
    mid = len(v) // 2
    return v[mid] if len(v) % 2 == 1 else 0.5 * (v[mid - 1] + v[mid])


class Outcome:
    """execute (cli.cpp:249-272): never raises; failures are recorded."""

    def __init__(self, x32: np.ndarray, cfg: SolverConfig):
        self.trace, self.ok, self.input_failure = None, False, False
        try:
            res = solve(x32, cfg)
            self.trace, self.ok = res.trace, True
            self.status, self.message = STATUS_NAMES[res.trace.status], res.trace.message
        except (ConfigError, InputError, IoError, UnsupportedError) as e:
            self.input_failure, self.status, self.message = True, "error", str(e)
        except Exception as e:  # noqa: BLE001 -- runtime failures are recorded, not raised
            self.status, self.message = "error", str(e)

    def final_error(self) -> float:
        if not self.ok or not self.trace.records:
            return float("nan")
        return self.trace.records[-1].error


def sanitize_cell(s: str) -> str:
    """cli.cpp:275-279."""
    return s.replace(",", ";").replace("\n", ";").replace("\r", ";")


def plan_exit_code(results: List[Outcome]) -> int:
    """cli.cpp:282-292: input problems dominate runtime failures."""
    any_input = any(not r.ok and r.input_failure for r in results)
    any_runtime = any((not r.ok and not r.input_failure) or
                      (r.ok and r.trace.status == ABORTED) for r in results)
    return 2 if any_input else 1 if any_runtime else 0


def report_failures(results: List[Outcome], labels: List[str]) -> None:
    for r, label in zip(results, labels):
        if not r.ok or r.trace.status == ABORTED:
            print(f"cnmf: {label}: {r.status}" + (f": {r.message}" if r.message else ""),
                  file=sys.stderr)


COMPARE_ORDER = ["mu", "hals", "fasthals", "mu-rp", "hals-rp", "fasthals-rp"]  # cli.cpp:334-336


def cmd_compare(o: Dict[str, object]) -> int:
    """cmd_compare (cli.cpp:328-409): every algorithm over every seed."""
    if not o["out"]:
        raise ConfigError("--out is required")
    x = load_dataset(o)
    d, n = x.shape
    x32 = device_input(x)
    plan = [(a, sd) for a in COMPARE_ORDER for sd in o["seeds"]]
    results = []
    for a, sd in plan:
        o2 = dict(o, algo=a)
        results.append(Outcome(x32, make_config(o2, sd)))
    runs = TRACE_HEADER
    summary = "algorithm,seed,final_error,gini_b,iterations_run,status\n"
    labels = []
    for (a, sd), r in zip(plan, results):
        labels.append(f"{a} seed {sd}")
        if r.ok:
            runs += trace_csv_rows(a, sd, r.trace)
        summary += (f"{a},{sd},{fmt(r.final_error())},"
                    f"{fmt(r.trace.gini_b if r.ok else float('nan'))},"
                    f"{r.trace.iterations_run if r.ok else 0},{sanitize_cell(r.status)}\n")
    table = "algorithm,flops_per_iter,median_seconds_per_update,memory_floats\n"
    for a in COMPARE_ORDER:
        flops = memory = float("nan")
        try:
            e = estimate_cost(a, d, n, o["k"], o["q"] if a.endswith("-rp") else 0)
            flops, memory = e.flops_per_iteration, e.memory_floats
        except Exception:  # noqa: BLE001 -- invalid geometry for this variant
            pass
        secs = [r.trace.update_seconds / r.trace.iterations_run
                for (pa, _), r in zip(plan, results)
                if pa == a and r.ok and r.trace.iterations_run > 0]
        table += f"{a},{fmt(flops)},{fmt(median(secs) if secs else float('nan'))},{fmt(memory)}\n"
    out = o["out"]
    os.makedirs(out, exist_ok=True)
    write_text_atomic(os.path.join(out, "runs.csv"), runs)
    write_text_atomic(os.path.join(out, "runs_summary.csv"), summary)
    write_text_atomic(os.path.join(out, "table.csv"), table)
    report_failures(results, labels)
    return plan_exit_code(results)


def cmd_sweep(o: Dict[str, object]) -> int:
    """cmd_sweep (cli.cpp:411-514): the (k, q, w, alpha, beta) grid of one
    algorithm over every seed, with per-cell medians."""
    if not o["out"]:
        raise ConfigError("--out is required")
    x = load_dataset(o)
    x32 = device_input(x)
    grid = lambda key, one: o[key] if o[key] else [o[one]]  # noqa: E731
    cells = [(k, q, w, al, be) for k in grid("k-grid", "k") for q in grid("q-grid", "q")
             for w in grid("w-grid", "w") for al in grid("alpha-grid", "alpha")
             for be in grid("beta-grid", "beta")]
    plan = [(ci, sd) for ci in range(len(cells)) for sd in o["seeds"]]
    name = CANONICAL[parse_algorithm(o["algo"])]
    results = []
    for ci, sd in plan:
        k, q, w, al, be = cells[ci]
        cfg = make_config(o, sd)
        cfg.k, cfg.sketch.q, cfg.sketch.power_iterations = k, q, w
        cfg.alpha, cfg.beta = float(al), float(be)
        results.append(Outcome(x32, cfg))

    def prefix(c):
        k, q, w, al, be = c
        return f"{name},{k},{q},{w},{fmt(float(al))},{fmt(float(be))}"

    raw = "algorithm,k,q,w,alpha,beta,seed,final_error,gini_b,iterations_run,status\n"
    labels = []
    for (ci, sd), r in zip(plan, results):
        labels.append(f"{name} k={cells[ci][0]} seed {sd}")
        raw += (f"{prefix(cells[ci])},{sd},{fmt(r.final_error())},"
                f"{fmt(r.trace.gini_b if r.ok else float('nan'))},"
                f"{r.trace.iterations_run if r.ok else 0},{sanitize_cell(r.status)}\n")
    sheet = "algorithm,k,q,w,alpha,beta,median_final_error,median_gini_b\n"
    for ci, c in enumerate(cells):
        errs = [r.final_error() for (pc, _), r in zip(plan, results)
                if pc == ci and r.ok and math.isfinite(r.final_error())]
        ginis = [r.trace.gini_b for (pc, _), r in zip(plan, results)
                 if pc == ci and r.ok and math.isfinite(r.trace.gini_b)]
        sheet += (f"{prefix(c)},{fmt(median(errs) if errs else float('nan'))},"
                  f"{fmt(median(ginis) if ginis else float('nan'))}\n")
    out = o["out"]
    os.makedirs(out, exist_ok=True)
    write_text_atomic(os.path.join(out, "sweep_runs.csv"), raw)
    write_text_atomic(os.path.join(out, "sweep.csv"), sheet)
    report_failures(results, labels)
    return plan_exit_code(results)


_COMMANDS = {"factorize": cmd_factorize, "project": cmd_project, "estimate": cmd_estimate,
             "compare": cmd_compare, "sweep": cmd_sweep}


def run(args: Sequence[str]) -> int:
    """cli::run (cli.cpp:759-799) for the subcommands above; returns the exit code."""
    args = list(args)
    if not args or args[0] in ("-h", "--help"):
        print(_usage())
        return 0 if args else 2
    sub, rest = args[0], args[1:]
    if sub not in SUBCOMMANDS:
        print(f"cnmf: unknown subcommand '{sub}'\n{_usage()}", file=sys.stderr)
        return 2
    try:
        vals, given = parse_args(sub, rest)
    except UsageError as e:
        print(f"cnmf: {e}\n{_usage(sub)}", file=sys.stderr)
        return 2
    except SystemExit as e:
        print(e.code)
        return 0
    try:
        apply_config(sub, vals, given)
        return _COMMANDS[sub](vals)
    except UsageError as e:
        print(f"cnmf: {e}", file=sys.stderr)
        return 2
    except (ConfigError, InputError, IoError, UnsupportedError) as e:
        print(f"cnmf: {e}", file=sys.stderr)
        return 2
    except (DimensionError, CudaError, RuntimeError, ValueError) as e:
        print(f"cnmf: {e}", file=sys.stderr)
        return 1


def main() -> None:
    sys.exit(run(sys.argv[1:]))


if __name__ == "__main__":
    main()
