#!/usr/bin/env python
"""bench.py -- compress+HALS seconds of the FastHALS-RP hot path on B200.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config c2] [--impl ours|reference]

A step is one pass of the hot path over the configuration's synthetic X:
build_projectors + compress_left/right (4w+4 X passes, Gaussian sketches
generated on the device) followed by `iters` FastHALS-RP iterations -- the
reference's cnmf::run(fasthals-rp) minus its untimed objective evaluations
(proj/src/solvers.cpp:213-284).  One JSON line on rank 0.

  value   compress+HALS seconds per step, device-timed (CUDA events inside the
          library on its stream), X resident in HBM.
  e2e     the same job through the public C ABI (cnmf_run) from pinned HOST
          memory: H2D of X, check, init, compress, HALS, the two objective
          evaluations run() always makes, Gini, D2H of A and B -- wall clock.
  roofline  the X-stream contraction kernel (the compression GEMM): algorithmic
          bytes per launch / CUDA-event launch time vs MEASURED_PEAKS.json HBM.
  cpu_baseline  the reference itself (oracle/_ref, compiled from its sources)
          on this host's cores, rank 0 at N=1 only.
"""
import argparse
import json
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "compress+HALS seconds, X-stream GB/s and % roofline at 1/2/4/8 B200"
L2_BYTES = 126 * 1024 * 1024


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="c4", choices=["c1", "c2", "c3", "c4", "c5"])
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    return ap.parse_args()


def fp64_peak_tflops():
    """FP64 tensor-core (DMMA) peak measured on this pool by tools/ubench_dmma.cu
    (profiles/fp64_peak.json); MEASURED_PEAKS.json carries no fp64 figure."""
    try:
        with open(os.path.join(ROOT, "profiles", "fp64_peak.json")) as f:
            p = json.load(f)
        return float(p["tflops"]), p.get("source", "profiles/fp64_peak.json")
    except Exception:
        return 37.0, "round-1 DMMA microbenchmark (tools/ubench_dmma.cu), not re-measured"


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def workload_desc(name, c):
    kinds = {0: "Uniform[0,1)", 1: "Exponential(1)", 2: "Gamma(0.3,1)"}
    noise = {0: "", 1: f" + |N(0,{c['sigma']})|", 2: " -> Poisson(W0 H0)"}[c["noise_kind"]]
    return (f"{name.upper()}: X {c['d']}x{c['n']} fp32 = W0 H0 ({kinds[c['factor_kind']]}, "
            f"rank {c['rank']}){noise}; k={c['k']}, l={c['q']}, q(power iters)={c['w']}, "
            f"{c['iters']} FastHALS-RP iterations")


# ----------------------------------------------------------------- clocks ---
class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu):
        self.gpu = gpu
        self.p = None

    def __enter__(self):
        try:
            self.p = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.p = None
        time.sleep(0.15)
        return self

    def __exit__(self, *a):
        self.lines = []
        if self.p is not None:
            time.sleep(0.15)
            self.p.terminate()
            try:
                out, _ = self.p.communicate(timeout=5)
            except Exception:
                self.p.kill()
                out, _ = self.p.communicate()
            self.lines = [ln for ln in out.splitlines() if ln.strip()]

    def summary(self):
        sm, mx, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            f = [t.strip() for t in ln.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                mx = max(mx, float(f[2]))
            except ValueError:
                continue
            for nm, v in zip(names, f[5:9]):
                if v.lower() == "active":
                    reasons.add(nm)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


# -------------------------------------------------------- CPU reference leg ---
def host_cpu():
    """CPU model and core count of this host (lscpu / nproc)."""
    model = "unknown"
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        for ln in out.splitlines():
            if ln.startswith("Model name:"):
                model = ln.split(":", 1)[1].strip()
                break
    except Exception:
        pass
    return model, os.cpu_count() or 1


class PinnedCore:
    """Pins this process to one host core for the single-threaded reference
    (taskset -c 0)."""

    def __init__(self, core=0):
        self.core = core

    def __enter__(self):
        try:
            self.old = os.sched_getaffinity(0)
            os.sched_setaffinity(0, {self.core})
        except Exception:
            self.old = None
        return self

    def __exit__(self, *a):
        if self.old is not None:
            os.sched_setaffinity(0, self.old)


def cpu_reference_sample(name, c, timed_steps=1):
    """The reference (oracle/_ref, its own sources) on one pinned host core:
    build_projectors + compress_left/right and `iters` fasthals_rp_step calls.

    C1/C2 run the full workload.  Larger configs are extrapolated from
    bounded samples, each operation's cost being linear in the dimension it
    is sliced along: the X contractions exactly as the reference calls them
    (compression.cpp:23-84: (1+2w) X*S, (1+2w) X^T*T, compress_left L^T X,
    compress_right X R^T) on a column slice, scaled by n / n_s; the (1+2w)
    thin_qr of d x q and of n x q bases on row slices, scaled by rows; the two
    Gaussian sketches on row slices; one fasthals_rp_step on a (d, n) / f
    shape, scaled by (d + n) / (d_s + n_s) (its cost is (d + n)(4lk + 2k^2) +
    O(lk^2)).  About 4-8 s of CPU per sample."""
    import numpy as np

    from oracle import REF_SO, Oracle, Reference
    o = Oracle()
    kind = "reference" if os.path.exists(REF_SO) else "port"
    r = Reference() if kind == "reference" else None
    impl = r if kind == "reference" else o
    d, n, k, q, w, iters = c["d"], c["n"], c["k"], c["q"], c["w"], c["iters"]
    full = d * n <= 6e7
    vals = []
    with PinnedCore(0):
        if full:
            x = o.synth_x(d, n, c["rank"], c["factor_kind"], c["noise_kind"], c["sigma"],
                          1).astype(np.float64)
        else:
            n_s = max(q + 1, min(n, int(4e6 // d) + 1))
            x = o.synth_x(d, n, c["rank"], c["factor_kind"], c["noise_kind"], c["sigma"], 1,
                          col_lo=0, col_hi=n_s).astype(np.float64)
        for _ in range(timed_steps):
            if full:
                if kind == "reference":
                    left, right, xhat, xcheck, t_comp = r.compress(x, q, w, 1)
                else:
                    t0 = time.perf_counter()
                    left, right = o.build_projectors(x, q, w, 1)
                    xhat, xcheck = o.compress(x, left, right)
                    t_comp = time.perf_counter() - t0
                a, b = o.initialize(d, n, k, 1)
                ah, bc = o.compress_factors(a, b, left, right)
                if kind == "reference":
                    t_h = r.fasthals_rp_steps(xhat, xcheck, left, right, a, b, ah, bc, 1, iters)
                else:
                    t0 = time.perf_counter()
                    rg = o.rng(1)
                    for _ in range(iters):
                        o.fasthals_rp_step(xhat, xcheck, a, b, ah, bc, left, right, True, 0.0,
                                           0.0, rg)
                    t_h = time.perf_counter() - t0
                vals.append(t_comp + t_h)
                continue
            rng = np.random.default_rng(0)

            def timed(f, *args, **kw):
                t0 = time.perf_counter()
                f(*args, **kw)
                return time.perf_counter() - t0

            s_n = rng.standard_normal((n_s, q))
            t_d = rng.standard_normal((d, q))
            r_s = rng.standard_normal((q, n_s))
            t_nn = timed(impl.matmul, x, s_n)                 # X * S      (matrix.cpp:105-116)
            t_tn = timed(impl.matmul, x, t_d, tl=True)        # X^T * T    (129-140)
            t_cl = timed(impl.matmul, t_d, x, tl=True)        # L^T X      (compress_left)
            t_cr = timed(impl.matmul, x, r_s, tr=True)        # X R^T      (compress_right, NT)
            t_x = ((1 + 2 * w) * (t_nn + t_tn) + t_cl + t_cr) * (n / n_s)
            rows_q = max(q + 1, int(1.5e6 // q))
            t_qr = 0.0
            for rows in (d, n):
                rs_ = min(rows, rows_q)
                t_qr += (1 + 2 * w) * timed(impl.thin_qr, rng.standard_normal((rs_, q))) * (rows / rs_)
            t_sk = 0.0
            for rows, seed in ((n, 2), (d, 3)):
                rs_ = min(rows, rows_q)
                t_sk += timed(impl.gaussian_sketch, rs_, q, seed) * (rows / rs_)
            t_comp = t_x + t_qr + t_sk
            f = max(1.0, ((d + n) * k * (4 * q + 2 * k)) / 2e9)
            ds, ns = max(q + 1, int(d / f)), max(q + 1, int(n / f))
            xh = rng.random((q, ns))
            xc = rng.random((ds, q))
            left = np.linalg.qr(rng.standard_normal((ds, q)))[0]
            right = np.linalg.qr(rng.standard_normal((ns, q)))[0].T.copy()
            a, b = o.initialize(ds, ns, k, 1)
            ah, bc = o.compress_factors(a, b, left, right)
            if kind == "reference":
                t_step = r.fasthals_rp_steps(xh, xc, left, right, a, b, ah, bc, 1, 1)
            else:
                t0 = time.perf_counter()
                o.fasthals_rp_step(xh, xc, a, b, ah, bc, left, right, True, 0.0, 0.0, o.rng(1))
                t_step = time.perf_counter() - t0
            vals.append(t_comp + t_step * ((d + n) / (ds + ns)) * iters)
    if full:
        sample = (f"full {name.upper()} workload: build_projectors+compress_left/right on the "
                  f"{d}x{n} X and {iters} fasthals_rp_step calls, one thread pinned to core 0 "
                  f"(the reference solver is single-threaded)")
    else:
        sample = (f"extrapolated from bounded samples on one pinned core: the reference's "
                  f"{4 * w + 4} X contractions ((1+2w) X*S, (1+2w) X^T*T, L^T X, X R^T) on a "
                  f"{d}x{n_s} column slice scaled by n/n_s; {2 + 4 * w} thin_qr and the two "
                  f"sketches on <= {rows_q}-row slices scaled by rows; one fasthals_rp_step at "
                  f"{ds}x{ns} scaled by (d+n)/(d_s+n_s), x {iters} iterations")
    return vals, kind, sample


def shared_config(name, c, world):
    """The config dict BOTH arms print, identical for the same workload and N
    (the driver's same_config); what each arm ran on is in its own keys
    (impl, cpu_baseline)."""
    x_bytes = 4.0 * c["d"] * ((c["n"] + world - 1) // world)  # per GPU
    big = x_bytes > L2_BYTES
    return config_dict(name, c, f"X column-sharded over {world} GPUs (NCCL)" if world > 1
                       else "1 GPU",
                       {"l2": ("inputs larger than L2 (X %.0f MB > 126 MB)" % (x_bytes / 1e6))
                        if big else "L2 flushed (256 MB write) between timed steps"})


def config_dict(name, c, parallelism, extra=None):
    """The workload description both arms print (same keys: same_config)."""
    out = {"workload": workload_desc(name, c), "d": c["d"], "n": c["n"], "k": c["k"],
           "l": c["q"], "power_iterations": c["w"], "iterations": c["iters"],
           "parallelism": parallelism}
    out.update(extra or {})
    return out


def run_reference_arm(args, name, c, rank):
    if rank != 0:
        return
    # one untimed tiny sample as warm-up (CPU code has no JIT/caches to warm)
    small = dict(c, d=200, n=150, rank=3, k=3, q=6, w=1, iters=2)
    for _ in range(max(1, min(args.warmup, 1))):
        cpu_reference_sample("warmup", small, 1)
    vals, kind, sample = cpu_reference_sample(name, c, args.steps)
    v = statistics.mean(vals)
    model, ncpu = host_cpu()
    line = {"metric": METRIC, "value": v, "unit": "s", "n_gpus": args.gpus, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": v * 1e3, "higher_is_better": False,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "impl": "reference",
            "config": shared_config(name, c, args.gpus),
            "cpu_baseline": {"value": v, "unit": "s", "cores": 1, "kind": kind,
                             "sample": sample, "host_cpu": model, "host_cores": ncpu,
                             "pinning": "sched_setaffinity core 0 (taskset -c 0)",
                             "note": "the reference solver is single-threaded (cli.cpp:231-247 "
                                     "only runs independent jobs in parallel)"},
            "e2e": {"value": v, "unit": "s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------ our arm -------
def run_ours(args, name, c, rank, world, local_rank):
    import numpy as np
    import torch

    import paper_1712_02248_b200 as cb

    torch.cuda.set_device(local_rank)
    d, n, k, q, w, iters = c["d"], c["n"], c["k"], c["q"], c["w"], c["iters"]
    if world > 1:
        # column-sharded run: this rank holds X[:, lo:hi] (synthesised locally)
        ctx = cb.ShardedContext.from_process_group(local_rank)
        lo, hi = cb.shard_range(n, rank, world)
    else:
        ctx = cb.Context(local_rank)
        lo, hi = 0, n
    nloc = hi - lo
    ldx = (nloc + 3) // 4 * 4
    x = torch.empty((d, ldx), dtype=torch.float32, device="cuda")
    ctx.synth_x(d, n, c["rank"], c["factor_kind"], c["noise_kind"], c["sigma"], 1, x, lo, hi)
    xv = x[:, :nloc]
    solve = (lambda xx, cc, aa=None, bb=None: ctx.run_sharded(xx, n, cc, aa, bb)) if world > 1 \
        else (lambda xx, cc, aa=None, bb=None: ctx.run_device(xx, cc, aa, bb))
    cfg = cb.SolverConfig(algorithm=cb.FASTHALS_RP, k=k, sketch=cb.SketchConfig(q, w, 1),
                          max_iterations=iters, error_interval=iters, rel_tolerance=1e-300,
                          seed=1)
    a = torch.empty((d, k), device="cuda")
    b = torch.empty((nloc, k), device="cuda")
    flush = torch.empty(2 * L2_BYTES // 4, dtype=torch.float32, device="cuda")
    stream = torch.cuda.ExternalStream(ctx.stream())
    x_bytes = 4.0 * d * nloc  # this GPU's X bytes
    big = x_bytes > L2_BYTES

    for _ in range(args.warmup):
        solve(xv, cfg, a, b)
    torch.cuda.synchronize()
    if world > 1:
        torch.distributed.barrier()
    steps, comp, upd, passes = [], [], [], []
    launches0 = cb.launch_count()
    with ClockSampler(local_rank) as clk:
        for i in range(args.steps):
            if not big:
                flush.fill_(float(i))
            torch.cuda.synchronize()
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            _, _, tr = solve(xv, cfg, a, b)
            e1.record(stream)
            e1.synchronize()
            steps.append(e0.elapsed_time(e1) * 1e-3)
            comp.append(tr.compress_seconds)
            upd.append(tr.update_seconds)
            passes.append(tr.x_passes)
            redraws = tr.redraws
    torch.cuda.synchronize()
    launches = cb.launch_count() - launches0
    if world > 1:
        torch.distributed.barrier()
    value = statistics.mean([cc + uu for cc, uu in zip(comp, upd)])
    ms_per_step = statistics.mean(steps) * 1e3
    if world > 1:
        t = torch.tensor([value, ms_per_step], dtype=torch.float64, device="cuda")
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        value, ms_per_step = t.tolist()

    # roofline of the dominant kernel: the persistent FastHALS-RP kernel (HALS is
    # 75-90% of `value` at C2-C4), fp64 on the FP64 tensor cores (DMMA); and of
    # the compression GEMM, the X-stream contraction (HBM-bound).
    hbm, src = peaks()
    fp64_peak, fp64_src = fp64_peak_tflops()
    upd_mean = statistics.mean(upd)
    hals_flops = (4.0 * (d + nloc) * q * k + 2.0 * (d + nloc) * k * k + 4.0 * q * k * k)
    hals_bytes = 4.0 * (2 * d * q + 2 * q * nloc) + 8.0 * 3 * (d + nloc) * k
    t_iter = upd_mean / iters
    t_nn = ctx.time_xstream(xv, q, 0, iters=10)
    t_tn = ctx.time_xstream(xv, q, 1, iters=10)
    alg_bytes = 4.0 * d * nloc + 4.0 * (d + nloc) * q
    # the exact-accumulation contraction (int8 digit slices): the compressed
    # views always, the range finder of an ill-conditioned sketch
    exact_traffic = None
    prof = os.path.join(ROOT, "profiles", f"traffic_exact_{name}.json")
    if os.path.exists(prof):
        try:
            exact_traffic = json.load(open(prof)).get("bytes_per_launch")
        except Exception:
            exact_traffic = None
    try:
        te_nn, pe_nn = ctx.time_xs_exact(xv, q, 0, iters=5)
        te_tn, pe_tn = ctx.time_xs_exact(xv, q, 1, iters=5)
        exact = {"bound": "hbm", "kernel": "xs_i8_kernel (tcgen05 kind::i8, int32 accumulators; X*S with fp64-grade accumulation)",
                 "achieved": alg_bytes / te_nn / 1e9, "peak": hbm, "unit": "GB/s",
                 "frac": alg_bytes / te_nn / 1e9 / hbm, "launch_seconds": te_nn, "x_reads_per_contraction": pe_nn,
                 "per_x_read_frac": pe_nn * alg_bytes / te_nn / 1e9 / hbm,
                 "tn_achieved": alg_bytes / te_tn / 1e9, "tn_frac": alg_bytes / te_tn / 1e9 / hbm,
                 "tn_launch_seconds": te_tn, "algorithmic_bytes": alg_bytes, "traffic": exact_traffic,
                 "note": "a contraction wider than one column chunk (80 columns; 64 for integer X) reads X once per chunk"}
    except Exception as e:  # shape outside the kernel's envelope
        exact = {"unavailable": str(e)}
    ach_nn = alg_bytes / t_nn / 1e9
    ach_tn = alg_bytes / t_tn / 1e9
    traffic = None
    prof = os.path.join(ROOT, "profiles", f"traffic_{name}.json")
    if os.path.exists(prof):
        try:
            traffic = json.load(open(prof)).get("bytes_per_launch")
        except Exception:
            traffic = None
    hals_traffic = None
    prof = os.path.join(ROOT, "profiles", f"hals_traffic_{name}.json")
    if os.path.exists(prof):
        try:
            hals_traffic = json.load(open(prof)).get("bytes_per_iteration")
        except Exception:
            hals_traffic = None
    mean_comp = statistics.mean(comp)
    xstream_gbs = passes[0] * 4.0 * d * n / mean_comp / 1e9  # whole-job X bytes
    peak_note = (f"{src} (MEASURED_PEAKS.json hbm_gbs)" if src == "measured"
                 else "fallback 6.65 TB/s (B200_PROFILING.md)")

    line = {"metric": METRIC, "value": value, "unit": "s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_per_step,
            "higher_is_better": False, "scaling": "strong", "vs_baseline": None,
            "dtype": "f32", "data": "synthetic",
            "config": shared_config(name, c, world),
            "compress_seconds": mean_comp, "hals_seconds": upd_mean,
            "hals_ms_per_iteration": t_iter * 1e3,
            "redraws_per_run": redraws,
            "x_passes": passes[0], "x_stream_gbs": xstream_gbs,
            "x_stream_gbs_fused_min": (2 * w + 2) * 4.0 * d * n / mean_comp / 1e9,
            "roofline": {"bound": "tensor",
                         "kernel": "hals_kernel / hals_resident_kernel (persistent FastHALS-RP "
                                   "iteration, fp64 DMMA)",
                         "unit": "TFLOP/s", "achieved": hals_flops / t_iter / 1e12,
                         "peak": fp64_peak, "frac": hals_flops / t_iter / 1e12 / fp64_peak,
                         "traffic": hals_traffic, "peak_source": fp64_src,
                         "per": "one HALS iteration (device time of the iteration range "
                                "/ iterations, redraw servicing included)",
                         "algorithmic_flops": hals_flops,
                         "hbm_view": {"algorithmic_bytes": hals_bytes,
                                      "achieved_gbs": hals_bytes / t_iter / 1e9, "peak": hbm,
                                      "frac": hals_bytes / t_iter / 1e9 / hbm}},
            "roofline_xstream": {"bound": "hbm", "kernel": "xs_tc_kernel (X*S, NN contraction)",
                                 "achieved": ach_nn, "peak": hbm, "unit": "GB/s",
                                 "frac": ach_nn / hbm, "traffic": traffic,
                                 "peak_source": peak_note,
                                 "launch_seconds": t_nn, "algorithmic_bytes": alg_bytes,
                                 "tn_achieved": ach_tn, "tn_frac": ach_tn / hbm,
                                 "tn_launch_seconds": t_tn},
            "roofline_exact": exact,
            "gpu_launches": int(launches),
            "clocks": clk.summary()}

    if not args.no_e2e:
        xh = torch.empty((d, nloc), dtype=torch.float32, pin_memory=True)
        xh.copy_(xv)
        if world == 1:
            xnp = xh.numpy()
            ctx.run(xnp, cfg)  # warm
        e2e = []
        for _ in range(max(1, min(args.steps, 3))):
            if world > 1:
                torch.distributed.barrier()
            t0 = time.perf_counter()
            if world == 1:
                ctx.run(xnp, cfg)
            else:  # host shard -> device, collective run, factors -> host
                xd = xh.to("cuda")
                aa, bb, _ = ctx.run_sharded(xd, n, cfg)
                aa.cpu(), bb.cpu()
            e2e.append(time.perf_counter() - t0)
        ev = statistics.mean(e2e)
        if world > 1:
            t = torch.tensor([ev], dtype=torch.float64, device="cuda")
            torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
            ev = t.item()
        line["e2e"] = {"value": ev, "unit": "s",
                       "h2d_bytes_per_step": int(4 * d * n),
                       "d2h_bytes_per_step": int(4 * (d * world + n) * k)}

    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        vals, kind, sample = cpu_reference_sample(name, c, 1)
        model, ncpu = host_cpu()
        line["cpu_baseline"] = {"value": vals[0], "unit": "s", "cores": 1, "kind": kind,
                                "sample": sample, "host_cpu": model, "host_cores": ncpu,
                                "pinning": "sched_setaffinity core 0 (taskset -c 0)"}
    if rank == 0:
        print(json.dumps(line), flush=True)


def self_launch(args):
    """--gpus N without torchrun: re-run this script as N ranks (one per GPU)."""
    import socket
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr=127.0.0.1",
           f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def main():
    args = parse()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(self_launch(args))
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    from paper_1712_02248_b200 import CONFIGS
    c = CONFIGS[args.config]
    if args.impl == "reference":
        run_reference_arm(args, args.config, c, rank)
        return
    if world > 1:
        import torch
        torch.cuda.set_device(local_rank)
        torch.distributed.init_process_group("nccl")
    run_ours(args, args.config, c, rank, world, local_rank)
    if world > 1:
        import torch
        torch.distributed.destroy_process_group()


if __name__ == "__main__":
    main()
