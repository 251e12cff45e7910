#!/usr/bin/env python
"""Benchmark of the Spar-Sink hot path on B200 (BASELINE.json metric:
"sparse Sinkhorn iters/s and achieved HBM GB/s vs peak; end-to-end solve time").

Default workload: config 4 (n = 1e6, balanced OT, fp32 sketch values, fp64
scalings, 300 iterations), the configuration the north-star target (>= 60% of
HBM on 1 GPU) is quoted on. A "step" is one full 300-iteration Sinkhorn solve
on the HBM-resident sketch (persistent loop kernel + residual readout).

  python bench.py [--gpus N --steps K --warmup W] [--config c1|c2|c3|c4|c5]
  python bench.py --impl reference ...   # the reference's CPU loop (oracle/_ref)

Prints ONE JSON line on rank 0.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "sparse Sinkhorn iters/s and achieved HBM GB/s vs peak; end-to-end solve time"


def peaks() -> tuple[float, str]:
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        return float(json.loads(p.read_text())["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.rows: list[list[str]] = []
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--id={self.device}", f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.th = threading.Thread(target=self._read, daemon=True)
            self.th.start()
        except FileNotFoundError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([c.strip() for c in line.split(",")])

    def __exit__(self, *exc):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self) -> dict:
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"], "samples": 0}
        sm = [float(r[1]) for r in self.rows if len(r) > 2 and r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in self.rows if len(r) > 2 and r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[k] for r in self.rows if len(r) >= 9 for k in range(4)
                          if r[5 + k].lower().startswith("active")})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


def dist_init():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if ws > 1 or (os.environ.get("SPK_SHARDED") == "1" and "MASTER_ADDR" in os.environ):
        import torch
        import torch.distributed as dist

        torch.cuda.set_device(local)
        backend = "nccl" if os.environ.get("SPK_BACKEND", "nccl") == "nccl" else "gloo"
        dist.init_process_group(backend=backend)
    return ws, rank, local


def barrier(ws):
    if ws > 1:
        import torch.distributed as dist

        dist.barrier()


def max_over_ranks(x: float, ws: int) -> float:
    if ws == 1:
        return x
    import torch
    import torch.distributed as dist

    t = torch.tensor([x], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def sum_over_ranks(x: float, ws: int) -> float:
    if ws == 1:
        return x
    import torch
    import torch.distributed as dist

    t = torch.tensor([float(x)], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return float(t.item())


def value_bytes(values: str) -> int:
    return 4 if values == "f32" else 8


def cpu_same_law_sketch(w, nnz_target: float, seed: int = 77):
    """A CPU-drawn sketch with config 4's sampling law (p uniform on the
    support, so each row keeps ~Binomial(n, p*) uniformly placed columns with
    values K_ij / p*). Used only by the reference arm, which must not run our
    GPU sampler."""
    n = w.n
    rng = np.random.default_rng(seed)
    ps = min(1.0, nnz_target / (float(n) * n))
    counts = rng.binomial(n, ps, size=n)
    rp = np.zeros(n + 1, np.int64)
    np.cumsum(counts, out=rp[1:])
    cols = np.empty(rp[-1], np.uint32)
    vals = np.empty(rp[-1])
    chunk = 20000
    for r0 in range(0, n, chunk):
        r1 = min(n, r0 + chunk)
        m = rp[r1] - rp[r0]
        c = rng.integers(0, n, size=m, dtype=np.int64)
        rows = np.repeat(np.arange(r0, r1), counts[r0:r1])
        # sort columns inside each row
        order = np.lexsort((c, rows))
        c = c[order]
        d2 = ((w.x[rows] - w.y[c]) ** 2).sum(axis=1)
        k = np.exp(-(d2 / w.scale) / w.eps)
        cols[rp[r0]:rp[r1]] = c
        vals[rp[r0]:rp[r1]] = (k / ps).astype(np.float32)
    return rp, cols, vals


def run_reference(args, ws, rank):
    """--impl reference: the reference's own CPU loop (sinkhorn_ot/uot<SparseKernel>,
    compiled from /root/reference by oracle/Makefile into oracle/_ref) on the
    box's host; a bounded number of iterations per step."""
    if rank != 0:
        return
    from oracle import Oracle, Reference
    from paper_2306_06581_b200 import workloads as W

    if args.config == "c3":
        return run_reference_c3(args)
    w = W.CONFIGS[args.config]()
    iters = args.ref_iters
    t0 = time.time()
    if args.config == "c4":
        csr = cpu_same_law_sketch(w, w.s)
        sample = f"{iters} iterations of sinkhorn_ot<SparseKernel> per step on a CPU-drawn C4-law sketch " \
                 f"(n=1e6, {csr[0][-1]} nnz, fp64 values)"
    else:
        # small configs: the reference builds its own dense K and sketch
        R = Reference()
        Cm, c0 = R.pairwise_cost(w.x, w.y, w.cost, w.eta)
        Cm /= (c0 if w.scale is None else w.scale)
        K, ratio = R.kernel_from_cost(Cm, w.eps)
        plan = "uot" if w.uot else "ot"
        csr = R.poisson_sparsify(plan, w.a, w.b, K, ratio, w.s, 7, w.lam, w.eps)
        sample = f"{iters} iterations of sinkhorn_{plan}<SparseKernel> per step on the reference's own sketch"
    prep = time.time() - t0
    if Reference.available():
        R = Reference()
        kind = "reference"

        def step():
            secs, _ = R.sparse_loop_seconds(csr, w.a, w.b, w.eps, iters, w.lam, w.uot)
            return secs
    else:
        O = Oracle()
        kind = "port"

        def step():
            t, _, _ = O.time_scaling_iters(csr, w.a, w.b, iters)
            return t * iters
    for _ in range(args.warmup):
        step()
    times = [step() for _ in range(args.steps)]
    total = sum(times)
    value = args.steps * iters / total
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "iters/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * total / args.steps,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": w.name, "n": w.n, "iterations_per_step": iters, "nnz": int(csr[0][-1])},
        "cpu_baseline": {"value": value, "unit": "iters/s", "cores": 1, "host_cores": os.cpu_count(), "kind": kind,
                         "sample": sample},
        "e2e": {"value": value, "unit": "iters/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "extra": {"prep_s": prep, "note": f"one solve is single-threaded in the reference (proj/CMakeLists.txt:19; "
                                          f"no OpenMP): 1 of {os.cpu_count()} host cores"},
    }
    print(json.dumps(line), flush=True)


def c3_reference_pool(P: int, iters: int, sketches=None):
    """Config 3 on the host as the reference runs it: independent frame pairs,
    one single-threaded reference solve (log-domain sinkhorn_uot<SparseKernel>)
    per host thread, P threads at once (ctypes drops the GIL). sketches: the
    first P pairs' CSR (default: the reference's own spar_sink sketches on
    its dense WFR kernel). Returns (step(), sample)."""
    from concurrent.futures import ThreadPoolExecutor

    from oracle import Reference
    from paper_2306_06581_b200 import api
    from paper_2306_06581_b200 import workloads as W

    R = Reference()
    coords, masses = W.c3_frames(3)
    n = coords.shape[0]
    pairs = api.frame_pairs(masses.shape[0])[:P]
    if sketches is None:
        Cm, _ = R.pairwise_cost(coords, coords, "wfr", 0.1)
        K, ratio = R.kernel_from_cost(Cm, 0.01)
        del Cm
        s = 10 * n * math.log(n)

        def draw(k):
            i, j = pairs[k]
            return R.poisson_sparsify("uot", masses[i], masses[j], K, ratio, s, api.mix_seed(3, k), 1.0, 0.01)

        with ThreadPoolExecutor(P) as ex:
            sketches = list(ex.map(draw, range(P)))
        del K
        src = "the reference's own sketches (poisson_sparsify on its dense WFR kernel)"
    else:
        src = "the GPU-built sketches copied to host"

    def one(k):
        i, j = pairs[k]
        secs, _ = R.sparse_loop_seconds(sketches[k], masses[i], masses[j], 0.01, iters, 1.0, True, stabilize=True)
        return secs

    def step():
        t0 = time.perf_counter()
        with ThreadPoolExecutor(P) as ex:
            list(ex.map(one, range(P)))
        return time.perf_counter() - t0

    sample = (f"{P} frame pairs at once (1 reference solve per host thread, {P} of {os.cpu_count()} cores), "
              f"{iters} log-domain iterations of sinkhorn_uot<SparseKernel> each per step, on {src}")
    return step, sample


def run_reference_c3(args):
    P = max(1, min(os.cpu_count() or 1, 496))
    iters = args.ref_iters
    t0 = time.time()
    step, sample = c3_reference_pool(P, iters)
    prep = time.time() - t0
    for _ in range(args.warmup):
        step()
    times = [step() for _ in range(args.steps)]
    total = sum(times)
    value = args.steps * P * iters / total
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "iters/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * total / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": "C3", "n": 12544, "pairs": 496, "pairs_timed": P, "iterations_per_step": P * iters},
        "cpu_baseline": {"value": value, "unit": "iters/s", "cores": P, "host_cores": os.cpu_count(),
                         "kind": "reference", "sample": sample},
        "e2e": {"value": value, "unit": "iters/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "extra": {"prep_s": prep, "all_496_pairs_1000_iterations_s_extrapolated": 496 * 1000 / value},
    }
    print(json.dumps(line), flush=True)


def run_ours(args, ws, rank, local):
    import torch

    import paper_2306_06581_b200 as spk
    from paper_2306_06581_b200 import workloads as W

    torch.cuda.set_device(local)
    w = W.CONFIGS[args.config]()
    iters = args.iters or w.max_iter
    ctx = spk.Context(local)
    if os.environ.get("SPK_BLOCKED") is not None:  # loop variant override (profiling)
        from paper_2306_06581_b200 import _lib as L

        ctx.set_option(L.OPT_BLOCKED_LOOP, int(os.environ["SPK_BLOCKED"]))
    if os.environ.get("SPK_SPLIT") is not None:  # column parts per row slab (profiling)
        from paper_2306_06581_b200 import _lib as L

        ctx.set_option(L.OPT_BLOCKED_SPLIT, int(os.environ["SPK_SPLIT"]))
    if os.environ.get("SPK_SPREAD") is not None:  # column-bank spreading of the layout (profiling)
        from paper_2306_06581_b200 import _lib as L

        ctx.set_option(L.OPT_BLOCKED_SPREAD, int(os.environ["SPK_SPREAD"]))
    if os.environ.get("SPK_SMALL") is not None:  # one-cluster loop for small sketches (profiling)
        from paper_2306_06581_b200 import _lib as L

        ctx.set_option(L.OPT_SMALL_LOOP, int(os.environ["SPK_SMALL"]))
    if os.environ.get("SPK_ROW_LANES") is not None:  # grid loop: lanes per row (profiling)
        from paper_2306_06581_b200 import _lib as L

        ctx.set_option(L.OPT_ROW_LANES, int(os.environ["SPK_ROW_LANES"]))
    if os.environ.get("SPK_SMALL_CS") is not None:
        from paper_2306_06581_b200 import _lib as L

        ctx.set_option(L.OPT_SMALL_CLUSTER, int(os.environ["SPK_SMALL_CS"]))
    if os.environ.get("SPK_CLUSTER") is not None:  # CTA pairs as clusters (profiling)
        from paper_2306_06581_b200 import _lib as L

        ctx.set_option(L.OPT_BLOCKED_CLUSTER, int(os.environ["SPK_CLUSTER"]))
    stream = torch.cuda.current_stream()
    ctx.set_stream(stream.cuda_stream)
    kernel = spk.Coords(w.x, w.y, w.cost, w.eta, scale=w.scale, eps=w.eps)
    opts = spk.SparSinkOptions(values=w.values)
    plan = "uot" if w.uot else "ot"

    # ---- setup: plan + sample + CSC on the device (kept resident) ----
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    sk = ctx.sketch(kernel, w.a, w.b, plan, w.lam, w.eps, w.s, 7, opts)
    torch.cuda.synchronize()
    setup_s = time.perf_counter() - t0
    cfg = spk.SolverConfig(w.eps, w.lam, w.delta, iters, w.stabilize)

    # ---- warm-up + timed region: K full solves on the resident sketch ----
    for _ in range(args.warmup):
        sk.solve(cfg, w.uot, want_scalings=False)
    launches0 = ctx.launches
    loop_s, iters_done = [], 0
    barrier(ws)
    torch.cuda.synchronize()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        ev0.record(stream)
        for _ in range(args.steps):
            res = sk.solve(cfg, w.uot, want_scalings=False)
            loop_s.append(res.report["t_loop_s"])
            iters_done += res.report["iterations"]
        ev1.record(stream)
        torch.cuda.synchronize()
    barrier(ws)
    elapsed = max_over_ranks(ev0.elapsed_time(ev1) * 1e-3, ws)
    launches = ctx.launches - launches0
    value = ws * iters_done / elapsed  # replicas: every rank runs the full problem

    # ---- roofline of the dominant kernel (the persistent loop) ----
    peak, peak_src = peaks()
    vb = value_bytes(w.values)
    b_iter = W.bytes_per_iteration(sk.n, sk.nnz, vb)
    per_launch_iters = iters_done / args.steps
    mean_loop = sum(loop_s) / len(loop_s)
    achieved = b_iter * per_launch_iters / mean_loop / 1e9
    # DRAM bytes per launch: NOT measured in this run (no profiler in a timed
    # run) -- the per-iteration DRAM bytes of the committed ncu --set full
    # capture of this loop, times this launch's iterations; labelled as such
    traffic, traffic_src = None, None
    prof = ROOT / "profiles" / f"r2_ncu_{w.name.lower()}_loop.json"  # latest committed capture of this loop
    if not prof.exists():
        prof = ROOT / "profiles" / f"ncu_{w.name.lower()}_loop.json"
    if prof.exists():
        k0 = json.loads(prof.read_text())["kernels"][0]
        if "dram_bytes_per_iteration" in k0:
            traffic = k0["dram_bytes_per_iteration"] * per_launch_iters
            traffic_src = f"copied from {prof.relative_to(ROOT)} ({k0.get('variant', 'ncu capture')}), not measured in this run"

    # ---- end to end through the C ABI with host buffers ----
    e2e = None
    if not args.no_e2e:
        # host inputs in pinned memory (the library's uploads are cudaMemcpyAsync from the caller's pointers)
        pins = [torch.from_numpy(np.ascontiguousarray(z)).pin_memory() for z in (w.x, w.y, w.a, w.b)]
        px, py, pa, pb = (t.numpy() for t in pins)
        kernel_h = spk.Coords(px, py, w.cost, w.eta, scale=w.scale, eps=w.eps)
        e2e_times = []
        for k in range(4):  # the first call grows the memory pool; the median of the other three is reported
            torch.cuda.synchronize()
            t1 = time.perf_counter()
            r = ctx.spar_sink(kernel_h, pa, pb, cfg, w.s, 7, opts, uot=w.uot)
            torch.cuda.synchronize()
            e2e_times.append(time.perf_counter() - t1)
        e2e_t = max_over_ranks(sorted(e2e_times[1:])[1], ws)
        h2d = w.x.nbytes + w.y.nbytes + w.a.nbytes + w.b.nbytes
        d2h = r.u.nbytes + r.v.nbytes + 8 * 4
        e2e = {"value": ws * r.report["iterations"] / e2e_t, "unit": "iters/s", "h2d_bytes_per_step": h2d,
               "d2h_bytes_per_step": d2h, "solve_s": e2e_t, "solve_s_all": [round(x, 4) for x in e2e_times],
               "objective": r.report["objective"],
               "phases_s": {"plan": r.report["t_plan_s"], "sample": r.report["t_sample_s"],
                            "loop": r.report["t_loop_s"], "readout": r.report["t_readout_s"]}}

    # ---- CPU baseline: the reference loop on this very sketch (rank 0, N=1) ----
    cpu = None
    parity = None
    if rank == 0 and ws == 1 and not args.no_cpu:
        from oracle import Oracle, Reference

        rp, ci, vv = sk.csr()
        k_cpu = args.cpu_iters
        if Reference.available():
            # the reference's sinkhorn_<plan><SparseKernel> on this very sketch for k_cpu
            # fixed iterations: its wall time is the CPU baseline, its scalings
            # the parity check of the production loop on the same iterations
            t0 = time.perf_counter()
            ru, rv, _, _, rrep = Reference().sinkhorn(w.a, w.b, w.eps, w.lam, -1.0, k_cpu, stabilize=w.stabilize,
                                                      policy="mask", uot=w.uot, csr=(rp, ci, vv))
            secs = rrep["wall_time_s"] if rrep.get("wall_time_s") else time.perf_counter() - t0
            kind = "reference"
            g = sk.solve(spk.SolverConfig(w.eps, w.lam, -1.0, k_cpu, w.stabilize), w.uot)
            rel = lambda a, b: float(np.max(np.abs(a - b) / np.maximum(np.abs(b), 1e-300)))  # noqa: E731
            parity = {"iterations": k_cpu, "max_rel_diff_u": rel(g.u, ru), "max_rel_diff_v": rel(g.v, rv),
                      "masked_rows_equal": g.report["masked_rows"] == rrep["masked_rows"],
                      "against": "reference sinkhorn on the same GPU-built sketch (oracle/_ref)"}
        else:
            t, _, _ = Oracle().time_scaling_iters((rp, ci, vv), w.a, w.b, k_cpu)
            secs, kind = t * k_cpu, "port"
            parity = None
        cpu = {"value": k_cpu / secs, "unit": "iters/s", "cores": 1, "host_cores": os.cpu_count(), "kind": kind,
               "sample": f"{k_cpu} of {iters} iterations of sinkhorn_{plan}<SparseKernel> on the GPU-built "
                         f"{w.name} sketch ({sk.nnz} nnz) copied to host, 1 of {os.cpu_count()} host cores "
                         f"(one reference solve is single-threaded)"}
        if args.config == "c4":
            # the reference cannot build config 4's dense K (8 TB); its sampler
            # (poisson_sparsify, sparsify.cpp:169-201) restated on coordinates
            # (oracle) on a row sample, extrapolated to all n rows (labelled)
            plan = sk.plan()
            ra = np.sqrt(w.a)
            sa = 0.0
            for t_ in ra.tolist():
                sa += t_
            rows = 100
            t0 = time.perf_counter()
            Oracle().sample_rows_coords(w.x, w.y, "sqeuclid", 0.0, w.scale, w.eps, "ot", plan["factorized"],
                                        ra / sa, ra / sa, 0.0, plan["inv"], w.s, 7, 0, rows)
            ts = time.perf_counter() - t0
            cpu["sampler"] = {"rows_timed": rows, "seconds": ts, "extrapolated_all_rows_s": ts * w.n / rows,
                              "kind": "port (oracle restatement of poisson_sparsify on coordinates), 1 core",
                              "gpu_sample_s": e2e["phases_s"]["sample"] if e2e else None}

    dense = None
    if args.config == "c5" and rank == 0:
        dense = c5_dense_comparison(ctx, w, kernel, iters, args.no_cpu)

    line = {
        "metric": METRIC, "value": value, "unit": "iters/s", "n_gpus": ws, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": 1e3 * elapsed / args.steps, "higher_is_better": True,
        "scaling": "strong" if args.config in ("c2", "c4") else "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic",
        "config": {"workload": w.name, "n": sk.n, "nnz": sk.nnz, "s": w.s, "epsilon": w.eps,
                   "lambda": w.lam if math.isfinite(w.lam) else "inf", "iterations_per_step": per_launch_iters,
                   "sketch_values": w.values, "scalings": "f64",
                   "parallelism": f"replicas{ws}" if ws > 1 else "single",
                   "l2": f"inputs larger than L2: sketch {(sk.nnz * 2 * (vb + 4)) / 1e9:.2f} GB"
                         if args.config == "c4" else "sketch L2-resident (config smaller than L2)"},
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                     "traffic": traffic, "traffic_source": traffic_src, "kernel": "loop_kernel (persistent, both halves)",
                     "bytes_per_iter": b_iter, "peak_source": peak_src},
        "cpu_baseline": cpu,
        "e2e": e2e,
        "gpu_launches": launches,
        "clocks": clk.summary(),
        "parity": parity,
        "dense_comparison": dense,
        "extra": {"setup_s": setup_s, "loop_ms_per_iter": 1e3 * mean_loop / per_launch_iters,
                  "kernel_nnz": sk.kernel_nnz, "factorized_plan": sk.factorized_plan},
    }
    if rank == 0:
        print(json.dumps(line), flush=True)
    sk.free()
    ctx.close()


def c5_dense_comparison(ctx, w, kernel, iters, no_cpu):
    """Config 5 as BASELINE.json states it: the classical Sinkhorn with K
    recomputed on the fly every iteration (the dense comparator, fp32 K) for
    `iters` iterations, and Spar-Sink at s = 4, 8, 16 n ln n with the
    objective error against it. The comparator's roofline is the measured
    MUFU.EX2 peak (2 n^2 exp2 per iteration). CPU: the reference's dense
    sinkhorn_ot<KernelMatrix> at n = 8000 (2 iterations, its K built by the
    reference) scaled by n^2 to config 5's n (labelled)."""
    import paper_2306_06581_b200 as spk

    MUFU_PEAK = 4.619e12  # profiles/microbench/r1_sfu_fma_peak_b200.txt (measured MUFU.EX2 / s)
    cfg = spk.SolverConfig(w.eps, w.lam, -1.0, iters)
    ctx.sinkhorn(kernel, w.a, w.b, spk.SolverConfig(w.eps, w.lam, -1.0, 5))  # warm-up
    d = ctx.sinkhorn(kernel, w.a, w.b, cfg)
    evals = 2.0 * w.n * w.n * d.report["iterations"] / d.report["t_loop_s"]
    out = {"n": w.n, "iterations": d.report["iterations"], "loop_s": d.report["t_loop_s"],
           "ms_per_iteration": 1e3 * d.report["t_loop_s"] / d.report["iterations"],
           "kernel_evals_per_s": evals, "mufu_ex2_peak_per_s": MUFU_PEAK, "frac_of_mufu_peak": evals / MUFU_PEAK,
           "objective": d.report["objective"], "spar_sink": []}
    for mult in (4, 8, 16):
        sp = ctx.spar_sink(kernel, w.a, w.b, cfg, mult * w.n * math.log(w.n), 7)
        out["spar_sink"].append({"s_over_nlogn": mult, "sketch_nnz": sp.report["sketch_nnz"],
                                 "objective": sp.report["objective"],
                                 "rel_error_vs_dense": abs(sp.report["objective"] - d.report["objective"]) /
                                 abs(d.report["objective"])})
    if not no_cpu:
        from oracle import Reference
        from paper_2306_06581_b200 import workloads as W

        if Reference.available():
            m = 8000
            ws = W.c5(n=m)
            R = Reference()
            Cm, c0 = R.pairwise_cost(ws.x, ws.y)
            Cm /= c0
            K, r = R.kernel_from_cost(Cm, ws.eps)
            del Cm
            _, _, _, _, rep = R.sinkhorn(ws.a, ws.b, ws.eps, ws.lam, -1.0, 2, K=K, nnz_ratio=r)
            per_it = rep["wall_time_s"] / 2
            out["cpu_reference_dense"] = {
                "n_timed": m, "s_per_iteration": per_it, "kind": "reference", "cores": 1,
                "extrapolated_s_per_iteration_at_n": per_it * (w.n / m) ** 2,
                "sample": f"2 iterations of the reference's dense sinkhorn_ot<KernelMatrix> at n = {m} "
                          f"(K built by the reference), scaled by n^2 to n = {w.n} (labelled extrapolation)"}
    return out


def run_sharded(args, ws, rank, local):
    """N > 1: config 4's rows and columns sharded across the N GPUs (SURVEY
    §8(e)) by the library's own driver (spk_sharded_*): NCCL loaded by the
    library, one all-gather per half-iteration, the whole iteration loop
    captured once as a CUDA graph and replayed per solve. Strong scaling: the
    same n = 1e6 problem at every N."""
    import torch
    import torch.distributed as dist

    import paper_2306_06581_b200 as spk
    from paper_2306_06581_b200 import sharded as S
    from paper_2306_06581_b200 import workloads as W

    torch.cuda.set_device(local)
    w = W.CONFIGS[args.config]()
    iters = args.iters or w.max_iter
    ctx = spk.Context(local)
    uid = [S.LibComm.unique_id(ctx.lib) if rank == 0 else None]
    dist.broadcast_object_list(uid, src=0)
    comm = S.LibComm.nccl(ctx, uid[0], ws, rank)
    kernel = spk.Coords(w.x, w.y, w.cost, w.eta, scale=w.scale, eps=w.eps)
    opts = spk.SparSinkOptions(values=w.values)
    plan = "uot" if w.uot else "ot"
    stream = torch.cuda.current_stream()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    sk = S.LibShardedSketch(comm, kernel, w.a, w.b, plan, w.lam, w.eps, w.s, 7, opts)
    torch.cuda.synchronize()
    setup_s = max_over_ranks(time.perf_counter() - t0, ws)
    cfg = spk.SolverConfig(w.eps, w.lam, w.delta, iters, w.stabilize)
    for _ in range(args.warmup):  # the first solve captures the loop graph
        sk.solve(cfg, w.uot, want_scalings=False)
    launches0 = ctx.launches
    iters_done = 0
    loop_s = []
    barrier(ws)
    torch.cuda.synchronize()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        ev0.record(stream)
        for _ in range(args.steps):
            res = sk.solve(cfg, w.uot, want_scalings=False)
            iters_done += res.report["iterations"]
            loop_s.append(res.report["t_loop_s"])
        ev1.record(stream)
        torch.cuda.synchronize()
    barrier(ws)
    # library calls synchronise their own stream before returning, so the
    # host-bracketed events cover them; the in-library loop time is event-timed
    elapsed = max_over_ranks(ev0.elapsed_time(ev1) * 1e-3, ws)
    mean_loop = max_over_ranks(sum(loop_s) / len(loop_s), ws)
    launches = ctx.launches - launches0
    value = iters_done / elapsed  # one problem shared by all ranks
    peak, peak_src = peaks()
    vb = value_bytes(w.values)
    b_iter = W.bytes_per_iteration(sk.info["n"], sk.info["nnz"], vb)
    achieved = b_iter * iters_done / args.steps / mean_loop / 1e9
    e2e = None
    if not args.no_e2e:
        torch.cuda.synchronize()
        barrier(ws)
        t1 = time.perf_counter()
        sk2 = S.LibShardedSketch(comm, kernel, w.a, w.b, plan, w.lam, w.eps, w.s, 7, opts)
        r = sk2.solve(cfg, w.uot)
        sk2.free()
        torch.cuda.synchronize()
        e2e_t = max_over_ranks(time.perf_counter() - t1, ws)
        h2d = w.x.nbytes + w.y.nbytes + w.a.nbytes + w.b.nbytes
        d2h = r.u.nbytes + r.v.nbytes + 8 * 4
        e2e = {"value": r.report["iterations"] / e2e_t, "unit": "iters/s", "h2d_bytes_per_step": h2d,
               "d2h_bytes_per_step": d2h, "solve_s": e2e_t, "objective": r.report["objective"],
               "note": "spar_sink over all ranks through the library driver, graph capture included"}
    line = {
        "metric": METRIC, "value": value, "unit": "iters/s", "n_gpus": ws, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": 1e3 * elapsed / args.steps, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": w.name, "n": sk.info["n"], "nnz": sk.info["nnz"], "s": w.s, "epsilon": w.eps,
                   "lambda": w.lam if math.isfinite(w.lam) else "inf", "iterations_per_step": iters_done / args.steps,
                   "sketch_values": w.values, "scalings": "f64", "parallelism": f"rowcol-shard{ws}",
                   "l2": f"inputs larger than L2: sketch {(sk.info['nnz'] * 2 * (vb + 4)) / 1e9:.2f} GB"},
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak * ws, "unit": "GB/s",
                     "frac": achieved / (peak * ws), "traffic": None,
                     "kernel": "captured loop graph: shard_half_kernel (slab x block, CTA-pair clusters) + NCCL "
                               "all-gather per half; whole job, max over ranks", "bytes_per_iter": b_iter,
                     "peak_source": f"{ws} x {peak_src}"},
        "cpu_baseline": None,
        "e2e": e2e,
        "gpu_launches": launches,
        "clocks": clk.summary(),
        "extra": {"setup_s": setup_s, "ms_per_iter": 1e3 * elapsed / iters_done,
                  "loop_ms_per_iter": 1e3 * mean_loop * args.steps / iters_done,
                  "kernel_nnz": sk.info["kernel_nnz"], "captured_launches_per_solve": sk.info["captured_launches"],
                  "driver": "library (spk_sharded_*, NCCL + CUDA graph)"},
    }
    if rank == 0:
        print(json.dumps(line), flush=True)
    sk.free()
    comm.close()
    ctx.close()


def run_c3_batch(args, ws, rank, local):
    """Config 3 as BASELINE.json states it: ALL 496 WFR frame pairs (32 synthetic
    frames of 112x112, n = 12,544, UOT lambda = 1, eps = 0.01, s = 10 n ln n,
    log domain, up to 1000 iterations, fp32 sketch values). A step = one
    spk_sketch_solve_batch over this rank's pairs (a CTA per pair); the pairs
    split round-robin over ranks with no communication (weak in the pairs:
    `value` = iterations of all pairs of all ranks / max rank time)."""
    import torch

    import paper_2306_06581_b200 as spk
    from paper_2306_06581_b200 import api
    from paper_2306_06581_b200 import workloads as W

    torch.cuda.set_device(local)
    coords, masses = W.c3_frames(3)
    n = coords.shape[0]
    pairs = api.frame_pairs(masses.shape[0])
    mine = list(range(rank, len(pairs), ws))
    iters = args.iters or 1000
    cfg = spk.SolverConfig(0.01, 1.0, 1e-6, iters, stabilize=True)
    s = 10 * n * math.log(n)
    kern = spk.Coords(coords, coords, "wfr", 0.1, scale=1.0, eps=0.01)
    opts = spk.SparSinkOptions(values="f32")
    ctx = spk.Context(local)
    from paper_2306_06581_b200 import _lib as L

    for env, key in (("SPK_BATCH_CS", L.OPT_BATCH_CLUSTER), ("SPK_BATCH_U", L.OPT_BATCH_UNROLL)):
        if os.environ.get(env) is not None:  # batched-loop variant override (profiling)
            ctx.set_option(key, int(os.environ[env]))
    stream = torch.cuda.current_stream()
    ctx.set_stream(stream.cuda_stream)
    t0 = time.perf_counter()
    sks = ctx.sketch_batch(kern, masses[[pairs[k][0] for k in mine]], masses[[pairs[k][1] for k in mine]], "uot",
                           1.0, 0.01, s, [api.mix_seed(3, k) for k in mine], opts)
    torch.cuda.synchronize()
    setup_s = time.perf_counter() - t0
    for _ in range(args.warmup):
        api.solve_batch(ctx, sks, cfg, uot=True)
    launches0 = ctx.launches
    iters_done = 0
    barrier(ws)
    torch.cuda.synchronize()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        ev0.record(stream)
        for _ in range(args.steps):
            reps = api.solve_batch(ctx, sks, cfg, uot=True)
            iters_done += sum(r["iterations"] for r in reps)
        ev1.record(stream)
        torch.cuda.synchronize()
    barrier(ws)
    elapsed = max_over_ranks(ev0.elapsed_time(ev1) * 1e-3, ws)
    total_iters = sum_over_ranks(iters_done, ws)
    value = total_iters / elapsed
    # algorithmic bytes: V + I = 8 bytes per entry and half (fp32
    # sketch: log K~ and the index travel as one u64 per entry)
    nnz = [sk.nnz for sk in sks]
    b_pair_iter = [W.bytes_per_iteration(n, z, 4) for z in nnz]
    per_step_bytes = sum(b * r["iterations"] for b, r in zip(b_pair_iter, reps))
    achieved = sum_over_ranks(per_step_bytes, ws) * args.steps / elapsed / 1e9
    peak, peak_src = peaks()
    # the CPU leg's inputs, then the timed part's sketches go back to the memory
    # pool (the end-to-end call draws its own 496)
    want_cpu = rank == 0 and ws == 1 and not args.no_cpu
    Pcpu = max(1, min(os.cpu_count() or 1, len(sks)))
    cpu_csr = [sks[k].csr() for k in range(Pcpu)] if want_cpu else None
    for sk in sks:
        sk.free()
    e2e = None
    if not args.no_e2e:
        torch.cuda.synchronize()
        barrier(ws)
        t1 = time.perf_counter()
        out = api.spar_sink_pairs(ctx, coords, masses, cfg, s, 3, 0.1, opts=opts, rank=rank, world=ws)
        torch.cuda.synchronize()
        e2e_t = max_over_ranks(time.perf_counter() - t1, ws)
        e2e = {"value": sum_over_ranks(sum(r["iterations"] for _, _, r in out), ws) / e2e_t, "unit": "iters/s",
               "h2d_bytes_per_step": int(masses.nbytes + 2 * coords.nbytes),
               "d2h_bytes_per_step": 8 * 16 * len(out), "solve_s": e2e_t,
               "pairs": len(pairs), "objective_pair0": out[0][2]["objective"] if out else None}
    cpu = None
    if want_cpu:
        P = Pcpu
        step, sample = c3_reference_pool(P, args.cpu_iters, cpu_csr)
        secs = step()
        cpu = {"value": P * args.cpu_iters / secs, "unit": "iters/s", "cores": P, "host_cores": os.cpu_count(),
               "kind": "reference", "sample": sample}
    line = {
        "metric": METRIC, "value": value, "unit": "iters/s", "n_gpus": ws, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": 1e3 * elapsed / args.steps, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": "C3", "n": n, "pairs": len(pairs), "pairs_this_rank": len(mine), "epsilon": 0.01,
                   "lambda": 1.0, "iterations_max": iters,
                   "sketch_values": "f32 (streamed as one u64 per entry: log K~ with a 37-bit mantissa | 16-bit index)",
                   "batch_cluster": ctx.get_option(L.OPT_BATCH_CLUSTER), "batch_unroll": ctx.get_option(L.OPT_BATCH_UNROLL),
                   "scalings": "f64 (shared memory)", "parallelism": f"pairs-round-robin{ws}" if ws > 1 else "single",
                   "l2": "inputs larger than L2: 496 sketches ~10 GB"},
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                     "traffic": None, "kernel": "batch_log_kernel (one cluster of CTAs per pair)",
                     "bytes_per_iter": "per pair: 2 nnz (4+4) + 2 (n+1) 8 + 64 n", "peak_source": peak_src},
        "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": ctx.launches - launches0, "clocks": clk.summary(),
        "extra": {"setup_s": setup_s, "iterations_per_step": total_iters / args.steps,
                  "converged_last_step": sum(r["converged"] for r in reps)},
    }
    if rank == 0:
        print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="c4", choices=["c1", "c2", "c3", "c4", "c5"])
    ap.add_argument("--iters", type=int, default=0, help="iterations per step (default: the config's)")
    ap.add_argument("--cpu-iters", type=int, default=10)
    ap.add_argument("--ref-iters", type=int, default=10)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3  # timing rule: >= 3 warm-up steps
    ws, rank, local = dist_init()
    if args.impl == "reference":
        run_reference(args, ws, rank)
    elif (ws > 1 and args.config in ("c2", "c4")) or os.environ.get("SPK_SHARDED") == "1":
        run_sharded(args, ws, rank, local)  # rows/columns of one problem across the GPUs
    elif args.config == "c3":
        run_c3_batch(args, ws, rank, local)  # all 496 frame pairs, batched, split over ranks
    else:
        run_ours(args, ws, rank, local)  # N = 1, or replicas for the small configs
    import torch.distributed as dist

    if dist.is_available() and dist.is_initialized():
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
