"""Config 5's dense on-the-fly comparator (K recomputed from coordinates every
iteration: 2 n^2 kernel evaluations per iteration) at n = 5e4, 200 iterations:
evaluations/s for the SFU/FMA roofline.  python profiles/scripts/c5_dense.py [n] [iters]"""
import json
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
import paper_2306_06581_b200 as spk  # noqa: E402
from paper_2306_06581_b200 import workloads as W  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 50_000
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 200
w = W.c5(n=n)
kern = spk.Coords(w.x, w.y, w.cost, w.eta, scale=w.scale, eps=w.eps)
cfg = spk.SolverConfig(w.eps, w.lam, -1.0, iters)
with spk.Context(0) as ctx:
    ctx.sinkhorn(kern, w.a, w.b, spk.SolverConfig(w.eps, w.lam, -1.0, 5))  # warm-up
    t0 = time.perf_counter()
    r = ctx.sinkhorn(kern, w.a, w.b, cfg)
    wall = time.perf_counter() - t0
rep = r.report
evals = 2.0 * n * n * rep["iterations"]
print(json.dumps({"n": n, "iterations": rep["iterations"], "loop_s": rep["t_loop_s"], "wall_s": wall,
                  "kernel_evals_per_s": evals / rep["t_loop_s"], "objective": rep["objective"],
                  "ms_per_iteration": 1e3 * rep["t_loop_s"] / rep["iterations"]}))
