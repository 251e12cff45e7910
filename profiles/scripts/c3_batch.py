"""Config 3 end to end on one GPU: 496 WFR frame pairs (32 frames of 112x112)
sketched, solved as ONE batch (a CTA per pair), objectives read out; plus the
one-pair-at-a-time path on the first P pairs for comparison.
  python profiles/scripts/c3_batch.py [pairs_for_sequential]"""
import json
import math
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
import paper_2306_06581_b200 as spk  # noqa: E402
from paper_2306_06581_b200 import api  # noqa: E402
from paper_2306_06581_b200 import workloads as W  # noqa: E402

P = int(sys.argv[1]) if len(sys.argv) > 1 else 8
coords, masses = W.c3_frames(3)
n = coords.shape[0]
cfg = spk.SolverConfig(0.01, 1.0, 1e-6, 1000, stabilize=True)
s = 10 * n * math.log(n)
pairs = api.frame_pairs(masses.shape[0])
kern = spk.Coords(coords, coords, "wfr", 0.1, scale=1.0, eps=0.01)
opts = spk.SparSinkOptions(values="f32")
with spk.Context(0) as ctx:
    ctx.sketch(kern, masses[0], masses[1], "uot", 1.0, 0.01, s, 1, opts).free()  # warm-up
    t0 = time.perf_counter()
    sks = [ctx.sketch(kern, masses[i], masses[j], "uot", 1.0, 0.01, s, api.mix_seed(3, k), opts)
           for k, (i, j) in enumerate(pairs)]
    t1 = time.perf_counter()
    reps = api.solve_batch(ctx, sks, cfg, uot=True)
    t2 = time.perf_counter()
    objs = [sk.readout(kern, uot=True, lambda_=1.0, epsilon=0.01)[2] for sk in sks]
    t3 = time.perf_counter()
    iters = sum(r["iterations"] for r in reps)
    for sk in sks:
        sk.free()
    t4 = time.perf_counter()
    seq = [ctx.spar_sink(kern, masses[i], masses[j], cfg, s, api.mix_seed(3, k), opts, uot=True)
           for k, (i, j) in enumerate(pairs[:P])]
    t5 = time.perf_counter()
    same = all(abs(r.report["objective"] - objs[k]) <= 1e-12 * abs(objs[k]) for k, r in enumerate(seq))
    print(json.dumps({"pairs": len(pairs), "n": n, "sketch_s": t1 - t0, "batch_loop_s": t2 - t1,
                      "readout_s": t3 - t2, "total_s": t3 - t0, "iterations_total": iters,
                      "iters_per_pair_mean": iters / len(pairs), "converged": sum(r["converged"] for r in reps),
                      "batch_iters_per_s": iters / (t2 - t1),
                      "sequential_pairs": P, "sequential_s_per_pair": (t5 - t4) / P,
                      "sequential_iters_per_s": sum(r.report["iterations"] for r in seq) / (t5 - t4),
                      "objectives_match_sequential": same}))
