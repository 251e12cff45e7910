"""ncu target: config 3 batch of P frame pairs, `iters` iterations (one launch).
  python profiles/scripts/c3_batch_prof.py [P] [iters]"""
import math
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
import paper_2306_06581_b200 as spk  # noqa: E402
from paper_2306_06581_b200 import api  # noqa: E402
from paper_2306_06581_b200 import workloads as W  # noqa: E402

P = int(sys.argv[1]) if len(sys.argv) > 1 else 148
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 50
coords, masses = W.c3_frames(3)
n = coords.shape[0]
s = 10 * n * math.log(n)
pairs = api.frame_pairs(masses.shape[0])[:P]
kern = spk.Coords(coords, coords, "wfr", 0.1, scale=1.0, eps=0.01)
with spk.Context(0) as ctx:
    sks = [ctx.sketch(kern, masses[i], masses[j], "uot", 1.0, 0.01, s, api.mix_seed(3, k),
                      spk.SparSinkOptions(values="f32")) for k, (i, j) in enumerate(pairs)]
    reps = api.solve_batch(ctx, sks, spk.SolverConfig(0.01, 1.0, -1.0, iters, stabilize=True), uot=True)
    print("loop_s", reps[0]["t_loop_s"] * P, "iters", iters)
