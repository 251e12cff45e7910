"""Config 3 batched sketch build (cached K / K^g_k path) timing / ncu target.
  python profiles/scripts/c3_sketch_batch.py [pairs]"""
import math, sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
import paper_2306_06581_b200 as spk
from paper_2306_06581_b200 import api
from paper_2306_06581_b200 import workloads as W
P = int(sys.argv[1]) if len(sys.argv) > 1 else 16
coords, masses = W.c3_frames(3)
n = coords.shape[0]; s = 10 * n * math.log(n)
pairs = api.frame_pairs(masses.shape[0])[:P]
kern = spk.Coords(coords, coords, "wfr", 0.1, scale=1.0, eps=0.01)
with spk.Context(0) as ctx:
    for rep in range(2):
        t0 = time.perf_counter()
        sks = ctx.sketch_batch(kern, masses[[i for i, _ in pairs]], masses[[j for _, j in pairs]], "uot", 1.0, 0.01, s,
                               [api.mix_seed(3, k) for k in range(P)], spk.SparSinkOptions(values="f32"))
        dt = time.perf_counter() - t0
        print(f"batch of {P}: {dt:.4f} s, {1e3 * dt / P:.3f} ms per sketch", file=sys.stderr)
        for sk in sks:
            sk.free()
