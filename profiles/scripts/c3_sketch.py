"""Config 3 sketch timing / ncu target: a few WFR frame-pair sketches (n = 12,544)."""
import math, sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
import paper_2306_06581_b200 as spk
from paper_2306_06581_b200 import api
from paper_2306_06581_b200 import workloads as W
coords, masses = W.c3_frames(3)
n = coords.shape[0]; s = 10 * n * math.log(n)
kern = spk.Coords(coords, coords, "wfr", 0.1, scale=1.0, eps=0.01)
with spk.Context(0) as ctx:
    for k in range(4):
        t0 = time.perf_counter()
        sk = ctx.sketch(kern, masses[0], masses[k + 1], "uot", 1.0, 0.01, s, k, spk.SparSinkOptions(values="f32"))
        print("sketch", time.perf_counter() - t0, sk.nnz, file=sys.stderr)
        sk.free()
