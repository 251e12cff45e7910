"""Build one config-4-law sketch (plan + sample + CSC) at a reduced n: the
sampler's ncu target (a full n = 1e6 launch is 10^12 draws; ncu replays it
~40 times).  python profiles/scripts/sketch_c4.py [n]"""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
import paper_2306_06581_b200 as spk  # noqa: E402
from paper_2306_06581_b200 import workloads as W  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 200_000
w = W.c4(n=n, pairs=1_000_000)
with spk.Context(0) as ctx:
    kern = spk.Coords(w.x, w.y, w.cost, w.eta, scale=w.scale, eps=w.eps)
    t0 = time.perf_counter()
    sk = ctx.sketch(kern, w.a, w.b, "ot", w.lam, w.eps, w.s, 7, spk.SparSinkOptions(values=w.values))
    print(f"n={n} nnz={sk.nnz} sketch {time.perf_counter() - t0:.3f} s")
