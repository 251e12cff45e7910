"""Small instances of every hand-synchronised kernel family, for
compute-sanitizer (memcheck / racecheck / synccheck / initcheck):

  * blocked loop  -- slab x block layout, TMA bulk copies + mbarrier ring,
                     CTA-pair clusters with DSMEM partial sums (forced at small n)
  * small loop    -- one cluster, DSMEM broadcast + cluster barrier per half
  * batched loop  -- a cluster of CTAs per sketch, DSMEM exchange
  * shard halves  -- the emulated-rank sharded solve (CSR and slab x block)
  * sampler, CSC build, readout, dense on-the-fly comparator

  compute-sanitizer --tool racecheck python profiles/scripts/sanitize.py
Exit status 0 = every solve matched its reference path."""
import math
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))

import paper_2306_06581_b200 as spk  # noqa: E402
from paper_2306_06581_b200 import _lib as L  # noqa: E402
from paper_2306_06581_b200 import api  # noqa: E402
from paper_2306_06581_b200 import sharded as S  # noqa: E402
from paper_2306_06581_b200 import workloads as W  # noqa: E402


def main() -> int:
    n = 600
    x = W.uniforms(3, 0, 3 * n).reshape(n, 3)
    y = 0.2 + W.uniforms(3, 1, 3 * n).reshape(n, 3)
    a = np.full(n, 1.0 / n)
    kern = spk.Coords(x, y, "sqeuclid", scale=None, eps=0.05)
    cfg = spk.SolverConfig(0.05, math.inf, -1.0, 12)
    s = 8 * n * math.log(n)
    res = {}
    with spk.Context(0) as ctx:
        ctx.set_option(L.OPT_SMALL_LOOP, 0)
        ctx.set_option(L.OPT_BLOCKED_LOOP, 0)
        res["csr"] = ctx.spar_sink(kern, a, a, cfg, s, 5, spk.SparSinkOptions(values="f32"))
        ctx.set_option(L.OPT_BLOCKED_LOOP, 1)
        ctx.set_option(L.OPT_BLOCKED_MAX_W, 64)  # many tiles per half: the mbarrier ring wraps
        res["blocked"] = ctx.spar_sink(kern, a, a, cfg, s, 5, spk.SparSinkOptions(values="f32"))
        ctx.set_option(L.OPT_BLOCKED_LOOP, 0)
        ctx.set_option(L.OPT_SMALL_LOOP, 1)
        ctx.set_option(L.OPT_SMALL_CLUSTER, 4)
        res["small"] = ctx.spar_sink(kern, a, a, cfg, s, 5, spk.SparSinkOptions(values="f32"))
        # batched log-domain loop over WFR frame pairs (cluster of 2 CTAs per pair)
        coords, masses = W.c3_frames(3, frames=4, side=24)
        m = coords.shape[0]
        pairs = api.frame_pairs(4)
        bcfg = spk.SolverConfig(0.01, 1.0, -1.0, 15, stabilize=True)
        out = api.spar_sink_pairs(ctx, coords, masses, bcfg, 10 * m * math.log(m), 3, 0.1,
                                  opts=spk.SparSinkOptions(values="f32"))
        assert all(np.isfinite(r["objective"]) for _, _, r in out)
        # dense on-the-fly comparator
        res["dense"] = ctx.sinkhorn(spk.Coords(x[:200], y[:200], "sqeuclid", scale=None, eps=0.05),
                                    np.full(200, 1 / 200), np.full(200, 1 / 200), spk.SolverConfig(0.05, math.inf, -1.0, 5))
    # sharded halves, 2 emulated ranks (CSR and slab x block layouts)
    for blocked in (0, 1):
        outs = S.run_emulated(2, lambda comm, shard: S.spar_sink_sharded(comm, shard, kern, a, a, cfg, s, 5,
                                                                          spk.SparSinkOptions(values="f32")),
                              options={L.OPT_BLOCKED_LOOP: blocked})
        res[f"shard{blocked}"] = outs[0]
    ref = res["csr"]
    for k, r in res.items():
        if k == "dense":
            continue
        if not np.allclose(r.u, ref.u, rtol=1e-4):
            print("MISMATCH", k)
            return 1
    print("sanitize workload ok:", ", ".join(res))
    return 0


if __name__ == "__main__":
    sys.exit(main())
