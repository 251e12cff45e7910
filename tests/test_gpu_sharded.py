"""GPU: the row/column-sharded path (spk_shard_* + sharded.py) at W = 2, 3, 4
emulated ranks on one GPU (threads with host-synchronised collectives; no
kernel waits on another rank's kernel), against the single-GPU path.

SURVEY §8(e): the union of the row slabs is the single-GPU sketch bit for bit
(per-row RNG streams, normaliser from the gathered per-row sums in fixed
order); the sharded loop matches the single-GPU loop to rounding (sums in a
different order), with identical iteration and mask counts.
"""
import math

import numpy as np
import pytest
import torch

import paper_2306_06581_b200 as spk
from paper_2306_06581_b200 import sharded as S
from paper_2306_06581_b200 import workloads as Wl

pytestmark = pytest.mark.gpu


def _c4_like(n=3000, seed=11):
    x = Wl.student_t3(seed, 0, 3 * n).reshape(n, 3)
    y = Wl.student_t3(seed, 1, 3 * n).reshape(n, 3)
    q = Wl.c4_quantile(x, y, seed, 200_000)
    a = np.full(n, 1.0 / n)
    return x, y, a, q


def _sketch_triplets(world, kern, a, b, plan_kind, lam, eps, s, seed, opts):
    """Each emulated rank builds its row slab; returns the union as sorted
    (row, col, value) arrays, taken from the column-exchange export."""

    def fn(comm, shard):
        kd, keep = kern.desc()
        n, W, r = int(kd.n), comm.world, comm.rank
        m, lo, hi = S.slab(n, W, r)
        shard.bind_stream()
        need, rs, rn = shard.plan_rows(kd, a, b, plan_kind, lam, eps, W, r, m)
        rs_all = rn_all = None
        if need:
            rs_all, rn_all = shard.zeros(W * m), shard.zeros(W * m, torch.int64)
            rs_all[r * m:(r + 1) * m].copy_(rs[:m])
            rn_all[r * m:(r + 1) * m].copy_(rn[:m])
            comm.all_gather(rs_all, m)
            comm.all_gather(rn_all, m)
        shard.create(kd, a, b, plan_kind, lam, eps, s, seed, opts, W, r, rs_all, rn_all)
        info = shard.info()
        counts, rows, vals, _ = shard.export(W, m, info["row_nnz"], info["value_bytes"])
        cols = np.repeat(np.arange(W * m), counts.cpu().numpy())
        return rows.cpu().numpy().astype(np.int64), cols, vals.cpu().numpy().astype(np.float64), info

    parts = S.run_emulated(world, fn)
    rows = np.concatenate([p[0] for p in parts])
    cols = np.concatenate([p[1] for p in parts])
    vals = np.concatenate([p[2] for p in parts])
    order = np.lexsort((cols, rows))
    return rows[order], cols[order], vals[order], [p[3] for p in parts]


@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("plan", ["ot", "uot"])
def test_shard_union_is_the_single_gpu_sketch(ctx, world, plan):
    x, y, a, q = _c4_like()
    b = a.copy() if plan == "ot" else a * 1.5
    kern = spk.Coords(x, y, scale=q, eps=0.05)
    lam = math.inf if plan == "ot" else 1.0
    n = len(a)
    s = 8 * n * math.log(n)
    sk = ctx.sketch(kern, a, b, plan, lam, 0.05, s, 21)
    rp, ci, vv = sk.csr()
    ref_rows = np.repeat(np.arange(n), np.diff(rp))
    kind = spk._lib.PLAN_UOT if plan == "uot" else spk._lib.PLAN_OT
    rows, cols, vals, infos = _sketch_triplets(world, kern, a, b, kind, lam, 0.05, s, 21, spk.SparSinkOptions())
    assert np.array_equal(rows, ref_rows) and np.array_equal(cols, ci.astype(np.int64))
    np.testing.assert_array_equal(vals, vv)  # same device arithmetic: bit-identical
    assert sum(i["row_nnz"] for i in infos) == len(ci)
    # the quantile scale forces the plan's support pass, so the per-row sums were
    # gathered across ranks; UOT is always a (normalised) grid plan
    assert infos[0]["factorized"] == (0 if plan == "uot" else infos[0]["factorized"])


@pytest.mark.parametrize("world", [1, 2, 3, 4])
def test_sharded_ot_matches_single_gpu(ctx, world):
    x, y, a, q = _c4_like()
    kern = spk.Coords(x, y, scale=q, eps=0.05)
    n = len(a)
    cfg = spk.SolverConfig(0.05, math.inf, -1.0, 40)
    s = 8 * n * math.log(n)
    opts = spk.SparSinkOptions(values="f32")
    ref = ctx.spar_sink(kern, a, a, cfg, s, 5, opts)
    outs = S.run_emulated(world, lambda comm, shard: S.spar_sink_sharded(comm, shard, kern, a, a, cfg, s, 5, opts))
    for r in outs:
        np.testing.assert_allclose(r.u, ref.u, rtol=1e-9)
        np.testing.assert_allclose(r.v, ref.v, rtol=1e-9)
        assert r.report["iterations"] == ref.report["iterations"] == 40
        assert r.report["sketch_nnz"] == ref.report["sketch_nnz"]
        assert r.report["objective"] == pytest.approx(ref.report["objective"], rel=1e-9)
        assert r.report["residual_row"] == pytest.approx(ref.report["residual_row"], rel=1e-6, abs=1e-15)
        assert r.report["kernel_mean"] == pytest.approx(ref.report["kernel_mean"], rel=1e-12)
    for r in outs[1:]:
        np.testing.assert_array_equal(r.u, outs[0].u)


@pytest.mark.parametrize("world,max_w", [(1, 256), (2, 256), (3, 64), (4, 4096)])
def test_sharded_blocked_matches_single_gpu(ctx, world, max_w):
    """The slab x block half-steps (CTA-pair clusters, TMA-staged tiles of the
    gathered vector, tails skipped) on every rank, forced at a small n, against
    the single-GPU solve."""
    from paper_2306_06581_b200 import _lib as L

    x, y, a, q = _c4_like()
    kern = spk.Coords(x, y, scale=q, eps=0.05)
    n = len(a)
    cfg = spk.SolverConfig(0.05, math.inf, -1.0, 40)
    s = 8 * n * math.log(n)
    opts = spk.SparSinkOptions(values="f32")
    ref = ctx.spar_sink(kern, a, a, cfg, s, 5, opts)
    o = {L.OPT_BLOCKED_LOOP: 1, L.OPT_BLOCKED_MAX_W: max_w}
    outs = S.run_emulated(world, lambda comm, shard: S.spar_sink_sharded(comm, shard, kern, a, a, cfg, s, 5, opts),
                          options=o)
    for r in outs:
        np.testing.assert_allclose(r.u, ref.u, rtol=1e-9)
        np.testing.assert_allclose(r.v, ref.v, rtol=1e-9)
        assert r.report["iterations"] == ref.report["iterations"] == 40
        assert r.report["objective"] == pytest.approx(ref.report["objective"], rel=1e-9)
    # UOT with a convergence stop
    b = a * 1.5
    cfg = spk.SolverConfig(0.05, 1.0, 1e-9, 500)
    ref = ctx.spar_sink(kern, a, b, cfg, s, 9, uot=True)
    outs = S.run_emulated(world, lambda comm, shard: S.spar_sink_sharded(comm, shard, kern, a, b, cfg, s, 9, uot=True,
                                                                           check_every=8), options=o)
    for r in outs:
        assert r.report["converged"] == ref.report["converged"] == 1
        assert abs(r.report["iterations"] - ref.report["iterations"]) <= 3  # delta stop: rounding noise of the residual
        np.testing.assert_allclose(r.u, ref.u, rtol=1e-6)
        np.testing.assert_allclose(r.v, ref.v, rtol=1e-6)


@pytest.mark.parametrize("stabilize", [False, True])
def test_sharded_uot_converges_like_single_gpu(ctx, stabilize):
    x, y, a, q = _c4_like(2000, 13)
    b = a * 1.5
    kern = spk.Coords(x, y, scale=q, eps=0.05)
    n = len(a)
    cfg = spk.SolverConfig(0.05, 1.0, 1e-9, 500, stabilize)
    s = 8 * n * math.log(n)
    ref = ctx.spar_sink(kern, a, b, cfg, s, 9, uot=True)
    outs = S.run_emulated(3, lambda comm, shard: S.spar_sink_sharded(comm, shard, kern, a, b, cfg, s, 9, uot=True,
                                                                       check_every=8))
    for r in outs:
        assert r.report["converged"] == ref.report["converged"] == 1
        # the delta stop: near convergence the residual sum_i |du_i| (~1e-9)
        # carries rounding noise of ~1e-16 u per atom, so another summation
        # order (3 ranks vs the one-cluster loop) may cross delta a few
        # iterations apart; the scalings below pin the result
        assert abs(r.report["iterations"] - ref.report["iterations"]) <= 3
        np.testing.assert_allclose(r.u, ref.u, rtol=1e-6)
        np.testing.assert_allclose(r.v, ref.v, rtol=1e-6)
        assert r.report["objective"] == pytest.approx(ref.report["objective"], rel=1e-7)


def test_sharded_strict_raises_on_every_rank(ctx):
    # a budget so small that rows go empty: strict mode -> DegenerateSketchError from every rank
    x, y, a, q = _c4_like(600, 17)
    kern = spk.Coords(x, y, scale=q, eps=0.05)
    cfg = spk.SolverConfig(0.05, math.inf, -1.0, 10)
    with pytest.raises(spk.api.ERRORS["DegenerateSketchError"]):
        S.run_emulated(2, lambda comm, shard: S.spar_sink_sharded(comm, shard, kern, a, a, cfg, 300.0, 3,
                                                                  spk.SparSinkOptions(strict=True)))
