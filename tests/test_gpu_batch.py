"""GPU: spk_sketch_solve_batch -- many log-domain sketches solved together,
one CTA per sketch with both log scalings in shared memory (config 3's 496
frame pairs, pairwise_wfr in proj/src/harness.cpp:349-406) -- against the
one-sketch-at-a-time solve of the same sketches (the row sums run in another
lane order: iteration counts equal at a fixed count, marginals and objectives
to 1e-12)."""
import math

import numpy as np
import pytest

import paper_2306_06581_b200 as spk
from paper_2306_06581_b200 import api
from paper_2306_06581_b200 import workloads as W

pytestmark = pytest.mark.gpu


def _pairs_sketches(ctx, side, npairs, cfg, seed=3):
    coords, masses = W.c3_frames(seed, frames=8, side=side)
    n = coords.shape[0]
    s = 10 * n * math.log(n)
    kern = spk.Coords(coords, coords, "wfr", 0.1, scale=1.0, eps=cfg.epsilon)
    pairs = api.frame_pairs(8)[:npairs]
    sks = [ctx.sketch(kern, masses[i], masses[j], "uot", cfg.lambda_, cfg.epsilon, s, api.mix_seed(seed, k))
           for k, (i, j) in enumerate(pairs)]
    return kern, sks


@pytest.mark.parametrize("side,npairs", [(40, 7), (112, 3)])
def test_batch_matches_one_at_a_time(ctx, side, npairs):
    cfg = spk.SolverConfig(0.01, 1.0, -1.0, 300 if side == 112 else 600, stabilize=True)
    kern, sks = _pairs_sketches(ctx, side, npairs, cfg)
    reps = api.solve_batch(ctx, sks, cfg, uot=True)
    got = [sk.readout(kern, uot=True, lambda_=cfg.lambda_, epsilon=cfg.epsilon) for sk in sks]
    for sk, rep, (rm, cm, obj, _) in zip(sks, reps, got):
        one = sk.solve(cfg, uot=True)
        rm1, cm1, obj1, _ = sk.readout(kern, uot=True, lambda_=cfg.lambda_, epsilon=cfg.epsilon)
        assert rep["iterations"] == one.report["iterations"]
        assert rep["converged"] == one.report["converged"]
        assert rep["masked_rows"] == one.report["masked_rows"] and rep["masked_cols"] == one.report["masked_cols"]
        np.testing.assert_allclose(rm, rm1, rtol=1e-11, atol=1e-300)
        np.testing.assert_allclose(cm, cm1, rtol=1e-11, atol=1e-300)
        assert obj == pytest.approx(obj1, rel=1e-12)
        assert rep["residual_row"] == pytest.approx(one.report["residual_row"], rel=1e-9, abs=1e-15)
    for sk in sks:
        sk.free()


def test_batch_pairs_driver_matches_unbatched(ctx):
    coords, masses = W.c3_frames(5, frames=5, side=36)
    n = coords.shape[0]
    cfg = spk.SolverConfig(0.01, 1.0, 1e-6, 400, stabilize=True)
    s = 10 * n * math.log(n)
    a = api.spar_sink_pairs(ctx, coords, masses, cfg, s, 5, 0.1, batched=True, chunk=4)
    b = api.spar_sink_pairs(ctx, coords, masses, cfg, s, 5, 0.1, batched=False)
    assert [k for k, _, _ in a] == [k for k, _, _ in b] == list(range(10))
    for (_, pa, ra), (_, pb, rb) in zip(a, b):
        assert pa == pb
        assert abs(ra["iterations"] - rb["iterations"]) <= 1  # residual within rounding of delta
        assert ra["sketch_nnz"] == rb["sketch_nnz"]
        assert ra["objective"] == pytest.approx(rb["objective"], rel=1e-12)


def test_batch_error_policy_and_linear_fallback(ctx, oracle):
    # a sketch with an empty row: Error policy raises ZeroDenominator naming the item
    n = 50
    x = oracle.rng_doubles(41, 0, 2 * n).reshape(n, 2)
    Cm, _ = oracle.pairwise_cost(x, x)
    K, r = oracle.kernel_from_cost(Cm, 0.05)
    K[3, :] = 0.0
    a = np.full(n, 1.0 / n)
    p = oracle.plan("ot", a, a, K, r)
    so = oracle.poisson_sparsify(K, p, 8 * n * math.log(n), 2)
    oracle.free_plan(p)
    good = ctx.sketch_from_csr(*oracle.poisson_sparsify(K + (K == 0) * 1e-3, oracle.plan("ot", a, a, K + (K == 0) * 1e-3, 1.0),
                                                        8 * n * math.log(n), 3))
    bad = ctx.sketch_from_csr(*so)
    cfg = spk.SolverConfig(0.05, math.inf, 1e-9, 200, stabilize=True)
    for sk in (good, bad):
        sk.solve(cfg, a=a, b=a)  # gives the sketches their marginals
    with pytest.raises(spk.ERRORS["ZeroDenominator"], match="batch item 1"):
        api.solve_batch(ctx, [good, bad], cfg, policy="error")
    # Mask policy: the batch runs; the linear domain falls back to one solve at a time
    reps = api.solve_batch(ctx, [good, bad], cfg)
    assert reps[1]["masked_rows"] >= 1
    lin = spk.SolverConfig(0.05, math.inf, 1e-9, 200)
    reps = api.solve_batch(ctx, [good, bad], lin)
    one = good.solve(lin)
    assert reps[0]["iterations"] == one.report["iterations"]
    # per-item outcomes (pairwise_wfr, harness.cpp:395-401): the failing item is
    # recorded, the others complete and keep their scalings
    for c in (cfg, lin):
        reps = api.solve_batch(ctx, [bad, good, bad], c, policy="error", per_item=True)
        assert [r["error"] for r in reps] == ["ZeroDenominator", None, "ZeroDenominator"]
        ref = good.solve(c)
        u, v, _, _ = api.solve_batch(ctx, [bad, good], c, policy="error", per_item=True) and good.scalings()
        np.testing.assert_allclose(u, ref.u, rtol=1e-12)
        np.testing.assert_allclose(v, ref.v, rtol=1e-12)
        with pytest.raises(spk.ERRORS["LengthMismatch"]):
            bad.scalings()  # no valid solve on the failed item


def test_sketch_batch_equals_one_at_a_time(ctx):
    """spk_sketch_build_batch (the kernel prepared once) draws the same sketches
    bit for bit as spk_sketch_build per pair."""
    coords, masses = W.c3_frames(7, frames=5, side=48)
    n = coords.shape[0]
    s = 10 * n * math.log(n)
    kern = spk.Coords(coords, coords, "wfr", 0.1, scale=1.0, eps=0.01)
    pairs = api.frame_pairs(5)
    seeds = [api.mix_seed(7, k) for k in range(len(pairs))]
    opts = spk.SparSinkOptions(values="f32")
    batch = ctx.sketch_batch(kern, masses[[i for i, _ in pairs]], masses[[j for _, j in pairs]], "uot", 1.0, 0.01, s,
                             seeds, opts)
    for (i, j), sd, sb in zip(pairs, seeds, batch):
        one = ctx.sketch(kern, masses[i], masses[j], "uot", 1.0, 0.01, s, sd, opts)
        for x, y in zip(sb.csr(), one.csr()):
            assert np.array_equal(x, y)
        one.free()
        sb.free()
