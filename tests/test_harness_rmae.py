"""the RMAE experiment on the GPU path against the
compiled reference's rmae_experiment on the same scenario (inputs from the
reference's own generate_scenario): the same replication seeds give the same
sketches, so every per-replication relative error matches."""
import math

import numpy as np
import pytest

import paper_2306_06581_b200 as spk
from paper_2306_06581_b200 import harness


def test_s_schedule_matches_reference_formula():
    b, clamped = harness.s_schedule(100, [1.0, 1e9])
    assert b[0] == pytest.approx(1e-3 * 100 * math.log(100) ** 4, rel=1e-15)
    assert clamped and b[1] == 100.0 * 100.0 * (1.0 - 1e-9)


@pytest.mark.gpu
@pytest.mark.parametrize("method", ["sparsink", "randsink"])
def test_rmae_matches_reference_balanced(reference, ctx, method):
    spec = {"scenario": "C1", "n": 80, "d": 3, "seed": 5}
    x, a, b, _ = reference.scenario(spec)
    budgets = [400.0, 1200.0]
    exact, errs, retried = reference.rmae(spec, method, budgets, 4, 0.5)
    rep = harness.rmae_experiment(ctx, x, a, b, spk.SolverConfig(0.5), budgets, 4, 5, method)
    assert rep["exact_objective"] == pytest.approx(exact, rel=1e-9)
    for k, row in enumerate(rep["rows"]):
        np.testing.assert_allclose(row["errors"], errs[k], rtol=1e-6, atol=1e-10)
        assert row["retried"] == retried[k]


@pytest.mark.gpu
def test_rmae_matches_reference_unbalanced_wfr(reference, ctx):
    spec = {"scenario": "C3", "n": 70, "d": 2, "seed": 9, "masses": (1.0, 1.5), "sparsity_target": 0.5}
    x, a, b, eta = reference.scenario(spec)
    budgets = [700.0]
    exact, errs, retried = reference.rmae(spec, "sparsink", budgets, 3, 0.2, lam=1.0)
    rep = harness.rmae_experiment(ctx, x, a, b, spk.SolverConfig(0.2, 1.0), budgets, 3, 9, eta=eta)
    assert rep["exact_objective"] == pytest.approx(exact, rel=1e-9)
    np.testing.assert_allclose(rep["rows"][0]["errors"], errs[0], rtol=1e-6, atol=1e-10)


@pytest.mark.parametrize("spec", [
    {"scenario": "C1", "n": 300, "d": 5, "seed": 3},
    {"scenario": "C2", "n": 257, "d": 4, "seed": 11},
    {"scenario": "C3", "n": 200, "d": 2, "seed": 9, "masses": (1.0, 1.5)},
    {"scenario": "C1", "n": 150, "d": 3, "seed": 2, "scale_param": 0.2, "scale_is_sd": True},
    {"scenario": "C3", "n": 90, "d": 2, "seed": 4, "masses": (2.0, 0.5), "sparsity_target": 0.3},
], ids=lambda s: f"{s['scenario']}-n{s['n']}")
def test_generate_scenario_bit_equal_to_reference(reference, spec):
    """generate_scenario (harness.cpp:85-126) and eta_for_sparsity
    (geometry.cpp:104-135) restated on the host: bit-equal to the reference."""
    x, a, b, eta = reference.scenario(spec)
    gx, ga, gb = harness.generate_scenario(spec["scenario"], spec["n"], spec["d"], spec["seed"], spec.get("masses"),
                                           spec.get("scale_param", 0.05), spec.get("scale_is_sd", False))
    assert np.array_equal(gx, x) and np.array_equal(ga, a) and np.array_equal(gb, b)
    if spec.get("sparsity_target") is not None:
        assert harness.eta_for_sparsity(gx, spec["sparsity_target"]) == eta


def test_loglog_slope_known_answers():
    xs = [1000, 2000, 4000, 8000]
    assert harness.loglog_slope(xs, [3e-9 * x ** 2 for x in xs]) == pytest.approx(2.0, rel=1e-12)
    assert harness.loglog_slope(xs, [5.0 * x for x in xs]) == pytest.approx(1.0, rel=1e-12)
    with pytest.raises(spk.ERRORS["LengthMismatch"]):
        harness.loglog_slope([1], [1.0])


@pytest.mark.gpu
def test_rmae_scenario_driver_matches_reference(reference, ctx):
    """rmae_experiment from a scenario spec, end to end on the GPU path
    (scenario + eta generated here), against the reference's rmae_experiment."""
    spec = {"scenario": "C3", "n": 70, "d": 2, "seed": 9, "masses": (1.0, 1.5), "sparsity_target": 0.5}
    exact, errs, retried = reference.rmae(spec, "sparsink", [700.0], 3, 0.2, lam=1.0)
    rep = harness.rmae_scenario(ctx, spec, "sparsink", [700.0], 3, spk.SolverConfig(0.2, 1.0))
    assert rep["exact_objective"] == pytest.approx(exact, rel=1e-9)
    np.testing.assert_allclose(rep["rows"][0]["errors"], errs[0], rtol=1e-6, atol=1e-10)


@pytest.mark.gpu
def test_timing_sweep_per_iteration_slopes(ctx):
    """Acceptance #9 (tests/acceptance.cpp:359-371) on the GPU: the dense
    per-iteration time grows like n^2, the Spar-Sink one sub-quadratically.
    The reference's sizes (1e3..1.6e4) sit on the GPU's latency floor, so the
    sweep starts where the dense loop is throughput-bound."""
    sizes = [16000, 32000, 64000, 128000]
    rows = harness.timing_sweep(ctx, sizes, 5, spk.SolverConfig(0.1), 8.0, 901, 3)
    dense = [r["per_iter_s"] for r in rows if r["method"] == "sinkhorn"]
    sparse = [r["per_iter_s"] for r in rows if r["method"] == "spar-sink"]
    ds, ss = harness.loglog_slope(sizes, dense), harness.loglog_slope(sizes, sparse)
    print(f"timing sweep: dense slope {ds:.3f} ({dense}), sparse slope {ss:.3f} ({sparse})")
    assert ds > 1.7 and ss < 1.5
