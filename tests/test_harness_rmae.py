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
