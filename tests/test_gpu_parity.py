"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle and the
reference-generated golden fixtures.

Bars (north star): sampled index sets bit-exact; sketch values within a few
ULP (CUDA exp/pow vs glibc); fp64 scalings/objective within 1e-6 relative
(measured far tighter and asserted tighter where the path is exact:
deterministic-mode OT scalings on a given sketch are bit-identical).
"""
import math
from pathlib import Path

import numpy as np
import pytest

import paper_2306_06581_b200 as spk

pytestmark = pytest.mark.gpu
GOLD = Path(__file__).resolve().parent / "golden"
# Sketch values K/p*: with an exact cost (squared Euclidean: IEEE ops in the
# reference order) only exp and the division round differently (a few ULP).
# WFR costs go through cos/log, whose ULP error is amplified by C/eps inside
# exp (up to ~745 at the underflow edge): ~C/eps * 4 ULP.
VALUE_RTOL = 1e-14
WFR_VALUE_RTOL = 5e-13
SUBNORMAL_ATOL = 1e-320


def value_rtol(kind: str) -> float:
    return WFR_VALUE_RTOL if kind == "wfr" else VALUE_RTOL


def _kernel_for(g, form):
    kind = str(g["kind"])
    if form == "coords":
        return spk.Coords(g["x"], g["y"], kind, float(g["eta"]), scale=1.0, eps=float(g["eps"]))
    return None


# ---- sampler ----------------------------------------------------------------------


@pytest.mark.parametrize("form", ["coords", "dense"])
@pytest.mark.parametrize("path", sorted(GOLD.glob("sketch_*.npz")), ids=lambda p: p.stem)
def test_sketch_matches_reference_fixture(ctx, oracle, path, form):
    g = np.load(path)
    plan = str(g["plan"])
    if form == "coords":
        kern = _kernel_for(g, "coords")
    else:
        Cm, _ = oracle.pairwise_cost(g["x"], g["y"], str(g["kind"]), float(g["eta"]))
        K, r = oracle.kernel_from_cost(Cm, float(g["eps"]))
        kern = spk.Dense(K, r)
    sk = ctx.sketch(kern, g["a"], g["b"], plan, float(g["lam"]), float(g["eps"]), float(g["s"]), int(g["seed"]),
                    spk.SparSinkOptions(theta=float(g["theta"])))
    rp, ci, vv = sk.csr()
    assert np.array_equal(rp, g["row_ptr"]), "row counts differ"
    assert np.array_equal(ci, g["col_idx"]), "index sets differ"
    rtol = value_rtol(str(g["kind"])) if form == "coords" else VALUE_RTOL
    # subnormal values carry few significant bits: allow a few subnormal ULPs
    np.testing.assert_allclose(vv, g["values"], rtol=rtol, atol=SUBNORMAL_ATOL)
    assert sk.factorized_plan == bool(g["factorized"])
    # CSC mirror = exact transpose, rows ascending inside each column
    cp, ri, vt = sk.csc()
    rows = np.repeat(np.arange(sk.n), np.diff(rp))
    order = np.lexsort((rows, ci))
    assert np.array_equal(ri, rows[order]) and np.array_equal(vt, vv[order])
    assert np.array_equal(cp, np.concatenate([[0], np.cumsum(np.bincount(ci, minlength=sk.n))]))


@pytest.mark.parametrize("path", sorted(GOLD.glob("sketch_*.npz")), ids=lambda p: p.stem)
def test_plan_probabilities_match_reference(ctx, path):
    g = np.load(path)
    n = len(g["a"])
    qi, qj = np.divmod(np.arange(n * n), n)
    probs, fac = ctx.plan_probs(_kernel_for(g, "coords"), g["a"], g["b"], str(g["plan"]), float(g["lam"]),
                                float(g["eps"]), float(g["theta"]), qi, qj)
    want = g["probs"].ravel()
    # UOT grids carry pow(K, g_k): K's cos/log/exp ULPs times g_k (< 1)
    np.testing.assert_allclose(probs, want, rtol=1e-13 if str(g["kind"]) != "wfr" else 5e-13, atol=0)
    assert fac == bool(g["factorized"])


def test_cost_kernel_entries(ctx, oracle):
    n = 50
    x = oracle.rng_doubles(5, 0, 3 * n).reshape(n, 3)
    y = oracle.rng_doubles(6, 0, 3 * n).reshape(n, 3)
    qi, qj = np.divmod(np.arange(n * n), n)
    for kind, eta in (("sqeuclid", 0.0), ("euclid", 0.0), ("wfr", 0.2)):
        Cm, c0 = oracle.pairwise_cost(x, y, kind, eta)
        K, _ = oracle.kernel_from_cost(Cm / c0, 0.05)
        cost, kern, c0g = ctx.cost_kernel(spk.Coords(x, y, kind, eta, scale=None, eps=0.05), qi, qj)
        assert c0g == c0
        if kind == "sqeuclid":
            assert np.array_equal(cost, (Cm / c0).ravel())  # exact IEEE ops in the reference order
        np.testing.assert_allclose(cost, (Cm / c0).ravel(), rtol=1e-14)
        np.testing.assert_allclose(kern, K.ravel(), rtol=1e-13)


def test_sampler_unbiased_monte_carlo(ctx, oracle):
    # test_sparsify.cpp:159-184 on the GPU sampler: E[K~_ij] = K_ij within 3 se
    n, s, reps = 8, 20.0, 4000
    pts = oracle.rng_doubles(17, 0, 2 * n).reshape(n, 2)
    Cm, _ = oracle.pairwise_cost(pts, pts)
    K, r = oracle.kernel_from_cost(Cm, 0.5)
    a = np.full(n, 1.0 / n)
    mean = np.zeros((n, n))
    for rep in range(reps):
        sk = ctx.sketch(spk.Dense(K, r), a, a, "uniform", math.inf, 0.5, s, 1000 + rep)
        rp, ci, vv = sk.csr()
        rows = np.repeat(np.arange(n), np.diff(rp))
        np.add.at(mean, (rows, ci.astype(np.int64)), vv)
        sk.free()
    mean /= reps
    pstar = np.minimum(1.0, s / (n * n))
    se = K * np.sqrt((1 - pstar) / pstar / reps)
    assert np.sum(np.abs(mean - K) <= 3 * se + 1e-15) >= 61


def test_tiled_sampler_inclusion_frequencies(ctx, oracle):
    """inclusion frequencies of the coordinate (tiled) sampler are
    consistent with p*_ij = min(1, s p_ij) for the factorized OT plan
    p_ij = ra_i cb_j (ra = sqrt(a) / sum sqrt(a), sparsify.cpp:71-91): 3000
    seeds, every entry's frequency within 4 standard errors (a 4-sigma miss
    has probability 6e-5 per entry), and the mean sketch size within 4 se of
    sum p*."""
    n, s, reps = 16, 60.0, 3000
    x = oracle.rng_doubles(23, 0, 2 * n).reshape(n, 2)
    y = oracle.rng_doubles(23, 1, 2 * n).reshape(n, 2)
    w = 0.1 + oracle.rng_doubles(23, 2, 2 * n)
    a, b = w[:n] / w[:n].sum(), w[n:] / w[n:].sum()
    kern = spk.Coords(x, y, "sqeuclid", scale=1.0, eps=1.0)  # K > 0 everywhere: factorized plan
    counts = np.zeros((n, n))
    sizes = np.zeros(reps)
    for rep in range(reps):
        sk = ctx.sketch(kern, a, b, "ot", math.inf, 1.0, s, 5000 + rep)
        assert sk.factorized_plan
        rp, ci, _ = sk.csr()
        rows = np.repeat(np.arange(n), np.diff(rp))
        np.add.at(counts, (rows, ci.astype(np.int64)), 1.0)
        sizes[rep] = len(ci)
        sk.free()
    ra = np.sqrt(a) / np.sqrt(a).sum()
    cb = np.sqrt(b) / np.sqrt(b).sum()
    pstar = np.minimum(1.0, s * np.outer(ra, cb))
    freq = counts / reps
    se = np.sqrt(pstar * (1 - pstar) / reps)
    assert np.all(np.abs(freq - pstar) <= 4 * se + 1e-12)
    tot_se = np.sqrt(np.sum(pstar * (1 - pstar)) / reps)
    assert abs(sizes.mean() - pstar.sum()) <= 4 * tot_se


def test_sampler_errors(ctx, oracle):
    n = 10
    x = oracle.rng_doubles(1, 0, 2 * n).reshape(n, 2)
    a = np.full(n, 0.1)
    kern = spk.Coords(x, x, "sqeuclid", scale=1.0, eps=0.5)
    with pytest.raises(spk.ERRORS["BudgetTooLarge"]):
        ctx.sketch(kern, a, a, "ot", math.inf, 0.5, 0.0, 1)
    with pytest.raises(spk.ERRORS["BudgetTooLarge"]):
        ctx.sketch(kern, a, a, "ot", math.inf, 0.5, float(n * n), 1)
    with pytest.raises(spk.ERRORS["ThetaOutOfRange"]):
        ctx.sketch(kern, a, a, "ot", math.inf, 0.5, 30.0, 1, spk.SparSinkOptions(theta=1.0))
    with pytest.raises(spk.SparsinkError) as e:
        ctx.sketch(kern, a, a, "uot", -1.0, 0.5, 30.0, 1)
    assert e.value.category == 4
    with pytest.raises(spk.ERRORS["AllZeroKernel"]):
        ctx.sketch(spk.Dense(np.zeros((n, n)), 0.0), a, a, "ot", math.inf, 0.5, 30.0, 1)
    with pytest.raises(spk.ERRORS["NonPositiveEta"]):
        ctx.sketch(spk.Coords(x, x, "wfr", 0.0, scale=1.0, eps=0.5), a, a, "ot", math.inf, 0.5, 30.0, 1)


# ---- loop -------------------------------------------------------------------------------


@pytest.mark.parametrize("path", sorted(GOLD.glob("sketch_*.npz")), ids=lambda p: p.stem)
def test_loop_deterministic_bit_identical(dctx, oracle, path):
    """Parity mode on the reference's own sketch: OT scalings and iteration
    counts bit-identical to sinkhorn_ot<SparseKernel>; UOT within pow ULPs."""
    g = np.load(path)
    csr = (g["row_ptr"], g["col_idx"], g["values"])
    uot = str(g["plan"]) == "uot"
    lam = float(g["lam"]) if uot else math.inf
    eps = float(g["eps"])
    ou, ov, _, _, ores = oracle.sinkhorn(g["a"], g["b"], eps, lam, 1e-10, 3000, policy="mask", uot=uot, csr=csr)
    sk = dctx.sketch_from_csr(*csr)
    res = sk.solve(spk.SolverConfig(eps, lam, 1e-10, 3000), uot=uot, a=g["a"], b=g["b"])
    rep = res.report
    assert rep["iterations"] == ores["iterations"]
    assert (rep["converged"], rep["diverged"]) == (ores["converged"], ores["diverged"])
    assert (rep["masked_rows"], rep["masked_cols"]) == (ores["masked_rows"], ores["masked_cols"])
    if not uot:
        assert np.array_equal(res.u, ou) and np.array_equal(res.v, ov)
        assert rep["residual_row"] == ores["residual_row"] and rep["residual_col"] == ores["residual_col"]
    else:
        np.testing.assert_allclose(res.u, ou, rtol=1e-12)
        np.testing.assert_allclose(res.v, ov, rtol=1e-12)
    assert rep["kernel_mean"] == ores["kernel_mean"]


@pytest.mark.parametrize("path", sorted(GOLD.glob("sketch_*.npz")), ids=lambda p: p.stem)
def test_loop_fast_mode_tolerance(ctx, oracle, path):
    g = np.load(path)
    csr = (g["row_ptr"], g["col_idx"], g["values"])
    uot = str(g["plan"]) == "uot"
    lam = float(g["lam"]) if uot else math.inf
    eps = float(g["eps"])
    cfg = spk.SolverConfig(eps, lam, -1.0, 150)  # fixed iteration count
    ou, ov, _, _, _ = oracle.sinkhorn(g["a"], g["b"], eps, lam, -1.0, 150, policy="mask", uot=uot, csr=csr)
    res = ctx.sketch_from_csr(*csr).solve(cfg, uot=uot, a=g["a"], b=g["b"])
    np.testing.assert_allclose(res.u, ou, rtol=1e-10)
    np.testing.assert_allclose(res.v, ov, rtol=1e-10)


@pytest.mark.parametrize("stab", [False, True])
@pytest.mark.parametrize("path", sorted(GOLD.glob("sketch_*.npz"))[:4], ids=lambda p: p.stem)
def test_log_domain_loop(dctx, ctx, oracle, path, stab):
    g = np.load(path)
    csr = (g["row_ptr"], g["col_idx"], g["values"])
    uot = str(g["plan"]) == "uot"
    lam = float(g["lam"]) if uot else math.inf
    eps = float(g["eps"])
    ou, ov, olu, olv, ores = oracle.sinkhorn(g["a"], g["b"], eps, lam, -1.0, 60, stabilize=True, policy="mask",
                                             uot=uot, csr=csr)
    c = dctx if stab else ctx
    res = c.sketch_from_csr(*csr).solve(spk.SolverConfig(eps, lam, -1.0, 60, True), uot=uot, a=g["a"], b=g["b"])
    assert res.report["log_domain"] == 1 and res.report["iterations"] == ores["iterations"]
    fin = np.isfinite(olu)
    assert np.array_equal(fin, np.isfinite(res.log_u))
    np.testing.assert_allclose(res.log_u[fin], olu[fin], rtol=1e-11, atol=1e-11)
    np.testing.assert_allclose(res.u, ou, rtol=1e-10)
    np.testing.assert_allclose(res.v, ov, rtol=1e-10)


@pytest.mark.parametrize("path", sorted(GOLD.glob("loop_*.npz")), ids=lambda p: p.stem)
def test_loop_failure_semantics(dctx, path):
    """Dynamic masking / divergence restore / ZeroDenominator (solvers.hpp:292-358)."""
    g = np.load(path)
    csr = (g["row_ptr"], g["col_idx"], g["values"])
    stab = bool(g["stabilize"]) if "stabilize" in g else False
    cfg = spk.SolverConfig(float(g["eps"]), float(g["lam"]), float(g["delta"]), int(g["max_iter"]), stab)
    sk = dctx.sketch_from_csr(*csr)
    if int(g["err"]):
        with pytest.raises(spk.SparsinkError) as e:
            sk.solve(cfg, uot=bool(g["uot"]), a=g["a"], b=g["b"], policy=str(g["policy"]))
        assert e.value.kind == int(g["err"])
        return
    res = sk.solve(cfg, uot=bool(g["uot"]), a=g["a"], b=g["b"], policy=str(g["policy"]))
    for k in ("iterations", "converged", "diverged", "masked_rows", "masked_cols"):
        assert res.report[k] == int(g[f"rep_{k}"]), k
    if bool(g["uot"]):
        np.testing.assert_allclose(res.u, g["u"], rtol=1e-12)
        np.testing.assert_allclose(res.v, g["v"], rtol=1e-12)
    else:
        assert np.array_equal(res.u, g["u"]) and np.array_equal(res.v, g["v"])


# ---- end to end ------------------------------------------------------------------------------


@pytest.mark.parametrize("path", sorted(GOLD.glob("solve_*.npz")), ids=lambda p: p.stem)
def test_spar_sink_end_to_end(dctx, ctx, path):
    g = np.load(path)
    probs = str(g["probs"])
    opts = spk.SparSinkOptions(probs=probs)
    cfg = spk.SolverConfig(float(g["eps"]), float(g["lam"]), float(g["delta"]), int(g["max_iter"]),
                           bool(g["stabilize"]))
    kern = spk.Coords(g["x"], g["y"], "sqeuclid", scale=1.0, eps=float(g["eps"]))
    for c in (dctx, ctx):
        r = c.spar_sink(kern, g["a"], g["b"], cfg, float(g["s"]), int(g["seed"]), opts, uot=bool(g["uot"]))
        rep = r.report
        assert rep["sketch_nnz"] == int(g["rep_sketch_nnz"])
        assert rep["iterations"] == int(g["rep_iterations"])
        for k in ("converged", "diverged", "masked_rows", "masked_cols"):
            assert rep[k] == int(g[f"rep_{k}"]), k
        assert rep["objective"] == pytest.approx(float(g["rep_objective"]), rel=1e-10)
        np.testing.assert_allclose(r.u, g["u"], rtol=1e-9)
        np.testing.assert_allclose(r.v, g["v"], rtol=1e-9)
        assert rep["kernel_mean"] == pytest.approx(float(g["rep_kernel_mean"]), rel=1e-13)


def test_strict_mode_raises_on_orphans(ctx, oracle):
    # test_solvers.cpp:189-204: ~3 entries per row -> empty rows are certain
    n = 80
    p = oracle.rng_doubles(59, 0, 2 * n).reshape(n, 2)
    w = 0.2 + oracle.rng_doubles(59, 0, 4 * n)[2 * n:]
    a, b = w[:n] / w[:n].sum(), w[n:] / w[n:].sum()
    kern = spk.Coords(p, p, "sqeuclid", scale=1.0, eps=0.5)
    cfg = spk.SolverConfig(0.5, math.inf, 1e-8, 200000)
    r = ctx.spar_sink(kern, a, b, cfg, 240.0, 7)
    assert r.report["masked_rows"] > 0 and math.isfinite(r.report["objective"])
    with pytest.raises(spk.ERRORS["DegenerateSketchError"]) as e:
        ctx.spar_sink(kern, a, b, cfg, 240.0, 7, spk.SparSinkOptions(strict=True))
    assert e.value.category == 3 and "orphaned atom" in str(e.value)


def test_solver_argument_errors(ctx, oracle):
    n = 20
    p = oracle.rng_doubles(3, 0, 2 * n).reshape(n, 2)
    a = np.full(n, 1.0 / n)
    kern = spk.Coords(p, p, "sqeuclid", scale=1.0, eps=0.5)
    with pytest.raises(spk.ERRORS["NotNormalized"]):
        ctx.spar_sink(kern, a * 1.5, a, spk.SolverConfig(0.5), 100.0, 1)
    with pytest.raises(spk.SparsinkError) as e:
        ctx.sinkhorn(kern, a, a, spk.SolverConfig(0.5), uot=True)  # lambda = inf
    assert e.value.category == 4 and type(e.value) is spk.SparsinkError


# ---- dense Sinkhorn (sinkhorn_ot/uot<KernelMatrix>) -------------------------------------------


def _dense_case(oracle, sup, eps):
    Cm, _ = oracle.pairwise_cost(sup, sup)
    K, r = oracle.kernel_from_cost(Cm, eps)
    return Cm, K, r


@pytest.mark.parametrize("form", ["dense", "coords"])
def test_dense_known_answers(dctx, oracle, form):
    sup = np.array([0.0, 1.0])
    Cm, K, r = _dense_case(oracle, sup, 1.0)
    kern = spk.Dense(K, r, Cm) if form == "dense" else spk.Coords(sup, sup, "sqeuclid", scale=1.0, eps=1.0)
    a = np.array([0.5, 0.5])
    res = dctx.sinkhorn(kern, a, a, spk.SolverConfig(1.0, math.inf, 1e-13, 200000))
    assert res.report["converged"]
    assert res.u[0] * K[0, 0] * res.v[0] == pytest.approx(0.36552928931500245, rel=1e-10)
    assert res.report["objective"] == pytest.approx(-2.006408868078168, rel=1e-10)
    # two-atom UOT (test_solvers.cpp:102-115)
    a2, b2 = np.array([0.7, 0.9]), np.array([0.4, 0.8])
    Cm, K, r = _dense_case(oracle, sup, 0.5)
    kern = spk.Dense(K, r, Cm) if form == "dense" else spk.Coords(sup, sup, "sqeuclid", scale=1.0, eps=0.5)
    res = dctx.sinkhorn(kern, a2, b2, spk.SolverConfig(0.5, 2.0, 1e-13, 200000), uot=True)
    assert res.u[0] * K[0, 0] * res.v[0] == pytest.approx(0.4880086699186626, rel=1e-9)
    assert res.report["objective"] == pytest.approx(-0.9506480667355813, rel=1e-9)
    # one atom (test_solvers.cpp:88-100)
    one = np.array([0.0])
    Cm, K, r = _dense_case(oracle, one, 1.0)
    kern = spk.Dense(K, r, Cm) if form == "dense" else spk.Coords(one, one, "sqeuclid", scale=1.0, eps=1.0)
    res = dctx.sinkhorn(kern, np.array([2.0]), np.array([8.0]), spk.SolverConfig(1.0, 1.0, 1e-13, 200000), uot=True)
    assert abs(res.u[0] * K[0, 0] * res.v[0] - 16 ** (1 / 3)) < 1e-8
    assert res.report["objective"] == pytest.approx(2.440473700630761, rel=1e-10)


def test_dense_matches_oracle(dctx, ctx, oracle):
    n = 150
    x = oracle.rng_doubles(41, 0, 2 * n).reshape(n, 2)
    w = 0.2 + oracle.rng_doubles(41, 1, 2 * n)
    a, b = w[:n] / w[:n].sum(), w[n:] / w[n:].sum()
    Cm, K, r = _dense_case(oracle, x, 0.1)
    for uot, lam in ((False, math.inf), (True, 0.6)):
        for stab in (False, True):
            ou, ov, _, _, ores = oracle.sinkhorn(a, b, 0.1, lam, 1e-10, 5000, stab, uot=uot, K=K)
            fu, fv, _, _, _ = oracle.sinkhorn(a, b, 0.1, lam, -1.0, 300, stab, uot=uot, K=K)
            cfg = spk.SolverConfig(0.1, lam, 1e-10, 5000, stab)
            for c, form in ((dctx, "dense"), (ctx, "dense"), (dctx, "coords"), (ctx, "coords")):
                kern = spk.Dense(K, r, Cm) if form == "dense" else spk.Coords(x, x, "sqeuclid", scale=1.0, eps=0.1)
                fp32 = c is ctx and form == "coords" and not stab
                if fp32:  # fp32 kernel values cannot reach delta=1e-10: compare at fixed iterations, fp32 bar
                    res = c.sinkhorn(kern, a, b, spk.SolverConfig(0.1, lam, -1.0, 300, stab), uot=uot)
                    np.testing.assert_allclose(res.u, fu, rtol=1e-4)
                    np.testing.assert_allclose(res.v, fv, rtol=1e-4)
                    continue
                res = c.sinkhorn(kern, a, b, cfg, uot=uot)
                if c is dctx and not uot and not stab and form == "dense":  # same K bits: exact order
                    assert np.array_equal(res.u, ou) and np.array_equal(res.v, ov)
                    assert res.report["iterations"] == ores["iterations"]
                np.testing.assert_allclose(res.u, ou, rtol=1e-9)
                np.testing.assert_allclose(res.v, ov, rtol=1e-9)


@pytest.mark.parametrize("max_w", [16, 64, 16384])
def test_blocked_loop_matches_csr(oracle, max_w):
    """The slab x block layout (TMA-staged tiles) against the CSR loop and the
    oracle, forcing many tiles per half with a small tile width."""
    from paper_2306_06581_b200 import _lib as L

    n = 700
    x = oracle.rng_doubles(77, 0, 2 * n).reshape(n, 2)
    w = 0.2 + oracle.rng_doubles(77, 1, 2 * n)
    a, b = w[:n] / w[:n].sum(), w[n:] / w[n:].sum()
    Cm, _ = oracle.pairwise_cost(x, x)
    K, r = oracle.kernel_from_cost(Cm, 0.02)
    for plan, lam in (("ot", math.inf), ("uot", 0.5)):
        p = oracle.plan(plan, a, b, K, r, lam, 0.02)
        so = oracle.poisson_sparsify(K, p, 10 * n * math.log(n), 5)
        oracle.free_plan(p)
        ou, ov, _, _, ores = oracle.sinkhorn(a, b, 0.02, lam, -1.0, 120, policy="mask", uot=plan == "uot", csr=so)
        for values in ("f64", "f32"):
            with spk.Context(0) as c:
                c.set_option(L.OPT_BLOCKED_LOOP, 1)
                c.set_option(L.OPT_BLOCKED_MAX_W, max_w)
                res = c.sketch_from_csr(*so, values_type=values).solve(spk.SolverConfig(0.02, lam, -1.0, 120),
                                                                         uot=plan == "uot", a=a, b=b)
                c.set_option(L.OPT_BLOCKED_LOOP, 0)
                ref = c.sketch_from_csr(*so, values_type=values).solve(spk.SolverConfig(0.02, lam, -1.0, 120),
                                                                         uot=plan == "uot", a=a, b=b)
            tol = 1e-10 if values == "f64" else 1e-4
            np.testing.assert_allclose(res.u, ref.u, rtol=tol)
            np.testing.assert_allclose(res.v, ref.v, rtol=tol)
            if values == "f64":
                np.testing.assert_allclose(res.u, ou, rtol=1e-10)
                np.testing.assert_allclose(res.v, ov, rtol=1e-10)
            assert res.report["masked_rows"] == ores["masked_rows"]


def test_blocked_layout_placements_agree():
    """The three chunk placements of the slab x block layout -- plain run
    placement (0), edge colouring of the row / column bank classes (1, the
    default: Kempe-chain flips, leftovers of over-full classes, per-class
    padding) and greedy column dealing (2) -- on a config-4-law sketch large
    enough for realistic segments (n = 1.5e5: ~180 rows per warp, several
    entries per row and block, both cluster and L2-swap pair exchange). Each
    must give the CSR loop's scalings: the same fp32 entries summed in fp64,
    only the order differs."""
    from paper_2306_06581_b200 import _lib as L
    from paper_2306_06581_b200 import workloads as W

    w = W.c4(n=150_000, pairs=1_000_000)
    cfg = spk.SolverConfig(w.eps, w.lam, -1.0, 12)
    with spk.Context(0) as c:
        kern = spk.Coords(w.x, w.y, w.cost, w.eta, scale=w.scale, eps=w.eps)
        c.set_option(L.OPT_BLOCKED_LOOP, 0)
        sk = c.sketch(kern, w.a, w.b, "ot", w.lam, w.eps, w.s, 7, spk.SparSinkOptions(values=w.values))
        ref = sk.solve(cfg)
        sk.free()
        for spread, cluster in ((0, 1), (1, 1), (1, 0), (2, 1)):
            c.set_option(L.OPT_BLOCKED_LOOP, 1)
            c.set_option(L.OPT_BLOCKED_SPREAD, spread)
            c.set_option(L.OPT_BLOCKED_CLUSTER, cluster)
            assert c.get_option(L.OPT_BLOCKED_SPREAD) == spread
            sk = c.sketch(kern, w.a, w.b, "ot", w.lam, w.eps, w.s, 7, spk.SparSinkOptions(values=w.values))
            res = sk.solve(cfg)
            sk.free()
            assert res.report["iterations"] == ref.report["iterations"] == 12
            assert res.report["masked_rows"] == ref.report["masked_rows"]
            np.testing.assert_allclose(res.u, ref.u, rtol=1e-11)
            np.testing.assert_allclose(res.v, ref.v, rtol=1e-11)


# ---- BASELINE configs at full size -------------------------------------------------------------


def test_config1_full_size(dctx, ctx, oracle):
    from paper_2306_06581_b200 import workloads as W

    w = W.c1()
    Cm, c0 = oracle.pairwise_cost(w.x, w.y)
    Cm /= c0
    K, r = oracle.kernel_from_cost(Cm, w.eps)
    assert r == 1.0
    p = oracle.plan("ot", w.a, w.b, K, r)
    so = oracle.poisson_sparsify(K, p, w.s, 7)
    oracle.free_plan(p)
    kern = spk.Coords(w.x, w.y, "sqeuclid", scale=None, eps=w.eps)
    sk = ctx.sketch(kern, w.a, w.b, "ot", w.lam, w.eps, w.s, 7)
    rp, ci, vv = sk.csr()
    assert np.array_equal(rp, so[0]) and np.array_equal(ci, so[1])
    np.testing.assert_allclose(vv, so[2], rtol=VALUE_RTOL)
    ou, ov, _, _, ores = oracle.sinkhorn(w.a, w.b, w.eps, w.lam, w.delta, w.max_iter, policy="mask", csr=so)
    res = dctx.sketch_from_csr(*so).solve(spk.SolverConfig(w.eps, w.lam, w.delta, w.max_iter), a=w.a, b=w.b)
    assert res.report["iterations"] == 200 == ores["iterations"]
    assert np.array_equal(res.u, ou) and np.array_equal(res.v, ov)
    r2 = ctx.spar_sink(kern, w.a, w.b, spk.SolverConfig(w.eps, w.lam, w.delta, w.max_iter), w.s, 7)
    _, _, oobj = oracle.readout(so, ou, ov, w.a, w.b, w.eps, Cm=Cm)
    assert r2.report["objective"] == pytest.approx(oobj, rel=1e-10)
    np.testing.assert_allclose(r2.u, ou, rtol=1e-10)


def test_config2_full_size(ctx, oracle):
    """UOT, n=1e4, grid plan with a 1e8-term normaliser: index sets must still
    match the oracle's sequential normaliser; scalings/objective to 1e-6."""
    from paper_2306_06581_b200 import workloads as W

    w = W.c2()
    Cm, c0 = oracle.pairwise_cost(w.x, w.y)
    Cm /= c0
    K, r = oracle.kernel_from_cost(Cm, w.eps)
    u, v, _, _, rep, so = oracle.spar_sink(K, r, Cm, w.a, w.b, w.eps, w.s, 7, w.lam, w.delta, w.max_iter,
                                           uot=True)
    del K
    kern = spk.Coords(w.x, w.y, "sqeuclid", scale=None, eps=w.eps)
    g = ctx.spar_sink(kern, w.a, w.b, spk.SolverConfig(w.eps, w.lam, w.delta, w.max_iter), w.s, 7, uot=True)
    sk = ctx.sketch(kern, w.a, w.b, "uot", w.lam, w.eps, w.s, 7)
    rp, ci, vv = sk.csr()
    mism = int(np.sum(rp != so[0]))
    assert mism == 0 and np.array_equal(ci, so[1]), "index sets differ from the oracle"
    np.testing.assert_allclose(vv, so[2], rtol=1e-12)
    assert abs(g.report["iterations"] - rep["iterations"]) <= 1
    assert g.report["objective"] == pytest.approx(rep["objective"], rel=1e-6)
    np.testing.assert_allclose(g.u, u, rtol=1e-6)
    np.testing.assert_allclose(g.v, v, rtol=1e-6)


def test_config4_rows_against_oracle(ctx, oracle):
    """n = 1e6 (the reference cannot hold K): full GPU sketch vs the oracle's
    coordinate restatement of poisson_sparsify on sampled rows, bit-exact
    indices; size-independent properties on the whole sketch."""
    from paper_2306_06581_b200 import workloads as W

    w = W.c4()
    kern = spk.Coords(w.x, w.y, "sqeuclid", scale=w.scale, eps=w.eps)
    sk = ctx.sketch(kern, w.a, w.b, "ot", w.lam, w.eps, w.s, 7, spk.SparSinkOptions(values="f32"))
    n = sk.n
    assert abs(sk.nnz - w.s) < 6 * math.sqrt(w.s)
    rp, ci, vv = sk.csr()
    cnt = np.diff(rp)
    assert cnt.min() >= 0 and rp[-1] == sk.nnz
    # strictly increasing columns inside rows
    d = np.diff(ci.astype(np.int64))
    starts = rp[1:-1]
    ok = np.ones(len(d), bool)
    ok[starts[(starts > 0) & (starts < len(ci))] - 1] = False
    assert np.all(d[ok] > 0)
    # row weights as the reference computes them (sparsify.cpp:76-82)
    ra = np.sqrt(w.a)
    sa = 0.0
    for t in ra.tolist():
        sa += t
    row_w = ra / sa
    assert sk.factorized_plan == (sk.kernel_nnz == n * n)
    plan = sk.plan()
    # heavy tails: some K underflow in fp64, so the reference's masked-grid
    # plan applies; its normaliser (a 1e12-term sum) comes from the device
    assert not plan["factorized"] and sk.kernel_nnz < n * n
    for i in [0, 1, 17, 4242, 99_999, 500_000, n - 1]:
        orp, oci, ovv = oracle.sample_rows_coords(w.x, w.y, "sqeuclid", 0.0, w.scale, w.eps, "ot",
                                                  plan["factorized"], row_w, row_w, 0.0, plan["inv"], w.s, 7, i,
                                                  i + 1)
        seg = slice(rp[i], rp[i + 1])
        assert np.array_equal(ci[seg], oci), f"row {i}"
        np.testing.assert_allclose(vv[seg], ovv.astype(np.float32).astype(np.float64), rtol=1e-6)
    # CSC mirror: same multiset of (i, j, value) -- integer checksums over 1.1e8 entries
    cp, ri, vt = sk.csc()
    assert np.array_equal(np.diff(cp), np.bincount(ci, minlength=n))
    rows = np.repeat(np.arange(n, dtype=np.uint64), cnt)
    cols = np.repeat(np.arange(n, dtype=np.uint64), np.diff(cp))
    key_r = rows * np.uint64(n) + ci.astype(np.uint64)
    key_c = ri.astype(np.uint64) * np.uint64(n) + cols
    assert np.sum(key_r) == np.sum(key_c) and np.sum(key_r * key_r) == np.sum(key_c * key_c)
    assert np.sum(vv * (key_r % np.uint64(9973))) == pytest.approx(np.sum(vt * (key_c % np.uint64(9973))), rel=1e-12)


def test_tiled_sampler_matches_two_pass(ctx, oracle):
    """The single-pass tiled sampler and the exact two-pass kernels give the
    same sketch (both against the oracle) on every plan kind."""
    from paper_2306_06581_b200 import _lib as L

    n = 500
    for d, kind, eta, eps in ((3, "sqeuclid", 0.0, 0.01), (2, "wfr", 0.1, 0.02), (5, "sqeuclid", 0.0, 0.2)):
        x = oracle.rng_doubles(300 + d, 0, d * n).reshape(n, d)
        y = oracle.rng_doubles(400 + d, 0, d * n).reshape(n, d)
        w = 0.2 + oracle.rng_doubles(500 + d, 1, 2 * n)
        a, b = w[:n] / w[:n].sum(), w[n:] / w[n:].sum()
        kern = spk.Coords(x, y, kind, eta, scale=1.0, eps=eps)
        Cm, _ = oracle.pairwise_cost(x, y, kind, eta)
        K, r = oracle.kernel_from_cost(Cm, eps)
        for plan, lam, theta in (("ot", math.inf, 0.0), ("uot", 0.7, 0.0), ("uniform", math.inf, 0.2),
                                 ("ot", math.inf, 0.3)):
            p = oracle.plan(plan, a, b, K, r, lam, eps, theta)
            so = oracle.poisson_sparsify(K, p, 8 * n * math.log(n), 9)
            oracle.free_plan(p)
            outs = []
            for two_pass in (0, 1):
                ctx.set_option(L.OPT_TWO_PASS_SAMPLER, two_pass)
                sk = ctx.sketch(kern, a, b, plan, lam, eps, 8 * n * math.log(n), 9,
                                spk.SparSinkOptions(theta=theta))
                outs.append(sk.csr())
            ctx.set_option(L.OPT_TWO_PASS_SAMPLER, 0)
            for rp, ci, vv in outs:
                assert np.array_equal(rp, so[0]) and np.array_equal(ci, so[1]), (kind, plan, theta)
                np.testing.assert_allclose(vv, so[2], rtol=value_rtol(kind), atol=SUBNORMAL_ATOL)
            assert np.array_equal(outs[0][2], outs[1][2])


def test_tiled_sampler_dense_budgets(ctx, oracle):
    """Budgets close to n^2: most p* reach 1 (every draw kept), so every 32-column
    step of a fully supported tile queues all its lanes for the exact decision
    (the candidate queue fills and drains several times per step). Tiled
    single-pass sampler against the exact two-pass kernels and the oracle."""
    from paper_2306_06581_b200 import _lib as L

    n = 416
    x = oracle.rng_doubles(31, 0, 3 * n).reshape(n, 3)
    y = oracle.rng_doubles(32, 0, 3 * n).reshape(n, 3)
    w = 0.05 + oracle.rng_doubles(33, 1, 2 * n)
    a, b = w[:n] / w[:n].sum(), w[n:] / w[n:].sum()
    kern = spk.Coords(x, y, "sqeuclid", 0.0, scale=1.0, eps=0.5)
    Cm, _ = oracle.pairwise_cost(x, y, "sqeuclid", 0.0)
    K, r = oracle.kernel_from_cost(Cm, 0.5)
    assert r == 1.0
    for frac in (0.3, 0.6, 0.95):
        s = frac * n * n
        p = oracle.plan("ot", a, b, K, r, math.inf, 0.5, 0.0)
        so = oracle.poisson_sparsify(K, p, s, 21)
        oracle.free_plan(p)
        outs = []
        for two_pass in (0, 1):
            ctx.set_option(L.OPT_TWO_PASS_SAMPLER, two_pass)
            outs.append(ctx.sketch(kern, a, b, "ot", math.inf, 0.5, s, 21).csr())
        ctx.set_option(L.OPT_TWO_PASS_SAMPLER, 0)
        for rp, ci, vv in outs:
            assert np.array_equal(rp, so[0]) and np.array_equal(ci, so[1]), frac
            np.testing.assert_allclose(vv, so[2], rtol=value_rtol("sqeuclid"), atol=SUBNORMAL_ATOL)
        assert np.array_equal(outs[0][2], outs[1][2])
        assert len(so[1]) > 0.25 * n * n * frac


def test_max_cost_tiled(ctx):
    """c0 = max finite cost of the C / max normalisation (geometry.cpp:61) from the
    tiled max-d2 pass (n >= 2048, squared-Euclidean and Euclidean costs): the
    same bits as the pairwise sequential-order computation, so every normalised
    cost is unchanged."""
    rng = np.random.default_rng(3)
    n = 3000
    x = rng.normal(size=(n, 3))
    y = rng.normal(size=(n, 3)) + 0.5
    s = np.zeros((n, n))
    for k in range(3):  # d2 summed over the dimensions in order, no FMA (geometry.cpp:16-59)
        diff = x[:, None, k] - y[None, :, k]
        s = s + diff * diff
    qi = np.arange(64, dtype=np.int64)
    qj = (qi * 7 + 3) % n
    for kind in ("sqeuclid", "euclid"):
        full = np.sqrt(s) if kind == "euclid" else s
        cost, _, c0 = ctx.cost_kernel(spk.Coords(x, y, kind, eps=0.1), qi, qj)
        assert c0 == full.max()
        assert np.array_equal(cost, full[qi, qj] / full.max())


def test_config3_frame_pair(ctx, oracle):
    """Config 3 (one WFR frame pair at full size, n = 12544): UOT grid plan on
    a 22%-support kernel, fp32 sketch values, log-domain loop. Index sets bit
    for bit against the oracle's dense path; values to one fp32 ulp; the
    log-domain solve against the oracle on the same sketch within the fp32
    bar (fp32 log K~ values)."""
    from paper_2306_06581_b200 import workloads as W

    w = W.c3()
    Cm, _ = oracle.pairwise_cost(w.x, w.y, "wfr", w.eta)
    K, r = oracle.kernel_from_cost(Cm, w.eps)
    del Cm
    plan = oracle.plan("uot", w.a, w.b, K, r, w.lam, w.eps)
    so = oracle.poisson_sparsify(K, plan, w.s, 7)
    oracle.free_plan(plan)
    del K
    kern = spk.Coords(w.x, w.y, "wfr", w.eta, scale=1.0, eps=w.eps)
    sk = ctx.sketch(kern, w.a, w.b, "uot", w.lam, w.eps, w.s, 7, spk.SparSinkOptions(values="f32"))
    rp, ci, vv = sk.csr()
    assert np.array_equal(rp, so[0]) and np.array_equal(ci, so[1]), "index sets differ from the oracle"
    np.testing.assert_allclose(vv, so[2].astype(np.float32).astype(np.float64), rtol=1.2e-7)
    cfg = spk.SolverConfig(w.eps, w.lam, -1.0, 150, stabilize=True)
    g = sk.solve(cfg, uot=True, a=w.a, b=w.b)
    _, _, olu, olv, ores = oracle.sinkhorn(w.a, w.b, w.eps, w.lam, -1.0, 150, stabilize=True, policy="mask",
                                           uot=True, csr=(rp, ci, vv))
    assert g.report["iterations"] == ores["iterations"] == 150
    fin = np.isfinite(olu)
    assert np.array_equal(fin, np.isfinite(g.log_u))
    # fp32 log K~ (|log K~| up to ~700): absolute error ~1e-4 in the log scalings
    np.testing.assert_allclose(g.log_u[fin], olu[fin], rtol=1e-5, atol=2e-3)
    fin = np.isfinite(olv)
    np.testing.assert_allclose(g.log_v[fin], olv[fin], rtol=1e-5, atol=2e-3)
    _, _, gobj, _ = sk.readout(kern, uot=True, lambda_=w.lam, epsilon=w.eps)
    _, _, oobj = oracle.readout((rp, ci, vv), np.exp(olu), np.exp(olv), w.a, w.b, w.eps, w.lam, True, lu=olu, lv=olv,
                                coords=(w.x, w.y, "wfr", w.eta, 1.0))
    assert gobj == pytest.approx(oobj, rel=1e-4)


def test_config5_dense_vs_sparse(ctx):
    """Config 5 at full size (n = 5e4): the dense on-the-fly comparator against
    Spar-Sink at s = 4, 8, 16 n ln n. The sketch estimate of the objective
    approaches the dense one as s grows (the paper's RMAE trend)."""
    from paper_2306_06581_b200 import workloads as W

    w = W.c5()
    kern = spk.Coords(w.x, w.y, "sqeuclid", scale=None, eps=w.eps)
    cfg = spk.SolverConfig(w.eps, w.lam, w.delta, w.max_iter)
    dense = ctx.sinkhorn(kern, w.a, w.b, cfg)
    assert dense.report["iterations"] == 200 and np.isfinite(dense.report["objective"])
    errs = []
    for mult in (4, 8, 16):
        sp = ctx.spar_sink(kern, w.a, w.b, cfg, mult * w.n * math.log(w.n), 7)
        errs.append(abs(sp.report["objective"] - dense.report["objective"]) / abs(dense.report["objective"]))
    # the entropic objective of a sketch plan converges slowly in s (measured
    # here: ~0.34 / 0.31 / 0.27 at 4 / 8 / 16 n ln n, eps = 0.05); the trend
    # must be monotone
    assert all(np.isfinite(errs)) and errs[0] < 0.5, errs
    assert errs[0] > errs[1] > errs[2], errs


def test_config3_pairs_batch_split_across_ranks(ctx):
    """Config 3's batch driver: pairs split round-robin over ranks give the
    same per-pair results as solving each pair alone with mix_seed(seed, k)."""
    from paper_2306_06581_b200 import api
    from paper_2306_06581_b200 import workloads as W

    coords, masses = W.c3_frames(3, frames=6, side=40)
    n = coords.shape[0]
    cfg = spk.SolverConfig(0.01, 1.0, 1e-6, 300, stabilize=True)
    s = 10 * n * math.log(n)
    pairs = api.frame_pairs(6)[:5]
    got = {}
    for r in range(2):
        for k, pr, rep in api.spar_sink_pairs(ctx, coords, masses, cfg, s, 3, 0.1, pairs=pairs, rank=r, world=2):
            got[k] = rep
    assert sorted(got) == list(range(5))
    kern = spk.Coords(coords, coords, "wfr", 0.1, scale=1.0, eps=0.01)
    for k, (i, j) in enumerate(pairs):
        one = ctx.spar_sink(kern, masses[i], masses[j], cfg, s, api.mix_seed(3, k), uot=True)
        assert one.report["objective"] == pytest.approx(got[k]["objective"], rel=1e-10)  # batched: other sum order
        assert one.report["sketch_nnz"] == got[k]["sketch_nnz"]
