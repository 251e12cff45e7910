"""Pin the CPU oracle (oracle/spk_oracle.c) before trusting it.

1. The reference's own known-answer values (proj/tests/test_sparsify.cpp,
   test_solvers.cpp, test_geometry.cpp), restated as numbers here.
2. The committed golden fixtures (tests/golden/*.npz, generated from the
   compiled reference by tests/golden/make_golden.py): bit-exact.
3. When oracle/_ref is built: fresh random cases, oracle vs reference, bit-exact.
"""
import math
from pathlib import Path

import numpy as np
import pytest

GOLD = Path(__file__).resolve().parent / "golden"


def dense_objective(u, v, K, Cm, eps):
    T = u[:, None] * K * v[None, :]
    m = T > 0
    t = T[m]
    return float(np.sum(t * Cm[m]) - eps * (-np.sum(t * (np.log(t) - 1.0))))


# ---- known-answer tests (reference unit tests) -------------------------------------


def test_kat_ot_probabilities(oracle):
    # test_sparsify.cpp:51-61
    pts = oracle.rng_doubles(3, 0, 4).reshape(2, 2)
    Cm, _ = oracle.pairwise_cost(pts, pts)
    K, r = oracle.kernel_from_cost(Cm, 1.0)
    p = oracle.plan("ot", np.array([0.25, 0.75]), np.array([0.5, 0.5]), K, r)
    probs = oracle.plan_probs(p)
    assert p.factorized == 1
    assert probs[0, 0] == pytest.approx(0.18301270189221933, rel=1e-14)
    assert probs[1, 1] == pytest.approx(0.31698729810778065, rel=1e-14)
    assert probs.sum() == pytest.approx(1.0, rel=1e-12)
    oracle.free_plan(p)


def test_kat_uot_probabilities(oracle):
    # test_sparsify.cpp:63-81: lambda = eps = 1 puts exponent 1/3 on both factors
    K = np.array([[1.0, 0.5], [0.25, 1.0]])
    p = oracle.plan("uot", np.array([0.3, 0.7]), np.array([0.4, 0.6]), K, 1.0, 1.0, 1.0)
    probs = oracle.plan_probs(p)
    want = [0.2346093653249565, 0.2131567545016285, 0.19602777445115938, 0.35620610572225564]
    assert probs.ravel() == pytest.approx(want, rel=1e-13)
    oracle.free_plan(p)


def test_kat_theta_shrink(oracle):
    # test_sparsify.cpp:95-108
    pts = oracle.rng_doubles(9, 0, 4).reshape(2, 2)
    Cm, _ = oracle.pairwise_cost(pts, pts)
    K, r = oracle.kernel_from_cost(Cm, 1.0)
    a, b = np.array([0.25, 0.75]), np.array([0.5, 0.5])
    p = oracle.plan("ot", a, b, K, r)
    q = oracle.plan("ot", a, b, K, r, theta=0.4)
    pp, qq = oracle.plan_probs(p), oracle.plan_probs(q)
    assert qq[0, 0] == pytest.approx(0.6 * pp[0, 0] + 0.4 / 4.0, rel=1e-14)
    assert qq.sum() == pytest.approx(1.0, rel=1e-12)
    from oracle import OracleError

    with pytest.raises(OracleError) as e:
        oracle.plan("ot", a, b, K, r, theta=1.0)
    assert e.value.kind == 12  # ThetaOutOfRange
    oracle.free_plan(p)
    oracle.free_plan(q)


def test_kat_wfr_cost_and_kernel(oracle):
    # test_geometry.cpp:47-72
    eta = 2.0
    x = np.array([0.0, 1.0, math.pi * eta + 0.5])
    Cm, c0 = oracle.pairwise_cost(x, x, "wfr", eta)
    assert Cm[0, 0] == 0.0
    assert Cm[0, 1] == pytest.approx(0.06316210249493931, rel=1e-14)
    assert math.isinf(Cm[0, 2]) and math.isfinite(c0)
    x2 = np.array([0.0, 1.0, 100.0])
    C2, _ = oracle.pairwise_cost(x2, x2, "wfr", 2.0)
    K, r = oracle.kernel_from_cost(C2, 0.5)
    assert K[0, 2] == 0.0 and K[0, 0] == 1.0
    assert r == pytest.approx(5.0 / 9.0)
    Cs, c0s = oracle.pairwise_cost(np.array([0.0, 3.0]), np.array([0.0, 3.0]))
    assert Cs[0, 1] == 9.0 and c0s == 9.0


def _dense_solve(oracle, sup, a, b, eps, lam=math.inf):
    Cm, _ = oracle.pairwise_cost(sup, sup)
    K, _ = oracle.kernel_from_cost(Cm, eps)
    u, v, _, _, rep = oracle.sinkhorn(a, b, eps, lam, 1e-13, 200000, uot=math.isfinite(lam), K=K)
    return u, v, K, Cm, rep


def test_kat_two_atom_ot(oracle):
    # test_solvers.cpp:60-73
    u, v, K, Cm, rep = _dense_solve(oracle, np.array([0.0, 1.0]), np.array([0.5, 0.5]), np.array([0.5, 0.5]), 1.0)
    assert rep["converged"]
    assert u[0] * K[0, 0] * v[0] == pytest.approx(0.36552928931500245, rel=1e-10)
    assert u[0] * K[0, 1] * v[1] == pytest.approx(0.13447071068499758, rel=1e-10)
    assert dense_objective(u, v, K, Cm, 1.0) == pytest.approx(-2.006408868078168, rel=1e-10)


def test_kat_three_atom_ot(oracle):
    # test_solvers.cpp:75-86
    u, v, K, Cm, _ = _dense_solve(oracle, np.array([0.0, 0.3, 1.0]), np.array([0.2, 0.3, 0.5]),
                                  np.array([0.4, 0.4, 0.2]), 0.5)
    assert u[0] * K[0, 0] * v[0] == pytest.approx(0.1269550276492255, rel=1e-9)
    assert dense_objective(u, v, K, Cm, 0.5) == pytest.approx(-1.2371064921733375, rel=1e-10)


def _uot_objective(u, v, K, Cm, a, b, lam, eps):
    T = u[:, None] * K * v[None, :]
    rm, cm = T.sum(1), T.sum(0)

    def kl(x, y):
        return float(np.sum(np.where(x > 0, x * np.log(np.where(x > 0, x, 1) / y) - x + y, y)))

    t = T[T > 0]
    return float(np.sum(t * Cm[T > 0]) + lam * kl(rm, a) + lam * kl(cm, b) + eps * np.sum(t * (np.log(t) - 1)))


def test_kat_single_atom_uot(oracle):
    # test_solvers.cpp:88-100
    a, b = np.array([2.0]), np.array([8.0])
    u, v, K, Cm, _ = _dense_solve(oracle, np.array([0.0]), a, b, 1.0, 1.0)
    assert abs(u[0] * K[0, 0] * v[0] - 16.0 ** (1 / 3)) < 1e-8
    assert _uot_objective(u, v, K, Cm, a, b, 1.0, 1.0) == pytest.approx(2.440473700630761, rel=1e-10)


def test_kat_two_atom_uot(oracle):
    # test_solvers.cpp:102-115
    a, b = np.array([0.7, 0.9]), np.array([0.4, 0.8])
    u, v, K, Cm, _ = _dense_solve(oracle, np.array([0.0, 1.0]), a, b, 0.5, 2.0)
    assert u[0] * K[0, 0] * v[0] == pytest.approx(0.4880086699186626, rel=1e-9)
    assert u[1] * K[1, 1] * v[1] == pytest.approx(0.7835780682111341, rel=1e-9)
    assert _uot_objective(u, v, K, Cm, a, b, 2.0, 0.5) == pytest.approx(-0.9506480667355813, rel=1e-9)


def test_kat_kl(oracle):
    # test_solvers.cpp:181-187
    import ctypes as C

    x = np.array([0.2, 0.0, 0.5])
    y = np.array([0.1, 0.3, 0.4])
    out = C.c_double()
    rc = oracle.lib.spko_kl_divergence(x.ctypes.data_as(C.POINTER(C.c_double)),
                                       y.ctypes.data_as(C.POINTER(C.c_double)), 3, C.byref(out))
    assert rc == 0 and out.value == pytest.approx(0.3502012117690939, rel=1e-14)
    bad = C.c_double()
    xx, yy = np.array([0.5]), np.array([0.0])
    assert oracle.lib.spko_kl_divergence(xx.ctypes.data_as(C.POINTER(C.c_double)),
                                         yy.ctypes.data_as(C.POINTER(C.c_double)), 1, C.byref(bad)) == 1


def test_saturated_budget_reproduces_kernel(oracle):
    # test_sparsify.cpp:110-135: with uniform weights on a truncated kernel the
    # masked plan is 1/nnz on the support and s slightly above nnz saturates
    n = 20
    p = oracle.rng_doubles(31, 0, 2 * n).reshape(n, 2)
    Cm, _ = oracle.pairwise_cost(p, p, "wfr", 0.12)
    K, r = oracle.kernel_from_cost(Cm, 0.5)
    assert r < 0.8
    u = np.full(n, 1.0 / n)
    plan = oracle.plan("ot", u, u, K, r)
    nnz = r * n * n
    rp, ci, vv = oracle.poisson_sparsify(K, plan, nnz * 1.01, 77)
    oracle.free_plan(plan)
    assert len(ci) == round(nnz)
    D = np.zeros((n, n))
    for i in range(n):
        D[i, ci[rp[i]:rp[i + 1]]] = vv[rp[i]:rp[i + 1]]
    assert np.array_equal(D, K)  # bit-identical, no rescaling


def test_sketch_seed_determinism_and_budget(oracle):
    # test_sparsify.cpp:137-157
    n = 40
    pts = oracle.rng_doubles(13, 0, 2 * n).reshape(n, 2)
    Cm, _ = oracle.pairwise_cost(pts, pts)
    K, r = oracle.kernel_from_cost(Cm, 0.5)
    w = 0.1 + oracle.rng_doubles(3, 1, n)
    a = w / w.sum()
    plan = oracle.plan("ot", a, a, K, r)
    s1 = oracle.poisson_sparsify(K, plan, 200.0, 42)
    s2 = oracle.poisson_sparsify(K, plan, 200.0, 42)
    s3 = oracle.poisson_sparsify(K, plan, 200.0, 43)
    assert all(np.array_equal(x, y) for x, y in zip(s1, s2))
    assert not np.array_equal(s1[1], s3[1]) if len(s1[1]) == len(s3[1]) else True
    assert len(s1[1]) < 200 + 5 * math.sqrt(200)
    from oracle import OracleError

    for bad in (0.0, float(n * n)):
        with pytest.raises(OracleError) as e:
            oracle.poisson_sparsify(K, plan, bad, 1)
        assert e.value.kind == 13  # BudgetTooLarge
    oracle.free_plan(plan)


def test_spmv_against_dense(oracle):
    # test_sparsify.cpp:186-211
    n = 30
    pts = oracle.rng_doubles(19, 0, 2 * n).reshape(n, 2)
    Cm, _ = oracle.pairwise_cost(pts, pts)
    K, r = oracle.kernel_from_cost(Cm, 0.5)
    plan = oracle.plan("uniform", None, None, K, r)
    csr = oracle.poisson_sparsify(K, plan, 300.0, 5)
    oracle.free_plan(plan)
    D = np.zeros((n, n))
    for i in range(n):
        D[i, csr[1][csr[0][i]:csr[0][i + 1]]] = csr[2][csr[0][i]:csr[0][i + 1]]
    v = oracle.rng_doubles(99, 0, n)
    assert oracle.spmv(csr, v) == pytest.approx(D @ v, rel=1e-12)
    assert oracle.spmv(csr, v, transpose=True) == pytest.approx(D.T @ v, rel=1e-12)


def test_log_domain_agrees_with_linear(oracle):
    # test_solvers.cpp:159-179
    n = 25
    p = oracle.rng_doubles(53, 0, 2 * n).reshape(n, 2)
    wa = 0.2 + oracle.rng_doubles(53, 0, 3 * n)[2 * n:]
    a = wa / wa.sum()
    Cm, _ = oracle.pairwise_cost(p, p)
    K, _ = oracle.kernel_from_cost(Cm, 0.2)
    for lam in (math.inf, 0.7):
        up, vp, _, _, _ = oracle.sinkhorn(a, a, 0.2, lam, 1e-13, 200000, uot=math.isfinite(lam), K=K)
        ul, vl, lu, lv, rep = oracle.sinkhorn(a, a, 0.2, lam, 1e-13, 200000, stabilize=True,
                                              uot=math.isfinite(lam), K=K)
        assert rep["log_domain"] == 1
        T1 = up[:, None] * K * vp[None, :]
        T2 = np.exp(lu[:, None] + np.log(K) + lv[None, :])
        assert T2 == pytest.approx(T1, rel=1e-6)


def test_input_validation(oracle):
    # test_solvers.cpp:189-204 (NotNormalized, UOT needs finite lambda)
    from oracle import OracleError

    K = np.eye(2) + 0.1
    with pytest.raises(OracleError) as e:
        oracle.sinkhorn(np.array([0.5, 0.6]), np.array([0.5, 0.5]), 0.5, K=K)
    assert e.value.kind == 4
    with pytest.raises(OracleError) as e:
        oracle.sinkhorn(np.array([0.5, 0.5]), np.array([0.5, 0.5]), 0.5, uot=True, K=K)
    assert e.value.kind == 1


# ---- golden fixtures generated by the reference itself ------------------------------


@pytest.mark.parametrize("path", sorted(GOLD.glob("sketch_*.npz")), ids=lambda p: p.stem)
def test_golden_sketch_bit_exact(oracle, path):
    g = np.load(path)
    kind, plan = str(g["kind"]), str(g["plan"])
    Cm, c0 = oracle.pairwise_cost(g["x"], g["y"], kind, float(g["eta"]))
    assert c0 == float(g["c0"])
    K, r = oracle.kernel_from_cost(Cm, float(g["eps"]))
    assert r == float(g["nnz_ratio"])
    p = oracle.plan(plan, g["a"], g["b"], K, r, float(g["lam"]), float(g["eps"]), float(g["theta"]))
    assert np.array_equal(oracle.plan_probs(p), g["probs"])
    rp, ci, vv = oracle.poisson_sparsify(K, p, float(g["s"]), int(g["seed"]))
    oracle.free_plan(p)
    assert np.array_equal(rp, g["row_ptr"])
    assert np.array_equal(ci, g["col_idx"])
    assert np.array_equal(vv, g["values"])


@pytest.mark.parametrize("path", sorted(GOLD.glob("solve_*.npz")), ids=lambda p: p.stem)
def test_golden_solve_bit_exact(oracle, path):
    g = np.load(path)
    Cm, c0 = oracle.pairwise_cost(g["x"], g["y"], "sqeuclid")
    K, r = oracle.kernel_from_cost(Cm, float(g["eps"]))
    u, v, lu, lv, rep, _ = oracle.spar_sink(K, r, Cm, g["a"], g["b"], float(g["eps"]), float(g["s"]), int(g["seed"]),
                                            float(g["lam"]), float(g["delta"]), int(g["max_iter"]),
                                            bool(g["stabilize"]), 0.0, str(g["probs"]), False, bool(g["uot"]))
    assert np.array_equal(u, g["u"]) and np.array_equal(v, g["v"])
    assert rep["iterations"] == int(g["rep_iterations"])
    assert rep["objective"] == float(g["rep_objective"])
    for k in ("converged", "diverged", "masked_rows", "masked_cols"):
        assert rep[k] == int(g[f"rep_{k}"]), k
    for k in ("residual_row", "residual_col", "kernel_mean"):
        assert rep[k] == float(g[f"rep_{k}"]), k


@pytest.mark.parametrize("path", sorted(GOLD.glob("loop_*.npz")), ids=lambda p: p.stem)
def test_golden_loop_outcomes(oracle, path):
    from oracle import OracleError

    g = np.load(path)
    csr = (g["row_ptr"], g["col_idx"], g["values"])
    stab = bool(g["stabilize"]) if "stabilize" in g else False
    kw = dict(lambda_=float(g["lam"]), delta=float(g["delta"]), max_iter=int(g["max_iter"]), stabilize=stab,
              policy=str(g["policy"]), uot=bool(g["uot"]), csr=csr)
    if int(g["err"]):
        with pytest.raises(OracleError) as e:
            oracle.sinkhorn(g["a"], g["b"], float(g["eps"]), **kw)
        assert e.value.kind == int(g["err"])
        return
    u, v, lu, lv, rep = oracle.sinkhorn(g["a"], g["b"], float(g["eps"]), **kw)
    assert np.array_equal(u, g["u"]) and np.array_equal(v, g["v"])
    for k in ("iterations", "converged", "diverged", "masked_rows", "masked_cols"):
        assert rep[k] == int(g[f"rep_{k}"]), k


# ---- fresh cases against the compiled reference -------------------------------------


@pytest.mark.parametrize("seed", [101, 202, 303])
def test_oracle_vs_reference_random(oracle, reference, seed):
    n = 120
    x = oracle.rng_doubles(seed, 0, 2 * n).reshape(n, 2)
    y = oracle.rng_doubles(seed, 1, 2 * n).reshape(n, 2)
    w = 0.3 + oracle.rng_doubles(seed, 2, 2 * n)
    a, b = w[:n] / w[:n].sum(), w[n:] / w[n:].sum()
    for kind, eta, eps in (("sqeuclid", 0.0, 0.05), ("wfr", 0.12, 0.02)):
        Co, _ = oracle.pairwise_cost(x, y, kind, eta)
        Cr, _ = reference.pairwise_cost(x, y, kind, eta)
        assert np.array_equal(Co, Cr)
        K, r = oracle.kernel_from_cost(Co, eps)
        for plan, lam in (("ot", math.inf), ("uot", 0.9), ("uniform", math.inf)):
            p = oracle.plan(plan, a, b, K, r, lam, eps, 0.2)
            so = oracle.poisson_sparsify(K, p, 6 * n * math.log(n), seed)
            oracle.free_plan(p)
            sr = reference.poisson_sparsify(plan, a, b, K, r, 6 * n * math.log(n), seed, lam, eps, 0.2)
            assert all(np.array_equal(s, t) for s, t in zip(so, sr)), (kind, plan)
            uo, vo, _, _, ro = oracle.sinkhorn(a, b, eps, lam, 1e-10, 3000, policy="mask",
                                               uot=math.isfinite(lam), csr=so)
            ur, vr, _, _, rr = reference.sinkhorn(a, b, eps, lam, 1e-10, 3000, policy="mask",
                                                  uot=math.isfinite(lam), csr=sr)
            assert np.array_equal(uo, ur) and np.array_equal(vo, vr)
            assert ro["iterations"] == rr["iterations"]
