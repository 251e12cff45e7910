"""GPU: the one-cluster Sinkhorn loop for small sketches (csrc/small.cu:
scalings in every CTA's shared memory, DSMEM broadcast, one cluster barrier
per half) against the oracle, the reference-generated loop fixtures
(dynamic masking, divergence restore, ZeroDenominator -- solvers.hpp:292-358)
and the persistent grid loop it replaces at configs 1 and 2."""
import math
from pathlib import Path

import numpy as np
import pytest

import paper_2306_06581_b200 as spk
from paper_2306_06581_b200 import _lib as L

pytestmark = pytest.mark.gpu
GOLD = Path(__file__).resolve().parent / "golden"
CLUSTERS = [1, 4, 16]


@pytest.fixture(scope="module")
def sctx():
    c = spk.Context(0)
    c.set_option(L.OPT_SMALL_LOOP, 1)
    yield c
    c.close()


@pytest.mark.parametrize("cs", CLUSTERS)
@pytest.mark.parametrize("path", sorted(GOLD.glob("loop_*.npz")), ids=lambda p: p.stem)
def test_small_loop_failure_semantics(sctx, path, cs):
    g = np.load(path)
    csr = (g["row_ptr"], g["col_idx"], g["values"])
    stab = bool(g["stabilize"]) if "stabilize" in g else False
    cfg = spk.SolverConfig(float(g["eps"]), float(g["lam"]), float(g["delta"]), int(g["max_iter"]), stab)
    sctx.set_option(L.OPT_SMALL_CLUSTER, cs)
    sk = sctx.sketch_from_csr(*csr)
    if int(g["err"]):
        with pytest.raises(spk.SparsinkError) as e:
            sk.solve(cfg, uot=bool(g["uot"]), a=g["a"], b=g["b"], policy=str(g["policy"]))
        assert e.value.kind == int(g["err"])
        return
    res = sk.solve(cfg, uot=bool(g["uot"]), a=g["a"], b=g["b"], policy=str(g["policy"]))
    for k in ("iterations", "converged", "diverged", "masked_rows", "masked_cols"):
        assert res.report[k] == int(g[f"rep_{k}"]), k
    np.testing.assert_allclose(res.u, g["u"], rtol=1e-10)
    np.testing.assert_allclose(res.v, g["v"], rtol=1e-10)


@pytest.mark.parametrize("cs", CLUSTERS)
@pytest.mark.parametrize("path", sorted(GOLD.glob("sketch_*.npz")), ids=lambda p: p.stem)
def test_small_loop_matches_oracle(sctx, oracle, path, cs):
    g = np.load(path)
    csr = (g["row_ptr"], g["col_idx"], g["values"])
    uot = str(g["plan"]) == "uot"
    lam = float(g["lam"]) if uot else math.inf
    eps = float(g["eps"])
    sctx.set_option(L.OPT_SMALL_CLUSTER, cs)
    for stab in (False, True):
        ou, ov, olu, _, ores = oracle.sinkhorn(g["a"], g["b"], eps, lam, -1.0, 150, stabilize=stab, policy="mask",
                                               uot=uot, csr=csr)
        for values in ("f64", "f32"):
            res = sctx.sketch_from_csr(*csr, values_type=values).solve(spk.SolverConfig(eps, lam, -1.0, 150, stab),
                                                                     uot=uot, a=g["a"], b=g["b"])
            assert res.report["iterations"] == ores["iterations"] == 150
            assert res.report["masked_rows"] == ores["masked_rows"]
            if values == "f32":  # fp32 sketch values (and, in the log domain, the fp32-accurate exp)
                np.testing.assert_allclose(res.u, ou, rtol=1e-4)
                np.testing.assert_allclose(res.v, ov, rtol=1e-4)
                continue
            np.testing.assert_allclose(res.u, ou, rtol=1e-10)
            np.testing.assert_allclose(res.v, ov, rtol=1e-10)
            if stab:
                fin = np.isfinite(olu)
                np.testing.assert_allclose(res.log_u[fin], olu[fin], rtol=1e-11, atol=1e-11)


@pytest.mark.parametrize("cfgname", ["c1", "c2"])
def test_small_loop_full_size_configs(oracle, cfgname):
    """Configs 1 and 2 at full size: the one-cluster loop against the
    persistent grid loop on the same sketch (same iterations, masks, and
    scalings to 1e-10) and against the oracle loop."""
    from paper_2306_06581_b200 import workloads as W

    w = W.CONFIGS[cfgname]()
    kern = spk.Coords(w.x, w.y, "sqeuclid", scale=None, eps=w.eps)
    plan = "uot" if w.uot else "ot"
    cfg = spk.SolverConfig(w.eps, w.lam, w.delta, w.max_iter)
    out = {}
    with spk.Context(0) as c:
        sk = c.sketch(kern, w.a, w.b, plan, w.lam, w.eps, w.s, 7)
        csr = sk.csr()
        for small in (1, 0):
            c.set_option(L.OPT_SMALL_LOOP, small)
            out[small] = sk.solve(cfg, uot=w.uot)
        sk.free()
    ou, ov, _, _, ores = oracle.sinkhorn(w.a, w.b, w.eps, w.lam, w.delta, w.max_iter, policy="mask", uot=w.uot,
                                         csr=csr)
    a, b = out[1], out[0]
    assert a.report["iterations"] == b.report["iterations"]
    assert abs(a.report["iterations"] - ores["iterations"]) <= 1  # delta stop within rounding
    for k in ("masked_rows", "masked_cols", "converged", "diverged"):
        assert a.report[k] == b.report[k], k
    np.testing.assert_allclose(a.u, b.u, rtol=1e-10)
    np.testing.assert_allclose(a.v, b.v, rtol=1e-10)
    np.testing.assert_allclose(a.u, ou, rtol=1e-8)
    assert a.report["residual_row"] == pytest.approx(b.report["residual_row"], rel=1e-6, abs=1e-15)
