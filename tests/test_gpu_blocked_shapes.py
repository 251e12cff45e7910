"""Slab x block loop on awkward shapes: forced at sizes where segments are
tiny, empty, over-full (plain placement fallback), or a column part is empty;
every placement mode and both pair exchanges must reproduce the CSR loop."""
import math

import numpy as np
import pytest

import paper_2306_06581_b200 as spk
from paper_2306_06581_b200 import _lib as L

pytestmark = pytest.mark.gpu


def _sketch_csr(rng, n, density, heavy_rows):
    """Random CSR with ascending columns; a few dense rows (long runs inside a block), some empty rows."""
    rows = []
    for i in range(n):
        if i % 11 == 7:
            k = 0
        elif i < heavy_rows:
            k = n
        else:
            k = min(n, rng.poisson(density * n))
        rows.append(np.sort(rng.choice(n, size=k, replace=False)).astype(np.uint32))
    rp = np.zeros(n + 1, np.int64)
    rp[1:] = np.cumsum([len(r) for r in rows])
    ci = np.concatenate(rows) if rp[-1] else np.zeros(0, np.uint32)
    vv = rng.uniform(0.1, 1.0, size=len(ci))
    return rp, ci, vv


@pytest.mark.parametrize("n,density,heavy,max_w", [(37, 0.5, 2, 16), (300, 0.08, 0, 16), (300, 0.3, 3, 64),
                                                    (1500, 0.05, 1, 4096), (2600, 0.02, 0, 256), (5000, 0.004, 0, 1024)])
def test_blocked_matches_csr_on_awkward_shapes(n, density, heavy, max_w):
    rng = np.random.default_rng(n)
    rp, ci, vv = _sketch_csr(rng, n, density, heavy)
    w = rng.uniform(0.5, 1.5, size=2 * n)
    a, b = w[:n] / w[:n].sum(), w[n:] / w[n:].sum()
    cfg = spk.SolverConfig(0.05, math.inf, -1.0, 25)
    with spk.Context(0) as c:
        c.set_option(L.OPT_SMALL_LOOP, 0)
        c.set_option(L.OPT_BLOCKED_LOOP, 0)
        ref = c.sketch_from_csr(rp, ci, vv).solve(cfg, a=a, b=b)
        for values in ("f64", "f32"):
            base = ref if values == "f64" else c.sketch_from_csr(rp, ci, vv, values_type="f32").solve(cfg, a=a, b=b)
            for split, spread, cluster in ((2, 1, 1), (2, 1, 0), (2, 0, 1), (2, 2, 1), (1, 1, 1)):
                c.set_option(L.OPT_BLOCKED_LOOP, 1)
                c.set_option(L.OPT_BLOCKED_MAX_W, max_w)
                c.set_option(L.OPT_BLOCKED_SPLIT, split)
                c.set_option(L.OPT_BLOCKED_SPREAD, spread)
                c.set_option(L.OPT_BLOCKED_CLUSTER, cluster)
                res = c.sketch_from_csr(rp, ci, vv, values_type=values).solve(cfg, a=a, b=b)
                c.set_option(L.OPT_BLOCKED_LOOP, 0)
                assert res.report["iterations"] == base.report["iterations"]
                assert res.report["masked_rows"] == base.report["masked_rows"]
                assert res.report["masked_cols"] == base.report["masked_cols"]
                np.testing.assert_allclose(res.u, base.u, rtol=1e-10, atol=0)
                np.testing.assert_allclose(res.v, base.v, rtol=1e-10, atol=0)
