"""IBP / Spar-IBP barycenters on the GPU (csrc/ibp.cu)
against the compiled, unmodified reference (oracle/_ref): q to pow()'s ULPs,
identical iteration counts; spar_ibp's sketches (column-constant plan, seeds
mix_seed(seed, k)) bit-identical, so the sparse barycenter matches too."""
import math

import numpy as np
import pytest

import paper_2306_06581_b200 as spk
from paper_2306_06581_b200 import api


def _problem(reference, n=60, eps=0.01):
    x = np.linspace(0.0, 1.0, n)[:, None]
    Cm, c0 = reference.pairwise_cost(x, x)
    K, r = reference.kernel_from_cost(Cm, eps)
    bs = []
    for mu, sd in ((0.2, 0.05), (0.5, 0.08), (0.8, 0.04)):
        g = np.exp(-0.5 * ((x[:, 0] - mu) / sd) ** 2) + 1e-3
        bs.append(g / g.sum())
    return x, K, r, np.stack(bs)


def test_reference_barycenter_shim_loads(reference):
    x, K, r, b = _problem(reference, n=20, eps=0.05)
    q, rep = reference.ibp(b, np.array([0.2, 0.5, 0.3]), Ks=[K] * 3, ratios=[r] * 3)
    assert rep["iterations"] >= 1 and abs(q.sum() - 1.0) < 0.1


@pytest.mark.gpu
def test_ibp_matches_reference(reference, ctx):
    x, K, r, b = _problem(reference)
    w = np.array([0.2, 0.5, 0.3])
    qr, rr = reference.ibp(b, w, 1e-9, 2000, Ks=[K] * 3, ratios=[r] * 3)
    rp = np.arange(0, 60 * 60 + 1, 60, dtype=np.int64)  # dense K as a full sketch (K > 0 everywhere here)
    ci = np.tile(np.arange(60, dtype=np.uint32), 60)
    sks = [ctx.sketch_from_csr(rp, ci, K.ravel()) for _ in range(3)]
    q, rep = api.ibp(ctx, sks, b, w, 1e-9, 2000)
    assert rep["iterations"] == rr["iterations"] and rep["converged"] == rr["converged"] == 1
    np.testing.assert_allclose(q, qr, rtol=1e-11, atol=1e-300)


@pytest.mark.gpu
@pytest.mark.parametrize("form", ["dense", "coords"])
def test_spar_ibp_matches_reference(reference, ctx, form):
    x, K, r, b = _problem(reference)
    w = np.array([0.3, 0.3, 0.4])
    n = len(x)
    s = 10 * n * math.log(n)
    qr, rr = reference.spar_ibp([K] * 3, [r] * 3, b, w, s, 77, 1e-9, 2000)
    kern = spk.Dense(K, r) if form == "dense" else spk.Coords(x, x, scale=1.0, eps=0.01)
    q, rep = api.spar_ibp(ctx, [kern] * 3, b, w, s, 77, 1e-9, 2000)
    assert rep["iterations"] == rr["iterations"]
    assert rep["masked_atoms"] == rr["masked_atoms"]
    np.testing.assert_allclose(q, qr, rtol=1e-10, atol=1e-300)


@pytest.mark.gpu
def test_ibp_argument_errors(reference, ctx):
    x, K, r, b = _problem(reference, n=20, eps=0.05)
    rp = np.arange(0, 400 + 1, 20, dtype=np.int64)
    ci = np.tile(np.arange(20, dtype=np.uint32), 20)
    sks = [ctx.sketch_from_csr(rp, ci, K.ravel()) for _ in range(3)]
    with pytest.raises(api.ERRORS["NotNormalized"]):
        api.ibp(ctx, sks, b, np.array([0.5, 0.5, 0.5]))
    with pytest.raises(api.ERRORS["NegativeWeight"]):
        api.ibp(ctx, sks, b, np.array([1.5, -0.5, 0.0]))
