"""the frame-pair caller (measure_from_image, mean_pool,
pairwise_wfr, predict_ed) against the compiled, unmodified reference
(oracle/_ref). Host helpers are bit-exact on CPU; pairwise_wfr runs the GPU
path (marked gpu) and matches the reference's own pairwise_wfr."""
import math

import numpy as np
import pytest

from paper_2306_06581_b200 import api, wfr


def blob(h, w, cr, cc, sigma):
    """harness.cpp:439-454 (test input generator)."""
    r, c = np.meshgrid(np.arange(h, dtype=float), np.arange(w, dtype=float), indexing="ij")
    return np.exp(-((r - cr) ** 2 + (c - cc) ** 2) / (2.0 * sigma * sigma))


def test_measure_from_image_matches_reference(reference):
    img = blob(7, 9, 3.0, 4.5, 1.7)
    coords, wts = wfr.measure_from_image(img, 7, 9)
    rc, rw = reference.measure_from_image(img.ravel(), 7, 9)
    assert np.array_equal(coords, rc) and np.array_equal(wts, rw)
    with pytest.raises(api.ERRORS["AllBlack"]):
        wfr.measure_from_image(np.zeros(4), 2, 2)
    with pytest.raises(api.ERRORS["NegativeWeight"]):
        wfr.measure_from_image(np.array([0.5, 1.5, 0.1, 0.2]), 2, 2)
    with pytest.raises(api.ERRORS["LengthMismatch"]):
        wfr.measure_from_image(np.ones(5), 2, 2)


@pytest.mark.parametrize("shape,filt,stride", [((8, 8), 2, 2), ((9, 7), 3, 2), ((10, 10), 4, 3)])
def test_mean_pool_matches_reference(reference, shape, filt, stride):
    img = np.random.default_rng(3).uniform(0, 1, shape)
    out, oh, ow = wfr.mean_pool(img, *shape, filt, stride)
    rout, roh, row = reference.mean_pool(img.ravel(), *shape, filt, stride)
    assert (oh, ow) == (roh, row) and np.array_equal(out, rout)
    with pytest.raises(api.ERRORS["EmptyOutput"]):
        wfr.mean_pool(img, *shape, 50, 1)
    with pytest.raises(api.ERRORS["LengthMismatch"]):
        wfr.mean_pool(img, *shape, 0, 1)


def test_predict_ed_matches_reference(reference):
    d = np.zeros((5, 5))
    d[0, 1:] = [0.1, 0.9, 0.9, 0.3]  # tie -> earliest index (test_harness.cpp:120-137)
    assert wfr.predict_ed(d, 0, 1, 4, 2) == reference.predict_ed(d, 0, 1, 4, 2) == (2, 0.0)
    assert wfr.predict_ed(d, 0, 1, 4, 4) == reference.predict_ed(d, 0, 1, 4, 4) == (2, 0.5)
    with pytest.raises(api.ERRORS["EmptyWindow"]):
        wfr.predict_ed(d, 0, 3, 7, 4)
    d[0, 1:] = math.nan
    with pytest.raises(api.ERRORS["EmptyWindow"]):
        wfr.predict_ed(d, 0, 1, 4, 4)
    assert wfr.s0_budget(100) == pytest.approx(1e-3 * 100 * math.log(100) ** 4, rel=1e-15)


def _frames():
    return [blob(10, 10, 4.5, 3.0 + sh, 1.2) for sh in (0.0, 1.5, 3.0, 4.5)]


@pytest.mark.gpu
def test_pairwise_wfr_exact_matches_reference(reference, ctx):
    fr = _frames()
    d, idx, failed = wfr.pairwise_wfr(ctx, fr, 2.0, 1.0, 0.01, 0.0, 1, exact=True)
    rd, rfailed = reference.pairwise_wfr(np.stack([f.ravel() for f in fr]), 10, 10, 2.0, 1.0, 0.01, 0.0, 1, 1,
                                         exact=True)
    assert failed == rfailed == 0 and idx == [0, 1, 2, 3]
    np.testing.assert_allclose(d, rd, rtol=1e-6, atol=1e-12)
    assert d[0, 3] > d[0, 2] > d[0, 1] > 0.0 and np.array_equal(d, d.T)
    ds, idx2, _ = wfr.pairwise_wfr(ctx, fr, 2.0, 1.0, 0.01, 0.0, 1, stride=2, exact=True)
    assert idx2 == [0, 2]


@pytest.mark.gpu
def test_pairwise_wfr_sparse_matches_reference_and_predicts_ed(reference, ctx):
    """Same pair seeds (mix_seed(seed, k)) -> the same sketches as the
    reference -> the same distances; ED = the farthest frame from ES."""
    fr = [blob(16, 16, 7.5, 3.0 + 1.5 * t, 1.5) for t in range(6)]
    d, _, failed = wfr.pairwise_wfr(ctx, fr, 5.0, 1.0, 0.02, 80.0, 1101)
    rd, rfailed = reference.pairwise_wfr(np.stack([f.ravel() for f in fr]), 16, 16, 5.0, 1.0, 0.02, 80.0, 1101, 1)
    assert failed == rfailed
    np.testing.assert_allclose(d, rd, rtol=1e-6, atol=1e-12)
    assert wfr.predict_ed(d, 0, 1, 5, 5) == reference.predict_ed(rd, 0, 1, 5, 5)
