"""Synthetic config generators: reference RNG addressing, determinism, shapes."""
import math

import numpy as np

from paper_2306_06581_b200 import workloads as W


def test_uniforms_are_the_reference_counter_rng(oracle):
    for seed, stream in ((7, 3), (0, 0), (2**63 + 5, 12345)):
        assert np.array_equal(W.uniforms(seed, stream, 257), oracle.rng_doubles(seed, stream, 257))
        assert W.mix_seed(seed, stream) == oracle.mix_seed(seed, stream)


def test_normals_follow_box_muller(oracle):
    d = W.normals(11, 2, 1001) - oracle.rng_normals(11, 2, 1001)
    assert np.max(np.abs(d)) < 1e-12  # numpy vs glibc transcendental ULPs only


def test_c1_c2_shapes_and_masses():
    w1 = W.c1()
    assert w1.x.shape == (1000, 5) and abs(w1.a.sum() - 1.0) < 1e-12 and not w1.uot
    assert w1.s == 8 * 1000 * math.log(1000) and w1.max_iter == 200 and w1.delta < 0
    w2 = W.c2()
    assert w2.x.shape == (10_000, 10) and abs(w2.a.sum() - 1.0) < 1e-12 and abs(w2.b.sum() - 1.5) < 1e-12
    assert w2.uot and w2.lam == 1.0 and w2.eps == 0.05 and w2.max_iter == 500


def test_c3_frames():
    coords, masses = W.c3_frames()
    assert coords.shape == (112 * 112, 2) and masses.shape == (32, 112 * 112)
    assert np.allclose(masses.sum(1), 1.0) and masses.min() > 0
    assert coords.min() == 0.0 and coords.max() == 1.0
    # periodic cycle: frame 0 and 32 coincide, neighbouring frames differ
    assert not np.allclose(masses[0], masses[1])


def test_c4_small_quantile_deterministic():
    w = W.c4(n=2000, pairs=100_000)
    w2 = W.c4(n=2000, pairs=100_000)
    assert np.array_equal(w.x, w2.x) and w.extra["q"] == w2.extra["q"] > 0
    d2 = ((w.x[:, None, :] - w.y[None, :, :]) ** 2).sum(-1)
    assert abs(np.mean(d2 <= w.extra["q"]) - 0.999) < 0.002


def test_bytes_per_iteration_formula():
    # C4 ~1.848 GB with fp32 values
    assert abs(W.bytes_per_iteration(10**6, 110_524_084, 4) / 1e9 - 1.848) < 0.01
    assert abs(W.bytes_per_iteration(1000, 55_262, 8) / 1e6 - 1.41) < 0.02


def test_pair_seeds_follow_the_reference_rng(oracle):
    """mix_seed(seed, k) (rng.hpp:17-19) is the per-pair seed of the batched
    frame pairs (harness.cpp:393): its first draw must equal the oracle's
    first draw of stream k."""
    from paper_2306_06581_b200 import api

    for seed, k in ((7, 0), (7, 5), (3, 495), (2**63 + 11, 17)):
        m = api.mix_seed(seed, k)
        x = (m + 0x9E3779B97F4A7C15) & api._M64
        x = ((x ^ (x >> 30)) * 0xBF58476D1CE4E5B9) & api._M64
        x = ((x ^ (x >> 27)) * 0x94D049BB133111EB) & api._M64
        x ^= x >> 31
        assert (x >> 11) * 2.0**-53 == oracle.rng_doubles(seed, k, 1)[0]
    pairs = api.frame_pairs(32)
    assert len(pairs) == 496 and pairs[0] == (0, 1) and pairs[-1] == (30, 31)
