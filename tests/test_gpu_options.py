"""GPU: context options read back (spk_ctx_get_option) and the callers that
change one temporarily restore the caller's value."""
import math

import pytest

import paper_2306_06581_b200 as spk
from paper_2306_06581_b200 import _lib as L
from paper_2306_06581_b200 import harness

pytestmark = pytest.mark.gpu


def test_option_round_trip_and_validation():
    with spk.Context(0) as c:
        assert c.get_option(L.OPT_BLOCKED_LOOP) == 2  # auto
        c.set_option(L.OPT_BLOCKED_MAX_W, 17)  # rounded down to a multiple of 16 (16-byte TMA sources)
        assert c.get_option(L.OPT_BLOCKED_MAX_W) == 16
        c.set_option(L.OPT_BLOCKED_MAX_W, 1000)
        assert c.get_option(L.OPT_BLOCKED_MAX_W) == 992
        for key, bad in ((L.OPT_BATCH_CLUSTER, 3), (L.OPT_BATCH_UNROLL, 5), (L.OPT_SMALL_CLUSTER, 12)):
            with pytest.raises(spk.SparsinkError):
                c.set_option(key, bad)
        c.set_option(L.OPT_SMALL_CLUSTER, 8)
        assert c.get_option(L.OPT_SMALL_CLUSTER) == 8
        with pytest.raises(spk.SparsinkError):
            c.get_option(999)


def test_rmae_restores_the_callers_setting():
    x, a, b = harness.generate_scenario("C1", 60, 2, 3)
    with spk.Context(0) as c:
        for prev in (0, 1):
            c.set_option(L.OPT_OTF_FP32, prev)
            harness.rmae_experiment(c, x, a, b, spk.SolverConfig(0.5), [200.0], 2, 3)
            assert c.get_option(L.OPT_OTF_FP32) == prev
