"""GPU: the multi-GPU path owned by the library (include/spk.h spk_comm_*,
spk_sharded_*, spk_spar_sink_multi) -- the driver a C / C++ caller uses.

Only one GPU is available, so: the emulated communicator runs W = 1..3 ranks
as threads sharing the GPU (host-synchronised copies; no kernel waits on
another rank); NCCL runs for real at W = 1 (the captured-graph loop, replayed
by a second solve); spk_spar_sink_multi runs over the one device. Every
result must equal the single-GPU solve of the same problem (the union of the
row slabs is the 1-GPU sketch bit for bit)."""
import math
import threading

import numpy as np
import pytest

import paper_2306_06581_b200 as spk
from paper_2306_06581_b200 import _lib as L
from paper_2306_06581_b200 import sharded as S

pytestmark = pytest.mark.gpu


def _problem(oracle, n=3000, uot=False):
    x = oracle.rng_doubles(201, 0, 3 * n).reshape(n, 3)
    y = 0.2 + oracle.rng_doubles(201, 1, 3 * n).reshape(n, 3)
    w = 0.3 + oracle.rng_doubles(201, 2, 2 * n)
    a = w[:n] / w[:n].sum()
    b = w[n:] / w[n:].sum() * (1.3 if uot else 1.0)
    kern = spk.Coords(x, y, "sqeuclid", scale=None, eps=0.02)
    lam = 1.0 if uot else math.inf
    cfg = spk.SolverConfig(0.02, lam, -1.0, 60)
    return kern, a, b, cfg, 8 * n * math.log(n)


def _emulated(world, fn, options=None):
    group = S.EmulatedGroup(world)
    out, err = [None] * world, [None] * world

    def body(r):
        ctx = comm = None
        try:
            ctx = spk.Context(0)
            for k, v in (options or {}).items():
                ctx.set_option(k, v)
            comm = S.LibComm.emulated(ctx, group.ptr, r)
            out[r] = fn(ctx, comm)
        except BaseException as e:  # noqa: BLE001
            err[r] = e
        finally:
            if comm:
                comm.close()
            if ctx:
                ctx.close()

    th = [threading.Thread(target=body, args=(r,)) for r in range(world)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    group.close()
    for e in err:
        if e is not None:
            raise e
    return out


@pytest.mark.parametrize("world", [1, 2, 3])
@pytest.mark.parametrize("case", ["ot_f32_blocked", "uot_f64", "ot_log"])
def test_library_driver_emulated_ranks(oracle, world, case):
    uot = case.startswith("uot")
    kern, a, b, cfg, s = _problem(oracle, uot=uot)
    opts = spk.SparSinkOptions(values="f32" if "f32" in case else "f64")
    if case == "ot_log":
        cfg = spk.SolverConfig(cfg.epsilon, cfg.lambda_, -1.0, 60, stabilize=True)
    options = {L.OPT_BLOCKED_LOOP: 1} if "blocked" in case else {L.OPT_BLOCKED_LOOP: 0}
    with spk.Context(0) as c:
        for k, v in options.items():
            c.set_option(k, v)
        ref = c.spar_sink(kern, a, b, cfg, s, 7, opts, uot=uot)

    def run(ctx, comm):
        sk = S.LibShardedSketch(comm, kern, a, b, "uot" if uot else "ot", cfg.lambda_, cfg.epsilon, s, 7, opts)
        r1 = sk.solve(cfg, uot)
        r2 = sk.solve(cfg, uot)  # the sketch is reusable
        sk.free()
        return r1, r2

    outs = _emulated(world, run, options)
    tol = 1e-4 if "f32" in case else 1e-9
    for r1, r2 in outs:
        assert r1.report["sketch_nnz"] == ref.report["sketch_nnz"]
        assert r1.report["iterations"] == ref.report["iterations"] == 60
        assert r1.report["masked_rows"] == ref.report["masked_rows"]
        assert r1.report["objective"] == pytest.approx(ref.report["objective"], rel=tol)
        np.testing.assert_allclose(r1.u, ref.u, rtol=tol)
        np.testing.assert_allclose(r1.v, ref.v, rtol=tol)
        assert np.array_equal(r1.u, r2.u) and r1.report["objective"] == r2.report["objective"]
    # every rank returns the same full scalings
    for r1, _ in outs[1:]:
        assert np.array_equal(r1.u, outs[0][0].u)


def test_library_driver_nccl_graph_world1(oracle):
    """NCCL (loaded by the library) at W = 1: the first solve captures the
    loop into a CUDA graph, the second replays it -- both equal the 1-GPU solve."""
    kern, a, b, cfg, s = _problem(oracle)
    opts = spk.SparSinkOptions(values="f32")
    with spk.Context(0) as c:
        c.set_option(L.OPT_BLOCKED_LOOP, 1)
        ref = c.spar_sink(kern, a, b, cfg, s, 7, opts)
        comm = S.LibComm.nccl(c, S.LibComm.unique_id(c.lib), 1, 0)
        assert comm.info() == {"world": 1, "rank": 0, "nccl": True}
        sk = S.LibShardedSketch(comm, kern, a, b, "ot", cfg.lambda_, cfg.epsilon, s, 7, opts)
        r1 = sk.solve(cfg)
        captured = sk.info["captured_launches"]
        l0 = c.launches
        r2 = sk.solve(cfg)
        assert captured >= 2 * cfg.max_iter  # two half kernels per iteration inside the graph
        assert c.launches - l0 >= captured
        cfg2 = spk.SolverConfig(cfg.epsilon, cfg.lambda_, -1.0, 30)  # another loop length: re-captured
        r3 = sk.solve(cfg2)
        sk.free()
        comm.close()
        one30 = c.spar_sink(kern, a, b, cfg2, s, 7, opts)
    for r in (r1, r2):
        assert r.report["sketch_nnz"] == ref.report["sketch_nnz"]
        assert r.report["iterations"] == 60
        np.testing.assert_allclose(r.u, ref.u, rtol=1e-10)
        assert r.report["objective"] == pytest.approx(ref.report["objective"], rel=1e-10)
    assert np.array_equal(r1.u, r2.u)
    assert r3.report["iterations"] == 30
    np.testing.assert_allclose(r3.u, one30.u, rtol=1e-10)


def test_spar_sink_multi_one_device(oracle):
    kern, a, b, cfg, s = _problem(oracle, uot=True)
    with spk.Context(0) as c:
        ref = c.spar_sink(kern, a, b, cfg, s, 7, uot=True)
    r = S.spar_sink_multi([0], kern, a, b, cfg, s, 7, uot=True)
    assert r.report["sketch_nnz"] == ref.report["sketch_nnz"]
    np.testing.assert_allclose(r.u, ref.u, rtol=1e-9)
    assert r.report["objective"] == pytest.approx(ref.report["objective"], rel=1e-9)
    with pytest.raises(spk.ERRORS["NotNormalized"]):  # the failing rank's error through spk_last_error(NULL)
        S.spar_sink_multi([0], kern, a, 2.0 * b, spk.SolverConfig(0.02, math.inf, -1.0, 10), s, 7)
