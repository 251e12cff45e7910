"""Multi-rank Spar-Sink driver over gloo on CPU (world 2 and 3).

The driver (paper_2306_06581_b200/sharded.py) runs unchanged -- plan row-sum
gather, column all-to-all, two all-gathers per iteration, tail-carried loop
decisions, readout reduction -- with a numpy stand-in for the CUDA shard
(tests/shard_cpu.py). Results must equal the single-process oracle solve on
the same sketch: scalings and objective to rounding,
iteration and mask counts exactly.
"""
import math
import os
import socket
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parent.parent


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _problem(case):
    from oracle import Oracle

    o = Oracle()
    n = {"ot": 240, "uot": 200, "ragged": 161}[case]
    x = o.rng_doubles(91, 0, 2 * n).reshape(n, 2)
    y = 0.3 + o.rng_doubles(91, 1, 2 * n).reshape(n, 2)
    w = 0.2 + o.rng_doubles(91, 2, 2 * n)
    a = w[:n] / w[:n].sum()
    b = w[n:] / w[n:].sum() * (1.5 if case == "uot" else 1.0)
    Cm, _ = o.pairwise_cost(x, y)
    scale = float(Cm.max())
    eps = 0.05
    K, r = o.kernel_from_cost(Cm / scale, eps)
    uot = case == "uot"
    lam = 1.0 if uot else math.inf
    p = o.plan("uot" if uot else "ot", a, b, K, r, lam, eps)
    csr = o.poisson_sparsify(K, p, 6 * n * math.log(n), 7)
    o.free_plan(p)
    delta, iters = (1e-9, 400) if uot else (-1.0, 60)
    return o, dict(x=x, y=y, a=a, b=b, scale=scale, eps=eps, lam=lam, uot=uot, csr=csr, delta=delta, iters=iters,
                   Cm=Cm / scale)


def _worker(rank, world, port, case, outdir):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    sys.path.insert(0, str(ROOT))
    sys.path.insert(0, str(ROOT / "tests"))
    import torch.distributed as dist

    from paper_2306_06581_b200 import api, sharded
    from shard_cpu import CpuShard

    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        _, P = _problem(case)
        shard = CpuShard(P["csr"], P["x"], P["y"], P["scale"])
        cfg = api.SolverConfig(P["eps"], P["lam"], P["delta"], P["iters"])
        res = sharded.spar_sink_sharded(sharded.TorchComm(), shard, api.Coords(P["x"], P["y"], scale=P["scale"]),
                                        P["a"], P["b"], cfg, 1.0, 7, uot=P["uot"], check_every=16)
        np.savez(Path(outdir) / f"r{rank}.npz", u=res.u, v=res.v,
                 rep=np.array([res.report["iterations"], res.report["converged"], res.report["masked_rows"],
                               res.report["masked_cols"], res.report["objective"], res.report["residual_row"],
                               res.report["residual_col"], res.report["sketch_nnz"]]))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("case,world", [("ot", 2), ("uot", 2), ("ragged", 3)])
def test_sharded_driver_gloo_matches_oracle(tmp_path, case, world):
    import torch.multiprocessing as mp

    mp.spawn(_worker, args=(world, _free_port(), case, str(tmp_path)), nprocs=world, join=True)
    o, P = _problem(case)
    ou, ov, _, _, ores = o.sinkhorn(P["a"], P["b"], P["eps"], P["lam"], P["delta"], P["iters"], policy="mask",
                                    uot=P["uot"], csr=P["csr"])
    _, _, oobj = o.readout(P["csr"], ou, ov, P["a"], P["b"], P["eps"], P["lam"], P["uot"], Cm=P["Cm"])
    outs = [np.load(tmp_path / f"r{r}.npz") for r in range(world)]
    for d in outs:  # every rank returns the whole answer
        np.testing.assert_allclose(d["u"], ou, rtol=1e-12)
        np.testing.assert_allclose(d["v"], ov, rtol=1e-12)
        it, conv, mr, mc, obj, rr, rc, nnz = d["rep"]
        assert int(it) == ores["iterations"] and int(conv) == ores["converged"]
        assert int(mr) == ores["masked_rows"] and int(mc) == ores["masked_cols"]
        assert obj == pytest.approx(oobj, rel=1e-11)
        assert int(nnz) == int(P["csr"][0][-1])
    for d in outs[1:]:
        np.testing.assert_array_equal(d["u"], outs[0]["u"])
        np.testing.assert_array_equal(d["rep"], outs[0]["rep"])


def _rmae_merge_worker(rank, world, port, outdir):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    sys.path.insert(0, str(ROOT))
    import torch.distributed as dist

    from paper_2306_06581_b200.harness import _merge_ranks

    dist.init_process_group("gloo", rank=rank, world_size=world)
    reps = 7
    # rank r ran replications r, r + world, ... (rmae_experiment's split)
    errors = [0.1 * (k + 1) if k % world == rank else math.nan for k in range(reps)]
    merged, retried = _merge_ranks(errors, rank + 1, world)
    np.save(Path(outdir) / f"m{rank}.npy", np.asarray(merged + [retried]))
    dist.destroy_process_group()


def test_rmae_ranks_merge_before_statistics(tmp_path):
    """rmae_experiment at world > 1: every rank ends with ALL replications'
    errors (so mean / std_error match the reference's single loop)."""
    import torch.multiprocessing as mp

    mp.spawn(_rmae_merge_worker, args=(2, _free_port(), str(tmp_path)), nprocs=2, join=True)
    for r in range(2):
        m = np.load(tmp_path / f"m{r}.npy")
        np.testing.assert_allclose(m[:-1], 0.1 * np.arange(1, 8))
        assert m[-1] == 3  # retried counts summed over ranks
