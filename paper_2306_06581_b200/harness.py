"""RMAE experiment on the GPU path: the reference's
rmae_experiment (proj/src/harness.cpp:150-232) and budget schedule (:128-149)
over given scenario data. The exact objective comes from the dense
on-the-fly Sinkhorn in fp64 (the reference's sinkhorn_ot/uot on K); every
replication r runs spar_sink_ot/uot (or Rand-Sink) with seed
mix_seed(seed, (r + 1) + attempt * 0x100000), retrying a failing draw up to
five times exactly as the reference does. Replications are independent, so
ranks can split them (rank/world)."""
from __future__ import annotations

import math

import numpy as np

from . import _lib as L
from .api import Context, Coords, SolverConfig, SparSinkOptions, SparsinkError, mix_seed


def s0_budget(n: int) -> float:
    """s0(n) = 1e-3 n ln^4 n (harness.cpp:128-131)."""
    ln = math.log(n)
    return 1e-3 * n * ln * ln * ln * ln


def s_schedule(n: int, multipliers) -> tuple[list[float], bool]:
    """(budgets, clamped) (harness.cpp:133-149)."""
    if n < 2:
        from .api import ERRORS
        raise ERRORS["LengthMismatch"]("LengthMismatch: s_schedule needs n >= 2")
    s0 = s0_budget(n)
    cap = float(n) * float(n) * (1.0 - 1e-9)
    out, clamped = [], False
    for m in multipliers:
        s = m * s0
        if s >= cap:
            s, clamped = cap, True
        out.append(s)
    return out, clamped


def rmae_experiment(ctx: Context, support, a, b, cfg: SolverConfig, budgets, replications: int, seed: int,
                    method: str = "sparsink", eta: float | None = None, rank: int = 0, world: int = 1) -> dict:
    """-> {"exact_objective", "rows": [{"budget", "errors", "mean", "std_error", "retried"}]}.
    eta given: WFR cost + UOT (cfg.lambda finite), else squared Euclidean + OT,
    both on the raw cost (no max-normalisation, like the reference)."""
    if replications < 1:
        from .api import ERRORS
        raise ERRORS["LengthMismatch"]("LengthMismatch: rmae_experiment needs replications >= 1")
    x = np.ascontiguousarray(support, dtype=np.float64)
    uot = eta is not None
    kern = Coords(x, x, "wfr" if uot else "sqeuclid", eta or 0.0, scale=1.0, eps=cfg.epsilon)
    prev_fp32 = ctx.get_option(L.OPT_OTF_FP32)
    ctx.set_option(L.OPT_OTF_FP32, 0)  # the exact baseline is the fp64 dense solve
    try:
        base = ctx.sinkhorn(kern, a, b, cfg, uot=uot)
    except SparsinkError as e:
        from .api import ERRORS
        raise ERRORS["BaselineFailed"](f"BaselineFailed: {e}")
    finally:
        ctx.set_option(L.OPT_OTF_FP32, prev_fp32)  # the caller's setting, not a default
    exact = base.report["objective"]
    if exact == 0.0:
        from .api import ERRORS
        raise ERRORS["BaselineFailed"]("BaselineFailed: exact objective is zero")
    opts = SparSinkOptions(probs="importance" if method == "sparsink" else "uniform")
    rows = []
    for s in budgets:
        errors, retried = [], 0
        for r in range(replications):
            if r % world != rank:
                errors.append(math.nan)
                continue
            attempt = 0
            while True:
                sd = mix_seed(seed, (r + 1) + attempt * 0x100000)
                try:
                    approx = ctx.spar_sink(kern, a, b, cfg, s, sd, opts, uot=uot).report["objective"]
                    break
                except SparsinkError:
                    attempt += 1
                    if attempt > 5:
                        raise
                    retried += 1
            errors.append(abs(approx - exact) / abs(exact))
        if world > 1:  # every rank computed a disjoint subset: merge before the statistics
            errors, retried = _merge_ranks(errors, retried, world)
        e = np.asarray([v for v in errors if not math.isnan(v)])
        mean = float(e.sum() / len(e)) if len(e) else math.nan
        var = float(((e - mean) ** 2).sum()) if len(e) else math.nan
        se = math.sqrt(var / (len(e) - 1) / len(e)) if len(e) > 1 else 0.0
        rows.append({"budget": s, "errors": errors, "mean": mean, "std_error": se, "retried": retried})
    return {"exact_objective": exact, "rows": rows, "replications": replications,
            "method": method}


def _merge_ranks(errors: list[float], retried: int, world: int) -> tuple[list[float], int]:
    """Replication r was run by rank r % world: gather every rank's errors
    (torch.distributed, any backend) so mean / std_error cover all
    replications as the reference's single loop does (harness.cpp:213-225)."""
    import torch.distributed as dist

    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() != world:
        raise RuntimeError("rmae_experiment with world > 1 needs an initialised torch.distributed group of that size")
    gathered: list = [None] * world
    dist.all_gather_object(gathered, (errors, retried))
    merged = [gathered[r % world][0][r] for r in range(len(errors))]
    return merged, int(sum(g[1] for g in gathered))
