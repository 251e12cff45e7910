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
import time

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


# ---- scenario generators (harness.cpp:14-126) -------------------------------------------
def _normal_density(x: float, mu: float, sigma: float) -> float:
    z = (x - mu) / sigma
    return math.exp(-0.5 * z * z) / sigma


def _t5_density(x: float, mu: float, sigma: float) -> float:
    z = (x - mu) / sigma
    return math.pow(1.0 + z * z / 5.0, -3.0) / sigma


def _grid_weights(n: int, density, total_mass: float) -> np.ndarray:
    """harness.cpp:26-37: density on the grid (i+1)/(n+1), scaled to total_mass
    (sequential sum, glibc exp/pow through math: bit-equal to the reference)."""
    w = [density(float(i + 1) / float(n + 1)) for i in range(n)]
    s = 0.0
    for v in w:
        s += v
    f = total_mass / s
    return np.asarray([v * f for v in w], dtype=np.float64)


def _counter_doubles(seed: int, count: int) -> np.ndarray:
    from .workloads import uniforms

    return uniforms(seed, 0, count)  # CounterRng(seed, 0).next_double() x count (integer ops only: exact)


def _counter_normals(seed: int, count: int) -> list[float]:
    """CounterRng(seed, 0).next_normal() x count (rng.cpp:7-21: Box-Muller, the
    sin value kept as the spare) with glibc log/cos/sin via math."""
    m = (count + 1) // 2
    u = _counter_doubles(seed, 2 * m).tolist()
    out = []
    two_pi = 2.0 * math.pi
    for k in range(m):
        u1 = max(u[2 * k], 1e-300)
        r = math.sqrt(-2.0 * math.log(u1))
        th = two_pi * u[2 * k + 1]
        out.append(r * math.cos(th))
        out.append(r * math.sin(th))
    return out[:count]


def generate_scenario(scenario: str = "C1", n: int = 1000, d: int = 5, seed: int = 1, masses=None,
                      scale_param: float = 0.05, scale_is_sd: bool = False):
    """generate_scenario (harness.cpp:85-126) -> (support (n, d), a, b): C1/C2
    normal-density weights at 1/3 and 1/2, C3 Student-t(5); C2 support
    N(0, 0.5^|j-k|) via its Cholesky factor, C1/C3 uniform on [0,1]^d; the
    reference's counter RNG. Bit-equal to the reference (tests/test_harness_rmae.py)."""
    from .api import ERRORS

    if n < 2 or d < 1:
        raise ERRORS["LengthMismatch"]("LengthMismatch: scenario needs n >= 2 and d >= 1")
    sigma = scale_param if scale_is_sd else math.sqrt(scale_param)
    ma, mb = (masses if masses is not None else (1.0, 1.0))
    if ma <= 0.0 or mb <= 0.0:
        raise ERRORS["NegativeWeight"]("NegativeWeight: total masses must be positive")
    dens = _t5_density if scenario == "C3" else _normal_density
    wa = _grid_weights(n, lambda x: dens(x, 1.0 / 3.0, sigma), ma)
    wb = _grid_weights(n, lambda x: dens(x, 0.5, sigma), mb)
    if scenario == "C2":  # ar_gaussian_support (harness.cpp:51-80)
        sig = [[math.pow(0.5, abs(j - k)) for k in range(d)] for j in range(d)]
        chol = [[0.0] * d for _ in range(d)]
        for j in range(d):
            for k in range(j + 1):
                acc = sig[j][k]
                for t in range(k):
                    acc -= chol[j][t] * chol[k][t]
                chol[j][k] = math.sqrt(acc) if j == k else acc / chol[k][k]
        z = _counter_normals(seed, n * d)
        pts = np.empty(n * d)
        for i in range(n):
            zi = z[i * d:(i + 1) * d]
            for j in range(d):
                acc = 0.0
                for k in range(j + 1):
                    acc += chol[j][k] * zi[k]
                pts[i * d + j] = acc
    else:
        pts = _counter_doubles(seed, n * d)
    support = pts.reshape(n, d)
    if masses is None:  # new_measure's simplex check (measures.cpp:12-34)
        for w in (wa, wb):
            t = 0.0
            for v in w.tolist():
                t += v
            if abs(t - 1.0) > 1e-8:
                raise ERRORS["NotNormalized"]("NotNormalized: scenario weights do not sum to 1")
    return support, wa, wb


def eta_for_sparsity(x, target_nnz_ratio: float) -> float:
    """eta_for_sparsity (geometry.cpp:104-135): the WFR eta whose cut pi*eta
    keeps the target fraction of the n^2 pairwise distances (sorted, the
    kept quantile and the next one averaged)."""
    from .api import ERRORS

    if not (0.0 < target_nnz_ratio <= 1.0):
        raise ERRORS["ThetaOutOfRange"]("ThetaOutOfRange: target nnz ratio must lie in (0,1]")
    x = np.ascontiguousarray(x, dtype=np.float64)
    n, d = x.shape
    if n < 2:
        raise ERRORS["DegenerateSupport"]("DegenerateSupport: need at least two points")
    d2 = np.zeros((n, n))
    for k in range(d):  # sq_dist in the reference's order (sequential over k, no FMA)
        diff = x[:, None, k] - x[None, :, k]
        d2 = d2 + diff * diff
    dists = np.sqrt(d2).ravel()
    dmax = float(dists.max())
    if dmax == 0.0:
        if target_nnz_ratio < 1.0:
            raise ERRORS["DegenerateSupport"]("DegenerateSupport: all points identical")
        return 1.0
    if target_nnz_ratio >= 1.0:
        return dmax / math.pi * 1.0001 + 1e-12
    dists.sort()
    keep = max(1, int(math.floor(target_nnz_ratio * float(n) * float(n) + 0.5)))  # llround
    q_in = float(dists[keep - 1])
    q_out = float(dists[keep]) if keep < len(dists) else q_in * 1.0001
    return (q_in * (1.0 + 1e-9) if q_in == q_out else 0.5 * (q_in + q_out)) / math.pi


def rmae_scenario(ctx: Context, spec: dict, method: str, budgets, replications: int, cfg: SolverConfig,
                  rank: int = 0, world: int = 1) -> dict:
    """rmae_experiment(spec, ...) (harness.cpp:151-232) from a scenario spec
    ({"scenario", "n", "d", "seed", "masses", "sparsity_target", "scale_param",
    "scale_is_sd"}): the scenario is generated here; a sparsity target selects
    the WFR cost (eta_for_sparsity) and UOT."""
    x, a, b = generate_scenario(spec.get("scenario", "C1"), spec.get("n", 1000), spec.get("d", 5),
                                spec.get("seed", 1), spec.get("masses"), spec.get("scale_param", 0.05),
                                spec.get("scale_is_sd", False))
    eta = None
    if spec.get("sparsity_target") is not None:
        eta = eta_for_sparsity(x, spec["sparsity_target"])
    rep = rmae_experiment(ctx, x, a, b, cfg, budgets, replications, spec.get("seed", 1), method, eta, rank, world)
    rep["scale_note"] = "scale_param read as sd" if spec.get("scale_is_sd") else "scale_param read as variance"
    return rep


# ---- timing sweep (harness.cpp:282-330) ---------------------------------------------------
def loglog_slope(x, y) -> float:
    """Least-squares slope of log y on log x (harness.cpp:332-346)."""
    if len(x) != len(y) or len(x) < 2:
        from .api import ERRORS
        raise ERRORS["LengthMismatch"]("LengthMismatch: loglog_slope needs matched samples")
    n = float(len(x))
    sx = sy = sxx = sxy = 0.0
    for xi, yi in zip(x, y):
        lx, ly = math.log(float(xi)), math.log(yi)
        sx += lx
        sy += ly
        sxx += lx * lx
        sxy += lx * ly
    return (n * sxy - sx * sy) / (n * sxx - sx * sx)


def timing_sweep(ctx: Context, sizes, d: int, cfg: SolverConfig, s_multiplier: float, seed: int,
                 iters_per_point: int = 5) -> list[dict]:
    """timing_sweep (harness.cpp:282-330) on the GPU: scenario C1 at each n;
    "sinkhorn" = the dense loop with K recomputed on the fly from coordinates
    (direct_sq_euclid_kernel's K = exp(-d^2/eps), no cost normalisation, fp32
    exp), "spar-sink" = plan + Poisson sketch at s = min(mult * s0(n),
    0.999 n^2) and the sparse loop. setup_s: device time to build the sketch
    (the dense loop needs none: its K is never materialised); per_iter_s:
    device loop time / iterations (fixed iteration counts, delta = -1)."""
    rows = []
    prev = ctx.get_option(L.OPT_OTF_FP32)
    ctx.set_option(L.OPT_OTF_FP32, 1)
    try:
        for n in sizes:
            x, a, b = generate_scenario("C1", int(n), d, seed)
            kern = Coords(x, x, "sqeuclid", 0.0, scale=1.0, eps=cfg.epsilon)
            dcfg = SolverConfig(cfg.epsilon, math.inf, -1.0, iters_per_point)
            r = ctx.sinkhorn(kern, a, b, dcfg)
            rows.append({"method": "sinkhorn", "n": int(n), "setup_s": 0.0,
                         "per_iter_s": r.report["t_loop_s"] / max(r.report["iterations"], 1),
                         "iters_timed": int(r.report["iterations"])})
            s = min(s_multiplier * s0_budget(int(n)), float(n) * float(n) * 0.999)
            t0 = time.perf_counter()
            sk = ctx.sketch(kern, a, b, "ot", math.inf, cfg.epsilon, s, seed)  # synchronous: returns when built
            setup = time.perf_counter() - t0
            scfg = SolverConfig(cfg.epsilon, math.inf, -1.0, iters_per_point * 50)  # O(s) iterations: average more
            res = sk.solve(scfg, want_scalings=False)
            rows.append({"method": "spar-sink", "n": int(n), "setup_s": setup,
                         "per_iter_s": res.report["t_loop_s"] / max(res.report["iterations"], 1),
                         "iters_timed": int(res.report["iterations"]), "nnz": sk.nnz})
            sk.free()
    finally:
        ctx.set_option(L.OPT_OTF_FP32, prev)
    return rows
