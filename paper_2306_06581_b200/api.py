"""Python host mirror of the reference's Spar-Sink interface over the C ABI.

Names and argument meanings follow proj/include/sparsink/solvers.hpp and
sparsify.hpp (SolverConfig, SparSinkOptions, spar_sink_ot/uot, sinkhorn_ot/uot,
poisson_sparsify, spmv/spmv_t, ot_objective/uot_objective); errors are raised
as exceptions named after the reference's classes (errors.hpp:30-47) carrying
the same category codes.
"""
from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass, field

import numpy as np

from . import _lib as L


# ---- exceptions (errors.hpp) ----------------------------------------------------
class SparsinkError(RuntimeError):
    """Base: sparsink::Error with an ErrorCategory (4 input, 3 degenerate, 2 solver; 5 device)."""

    category = 4
    kind = 1


ERRORS: dict[str, type] = {"Error": SparsinkError}
for _kind, _name in L.ERROR_CLASSES.items():
    if _name != "Error":
        ERRORS[_name] = type(_name, (SparsinkError,), {"kind": _kind})
globals().update({k: v for k, v in ERRORS.items() if k != "Error"})


def _raise(ctx_ptr, rc: int) -> None:
    if rc == L.SPK_OK:
        return
    lib = L.load()
    cat, kind = C.c_int(0), C.c_int(0)
    buf = C.create_string_buffer(1024)
    lib.spk_last_error(ctx_ptr, C.byref(cat), C.byref(kind), buf, len(buf))
    cls = ERRORS.get(L.ERROR_CLASSES.get(kind.value, "Error"), SparsinkError)
    err = cls(buf.value.decode(errors="replace"))
    err.category = cat.value or rc
    err.kind = kind.value
    raise err


# ---- configuration (solvers.hpp:20-26, 151-157) -----------------------------------
@dataclass
class SolverConfig:
    epsilon: float = 1.0
    lambda_: float = math.inf  # inf = balanced
    delta: float = 1e-6
    max_iter: int = 1000
    stabilize: bool = False

    def c(self, policy: int) -> L.SolverCfg:
        return L.SolverCfg(self.epsilon, self.lambda_, self.delta, int(self.max_iter), int(self.stabilize), policy)


@dataclass
class SparSinkOptions:
    theta: float = 0.0
    probs: str = "importance"  # or "uniform" (Rand-Sink)
    strict: bool = False
    values: str = "f64"        # sketch value storage: "f64" or "f32"

    def c(self) -> L.SketchOpts:
        return L.SketchOpts(self.theta, L.PROBS_UNIFORM if self.probs == "uniform" else L.PROBS_IMPORTANCE,
                            int(self.strict), L.VALUES_F32 if self.values == "f32" else L.VALUES_F64, 0)


# ---- kernel descriptions ------------------------------------------------------------
_COST = {"sqeuclid": L.COST_SQEUCLID, "euclid": L.COST_EUCLID, "wfr": L.COST_WFR}


@dataclass
class Coords:
    """Kernel from point coordinates: C = cost(x_i, y_j) / scale (scale=None:
    divide by the max finite cost c0), K = exp(-C/eps) (eps=None: the solver's)."""

    x: np.ndarray
    y: np.ndarray
    cost: str = "sqeuclid"
    eta: float = 0.0
    scale: float | None = None
    eps: float | None = None

    def desc(self) -> tuple[L.KernelDesc, tuple]:
        x = np.ascontiguousarray(self.x, dtype=np.float64)
        y = np.ascontiguousarray(self.y, dtype=np.float64)
        if x.ndim == 1:
            x = x[:, None]
        if y.ndim == 1:
            y = y[:, None]
        d = L.KernelDesc()
        d.n = x.shape[0]
        d.x, d.y = L.dptr(x), L.dptr(y)
        d.dim = x.shape[1] if x.shape[1] == y.shape[1] else -1
        d.cost_kind = _COST[self.cost]
        d.eta = self.eta
        d.cost_scale = 0.0 if self.scale is None else float(self.scale)
        d.kernel_epsilon = 0.0 if self.eps is None else float(self.eps)
        return d, (x, y)


@dataclass
class Dense:
    """KernelMatrix (+ optional CostMatrix) given densely (geometry.hpp:13-26)."""

    K: np.ndarray
    nnz_ratio: float | None = None
    C: np.ndarray | None = None

    def desc(self) -> tuple[L.KernelDesc, tuple]:
        K = np.ascontiguousarray(self.K, dtype=np.float64)
        Cm = None if self.C is None else np.ascontiguousarray(self.C, dtype=np.float64)
        d = L.KernelDesc()
        d.n = K.shape[0]
        d.K = L.dptr(K)
        d.nnz_ratio = float(np.count_nonzero(K > 0) / K.size) if self.nnz_ratio is None else float(self.nnz_ratio)
        d.C = L.dptr(Cm)
        return d, (K, Cm)


@dataclass
class Result:
    u: np.ndarray
    v: np.ndarray
    log_u: np.ndarray | None
    log_v: np.ndarray | None
    report: dict = field(default_factory=dict)


def _vec(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float64)


class Context:
    """One device context (spk_ctx): stream, options, scratch."""

    def __init__(self, device: int = 0, deterministic: bool = False):
        self.lib = L.load()
        p = C.c_void_p()
        rc = self.lib.spk_ctx_create(device, C.byref(p))
        if rc != 0:
            raise ERRORS["DeviceError"](f"spk_ctx_create(device={device}) failed with status {rc}")
        self.ptr = p
        if deterministic:
            self.set_option(L.OPT_DETERMINISTIC, 1)

    def close(self) -> None:
        if getattr(self, "ptr", None):
            self.lib.spk_ctx_destroy(self.ptr)
            self.ptr = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    def set_option(self, key: int, value: int) -> None:
        _raise(self.ptr, self.lib.spk_ctx_set_option(self.ptr, key, int(value)))

    def get_option(self, key: int) -> int:
        v = C.c_int64()
        _raise(self.ptr, self.lib.spk_ctx_get_option(self.ptr, key, C.byref(v)))
        return v.value

    def set_stream(self, stream_ptr: int | None) -> None:
        _raise(self.ptr, self.lib.spk_ctx_set_stream(self.ptr, C.c_void_p(stream_ptr) if stream_ptr else None))

    @property
    def launches(self) -> int:
        return int(self.lib.spk_ctx_launch_count(self.ptr))

    # -- solvers ------------------------------------------------------------------
    def spar_sink(self, kernel, a, b, cfg: SolverConfig, s: float, seed: int, opts: SparSinkOptions | None = None,
                  uot: bool = False) -> Result:
        """spar_sink_ot / spar_sink_uot (solvers.hpp:159-167)."""
        a, b = _vec(a), _vec(b)
        kd, keep = kernel.desc()
        n = kd.n
        u, v, lu, lv = (np.empty(n) for _ in range(4))
        rep = L.Report()
        o = (opts or SparSinkOptions()).c()
        c = cfg.c(L.POLICY_MASK)
        rc = self.lib.spk_spar_sink(self.ptr, C.byref(kd), L.dptr(a), L.dptr(b), C.byref(c), float(s),
                                    C.c_uint64(seed & 0xFFFFFFFFFFFFFFFF), C.byref(o), int(uot), L.dptr(u),
                                    L.dptr(v), L.dptr(lu), L.dptr(lv), C.byref(rep))
        _raise(self.ptr, rc)
        log = bool(rep.log_domain)
        return Result(u, v, lu if log else None, lv if log else None, rep.as_dict())

    def sinkhorn(self, kernel, a, b, cfg: SolverConfig, uot: bool = False, policy: str = "error") -> Result:
        """sinkhorn_ot / sinkhorn_uot on a dense or on-the-fly kernel (solvers.hpp:137-147)."""
        a, b = _vec(a), _vec(b)
        kd, keep = kernel.desc()
        n = kd.n
        u, v, lu, lv = (np.empty(n) for _ in range(4))
        rep = L.Report()
        c = cfg.c(L.POLICY_MASK if policy == "mask" else L.POLICY_ERROR)
        rc = self.lib.spk_sinkhorn(self.ptr, C.byref(kd), L.dptr(a), L.dptr(b), C.byref(c), int(uot), L.dptr(u),
                                   L.dptr(v), L.dptr(lu), L.dptr(lv), C.byref(rep))
        _raise(self.ptr, rc)
        log = bool(rep.log_domain)
        return Result(u, v, lu if log else None, lv if log else None, rep.as_dict())

    # -- sketches -------------------------------------------------------------------
    def sketch(self, kernel, a, b, plan: str, lambda_: float, epsilon: float, s: float, seed: int,
               opts: SparSinkOptions | None = None) -> "Sketch":
        """Plan + [theta] + poisson_sparsify on the device (sparsify.hpp:74-95)."""
        a, b = _vec(a), _vec(b)
        kd, keep = kernel.desc()
        kind = {"ot": L.PLAN_OT, "uot": L.PLAN_UOT, "uniform": L.PLAN_UNIFORM, "barycenter": L.PLAN_BARYCENTER}[plan]
        o = (opts or SparSinkOptions()).c()
        p = C.c_void_p()
        rc = self.lib.spk_sketch_build(self.ptr, C.byref(kd), L.dptr(a), L.dptr(b), kind, float(lambda_),
                                       float(epsilon), float(s), C.c_uint64(seed & 0xFFFFFFFFFFFFFFFF), C.byref(o),
                                       C.byref(p))
        _raise(self.ptr, rc)
        return Sketch(self, p)

    def sketch_batch(self, kernel, A, B, plan: str, lambda_: float, epsilon: float, s: float, seeds,
                     opts: SparSinkOptions | None = None) -> list["Sketch"]:
        """spk_sketch_build for many measure pairs on one kernel (rows of A, B:
        count x n), preparing the kernel once."""
        A = np.ascontiguousarray(A, dtype=np.float64)
        B = np.ascontiguousarray(B, dtype=np.float64)
        m = A.shape[0]
        kd, keep = kernel.desc()
        kind = {"ot": L.PLAN_OT, "uot": L.PLAN_UOT, "uniform": L.PLAN_UNIFORM, "barycenter": L.PLAN_BARYCENTER}[plan]
        o = (opts or SparSinkOptions()).c()
        sd = (C.c_uint64 * max(m, 1))(*[int(x) & 0xFFFFFFFFFFFFFFFF for x in seeds])
        out = (C.c_void_p * max(m, 1))()
        rc = self.lib.spk_sketch_build_batch(self.ptr, C.byref(kd), m, L.dptr(A), L.dptr(B), kind, float(lambda_),
                                             float(epsilon), float(s), sd, C.byref(o), out)
        _raise(self.ptr, rc)
        return [Sketch(self, C.c_void_p(out[k])) for k in range(m)]

    def sketch_from_csr(self, row_ptr, col_idx, values, values_type: str = "f64") -> "Sketch":
        rp = np.ascontiguousarray(row_ptr, dtype=np.int64)
        ci = np.ascontiguousarray(col_idx, dtype=np.uint32)
        vv = _vec(values)
        p = C.c_void_p()
        rc = self.lib.spk_sketch_from_csr(self.ptr, len(rp) - 1, L.i64ptr(rp), L.u32ptr(ci), L.dptr(vv),
                                          L.VALUES_F32 if values_type == "f32" else L.VALUES_F64, C.byref(p))
        _raise(self.ptr, rc)
        return Sketch(self, p)

    def plan_probs(self, kernel, a, b, plan: str, lambda_: float, epsilon: float, theta: float, qi, qj):
        """SamplingPlan::prob(i, j) for query pairs (sparsify.hpp:28-34)."""
        a, b = _vec(a), _vec(b)
        kd, keep = kernel.desc()
        kind = {"ot": L.PLAN_OT, "uot": L.PLAN_UOT, "uniform": L.PLAN_UNIFORM, "barycenter": L.PLAN_BARYCENTER}[plan]
        qi = np.ascontiguousarray(qi, dtype=np.int64)
        qj = np.ascontiguousarray(qj, dtype=np.int64)
        out = np.empty(len(qi))
        fac = C.c_int32(0)
        rc = self.lib.spk_plan_probs(self.ptr, C.byref(kd), L.dptr(a), L.dptr(b), kind, float(lambda_),
                                     float(epsilon), float(theta), len(qi), L.i64ptr(qi), L.i64ptr(qj), L.dptr(out),
                                     C.byref(fac))
        _raise(self.ptr, rc)
        return out, bool(fac.value)

    def cost_kernel(self, kernel: Coords, qi, qj):
        kd, keep = kernel.desc()
        qi = np.ascontiguousarray(qi, dtype=np.int64)
        qj = np.ascontiguousarray(qj, dtype=np.int64)
        cost, kern, c0 = np.empty(len(qi)), np.empty(len(qi)), C.c_double(0)
        rc = self.lib.spk_cost_kernel(self.ptr, C.byref(kd), len(qi), L.i64ptr(qi), L.i64ptr(qj), L.dptr(cost),
                                      L.dptr(kern), C.byref(c0))
        _raise(self.ptr, rc)
        return cost, kern, c0.value


class Sketch:
    """Device-resident sketch (CSR + CSC mirror); mirrors SparseKernel."""

    def __init__(self, ctx: Context, ptr):
        self.ctx, self.ptr, self.lib = ctx, ptr, ctx.lib
        n, nnz, knnz, fac, km = C.c_int64(), C.c_int64(), C.c_int64(), C.c_int32(), C.c_double()
        self.lib.spk_sketch_info(ptr, C.byref(n), C.byref(nnz), C.byref(knnz), C.byref(fac), C.byref(km))
        self.n, self.nnz, self.kernel_nnz = n.value, nnz.value, knnz.value
        self.factorized_plan, self.kernel_mean = bool(fac.value), km.value

    def free(self) -> None:
        if self.ptr:
            self.lib.spk_sketch_free(self.ptr)
            self.ptr = None

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass

    def plan(self) -> dict:
        """The sampling plan the sketch was drawn from (kind, factorized, 1/total, g_k, theta)."""
        kind, fac = C.c_int32(), C.c_int32()
        inv, gk, th = C.c_double(), C.c_double(), C.c_double()
        _raise(self.ctx.ptr, self.lib.spk_sketch_plan(self.ptr, C.byref(kind), C.byref(fac), C.byref(inv),
                                                      C.byref(gk), C.byref(th)))
        return {"kind": kind.value, "factorized": bool(fac.value), "inv": inv.value, "g_k": gk.value,
                "theta": th.value}

    def csr(self):
        rp = np.empty(self.n + 1, np.int64)
        ci = np.empty(max(self.nnz, 1), np.uint32)
        vv = np.empty(max(self.nnz, 1))
        _raise(self.ctx.ptr, self.lib.spk_sketch_copy_csr(self.ptr, L.i64ptr(rp), L.u32ptr(ci), L.dptr(vv)))
        return rp, ci[: self.nnz], vv[: self.nnz]

    def csc(self):
        cp = np.empty(self.n + 1, np.int64)
        ri = np.empty(max(self.nnz, 1), np.uint32)
        vv = np.empty(max(self.nnz, 1))
        _raise(self.ctx.ptr, self.lib.spk_sketch_copy_csc(self.ptr, L.i64ptr(cp), L.u32ptr(ri), L.dptr(vv)))
        return cp, ri[: self.nnz], vv[: self.nnz]

    def spmv(self, x, transpose: bool = False) -> np.ndarray:
        x = _vec(x)
        if len(x) != self.n:
            raise ERRORS["LengthMismatch"]("LengthMismatch: spmv vector length")
        y = np.empty(self.n)
        _raise(self.ctx.ptr, self.lib.spk_sketch_spmv(self.ptr, L.dptr(x), L.dptr(y), int(transpose)))
        return y

    def solve(self, cfg: SolverConfig, uot: bool = False, a=None, b=None, policy: str = "mask",
              want_scalings: bool = True) -> Result:
        """sinkhorn_ot / sinkhorn_uot on this sketch (SparseKernel instantiation)."""
        a = None if a is None else _vec(a)
        b = None if b is None else _vec(b)
        n = self.n
        u, v, lu, lv = ((np.empty(n) for _ in range(4)) if want_scalings else (None,) * 4)
        rep = L.Report()
        c = cfg.c(L.POLICY_MASK if policy == "mask" else L.POLICY_ERROR)
        rc = self.lib.spk_sketch_solve(self.ctx.ptr, self.ptr, L.dptr(a), L.dptr(b), C.byref(c), int(uot),
                                       L.dptr(u), L.dptr(v), L.dptr(lu), L.dptr(lv), C.byref(rep))
        _raise(self.ctx.ptr, rc)
        log = bool(rep.log_domain)
        return Result(u, v, lu if log else None, lv if log else None, rep.as_dict())

    def scalings(self):
        """(u, v, log_u, log_v) of the last solve (log_* None after a linear-domain solve)."""
        n = self.n
        u, v, lu, lv = (np.empty(n) for _ in range(4))
        _raise(self.ctx.ptr, self.lib.spk_sketch_scalings(self.ptr, L.dptr(u), L.dptr(v), L.dptr(lu), L.dptr(lv)))
        return u, v, lu, lv

    def readout(self, kernel=None, uot: bool = False, lambda_: float = math.inf, epsilon: float = 1.0,
                objective: bool = True):
        """Marginals + ot_objective / uot_objective of the last solve."""
        n = self.n
        rm, cm = np.empty(n), np.empty(n)
        obj = C.c_double(math.nan)
        rep = L.Report()
        if kernel is not None:
            kd, keep = kernel.desc()
            kdp = C.byref(kd)
        else:
            kdp = None
        rc = self.lib.spk_sketch_readout(self.ctx.ptr, self.ptr, kdp, int(uot), float(lambda_), float(epsilon),
                                         L.dptr(rm), L.dptr(cm), C.byref(obj) if objective else None, C.byref(rep))
        _raise(self.ctx.ptr, rc)
        return rm, cm, obj.value, rep.as_dict()


def solve_batch(ctx: Context, sketches, cfg: SolverConfig, uot: bool = False, policy: str = "mask",
                per_item: bool = False) -> list[dict]:
    """sinkhorn_ot / sinkhorn_uot on many independent sketches at once
    (spk_sketch_solve_batch: log-domain sketches that fit one CTA's shared
    memory run one CTA each, in a single launch). Scalings stay on the
    sketches (Sketch.readout / Sketch.scalings). Returns the per-sketch
    reports. per_item=False: the first failing item raises (its class);
    per_item=True: a failing item gets report["error"] = its exception class
    name and the others complete (pairwise_wfr, harness.cpp:395-401)."""
    m = len(sketches)
    ptrs = (C.c_void_p * max(m, 1))(*[sk.ptr for sk in sketches])
    reps = (L.Report * max(m, 1))()
    errs = (C.c_int32 * max(m, 1))()
    c = cfg.c(L.POLICY_MASK if policy == "mask" else L.POLICY_ERROR)
    _raise(ctx.ptr, ctx.lib.spk_sketch_solve_batch(ctx.ptr, ptrs, m, C.byref(c), int(uot), reps,
                                                   errs if per_item else None))
    out = []
    for k in range(m):
        d = reps[k].as_dict()
        d["error"] = L.ERROR_CLASSES.get(errs[k]) if errs[k] else None
        out.append(d)
    return out


_default: Context | None = None


def default_context() -> Context:
    global _default
    if _default is None:
        _default = Context(0)
    return _default


def spar_sink_ot(kernel, a, b, cfg: SolverConfig, s: float, seed: int, opts: SparSinkOptions | None = None,
                 ctx: Context | None = None) -> Result:
    return (ctx or default_context()).spar_sink(kernel, a, b, cfg, s, seed, opts, uot=False)


def spar_sink_uot(kernel, a, b, cfg: SolverConfig, s: float, seed: int, opts: SparSinkOptions | None = None,
                  ctx: Context | None = None) -> Result:
    return (ctx or default_context()).spar_sink(kernel, a, b, cfg, s, seed, opts, uot=True)


def sinkhorn_ot(kernel, a, b, cfg: SolverConfig, policy: str = "error", ctx: Context | None = None) -> Result:
    return (ctx or default_context()).sinkhorn(kernel, a, b, cfg, uot=False, policy=policy)


def sinkhorn_uot(kernel, a, b, cfg: SolverConfig, policy: str = "error", ctx: Context | None = None) -> Result:
    return (ctx or default_context()).sinkhorn(kernel, a, b, cfg, uot=True, policy=policy)


# ---- batched frame pairs (config 3) ----------------------------------------------
_M64 = 0xFFFFFFFFFFFFFFFF


def _splitmix64(x: int) -> int:
    x = (x + 0x9E3779B97F4A7C15) & _M64
    x = ((x ^ (x >> 30)) * 0xBF58476D1CE4E5B9) & _M64
    x = ((x ^ (x >> 27)) * 0x94D049BB133111EB) & _M64
    return x ^ (x >> 31)


def mix_seed(seed: int, stream: int) -> int:
    """rng.hpp:17-19: the per-stream seed (also the per-pair seed of pairwise_wfr)."""
    return _splitmix64((seed & _M64) ^ _splitmix64((stream + 0x632BE59BD9B4E019) & _M64))


def frame_pairs(frames: int) -> list[tuple[int, int]]:
    """All unordered pairs i < j in the reference's pairwise_wfr order (harness.cpp:387-393)."""
    return [(i, j) for i in range(frames) for j in range(i + 1, frames)]


def spar_sink_pairs(ctx: Context, coords, masses, cfg: SolverConfig, s: float, seed: int, eta: float,
                    opts: SparSinkOptions | None = None, pairs=None, rank: int = 0, world: int = 1,
                    scale: float = 1.0, batched: bool = True,
                    chunk: int = 512) -> list[tuple[int, tuple[int, int], dict]]:
    """Config 3's batch: spar_sink_uot with the WFR cost between frame pairs
    (pairwise_wfr, proj/src/harness.cpp:349-406). Pair k (in frame_pairs
    order) uses seed mix_seed(seed, k) as the reference does (:393). Pairs are
    independent: rank r of `world` takes pairs k = r, r + world, ... (no
    communication). batched (log domain): the rank's pairs are sketched, then
    solved together by spk_sketch_solve_batch (chunks of `chunk` pairs).
    Returns (k, pair, report) for this rank's pairs."""
    pairs = pairs if pairs is not None else frame_pairs(masses.shape[0])
    kern = Coords(coords, coords, "wfr", eta, scale=scale, eps=cfg.epsilon)
    mine = list(range(rank, len(pairs), world))
    if batched and cfg.stabilize and not (opts and opts.strict):
        # every sketch first, then ONE batched loop (a CTA per pair), then the
        # per-pair objectives: spar_sink_uot's steps (solvers.cpp:360-378)
        out = []
        for c0 in range(0, len(mine), chunk):
            ks = mine[c0:c0 + chunk]
            sks = ctx.sketch_batch(kern, masses[[pairs[k][0] for k in ks]], masses[[pairs[k][1] for k in ks]], "uot",
                                   cfg.lambda_, cfg.epsilon, s, [mix_seed(seed, k) for k in ks], opts)
            try:
                reps = solve_batch(ctx, sks, cfg, uot=True, policy="mask", per_item=True)
                for k, sk, rep in zip(ks, sks, reps):
                    rep = dict(rep)
                    if rep["error"] is None:
                        _, _, obj, rr = sk.readout(kern, uot=True, lambda_=cfg.lambda_, epsilon=cfg.epsilon)
                        rep["objective"] = obj
                    else:  # the reference records a failed pair as NaN (harness.cpp:395-401)
                        rep["objective"] = math.nan
                    rep["seed"] = mix_seed(seed, k)
                    out.append((k, pairs[k], rep))
            finally:
                for sk in sks:
                    sk.free()
        return out
    out = []
    for k in mine:
        i, j = pairs[k]
        try:
            r = ctx.spar_sink(kern, masses[i], masses[j], cfg, s, mix_seed(seed, k), opts, uot=True)
            rep = dict(r.report)
            rep["error"] = None
        except SparsinkError as e:
            if isinstance(e, ERRORS["DeviceError"]):
                raise
            rep = {"objective": math.nan, "error": type(e).__name__, "seed": mix_seed(seed, k)}
        out.append((k, (i, j), rep))
    return out


def failed_pairs(results) -> int:
    """Pairs whose solve failed (NaN objective), as pairwise_wfr's failed_pairs."""
    return sum(1 for _, _, rep in results if rep.get("error"))


# ---- barycenters (ibp / spar_ibp, include/sparsink/barycenter.hpp) ------------------
def ibp(ctx: Context, sketches, b, w, delta: float = 1e-6, max_iter: int = 1000, policy: str = "error"):
    """ibp<SparseKernel> (barycenter.hpp:48-206) on device sketches (Sketch
    objects of one dimension n); b: (m, n) measure weights, w: m weights.
    Returns (q, report)."""
    b = np.ascontiguousarray(b, dtype=np.float64)
    w = np.ascontiguousarray(w, dtype=np.float64)
    m = len(sketches)
    ptrs = (C.c_void_p * m)(*[sk.ptr for sk in sketches])
    q = np.empty(b.shape[1])
    rep = L.IbpReport()
    _raise(ctx.ptr, ctx.lib.spk_ibp(ctx.ptr, ptrs, m, L.dptr(b), L.dptr(w), float(delta), int(max_iter),
                                    L.POLICY_MASK if policy == "mask" else L.POLICY_ERROR, L.dptr(q),
                                    C.byref(rep)))
    return q, rep.as_dict()


def spar_ibp(ctx: Context, kernels, b, w, s: float, seed: int, delta: float = 1e-6, max_iter: int = 1000,
             strict: bool = False, values: str = "f64"):
    """spar_ibp (barycenter.cpp:8-40): one sketch per kernel (column-constant
    plan, seed mix_seed(seed, k)), then ibp. kernels: Dense or Coords (with
    eps) of one dimension n. Returns (q, report)."""
    b = np.ascontiguousarray(b, dtype=np.float64)
    w = np.ascontiguousarray(w, dtype=np.float64)
    m = len(kernels)
    descs = (L.KernelDesc * m)()
    keep = []
    for k, kern in enumerate(kernels):
        d, kk = kern.desc()
        descs[k] = d
        keep.append(kk)
    q = np.empty(b.shape[1])
    rep = L.IbpReport()
    _raise(ctx.ptr, ctx.lib.spk_spar_ibp(ctx.ptr, descs, m, L.dptr(b), L.dptr(w), float(delta), int(max_iter),
                                         float(s), C.c_uint64(seed & _M64), int(strict),
                                         L.VALUES_F32 if values == "f32" else L.VALUES_F64, L.dptr(q),
                                         C.byref(rep)))
    return q, rep.as_dict()
