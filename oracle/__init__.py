"""Test oracle (CHECKER ONLY -- never on the product path).

Two ctypes bindings:
  Oracle     oracle/_build/libspk_oracle.so -- our C restatement (spk_oracle.c)
  Reference  oracle/_ref/libsparsink_ref.so -- the unmodified reference sources
             compiled by oracle/Makefile (absent unless built where
             /root/reference exists; the built .so travels to the GPU box).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
reference legs import this package.
"""
from __future__ import annotations

import ctypes as C
import math
import subprocess
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
ORACLE_SO = HERE / "_build" / "libspk_oracle.so"
REF_SO = HERE / "_ref" / "libsparsink_ref.so"

DP = C.POINTER(C.c_double)
I64P = C.POINTER(C.c_int64)
U32P = C.POINTER(C.c_uint32)


def build(quiet: bool = True) -> None:
    """make -C oracle (restatement always; reference only if its sources exist)."""
    res = subprocess.run(["make", "-C", str(HERE)], capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError(res.stdout + res.stderr)
    if not quiet:
        print(res.stdout)


def _d(a):
    return None if a is None else np.ascontiguousarray(a, dtype=np.float64).ctypes.data_as(DP)


class OracleError(RuntimeError):
    def __init__(self, kind: int, msg: str):
        super().__init__(f"[kind {kind}] {msg}")
        self.kind = kind
        self.msg = msg


class spko_plan(C.Structure):
    _fields_ = [("kind", C.c_int), ("n", C.c_int64), ("factorized", C.c_int), ("theta", C.c_double),
                ("kernel_nnz", C.c_int64), ("grid", DP), ("row_w", DP), ("col_w", DP)]


class spko_csr(C.Structure):
    _fields_ = [("n", C.c_int64), ("nnz", C.c_int64), ("row_ptr", I64P), ("col_idx", U32P), ("values", DP)]


class spko_cfg(C.Structure):
    _fields_ = [("epsilon", C.c_double), ("lambda_", C.c_double), ("delta", C.c_double), ("max_iter", C.c_int64),
                ("stabilize", C.c_int)]


class spko_result(C.Structure):
    _fields_ = [("iterations", C.c_int64), ("converged", C.c_int), ("diverged", C.c_int), ("log_domain", C.c_int),
                ("masked_rows", C.c_int64), ("masked_cols", C.c_int64), ("residual_row", C.c_double),
                ("residual_col", C.c_double), ("kernel_mean", C.c_double)]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_}


class ref_result(C.Structure):
    _fields_ = [("iterations", C.c_int64), ("converged", C.c_int32), ("diverged", C.c_int32),
                ("log_domain", C.c_int32), ("pad", C.c_int32), ("masked_rows", C.c_int64),
                ("masked_cols", C.c_int64), ("residual_row", C.c_double), ("residual_col", C.c_double),
                ("kernel_mean", C.c_double), ("objective", C.c_double), ("wall_time_s", C.c_double),
                ("sketch_nnz", C.c_int64)]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_ if k != "pad"}


PLAN = {"ot": 0, "uot": 1, "barycenter": 2, "uniform": 3}
COST = {"sqeuclid": 0, "euclid": 1, "wfr": 2}


def _csr_from(c: spko_csr):
    n, nnz = c.n, c.nnz
    rp = np.ctypeslib.as_array(c.row_ptr, shape=(n + 1,)).copy()
    ci = np.ctypeslib.as_array(c.col_idx, shape=(max(nnz, 1),))[:nnz].copy()
    vv = np.ctypeslib.as_array(c.values, shape=(max(nnz, 1),))[:nnz].copy()
    return rp, ci, vv


class Oracle:
    """ctypes view of the C restatement."""

    def __init__(self):
        if not ORACLE_SO.exists():
            build()
        self.lib = C.CDLL(str(ORACLE_SO))
        L = self.lib
        L.spko_splitmix64.restype = C.c_uint64
        L.spko_splitmix64.argtypes = [C.c_uint64]
        L.spko_mix_seed.restype = C.c_uint64
        L.spko_mix_seed.argtypes = [C.c_uint64, C.c_uint64]
        L.spko_counter_draw.restype = C.c_double
        L.spko_counter_draw.argtypes = [C.c_uint64, C.c_uint64, C.c_uint64]
        L.spko_rng_doubles.argtypes = [C.c_uint64, C.c_uint64, C.c_int64, DP]
        L.spko_rng_normals.argtypes = [C.c_uint64, C.c_uint64, C.c_int64, DP]
        L.spko_new_measure.argtypes = [DP, C.c_int64, C.c_int, DP]
        L.spko_cost_entry.restype = C.c_double
        L.spko_cost_entry.argtypes = [DP, DP, C.c_int, C.c_int, C.c_double]
        L.spko_pairwise_cost.argtypes = [DP, C.c_int64, DP, C.c_int64, C.c_int, C.c_int, C.c_double, DP, DP]
        L.spko_kernel_from_cost.argtypes = [DP, C.c_int64, C.c_int64, C.c_double, DP, DP]
        L.spko_plan_free.argtypes = [C.POINTER(spko_plan)]
        L.spko_plan_prob.restype = C.c_double
        L.spko_plan_prob.argtypes = [C.POINTER(spko_plan), C.c_int64, C.c_int64]
        L.spko_ot_probabilities.argtypes = [DP, DP, C.c_int64, DP, C.c_double, C.POINTER(spko_plan)]
        L.spko_uot_probabilities.argtypes = [DP, DP, C.c_int64, DP, C.c_double, C.c_double, C.c_double,
                                             C.POINTER(spko_plan)]
        L.spko_uniform_probabilities.argtypes = [C.c_int64, DP, C.c_double, C.POINTER(spko_plan)]
        L.spko_shrink_with_uniform.argtypes = [C.POINTER(spko_plan), C.c_double]
        L.spko_csr_free.argtypes = [C.POINTER(spko_csr)]
        L.spko_poisson_sparsify.argtypes = [DP, C.c_int64, C.POINTER(spko_plan), C.c_double, C.c_uint64,
                                            C.POINTER(spko_csr)]
        L.spko_spmv.argtypes = [C.POINTER(spko_csr), DP, DP]
        L.spko_spmv_t.argtypes = [C.POINTER(spko_csr), DP, DP]
        L.spko_sample_rows_coords.argtypes = [DP, DP, C.c_int64, C.c_int, C.c_int, C.c_double, C.c_double,
                                              C.c_double, C.c_int, C.c_int, DP, DP, C.c_double, C.c_double,
                                              C.c_double, C.c_uint64, C.c_int64, C.c_int64, C.POINTER(spko_csr)]
        L.spko_sinkhorn.argtypes = [C.POINTER(spko_csr), DP, C.c_int64, DP, DP, C.c_double, C.c_double,
                                    C.POINTER(spko_cfg), C.c_int, C.c_int, DP, DP, DP, DP, C.POINTER(spko_result),
                                    C.c_char_p, C.c_size_t]
        L.spko_time_scaling_iters.restype = C.c_double
        L.spko_time_scaling_iters.argtypes = [C.POINTER(spko_csr), DP, DP, C.c_int64, DP, DP]
        L.spko_readout.argtypes = [C.POINTER(spko_csr), DP, C.c_int64, DP, DP, DP, DP, C.c_int, DP, DP, DP, C.c_int,
                                   C.c_int, C.c_double, C.c_double, DP, DP, C.c_int, C.c_double, C.c_double, DP, DP,
                                   DP, C.c_char_p, C.c_size_t]
        L.spko_kl_divergence.argtypes = [DP, DP, C.c_int64, DP]
        L.spko_spar_sink.argtypes = [DP, C.c_double, DP, C.c_int64, DP, DP, C.c_double, C.c_double,
                                     C.POINTER(spko_cfg), C.c_double, C.c_uint64, C.c_double, C.c_int, C.c_int,
                                     C.c_int, DP, DP, DP, DP, C.POINTER(spko_result), DP, I64P,
                                     C.POINTER(spko_csr), C.c_char_p, C.c_size_t]

    # -- rng ------------------------------------------------------------------------
    def splitmix64(self, x: int) -> int:
        return self.lib.spko_splitmix64(x)

    def mix_seed(self, seed: int, stream: int) -> int:
        return self.lib.spko_mix_seed(seed, stream)

    def rng_doubles(self, seed: int, stream: int, count: int) -> np.ndarray:
        out = np.empty(count)
        self.lib.spko_rng_doubles(seed, stream, count, out.ctypes.data_as(DP))
        return out

    def rng_normals(self, seed: int, stream: int, count: int) -> np.ndarray:
        out = np.empty(count)
        self.lib.spko_rng_normals(seed, stream, count, out.ctypes.data_as(DP))
        return out

    # -- geometry -------------------------------------------------------------------
    def pairwise_cost(self, x, y, kind="sqeuclid", eta=0.0):
        x = np.ascontiguousarray(x, dtype=np.float64)
        y = np.ascontiguousarray(y, dtype=np.float64)
        if x.ndim == 1:
            x, y = x[:, None], y[:, None]
        Cm = np.empty((x.shape[0], y.shape[0]))
        c0 = C.c_double()
        rc = self.lib.spko_pairwise_cost(x.ctypes.data_as(DP), x.shape[0], y.ctypes.data_as(DP), y.shape[0],
                                         x.shape[1], COST[kind], eta, Cm.ctypes.data_as(DP), C.byref(c0))
        if rc:
            raise OracleError(rc, "pairwise_cost")
        return Cm, c0.value

    def kernel_from_cost(self, Cm, eps):
        Cm = np.ascontiguousarray(Cm, dtype=np.float64)
        K = np.empty_like(Cm)
        r = C.c_double()
        rc = self.lib.spko_kernel_from_cost(Cm.ctypes.data_as(DP), Cm.shape[0], Cm.shape[1], eps,
                                            K.ctypes.data_as(DP), C.byref(r))
        if rc:
            raise OracleError(rc, "kernel_from_cost")
        return K, r.value

    # -- plans ----------------------------------------------------------------------
    def plan(self, kind, a, b, K, nnz_ratio, lambda_=math.inf, eps=1.0, theta=0.0) -> spko_plan:
        p = spko_plan()
        K = np.ascontiguousarray(K, dtype=np.float64)
        n = K.shape[0]
        if kind == "ot":
            rc = self.lib.spko_ot_probabilities(_d(a), _d(b), n, K.ctypes.data_as(DP), nnz_ratio, C.byref(p))
        elif kind == "uot":
            rc = self.lib.spko_uot_probabilities(_d(a), _d(b), n, K.ctypes.data_as(DP), nnz_ratio, lambda_, eps,
                                                 C.byref(p))
        else:
            rc = self.lib.spko_uniform_probabilities(n, K.ctypes.data_as(DP), nnz_ratio, C.byref(p))
        if rc:
            raise OracleError(rc, f"{kind}_probabilities")
        if theta > 0.0:
            rc = self.lib.spko_shrink_with_uniform(C.byref(p), theta)
            if rc:
                self.lib.spko_plan_free(C.byref(p))
                raise OracleError(rc, "shrink_with_uniform")
        return p

    def plan_probs(self, p: spko_plan) -> np.ndarray:
        n = p.n
        out = np.empty((n, n))
        for i in range(n):
            for j in range(n):
                out[i, j] = self.lib.spko_plan_prob(C.byref(p), i, j)
        return out

    def free_plan(self, p: spko_plan) -> None:
        self.lib.spko_plan_free(C.byref(p))

    # -- sampler ----------------------------------------------------------------------
    def poisson_sparsify(self, K, plan: spko_plan, s, seed):
        K = np.ascontiguousarray(K, dtype=np.float64)
        c = spko_csr()
        rc = self.lib.spko_poisson_sparsify(K.ctypes.data_as(DP), K.shape[0], C.byref(plan), s, seed, C.byref(c))
        if rc:
            raise OracleError(rc, "poisson_sparsify")
        out = _csr_from(c)
        self.lib.spko_csr_free(C.byref(c))
        return out

    def sample_rows_coords(self, x, y, cost_kind, eta, scale, eps, plan_kind, factorized, row_w, col_w, g_k, inv,
                           s, seed, r0, r1):
        x = np.ascontiguousarray(x, dtype=np.float64)
        y = np.ascontiguousarray(y, dtype=np.float64)
        c = spko_csr()
        rc = self.lib.spko_sample_rows_coords(x.ctypes.data_as(DP), y.ctypes.data_as(DP), x.shape[0], x.shape[1],
                                              COST[cost_kind], eta, scale, eps, PLAN[plan_kind], int(factorized),
                                              _d(row_w), _d(col_w), g_k, inv, s, seed, r0, r1, C.byref(c))
        if rc:
            raise OracleError(rc, "sample_rows_coords")
        out = _csr_from(c)
        self.lib.spko_csr_free(C.byref(c))
        return out

    @staticmethod
    def _csr_struct(rp, ci, vv):
        rp = np.ascontiguousarray(rp, dtype=np.int64)
        ci = np.ascontiguousarray(ci, dtype=np.uint32)
        vv = np.ascontiguousarray(vv, dtype=np.float64)
        c = spko_csr(len(rp) - 1, int(rp[-1]), rp.ctypes.data_as(I64P), ci.ctypes.data_as(U32P),
                     vv.ctypes.data_as(DP))
        return c, (rp, ci, vv)

    def spmv(self, csr, x, transpose=False):
        c, keep = self._csr_struct(*csr)
        x = np.ascontiguousarray(x, dtype=np.float64)
        y = np.empty(c.n)
        (self.lib.spko_spmv_t if transpose else self.lib.spko_spmv)(C.byref(c), x.ctypes.data_as(DP),
                                                                      y.ctypes.data_as(DP))
        return y

    # -- solvers --------------------------------------------------------------------
    def sinkhorn(self, a, b, eps, lambda_=math.inf, delta=1e-6, max_iter=1000, stabilize=False, policy="error",
                 uot=False, csr=None, K=None):
        a = np.ascontiguousarray(a, dtype=np.float64)
        b = np.ascontiguousarray(b, dtype=np.float64)
        n = len(a)
        cfg = spko_cfg(eps, lambda_, delta, max_iter, int(stabilize))
        u, v, lu, lv = (np.empty(n) for _ in range(4))
        res = spko_result()
        msg = C.create_string_buffer(512)
        if csr is not None:
            c, keep = self._csr_struct(*csr)
            cp, Kp = C.byref(c), None
        else:
            K = np.ascontiguousarray(K, dtype=np.float64)
            cp, Kp = None, K.ctypes.data_as(DP)
        rc = self.lib.spko_sinkhorn(cp, Kp, n, a.ctypes.data_as(DP), b.ctypes.data_as(DP), _seq(a), _seq(b),
                                    C.byref(cfg), 1 if policy == "mask" else 0, int(uot),
                                    u.ctypes.data_as(DP), v.ctypes.data_as(DP), lu.ctypes.data_as(DP),
                                    lv.ctypes.data_as(DP), C.byref(res), msg, len(msg))
        if rc:
            raise OracleError(rc, msg.value.decode())
        return u, v, (lu if res.log_domain else None), (lv if res.log_domain else None), res.as_dict()

    def time_scaling_iters(self, csr, a, b, iters):
        c, keep = self._csr_struct(*csr)
        n = c.n
        u, v = np.empty(n), np.empty(n)
        t = self.lib.spko_time_scaling_iters(C.byref(c), _d(a), _d(b), iters, u.ctypes.data_as(DP),
                                             v.ctypes.data_as(DP))
        return t, u, v

    def readout(self, csr, u, v, a, b, eps, lambda_=math.inf, uot=False, lu=None, lv=None, Cm=None, coords=None):
        """Objective + marginals. coords = (x, y, kind, eta, scale) recomputes costs."""
        c, keep = self._csr_struct(*csr)
        n = c.n
        rm, cm = np.empty(n), np.empty(n)
        obj = C.c_double(math.nan)
        msg = C.create_string_buffer(512)
        x = y = None
        kind, eta, scale, dim = 0, 0.0, 1.0, 0
        if coords is not None:
            x, y, kindname, eta, scale = coords
            x = np.ascontiguousarray(x, dtype=np.float64)
            y = np.ascontiguousarray(y, dtype=np.float64)
            dim, kind = x.shape[1], COST[kindname]
        log = lu is not None
        rc = self.lib.spko_readout(C.byref(c), None, n, _d(u), _d(v), _d(lu), _d(lv), int(log), _d(Cm), _d(x), _d(y),
                                   dim, kind, eta, scale, _d(a), _d(b), int(uot), lambda_, eps,
                                   rm.ctypes.data_as(DP), cm.ctypes.data_as(DP), C.byref(obj), msg, len(msg))
        if rc:
            raise OracleError(rc, msg.value.decode())
        return rm, cm, obj.value

    def spar_sink(self, K, nnz_ratio, Cm, a, b, eps, s, seed, lambda_=math.inf, delta=1e-6, max_iter=1000,
                  stabilize=False, theta=0.0, probs="importance", strict=False, uot=False):
        K = np.ascontiguousarray(K, dtype=np.float64)
        Cm = np.ascontiguousarray(Cm, dtype=np.float64)
        a = np.ascontiguousarray(a, dtype=np.float64)
        b = np.ascontiguousarray(b, dtype=np.float64)
        n = len(a)
        cfg = spko_cfg(eps, lambda_, delta, max_iter, int(stabilize))
        u, v, lu, lv = (np.empty(n) for _ in range(4))
        res = spko_result()
        obj = C.c_double()
        nnz = C.c_int64()
        sk = spko_csr()
        msg = C.create_string_buffer(512)
        rc = self.lib.spko_spar_sink(K.ctypes.data_as(DP), nnz_ratio, Cm.ctypes.data_as(DP), n, a.ctypes.data_as(DP),
                                     b.ctypes.data_as(DP), _seq(a), _seq(b), C.byref(cfg), s, seed, theta,
                                     1 if probs == "uniform" else 0, int(strict), int(uot), u.ctypes.data_as(DP),
                                     v.ctypes.data_as(DP), lu.ctypes.data_as(DP), lv.ctypes.data_as(DP),
                                     C.byref(res), C.byref(obj), C.byref(nnz), C.byref(sk), msg, len(msg))
        if rc:
            raise OracleError(rc, msg.value.decode())
        csr = _csr_from(sk)
        self.lib.spko_csr_free(C.byref(sk))
        d = res.as_dict()
        d["objective"] = obj.value
        d["sketch_nnz"] = nnz.value
        return u, v, (lu if res.log_domain else None), (lv if res.log_domain else None), d, csr


def _seq(w) -> float:
    """Sequential total exactly as new_measure (measures.cpp:18-23)."""
    t = 0.0
    for x in np.asarray(w, dtype=np.float64).tolist():
        t += x
    return t


class ref_ibp_result(C.Structure):
    _fields_ = [("iterations", C.c_int64), ("converged", C.c_int32), ("diverged", C.c_int32),
                ("masked_atoms", C.c_int64)]


class Reference:
    """ctypes view of the compiled, unmodified reference (oracle/_ref)."""

    @staticmethod
    def available() -> bool:
        return REF_SO.exists()

    def __init__(self):
        if not REF_SO.exists():
            raise FileNotFoundError(f"{REF_SO} not built (needs /root/reference at build time)")
        self.lib = C.CDLL(str(REF_SO))
        L = self.lib
        L.ref_last_error.restype = C.c_char_p
        L.ref_last_error.argtypes = [C.POINTER(C.c_int)]
        L.ref_free.argtypes = [C.c_void_p]
        L.ref_mix_seed.restype = C.c_uint64
        L.ref_mix_seed.argtypes = [C.c_uint64, C.c_uint64]
        L.ref_rng_doubles.argtypes = [C.c_uint64, C.c_uint64, C.c_int64, DP]
        L.ref_rng_normals.argtypes = [C.c_uint64, C.c_uint64, C.c_int64, DP]
        L.ref_pairwise_cost.argtypes = [DP, C.c_int64, DP, C.c_int64, C.c_int, C.c_int, C.c_double, DP, DP]
        L.ref_kernel_from_cost.argtypes = [DP, C.c_int64, C.c_double, DP, DP]
        L.ref_plan_probs.argtypes = [C.c_int, DP, DP, C.c_int64, DP, C.c_double, C.c_double, C.c_double, C.c_double,
                                     DP, C.POINTER(C.c_int)]
        L.ref_poisson_sparsify.argtypes = [C.c_int, DP, DP, C.c_int64, DP, C.c_double, C.c_double, C.c_double,
                                           C.c_double, C.c_double, C.c_uint64, C.POINTER(I64P), C.POINTER(U32P),
                                           C.POINTER(DP), I64P]
        L.ref_spmv.argtypes = [C.c_int64, I64P, U32P, DP, DP, C.c_int, DP]
        L.ref_sinkhorn.argtypes = [C.c_int64, I64P, U32P, DP, DP, C.c_double, DP, DP, C.c_double, C.c_double,
                                   C.c_double, C.c_int64, C.c_int, C.c_int, C.c_int, DP, DP, DP, DP,
                                   C.POINTER(ref_result)]
        L.ref_spar_sink.argtypes = [C.c_int64, DP, C.c_double, DP, DP, DP, C.c_double, C.c_double, C.c_double,
                                    C.c_int64, C.c_int, C.c_double, C.c_uint64, C.c_double, C.c_int, C.c_int, C.c_int,
                                    DP, DP, DP, DP, C.POINTER(ref_result)]
        L.ref_readout.argtypes = [C.c_int64, I64P, U32P, DP, DP, DP, DP, DP, C.c_int, DP, DP, DP, C.c_int, C.c_double,
                                  C.c_double, DP, DP, DP]
        L.ref_time_scaling_iters.restype = C.c_double
        L.ref_time_scaling_iters.argtypes = [C.c_int64, I64P, U32P, DP, DP, DP, C.c_int64, DP, DP]
        L.ref_sparse_loop_timed.argtypes = [C.c_int64, I64P, U32P, DP, DP, DP, C.c_double, C.c_double, C.c_int64,
                                            C.c_int, DP, C.POINTER(ref_result)]
        L.ref_sparse_loop_timed_stab.argtypes = [C.c_int64, I64P, U32P, DP, DP, DP, C.c_double, C.c_double,
                                                 C.c_int64, C.c_int, C.c_int, DP, C.POINTER(ref_result)]
        L.ref_measure_from_image.argtypes = [DP, C.c_int64, C.c_int64, DP, DP]
        L.ref_mean_pool.argtypes = [DP, C.c_int64, C.c_int64, C.c_int64, C.c_int64, DP, I64P, I64P]
        L.ref_pairwise_wfr.argtypes = [DP, C.c_int64, C.c_int64, C.c_int64, C.c_double, C.c_double, C.c_double,
                                       C.c_double, C.c_uint64, C.c_int64, C.c_int, DP, I64P, I64P]
        L.ref_predict_ed.argtypes = [DP, C.c_int64, C.c_int64, C.c_int64, C.c_int64, C.c_int64, I64P, DP]
        L.ref_ibp.argtypes = [C.c_int32, C.c_int64, DP, DP, I64P, U32P, DP, I64P, DP, DP, C.c_double, C.c_int64,
                              C.c_int, DP, C.POINTER(ref_ibp_result)]
        L.ref_save_triplet_csv.argtypes = [C.c_int64, I64P, U32P, DP, C.c_char_p]
        L.ref_save_metadata_json.argtypes = [C.c_int64, I64P, C.c_uint64, C.c_double, C.c_double, C.c_int,
                                             C.c_char_p]
        L.ref_report_json.argtypes = [C.c_double, C.c_int64, C.c_double, C.c_double, C.c_double, C.c_int64, C.c_int,
                                      C.c_int, C.c_uint64, C.c_char_p, C.c_int64]
        L.ref_write_measure_csv.argtypes = [DP, DP, C.c_int64, C.c_int, C.c_char_p]
        L.ref_read_measure_csv.argtypes = [C.c_char_p, C.c_int, DP, DP, C.c_int64, I64P, C.POINTER(C.c_int)]
        L.ref_matrix_save.argtypes = [DP, C.c_int64, C.c_int64, C.c_char_p, C.c_char_p]
        L.ref_scenario.argtypes = [C.c_int, C.c_int64, C.c_int64, C.c_uint64, C.c_int, C.c_double, C.c_double,
                                   C.c_int, C.c_double, C.c_double, C.c_int, DP, DP, DP, DP]
        L.ref_rmae.argtypes = [C.c_int, C.c_int64, C.c_int64, C.c_uint64, C.c_int, C.c_double, C.c_double, C.c_int,
                               C.c_double, C.c_double, C.c_int, C.c_int, DP, C.c_int64, C.c_int64, C.c_double,
                               C.c_double, C.c_double, C.c_int64, DP, DP, I64P]
        L.ref_spar_ibp.argtypes = [C.c_int32, C.c_int64, DP, DP, DP, DP, C.c_double, C.c_int64, C.c_double,
                                   C.c_uint64, C.c_int, DP, C.POINTER(ref_ibp_result)]

    def _check(self, rc):
        if rc:
            cat = C.c_int()
            msg = self.lib.ref_last_error(C.byref(cat)).decode()
            raise OracleError(rc, msg)

    # -- frame-pair caller (measures.cpp:36-85, harness.cpp:349-437) ---------------
    def measure_from_image(self, px, h, w):
        px = np.ascontiguousarray(px, dtype=np.float64)
        coords, weights = np.empty(2 * h * w), np.empty(h * w)
        self._check(self.lib.ref_measure_from_image(px.ctypes.data_as(DP), h, w, coords.ctypes.data_as(DP),
                                                    weights.ctypes.data_as(DP)))
        return coords.reshape(h * w, 2), weights

    def mean_pool(self, px, h, w, filt, stride):
        px = np.ascontiguousarray(px, dtype=np.float64)
        out = np.empty(h * w)
        oh, ow = np.zeros(1, np.int64), np.zeros(1, np.int64)
        self._check(self.lib.ref_mean_pool(px.ctypes.data_as(DP), h, w, filt, stride, out.ctypes.data_as(DP),
                                           oh.ctypes.data_as(I64P), ow.ctypes.data_as(I64P)))
        return out[:int(oh[0]) * int(ow[0])].copy(), int(oh[0]), int(ow[0])

    def pairwise_wfr(self, frames, h, w, eta, lam, eps, s_mult, seed, stride=1, exact=False):
        fr = np.ascontiguousarray(frames, dtype=np.float64)
        nf = fr.shape[0]
        d = np.empty(nf * nf)
        m, failed = np.zeros(1, np.int64), np.zeros(1, np.int64)
        self._check(self.lib.ref_pairwise_wfr(fr.ctypes.data_as(DP), nf, h, w, eta, lam, eps, s_mult, seed, stride,
                                              int(exact), d.ctypes.data_as(DP), m.ctypes.data_as(I64P),
                                              failed.ctypes.data_as(I64P)))
        mm = int(m[0])
        return d[:mm * mm].reshape(mm, mm).copy(), int(failed[0])

    def ibp(self, b, w, delta=1e-6, max_iter=1000, policy="error", Ks=None, ratios=None, sketches=None):
        """ibp on m dense kernels (Ks, ratios) or m CSR sketches [(rp, ci, val), ...]."""
        b = np.ascontiguousarray(b, dtype=np.float64)
        w = np.ascontiguousarray(w, dtype=np.float64)
        m, n = b.shape
        q = np.empty(n)
        res = ref_ibp_result()
        pol = 1 if policy == "mask" else 0
        if sketches is not None:
            rp = np.ascontiguousarray(np.concatenate([s[0] for s in sketches]), dtype=np.int64)
            ci = np.ascontiguousarray(np.concatenate([s[1] for s in sketches]), dtype=np.uint32)
            val = np.ascontiguousarray(np.concatenate([s[2] for s in sketches]), dtype=np.float64)
            nnz = np.array([len(s[1]) for s in sketches], dtype=np.int64)
            self._check(self.lib.ref_ibp(m, n, None, None, rp.ctypes.data_as(I64P), ci.ctypes.data_as(U32P),
                                         val.ctypes.data_as(DP), nnz.ctypes.data_as(I64P), b.ctypes.data_as(DP),
                                         w.ctypes.data_as(DP), delta, max_iter, pol, q.ctypes.data_as(DP),
                                         C.byref(res)))
        else:
            K = np.ascontiguousarray(np.stack(Ks), dtype=np.float64)
            r = np.ascontiguousarray(ratios, dtype=np.float64)
            self._check(self.lib.ref_ibp(m, n, K.ctypes.data_as(DP), r.ctypes.data_as(DP), None, None, None, None,
                                         b.ctypes.data_as(DP), w.ctypes.data_as(DP), delta, max_iter, pol,
                                         q.ctypes.data_as(DP), C.byref(res)))
        return q, {k: getattr(res, k) for k, _ in res._fields_}

    def spar_ibp(self, Ks, ratios, b, w, s, seed, delta=1e-6, max_iter=1000, strict=False):
        b = np.ascontiguousarray(b, dtype=np.float64)
        w = np.ascontiguousarray(w, dtype=np.float64)
        m, n = b.shape
        K = np.ascontiguousarray(np.stack(Ks), dtype=np.float64)
        r = np.ascontiguousarray(ratios, dtype=np.float64)
        q = np.empty(n)
        res = ref_ibp_result()
        self._check(self.lib.ref_spar_ibp(m, n, K.ctypes.data_as(DP), r.ctypes.data_as(DP), b.ctypes.data_as(DP),
                                          w.ctypes.data_as(DP), delta, max_iter, s, seed, int(strict),
                                          q.ctypes.data_as(DP), C.byref(res)))
        return q, {k: getattr(res, k) for k, _ in res._fields_}

    # -- RMAE harness ----------------------------------------------------------------
    def _spec(self, spec):
        m = spec.get("masses")
        t = spec.get("sparsity_target")
        return ({"C1": 0, "C2": 1, "C3": 2}[spec.get("scenario", "C1")], spec.get("n", 1000), spec.get("d", 5),
                spec.get("seed", 1), int(m is not None), m[0] if m else 1.0, m[1] if m else 1.0, int(t is not None),
                t or 0.0, spec.get("scale_param", 0.05), int(spec.get("scale_is_sd", False)))

    def scenario(self, spec):
        sp = self._spec(spec)
        n, d = sp[1], sp[2]
        x, a, b, eta = np.empty(n * d), np.empty(n), np.empty(n), C.c_double()
        self._check(self.lib.ref_scenario(*sp, x.ctypes.data_as(DP), a.ctypes.data_as(DP), b.ctypes.data_as(DP),
                                          C.byref(eta)))
        return x.reshape(n, d), a, b, eta.value

    def rmae(self, spec, method, budgets, reps, eps, lam=math.inf, delta=1e-6, max_iter=1000):
        sp = self._spec(spec)
        bud = np.ascontiguousarray(budgets, dtype=np.float64)
        exact = C.c_double()
        errs = np.empty(len(bud) * reps)
        retr = np.zeros(len(bud), np.int64)
        self._check(self.lib.ref_rmae(*sp, 1 if method == "randsink" else 0, bud.ctypes.data_as(DP), len(bud), reps,
                                      eps, lam, delta, max_iter, C.byref(exact), errs.ctypes.data_as(DP),
                                      retr.ctypes.data_as(I64P)))
        return exact.value, errs.reshape(len(bud), reps), retr

    # -- formats ---------------------------------------------------------------------
    def save_triplet_csv(self, csr, path):
        rp, ci, vv = (np.ascontiguousarray(csr[0], dtype=np.int64), np.ascontiguousarray(csr[1], dtype=np.uint32),
                      np.ascontiguousarray(csr[2], dtype=np.float64))
        self._check(self.lib.ref_save_triplet_csv(len(rp) - 1, rp.ctypes.data_as(I64P), ci.ctypes.data_as(U32P),
                                                  vv.ctypes.data_as(DP), str(path).encode()))

    def save_metadata_json(self, row_ptr, seed, s, theta, kind, path):
        rp = np.ascontiguousarray(row_ptr, dtype=np.int64)
        self._check(self.lib.ref_save_metadata_json(len(rp) - 1, rp.ctypes.data_as(I64P), seed, s, theta,
                                                    {"ot": 0, "uot": 1, "barycenter": 2, "uniform": 3}[kind],
                                                    str(path).encode()))

    def report_json(self, objective, iterations, rr, rc, wall, sketch_nnz, converged, diverged, seed):
        buf = C.create_string_buffer(4096)
        self._check(self.lib.ref_report_json(objective, iterations, rr, rc, wall, sketch_nnz, int(converged),
                                             int(diverged), seed, buf, len(buf)))
        return buf.value.decode()

    def write_measure_csv(self, w, x, path):
        w = np.ascontiguousarray(w, dtype=np.float64)
        x = np.ascontiguousarray(x, dtype=np.float64)
        self._check(self.lib.ref_write_measure_csv(w.ctypes.data_as(DP), x.ctypes.data_as(DP), len(w),
                                                   x.size // len(w), str(path).encode()))

    def read_measure_csv(self, path, simplex=False, cap=1 << 20):
        w, x = np.empty(cap), np.empty(cap)
        n, dim = np.zeros(1, np.int64), C.c_int(0)
        self._check(self.lib.ref_read_measure_csv(str(path).encode(), int(simplex), w.ctypes.data_as(DP),
                                                  x.ctypes.data_as(DP), cap, n.ctypes.data_as(I64P), C.byref(dim)))
        nn, d = int(n[0]), dim.value
        return w[:nn].copy(), x[:nn * d].reshape(nn, d).copy()

    def matrix_save(self, a, bin_path=None, csv_path=None):
        a = np.ascontiguousarray(a, dtype=np.float64)
        self._check(self.lib.ref_matrix_save(a.ctypes.data_as(DP), a.shape[0], a.shape[1],
                                             str(bin_path).encode() if bin_path else None,
                                             str(csv_path).encode() if csv_path else None))

    def predict_ed(self, d, t_es, lo, hi, t_true):
        d = np.ascontiguousarray(d, dtype=np.float64)
        th, err = np.zeros(1, np.int64), np.zeros(1)
        self._check(self.lib.ref_predict_ed(d.ctypes.data_as(DP), d.shape[0], t_es, lo, hi, t_true,
                                            th.ctypes.data_as(I64P), err.ctypes.data_as(DP)))
        return int(th[0]), float(err[0])

    def rng_doubles(self, seed, stream, count):
        out = np.empty(count)
        self.lib.ref_rng_doubles(seed, stream, count, out.ctypes.data_as(DP))
        return out

    def rng_normals(self, seed, stream, count):
        out = np.empty(count)
        self.lib.ref_rng_normals(seed, stream, count, out.ctypes.data_as(DP))
        return out

    def pairwise_cost(self, x, y, kind="sqeuclid", eta=0.0):
        x = np.ascontiguousarray(x, dtype=np.float64)
        y = np.ascontiguousarray(y, dtype=np.float64)
        if x.ndim == 1:
            x, y = x[:, None], y[:, None]
        Cm = np.empty((x.shape[0], y.shape[0]))
        c0 = C.c_double()
        self._check(self.lib.ref_pairwise_cost(x.ctypes.data_as(DP), x.shape[0], y.ctypes.data_as(DP), y.shape[0],
                                               x.shape[1], COST[kind], eta, Cm.ctypes.data_as(DP), C.byref(c0)))
        return Cm, c0.value

    def kernel_from_cost(self, Cm, eps):
        Cm = np.ascontiguousarray(Cm, dtype=np.float64)
        K = np.empty_like(Cm)
        r = C.c_double()
        self._check(self.lib.ref_kernel_from_cost(Cm.ctypes.data_as(DP), Cm.shape[0], eps, K.ctypes.data_as(DP),
                                                  C.byref(r)))
        return K, r.value

    def plan_probs(self, kind, a, b, K, nnz_ratio, lambda_=math.inf, eps=1.0, theta=0.0):
        K = np.ascontiguousarray(K, dtype=np.float64)
        n = K.shape[0]
        out = np.empty((n, n))
        fac = C.c_int()
        self._check(self.lib.ref_plan_probs(PLAN[kind], _d(a), _d(b), n, K.ctypes.data_as(DP), nnz_ratio, lambda_,
                                            eps, theta, out.ctypes.data_as(DP), C.byref(fac)))
        return out, bool(fac.value)

    def poisson_sparsify(self, kind, a, b, K, nnz_ratio, s, seed, lambda_=math.inf, eps=1.0, theta=0.0):
        K = np.ascontiguousarray(K, dtype=np.float64)
        n = K.shape[0]
        rp, ci, vv, nnz = I64P(), U32P(), DP(), C.c_int64()
        self._check(self.lib.ref_poisson_sparsify(PLAN[kind], _d(a), _d(b), n, K.ctypes.data_as(DP), nnz_ratio,
                                                  lambda_, eps, theta, s, seed, C.byref(rp), C.byref(ci),
                                                  C.byref(vv), C.byref(nnz)))
        m = nnz.value
        out = (np.ctypeslib.as_array(rp, shape=(n + 1,)).copy(),
               np.ctypeslib.as_array(ci, shape=(m + 1,))[:m].copy(),
               np.ctypeslib.as_array(vv, shape=(m + 1,))[:m].copy())
        for p in (rp, ci, vv):
            self.lib.ref_free(C.cast(p, C.c_void_p))
        return out

    @staticmethod
    def _csr(csr):
        rp = np.ascontiguousarray(csr[0], dtype=np.int64)
        ci = np.ascontiguousarray(csr[1], dtype=np.uint32)
        vv = np.ascontiguousarray(csr[2], dtype=np.float64)
        return rp, ci, vv

    def spmv(self, csr, x, transpose=False):
        rp, ci, vv = self._csr(csr)
        n = len(rp) - 1
        y = np.empty(n)
        self._check(self.lib.ref_spmv(n, rp.ctypes.data_as(I64P), ci.ctypes.data_as(U32P), vv.ctypes.data_as(DP),
                                      _d(x), int(transpose), y.ctypes.data_as(DP)))
        return y

    def sinkhorn(self, a, b, eps, lambda_=math.inf, delta=1e-6, max_iter=1000, stabilize=False, policy="error",
                 uot=False, csr=None, K=None, nnz_ratio=1.0):
        n = len(a)
        u, v, lu, lv = (np.empty(n) for _ in range(4))
        res = ref_result()
        if csr is not None:
            rp, ci, vv = self._csr(csr)
            args = (rp.ctypes.data_as(I64P), ci.ctypes.data_as(U32P), vv.ctypes.data_as(DP), None)
        else:
            K = np.ascontiguousarray(K, dtype=np.float64)
            args = (None, None, None, K.ctypes.data_as(DP))
        self._check(self.lib.ref_sinkhorn(n, *args, nnz_ratio, _d(a), _d(b), eps, lambda_, delta, max_iter,
                                          int(stabilize), 1 if policy == "mask" else 0, int(uot),
                                          u.ctypes.data_as(DP), v.ctypes.data_as(DP), lu.ctypes.data_as(DP),
                                          lv.ctypes.data_as(DP), C.byref(res)))
        return u, v, (lu if res.log_domain else None), (lv if res.log_domain else None), res.as_dict()

    def spar_sink(self, K, nnz_ratio, Cm, a, b, eps, s, seed, lambda_=math.inf, delta=1e-6, max_iter=1000,
                  stabilize=False, theta=0.0, probs="importance", strict=False, uot=False):
        K = np.ascontiguousarray(K, dtype=np.float64)
        Cm = np.ascontiguousarray(Cm, dtype=np.float64)
        n = len(a)
        u, v, lu, lv = (np.empty(n) for _ in range(4))
        res = ref_result()
        self._check(self.lib.ref_spar_sink(n, K.ctypes.data_as(DP), nnz_ratio, Cm.ctypes.data_as(DP), _d(a), _d(b),
                                           eps, lambda_, delta, max_iter, int(stabilize), s, seed, theta,
                                           1 if probs == "uniform" else 0, int(strict), int(uot),
                                           u.ctypes.data_as(DP), v.ctypes.data_as(DP), lu.ctypes.data_as(DP),
                                           lv.ctypes.data_as(DP), C.byref(res)))
        return u, v, (lu if res.log_domain else None), (lv if res.log_domain else None), res.as_dict()

    def readout(self, csr, u, v, a, b, Cm, eps, lambda_=math.inf, uot=False, lu=None, lv=None):
        rp, ci, vv = self._csr(csr)
        n = len(rp) - 1
        rm, cm, obj = np.empty(n), np.empty(n), C.c_double()
        self._check(self.lib.ref_readout(n, rp.ctypes.data_as(I64P), ci.ctypes.data_as(U32P), vv.ctypes.data_as(DP),
                                         _d(u), _d(v), _d(lu), _d(lv), int(lu is not None), _d(Cm), _d(a), _d(b),
                                         int(uot), lambda_, eps, rm.ctypes.data_as(DP), cm.ctypes.data_as(DP),
                                         C.byref(obj)))
        return rm, cm, obj.value

    def sparse_loop_seconds(self, csr, a, b, eps, iters, lambda_=math.inf, uot=False, stabilize=False):
        """The reference's own sinkhorn_ot/uot<SparseKernel> for `iters` fixed iterations (delta=-1),
        linear or log domain (SolverConfig::stabilize)."""
        rp, ci, vv = self._csr(csr)
        n = len(rp) - 1
        secs = C.c_double()
        res = ref_result()
        self._check(self.lib.ref_sparse_loop_timed_stab(n, rp.ctypes.data_as(I64P), ci.ctypes.data_as(U32P),
                                                        vv.ctypes.data_as(DP), _d(a), _d(b), eps, lambda_, iters,
                                                        int(uot), int(stabilize), C.byref(secs), C.byref(res)))
        return secs.value, res.as_dict()
