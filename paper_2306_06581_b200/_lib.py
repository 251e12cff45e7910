"""ctypes binding of the C ABI (include/spk.h) -- the same stub a Python
caller of the drop-in boundary would write.

Loading is strict: if libspk_b200.so is missing or cannot be loaded the
import fails loudly; there is no CPU fallback anywhere in this package.
"""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

import numpy as np

PKG = Path(__file__).resolve().parent
LIB_PATH = Path(os.environ.get("SPK_LIB_PATH", str(PKG / "libspk_b200.so")))  # override: variant builds (profiling)

# ---- enums (spk.h) ------------------------------------------------------------
SPK_OK = 0
COST_SQEUCLID, COST_EUCLID, COST_WFR = 0, 1, 2
PLAN_OT, PLAN_UOT, PLAN_BARYCENTER, PLAN_UNIFORM = 0, 1, 2, 3
POLICY_ERROR, POLICY_MASK = 0, 1
PROBS_IMPORTANCE, PROBS_UNIFORM = 0, 1
VALUES_F64, VALUES_F32 = 0, 1
OPT_DETERMINISTIC, OPT_LOOP_BLOCKS_PER_SM, OPT_OTF_FP32, OPT_BLOCKED_LOOP, OPT_BLOCKED_MAX_W = 1, 2, 3, 4, 5
OPT_TWO_PASS_SAMPLER = 6
OPT_BLOCKED_SPLIT = 7
OPT_BLOCKED_SPREAD = 8
OPT_BLOCKED_CLUSTER = 9
OPT_BATCH_CLUSTER = 10
OPT_BATCH_UNROLL = 11
OPT_SMALL_LOOP = 12
OPT_SMALL_CLUSTER = 13
OPT_SMALL_MAX_NNZ = 14
OPT_ROW_LANES = 15

ERROR_CLASSES = {
    1: "Error", 2: "NegativeWeight", 3: "LengthMismatch", 4: "NotNormalized", 5: "AllBlack",
    6: "EmptyOutput", 7: "DimensionMismatch", 8: "NonPositiveEta", 9: "NonPositiveEpsilon",
    10: "DegenerateSupport", 11: "AllZeroKernel", 12: "ThetaOutOfRange", 13: "BudgetTooLarge",
    14: "EmptyWindow", 15: "InfiniteCostOnSupport", 16: "IoError", 17: "ZeroDenominator",
    18: "BaselineFailed", 19: "DegenerateSketchError", 20: "DeviceError",
}

DP = C.POINTER(C.c_double)
I64P = C.POINTER(C.c_int64)
U32P = C.POINTER(C.c_uint32)


class KernelDesc(C.Structure):
    _fields_ = [("n", C.c_int64), ("K", DP), ("nnz_ratio", C.c_double), ("C", DP), ("x", DP), ("y", DP),
                ("dim", C.c_int32), ("cost_kind", C.c_int32), ("eta", C.c_double), ("cost_scale", C.c_double),
                ("kernel_epsilon", C.c_double)]


class SolverCfg(C.Structure):
    _fields_ = [("epsilon", C.c_double), ("lambda_", C.c_double), ("delta", C.c_double), ("max_iter", C.c_int64),
                ("stabilize", C.c_int32), ("empty_policy", C.c_int32)]


class SketchOpts(C.Structure):
    _fields_ = [("theta", C.c_double), ("probs", C.c_int32), ("strict", C.c_int32), ("value_type", C.c_int32),
                ("reserved", C.c_int32)]


class Report(C.Structure):
    _fields_ = [("objective", C.c_double), ("iterations", C.c_int64), ("residual_row", C.c_double),
                ("residual_col", C.c_double), ("wall_time_s", C.c_double), ("sketch_nnz", C.c_int64),
                ("converged", C.c_int32), ("diverged", C.c_int32), ("seed", C.c_uint64),
                ("kernel_mean", C.c_double), ("masked_rows", C.c_int64), ("masked_cols", C.c_int64),
                ("log_domain", C.c_int32), ("factorized_plan", C.c_int32), ("kernel_nnz", C.c_int64),
                ("t_plan_s", C.c_double), ("t_sample_s", C.c_double), ("t_loop_s", C.c_double),
                ("t_readout_s", C.c_double)]

    def as_dict(self) -> dict:
        return {name: getattr(self, name) for name, _ in self._fields_}


# every symbol include/spk.h declares: name -> (restype, argtypes)
SIGNATURES = {
    "spk_ctx_create": (C.c_int, [C.c_int, C.POINTER(C.c_void_p)]),
    "spk_ctx_destroy": (None, [C.c_void_p]),
    "spk_ctx_set_stream": (C.c_int, [C.c_void_p, C.c_void_p]),
    "spk_ctx_stream": (C.c_void_p, [C.c_void_p]),
    "spk_ctx_set_option": (C.c_int, [C.c_void_p, C.c_int, C.c_int64]),
    "spk_ctx_get_option": (C.c_int, [C.c_void_p, C.c_int, C.POINTER(C.c_int64)]),
    "spk_last_error": (C.c_int, [C.c_void_p, C.POINTER(C.c_int), C.POINTER(C.c_int), C.c_char_p, C.c_size_t]),
    "spk_ctx_launch_count": (C.c_int64, [C.c_void_p]),
    "spk_spar_sink": (C.c_int, [C.c_void_p, C.POINTER(KernelDesc), DP, DP, C.POINTER(SolverCfg), C.c_double,
                                C.c_uint64, C.POINTER(SketchOpts), C.c_int, DP, DP, DP, DP, C.POINTER(Report)]),
    "spk_sinkhorn": (C.c_int, [C.c_void_p, C.POINTER(KernelDesc), DP, DP, C.POINTER(SolverCfg), C.c_int, DP, DP,
                               DP, DP, C.POINTER(Report)]),
    "spk_sketch_build": (C.c_int, [C.c_void_p, C.POINTER(KernelDesc), DP, DP, C.c_int, C.c_double, C.c_double,
                                   C.c_double, C.c_uint64, C.POINTER(SketchOpts), C.POINTER(C.c_void_p)]),
    "spk_sketch_build_batch": (C.c_int, [C.c_void_p, C.POINTER(KernelDesc), C.c_int, DP, DP, C.c_int, C.c_double,
                                         C.c_double, C.c_double, C.POINTER(C.c_uint64), C.POINTER(SketchOpts),
                                         C.POINTER(C.c_void_p)]),
    "spk_sketch_from_csr": (C.c_int, [C.c_void_p, C.c_int64, I64P, U32P, DP, C.c_int, C.POINTER(C.c_void_p)]),
    "spk_sketch_free": (None, [C.c_void_p]),
    "spk_sketch_info": (C.c_int, [C.c_void_p, I64P, I64P, I64P, C.POINTER(C.c_int32), DP]),
    "spk_sketch_plan": (C.c_int, [C.c_void_p, C.POINTER(C.c_int32), C.POINTER(C.c_int32), DP, DP, DP]),
    "spk_sketch_copy_csr": (C.c_int, [C.c_void_p, I64P, U32P, DP]),
    "spk_sketch_copy_csc": (C.c_int, [C.c_void_p, I64P, U32P, DP]),
    "spk_sketch_spmv": (C.c_int, [C.c_void_p, DP, DP, C.c_int]),
    "spk_sketch_solve": (C.c_int, [C.c_void_p, C.c_void_p, DP, DP, C.POINTER(SolverCfg), C.c_int, DP, DP, DP, DP,
                                   C.POINTER(Report)]),
    "spk_sketch_solve_batch": (C.c_int, [C.c_void_p, C.POINTER(C.c_void_p), C.c_int, C.POINTER(SolverCfg), C.c_int,
                                         C.POINTER(Report), C.POINTER(C.c_int32)]),
    "spk_sketch_scalings": (C.c_int, [C.c_void_p, DP, DP, DP, DP]),
    "spk_sketch_readout": (C.c_int, [C.c_void_p, C.c_void_p, C.POINTER(KernelDesc), C.c_int, C.c_double,
                                     C.c_double, DP, DP, DP, C.POINTER(Report)]),
    "spk_plan_readout": (C.c_int, [C.c_void_p, C.POINTER(KernelDesc), C.c_int64, I64P, U32P, DP, DP, DP, DP, DP,
                                   C.c_int, DP, DP, C.c_int, C.c_double, C.c_double, DP, DP, DP, DP, DP]),
    "spk_plan_probs": (C.c_int, [C.c_void_p, C.POINTER(KernelDesc), DP, DP, C.c_int, C.c_double, C.c_double,
                                 C.c_double, C.c_int64, I64P, I64P, DP, C.POINTER(C.c_int32)]),
    "spk_kernel_from_cost": (C.c_int, [C.c_void_p, DP, C.c_int64, C.c_double, DP, I64P]),
    "spk_cost_kernel": (C.c_int, [C.c_void_p, C.POINTER(KernelDesc), C.c_int64, I64P, I64P, DP, DP, DP]),
    # row/column-sharded solve (device pointers travel as c_void_p)
    "spk_shard_plan_rows": (C.c_int, [C.c_void_p, C.POINTER(KernelDesc), DP, DP, C.c_int, C.c_double, C.c_double,
                                      C.c_int32, C.c_int32, C.c_void_p, C.c_void_p, C.POINTER(C.c_int32)]),
    "spk_shard_create": (C.c_int, [C.c_void_p, C.POINTER(KernelDesc), DP, DP, C.c_int, C.c_double, C.c_double,
                                   C.c_double, C.c_uint64, C.POINTER(SketchOpts), C.c_int32, C.c_int32, C.c_void_p,
                                   C.c_void_p, C.POINTER(C.c_void_p)]),
    "spk_shard_free": (None, [C.c_void_p]),
    "spk_shard_info": (C.c_int, [C.c_void_p, I64P, I64P, I64P, I64P, I64P, I64P, I64P, C.POINTER(C.c_int32), DP, I64P,
                                 C.POINTER(C.c_int32)]),
    "spk_shard_export": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, I64P]),
    "spk_shard_import": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int64]),
    "spk_shard_coverage": (C.c_int, [C.c_void_p, I64P, I64P]),
    # communicators + the library's sharded driver
    "spk_comm_unique_id": (C.c_int, [C.c_char_p]),
    "spk_comm_init": (C.c_int, [C.c_void_p, C.c_char_p, C.c_int, C.c_int, C.POINTER(C.c_void_p)]),
    "spk_comm_init_all": (C.c_int, [C.POINTER(C.c_int), C.c_int, C.POINTER(C.c_void_p), C.POINTER(C.c_void_p)]),
    "spk_comm_group_create": (C.c_int, [C.c_int, C.POINTER(C.c_void_p)]),
    "spk_comm_group_destroy": (None, [C.c_void_p]),
    "spk_comm_init_emulated": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int, C.POINTER(C.c_void_p)]),
    "spk_comm_destroy": (None, [C.c_void_p]),
    "spk_comm_info": (C.c_int, [C.c_void_p, C.POINTER(C.c_int), C.POINTER(C.c_int), C.POINTER(C.c_int)]),
    "spk_sharded_build": (C.c_int, [C.c_void_p, C.POINTER(KernelDesc), DP, DP, C.c_int, C.c_double, C.c_double,
                                    C.c_double, C.c_uint64, C.POINTER(SketchOpts), C.POINTER(C.c_void_p)]),
    "spk_sharded_solve": (C.c_int, [C.c_void_p, C.POINTER(SolverCfg), C.c_int, DP, DP, DP, DP, C.POINTER(Report)]),
    "spk_sharded_info": (C.c_int, [C.c_void_p, I64P, I64P, I64P, I64P, I64P, I64P]),
    "spk_sharded_free": (None, [C.c_void_p]),
    "spk_spar_sink_sharded": (C.c_int, [C.c_void_p, C.POINTER(KernelDesc), DP, DP, C.POINTER(SolverCfg), C.c_double,
                                        C.c_uint64, C.POINTER(SketchOpts), C.c_int, DP, DP, DP, DP,
                                        C.POINTER(Report)]),
    "spk_spar_sink_multi": (C.c_int, [C.POINTER(C.c_int), C.c_int, C.POINTER(KernelDesc), DP, DP,
                                      C.POINTER(SolverCfg), C.c_double, C.c_uint64, C.POINTER(SketchOpts), C.c_int,
                                      DP, DP, DP, DP, C.POINTER(Report)]),
    "spk_shard_begin": (C.c_int, [C.c_void_p, C.POINTER(SolverCfg), C.c_int, C.c_int, C.c_int64, C.c_int64, C.c_void_p,
                                  C.c_void_p]),
    "spk_shard_half": (C.c_int, [C.c_void_p, C.c_int, C.c_int64, C.c_void_p, C.c_void_p, C.c_void_p]),
    "spk_shard_finish": (C.c_int, [C.c_void_p, C.c_int64, C.c_void_p]),
    "spk_shard_status": (C.c_int, [C.c_void_p, C.POINTER(Report), C.POINTER(C.c_int32), C.POINTER(C.c_int32)]),
    "spk_shard_readout": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int, C.c_int, C.c_int, DP]),
}
SHARD_TAIL = 8  # SPK_SHARD_TAIL


class IbpReport(C.Structure):
    _fields_ = [("iterations", C.c_int64), ("converged", C.c_int32), ("diverged", C.c_int32),
                ("masked_atoms", C.c_int64), ("wall_time_s", C.c_double)]

    def as_dict(self) -> dict:
        return {k: getattr(self, k) for k, _ in self._fields_}


SIGNATURES["spk_ibp"] = (C.c_int, [C.c_void_p, C.POINTER(C.c_void_p), C.c_int32, DP, DP, C.c_double, C.c_int64,
                                   C.c_int32, DP, C.POINTER(IbpReport)])
SIGNATURES["spk_spar_ibp"] = (C.c_int, [C.c_void_p, C.POINTER(KernelDesc), C.c_int32, DP, DP, C.c_double, C.c_int64,
                                        C.c_double, C.c_uint64, C.c_int32, C.c_int32, DP, C.POINTER(IbpReport)])

_lib = None


def load() -> C.CDLL:
    """Load libspk_b200.so (raises if absent -- the product has no fallback)."""
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            raise ImportError(f"{LIB_PATH} is missing: run `python -c 'import __graft_entry__ as g; g.build()'`")
        lib = C.CDLL(str(LIB_PATH))
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
    return _lib


def dptr(a: np.ndarray | None):
    if a is None:
        return None
    assert a.dtype == np.float64 and a.flags.c_contiguous
    return a.ctypes.data_as(DP)


def i64ptr(a: np.ndarray | None):
    if a is None:
        return None
    assert a.dtype == np.int64 and a.flags.c_contiguous
    return a.ctypes.data_as(I64P)


def u32ptr(a: np.ndarray | None):
    if a is None:
        return None
    assert a.dtype == np.uint32 and a.flags.c_contiguous
    return a.ctypes.data_as(U32P)
