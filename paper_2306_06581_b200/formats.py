"""Wire / disk formats of the Spar-Sink path, written
byte-for-byte like the reference so GPU sketches and reports can be diffed
against the CPU tools:

  sketch triplet CSV     SparseKernel::save_triplet_csv   sparsify.cpp:236-244
  sketch metadata JSON   SparseKernel::save_metadata_json sparsify.cpp:246-263
  SolveReport JSON       SolveReport::to_json             solvers.cpp:227-242
  measure CSV            read/write_measure_csv           measures.cpp:87-141
  SPKM matrix            Matrix::save_binary/load_binary  matrix.cpp:15-42, save_csv :44-55

Numbers follow the reference's streams: `precision(17)` (%.17g) for CSVs and
nlohmann::json's shortest round-trip doubles (Python repr) with keys sorted,
2-space indent, for JSON.
"""
from __future__ import annotations

import json
import math
import struct

import numpy as np

from .api import ERRORS

_KIND = {0: "ot", 1: "uot", 2: "barycenter", 3: "uniform", "ot": "ot", "uot": "uot", "barycenter": "barycenter",
         "uniform": "uniform"}


def _g17(v: float) -> str:
    """std::ostream << double with precision(17), default floatfield (%.17g)."""
    if math.isnan(v):
        return "nan" if math.copysign(1.0, v) > 0 else "-nan"
    if math.isinf(v):
        return "inf" if v > 0 else "-inf"
    return "%.17g" % v


def _io_error(msg: str):
    return ERRORS["IoError"]("IoError: " + msg)


def save_triplet_csv(path: str, row_ptr, col_idx, values) -> None:
    rp = np.asarray(row_ptr, dtype=np.int64)
    ci = np.asarray(col_idx)
    vv = np.asarray(values, dtype=np.float64)
    try:
        f = open(path, "w")
    except OSError:
        raise _io_error(f"cannot open {path} for writing")
    with f:
        f.write("row,col,value\n")
        for i in range(len(rp) - 1):
            for p in range(rp[i], rp[i + 1]):
                f.write(f"{i},{int(ci[p])},{_g17(float(vv[p]))}\n")


def _json(obj) -> str:
    """nlohmann::json::dump(2) of a flat object: sorted keys, shortest doubles."""
    def val(v):
        if v is None:
            return "null"
        if isinstance(v, bool):
            return "true" if v else "false"
        if isinstance(v, (int, np.integer)):
            return str(int(v))
        if isinstance(v, str):
            return json.dumps(v)
        v = float(v)
        if not math.isfinite(v):
            return "null"  # nlohmann writes NaN / inf as null
        r = repr(v)
        return r if ("." in r or "e" in r or "n" in r) else r + ".0"
    body = ",\n".join(f'  "{k}": {val(obj[k])}' for k in sorted(obj))
    return "{\n" + body + "\n}"


def save_metadata_json(path: str, seed: int, s: float, theta: float, kind, realized_nnz: int, n: int) -> None:
    doc = {"seed": int(seed), "s": float(s), "theta": float(theta), "kind": _KIND[kind],
           "realized_nnz": int(realized_nnz), "n": int(n)}
    try:
        f = open(path, "w")
    except OSError:
        raise _io_error(f"cannot open {path} for writing")
    with f:
        f.write(_json(doc) + "\n")


def report_json(report: dict) -> str:
    """SolveReport::to_json (sketch_nnz null for dense solves)."""
    nnz = report.get("sketch_nnz", -1)
    doc = {"objective": report["objective"], "iterations": int(report["iterations"]),
           "residual_row": report["residual_row"], "residual_col": report["residual_col"],
           "wall_time_s": report["wall_time_s"], "sketch_nnz": None if nnz is None or nnz < 0 else int(nnz),
           "converged": bool(report["converged"]), "diverged": bool(report["diverged"]),
           "seed": int(report.get("seed", 0))}
    return _json(doc)


def write_measure_csv(path: str, weights, coords) -> None:
    w = np.asarray(weights, dtype=np.float64)
    x = np.asarray(coords, dtype=np.float64).reshape(len(w), -1)
    try:
        f = open(path, "w")
    except OSError:
        raise _io_error(f"cannot open {path} for writing")
    with f:
        f.write("weight" + "".join(f",x{k}" for k in range(1, x.shape[1] + 1)) + "\n")
        for i in range(len(w)):
            f.write(_g17(float(w[i])) + "".join("," + _g17(float(v)) for v in x[i]) + "\n")


def read_measure_csv(path: str, require_simplex: bool = False):
    """-> (weights, coords (n, d)); the reference's IoError cases, then
    new_measure's checks (measures.cpp:12-34)."""
    try:
        f = open(path)
    except OSError:
        raise _io_error(f"cannot open {path}")
    with f:
        lines = f.read().split("\n")
    if not lines or (len(lines) == 1 and lines[0] == ""):
        raise _io_error(f"empty file: {path}")
    head = lines[0].split(",")
    if head[0] != "weight":
        raise _io_error("expected 'weight' header column")
    dim = len(head) - 1
    if dim == 0:
        raise _io_error("measure CSV needs at least one coordinate")
    w, x = [], []
    for line in lines[1:]:
        if not line:
            continue
        tok = line.split(",")
        w.append(float(tok[0]))
        if len(tok) < dim + 1:
            raise _io_error(f"short row in {path}")
        x.extend(float(t) for t in tok[1:dim + 1])
    # new_measure (measures.cpp:12-34)
    if not w:
        raise ERRORS["LengthMismatch"]("LengthMismatch: measure must have atoms")
    total, any_pos = 0.0, False
    for v in w:
        if v < 0.0 or not math.isfinite(v):
            raise ERRORS["NegativeWeight"](f"NegativeWeight: weight {v:f}")
        any_pos = any_pos or v > 0.0
        total += v
    if not any_pos:
        raise ERRORS["NegativeWeight"]("NegativeWeight: all weights are zero")
    if require_simplex and abs(total - 1.0) > 1e-8:
        raise ERRORS["NotNormalized"](f"NotNormalized: weights sum to {total:f}")
    w = np.asarray(w)
    return w, np.asarray(x).reshape(len(w), dim)


def save_matrix_binary(path: str, m) -> None:
    a = np.ascontiguousarray(m, dtype=np.float64)
    try:
        f = open(path, "wb")
    except OSError:
        raise _io_error(f"cannot open {path} for writing")
    with f:
        f.write(b"SPKM" + struct.pack("<QQ", a.shape[0], a.shape[1]) + a.tobytes())


def load_matrix_binary(path: str) -> np.ndarray:
    try:
        f = open(path, "rb")
    except OSError:
        raise _io_error(f"cannot open {path}")
    with f:
        data = f.read()
    if len(data) < 4 or data[:4] != b"SPKM":
        raise _io_error(f"bad magic in {path}")
    r, c = struct.unpack("<QQ", data[4:20])
    body = data[20:]
    if len(body) < 8 * r * c:
        raise _io_error(f"truncated matrix file: {path}")
    return np.frombuffer(body[:8 * r * c], dtype=np.float64).reshape(r, c).copy()


def save_matrix_csv(path: str, m) -> None:
    a = np.asarray(m, dtype=np.float64)
    try:
        f = open(path, "w")
    except OSError:
        raise _io_error(f"cannot open {path} for writing")
    with f:
        for row in a:
            f.write(",".join(_g17(float(v)) for v in row) + "\n")
