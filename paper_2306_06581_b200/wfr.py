"""Frame-pair caller of the Spar-Sink path: pairwise
WFR distances between grayscale frames and end-diastole (ED) prediction.

Reference semantics (proj/src):
  measure_from_image  measures.cpp:36-60   atoms at (row, col), weights p/total
  mean_pool           measures.cpp:62-85
  s0_budget           harness.cpp:128-131  1e-3 n ln^4 n
  pairwise_wfr        harness.cpp:349-406  one WFR cost/kernel on the shared
                                           pixel grid; pair k (i < j, in order)
                                           solved by spar_sink_uot with seed
                                           mix_seed(seed, k), or by dense
                                           sinkhorn_uot when exact; distance
                                           wfr_from_uot (solvers.hpp:186-188);
                                           a failing pair -> NaN, counted
  predict_ed          harness.cpp:408-437  argmax over the window, earliest
                                           index on ties

The per-pair work is the GPU path (spk_spar_sink / spk_sinkhorn on the
coordinate form -- no n^2 host matrices); pairs are independent, so ranks take
them round-robin and one all-reduce assembles the matrix.
"""
from __future__ import annotations

import math

import numpy as np

from .api import ERRORS, Context, Coords, SolverConfig, SparsinkError, frame_pairs, mix_seed
from .harness import s0_budget  # noqa: F401 (harness.cpp:128-131; re-exported)


def measure_from_image(pixels, height: int, width: int) -> tuple[np.ndarray, np.ndarray]:
    """(coords (n, 2) as (row, col), weights) of a frame (measures.cpp:36-60)."""
    px = np.ascontiguousarray(pixels, dtype=np.float64).ravel()
    if px.size != height * width or px.size == 0:
        raise ERRORS["LengthMismatch"]("LengthMismatch: image dimensions do not match pixel count")
    total = 0.0
    for p in px:  # sequential, first offending pixel raises (measures.cpp:39-43)
        if p < 0.0 or p > 1.0:
            raise ERRORS["NegativeWeight"]("NegativeWeight: gray level out of [0,1]")
        total += p
    if total <= 0.0:
        raise ERRORS["AllBlack"]("AllBlack: image has no mass")
    r, c = np.meshgrid(np.arange(height, dtype=np.float64), np.arange(width, dtype=np.float64), indexing="ij")
    return np.stack([r.ravel(), c.ravel()], axis=1), px / total


def mean_pool(pixels, height: int, width: int, filt: int, stride: int) -> tuple[np.ndarray, int, int]:
    """Average pooling (measures.cpp:62-85): window sums in (dr, dc) order."""
    if filt < 1 or stride < 1:
        raise ERRORS["LengthMismatch"]("LengthMismatch: filter and stride must be positive")
    if height < filt or width < filt:
        raise ERRORS["EmptyOutput"]("EmptyOutput: pooling window larger than image")
    oh, ow = (height - filt) // stride + 1, (width - filt) // stride + 1
    img = np.ascontiguousarray(pixels, dtype=np.float64).reshape(height, width)
    out = np.zeros((oh, ow))
    for dr in range(filt):
        for dc in range(filt):
            out += img[dr:dr + stride * (oh - 1) + 1:stride, dc:dc + stride * (ow - 1) + 1:stride]
    return (out / float(filt * filt)).ravel(), oh, ow


def wfr_from_uot(value: float) -> float:
    return math.sqrt(max(value, 0.0))


def pairwise_wfr(ctx: Context, frames, eta: float, lambda_: float, epsilon: float, s_multiplier: float, seed: int,
                 stride: int = 1, exact: bool = False, rank: int = 0, world: int = 1, comm=None):
    """-> (distances (m, m), frame_indices, failed_pairs). `frames`: 2-D arrays
    (height, width) of gray levels. With world > 1 this rank solves pairs
    k = rank, rank + world, ...; `comm` (sharded.Comm) then sums the partial
    matrices so every rank returns the whole result."""
    if len(frames) < 2:
        raise ERRORS["LengthMismatch"]("LengthMismatch: need at least two frames")
    if stride < 1:
        raise ERRORS["LengthMismatch"]("LengthMismatch: stride must be >= 1")
    h, w = np.shape(frames[0])
    for f in frames:
        if np.shape(f) != (h, w):
            raise ERRORS["DimensionMismatch"]("DimensionMismatch: frames must share dimensions")
    idx = list(range(0, len(frames), stride))
    measures = [measure_from_image(frames[k], h, w) for k in idx]
    coords = measures[0][0]
    kern = Coords(coords, coords, "wfr", eta, scale=1.0, eps=epsilon)
    s = s_multiplier * s0_budget(coords.shape[0])
    cfg = SolverConfig(epsilon, lambda_)
    m = len(idx)
    dist = np.zeros((m, m))
    failed = 0
    for k, (i, j) in enumerate(frame_pairs(m)):
        if k % world != rank:
            continue
        try:
            if exact:
                res = ctx.sinkhorn(kern, measures[i][1], measures[j][1], cfg, uot=True)
            else:
                res = ctx.spar_sink(kern, measures[i][1], measures[j][1], cfg, s, mix_seed(seed, k), uot=True)
            d = wfr_from_uot(res.report["objective"])
        except SparsinkError:
            d = math.nan
            failed += 1
        dist[i, j] = dist[j, i] = d
    if world > 1:
        import torch

        buf = torch.zeros(m * m + 1, dtype=torch.float64)
        buf[:m * m] = torch.from_numpy(np.nan_to_num(dist, nan=0.0).ravel())
        nanmask = torch.from_numpy(np.isnan(dist).ravel().astype(np.float64))
        buf[m * m] = failed
        if comm is None:
            raise ValueError("world > 1 needs a comm")
        dev = "cuda" if torch.cuda.is_available() and getattr(comm, "inplace", False) else "cpu"
        buf, nanmask = buf.to(dev), nanmask.to(dev)
        comm.all_reduce_sum(buf)
        comm.all_reduce_sum(nanmask)
        out = buf[:m * m].cpu().numpy().reshape(m, m).copy()
        out[nanmask.cpu().numpy().reshape(m, m) > 0] = math.nan
        return out, idx, int(buf[m * m].item())
    return dist, idx, failed


def predict_ed(distances, t_es: int, window_lo: int, window_hi: int, t_ed_true: int) -> tuple[int, float]:
    """-> (t_ed_hat, |1 - (t_hat - t_es)/(t_true - t_es)|) (harness.cpp:408-437)."""
    d = np.asarray(distances, dtype=np.float64)
    m = d.shape[0]
    if t_es >= m or window_lo > window_hi or window_hi >= m:
        raise ERRORS["EmptyWindow"]("EmptyWindow: prediction window out of bounds")
    best, best_idx, found = -1.0, window_lo, False
    for t in range(window_lo, window_hi + 1):
        v = d[t_es, t]
        if math.isnan(v):
            continue
        if v > best:
            best, best_idx, found = v, t, True
    if not found:
        raise ERRORS["EmptyWindow"]("EmptyWindow: no finite distances in window")
    den = float(t_ed_true) - float(t_es)
    if den == 0.0:
        raise ERRORS["EmptyWindow"]("EmptyWindow: true ED equals ES")
    return best_idx, abs(1.0 - (float(best_idx) - float(t_es)) / den)
