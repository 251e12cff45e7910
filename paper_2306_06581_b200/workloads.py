"""Seeded synthetic inputs for BASELINE.json's five configs (no datasets).

All randomness is the reference's counter generator (proj/include/sparsink/rng.hpp):
draw t of stream (seed, k) = splitmix64 finalizer(mix_seed(seed, k) + t*golden),
top 53 bits; normals by Box-Muller as CounterRng::next_normal (rng.cpp:7-21).
Vectorised in numpy so n = 1e6 inputs take seconds. The same arrays feed the
GPU path and the CPU oracle/reference in one process.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

GOLDEN = np.uint64(0x9E3779B97F4A7C15)
M1 = np.uint64(0xBF58476D1CE4E5B9)
M2 = np.uint64(0x94D049BB133111EB)


def _finalize(x: np.ndarray) -> np.ndarray:
    x = (x ^ (x >> np.uint64(30))) * M1
    x = (x ^ (x >> np.uint64(27))) * M2
    return x ^ (x >> np.uint64(31))


def _splitmix(x):
    return _finalize(np.asarray(x, dtype=np.uint64) + GOLDEN)


def mix_seed(seed: int, stream: int) -> int:
    with np.errstate(over="ignore"):
        inner = _splitmix(np.uint64((stream + 0x632BE59BD9B4E019) & 0xFFFFFFFFFFFFFFFF))
        return int(_splitmix(np.uint64(seed) ^ inner))


def uniforms(seed: int, stream: int, count: int) -> np.ndarray:
    """CounterRng(seed, stream).next_double() x count (rng.hpp:38-40)."""
    with np.errstate(over="ignore"):
        t = np.arange(1, count + 1, dtype=np.uint64)
        x = _finalize(np.uint64(mix_seed(seed, stream)) + t * GOLDEN)
    return (x >> np.uint64(11)).astype(np.float64) * 2.0 ** -53


def normals(seed: int, stream: int, count: int) -> np.ndarray:
    """CounterRng::next_normal sequence (Box-Muller, cos then the sin spare)."""
    m = (count + 1) // 2
    u = uniforms(seed, stream, 2 * m)
    u1 = np.maximum(u[0::2], 1e-300)
    u2 = u[1::2]
    r = np.sqrt(-2.0 * np.log(u1))
    th = 2.0 * math.pi * u2
    out = np.empty(2 * m)
    out[0::2] = r * np.cos(th)
    out[1::2] = r * np.sin(th)
    return out[:count]


@dataclass
class Workload:
    name: str
    x: np.ndarray
    y: np.ndarray
    a: np.ndarray
    b: np.ndarray
    cost: str
    eta: float
    scale: float | None  # None = divide by max cost (c0)
    eps: float
    lam: float
    s: float
    delta: float
    max_iter: int
    values: str
    stabilize: bool = False
    extra: dict = field(default_factory=dict)

    @property
    def n(self) -> int:
        return self.x.shape[0]

    @property
    def uot(self) -> bool:
        return math.isfinite(self.lam)


def c1(seed: int = 1) -> Workload:
    """Balanced OT, n=1000 in R^5, X~N(0,I), Y~N(1,I), a=b=1/n, C/max, eps=0.1,
    s=8 n ln n, fixed 200 iterations (delta=-1), fp64."""
    n, d = 1000, 5
    x = normals(seed, 0, n * d).reshape(n, d)
    y = 1.0 + normals(seed, 1, n * d).reshape(n, d)
    a = np.full(n, 1.0 / n)
    return Workload("C1", x, y, a, a.copy(), "sqeuclid", 0.0, None, 0.1, math.inf, 8 * n * math.log(n), -1.0, 200,
                    "f64")


def c2(seed: int = 2) -> Workload:
    """UOT lambda=1, eps=0.05, n=1e4 in R^10, X~U[0,1]^10, Y~N(0.5, 0.1^2 I);
    a~U(.5,1.5) normalised to 1, b~U(.5,1.5) normalised to 1.5; C/max;
    s=16 n ln n; <=500 iterations or delta=1e-8; fp64."""
    n, d = 10_000, 10
    x = uniforms(seed, 0, n * d).reshape(n, d)
    y = 0.5 + 0.1 * normals(seed, 1, n * d).reshape(n, d)
    a = 0.5 + uniforms(seed, 2, n)
    b = 0.5 + uniforms(seed, 3, n)
    a = a / a.sum()
    b = 1.5 * b / b.sum()
    return Workload("C2", x, y, a, b, "sqeuclid", 0.0, None, 0.05, 1.0, 16 * n * math.log(n), 1e-8, 500, "f64")


def c3_frames(seed: int = 3, frames: int = 32, side: int = 112) -> tuple[np.ndarray, np.ndarray]:
    """Synthetic echo-like cycle: 3-6 anisotropic Gaussian blobs whose centres
    move along a periodic 32-frame cycle; background 1e-4; each frame
    normalised to mass 1. Returns (coords (side^2, 2) on [0,1]^2, masses
    (frames, side^2))."""
    r, c = np.meshgrid(np.arange(side), np.arange(side), indexing="ij")
    coords = np.stack([r.ravel() / (side - 1), c.ravel() / (side - 1)], axis=1)
    u = uniforms(seed, 0, 64)
    nblob = 3 + int(u[0] * 4)
    masses = np.empty((frames, side * side))
    for f in range(frames):
        ph = 2.0 * math.pi * f / frames
        img = np.full(side * side, 1e-4)
        for k in range(nblob):
            q = u[1 + 8 * k: 9 + 8 * k]
            cy = 0.25 + 0.5 * q[0] + 0.08 * math.sin(ph + 2 * math.pi * q[1])
            cx = 0.25 + 0.5 * q[2] + 0.08 * math.cos(ph + 2 * math.pi * q[3])
            sy = 0.04 + 0.06 * q[4]
            sx = 0.04 + 0.06 * q[5]
            amp = (0.5 + q[6]) * (1.0 + 0.3 * math.sin(ph + 2 * math.pi * q[7]))
            img += amp * np.exp(-0.5 * (((coords[:, 0] - cy) / sy) ** 2 + ((coords[:, 1] - cx) / sx) ** 2))
        masses[f] = img / img.sum()
    return coords, masses


def c3(seed: int = 3, pair: tuple[int, int] = (0, 16)) -> Workload:
    """One WFR UOT frame pair of config 3: eta=0.1, eps=0.01, lambda=1,
    s=10 n ln n, log domain, fp32 values."""
    coords, masses = c3_frames(seed)
    n = coords.shape[0]
    return Workload("C3", coords, coords.copy(), masses[pair[0]].copy(), masses[pair[1]].copy(), "wfr", 0.1, 1.0,
                    0.01, 1.0, 10 * n * math.log(n), 1e-6, 1000, "f32", stabilize=True,
                    extra={"pair": pair, "masses": masses})


def student_t3(seed: int, stream: int, count: int) -> np.ndarray:
    z = normals(seed, stream, count)
    g = normals(seed, stream + 100, 3 * count).reshape(count, 3)
    v = (g * g).sum(axis=1)
    return z / np.sqrt(v / 3.0)


def c4_quantile(x: np.ndarray, y: np.ndarray, seed: int, pairs: int = 10_000_000, q: float = 0.999) -> float:
    """Deterministic estimate of the 99.9th percentile of ||x_i - y_j||^2 from a
    fixed-seed sample of pairs (then treated as an input)."""
    n = x.shape[0]
    ii = np.minimum((uniforms(seed, 50, pairs) * n).astype(np.int64), n - 1)
    jj = np.minimum((uniforms(seed, 51, pairs) * n).astype(np.int64), n - 1)
    d2 = np.zeros(pairs)
    for k in range(x.shape[1]):
        diff = x[ii, k] - y[jj, k]
        d2 += diff * diff
    kth = int(math.floor(q * (pairs - 1)))
    return float(np.partition(d2, kth)[kth])


def c4(seed: int = 4, n: int = 1_000_000, pairs: int = 10_000_000) -> Workload:
    """Large balanced OT: n=1e6 in R^3, i.i.d. Student-t(3) coordinates, a=b=1/n,
    C = ||x-y||^2 / q (q = 99.9th percentile), eps=0.05, s=8 n ln n,
    fp32 kernel values, fp64 scalings, 300 fixed iterations."""
    d = 3
    x = student_t3(seed, 0, n * d).reshape(n, d)
    y = student_t3(seed, 1, n * d).reshape(n, d)
    q = c4_quantile(x, y, seed, pairs)
    a = np.full(n, 1.0 / n)
    return Workload("C4", x, y, a, a.copy(), "sqeuclid", 0.0, q, 0.05, math.inf, 8 * n * math.log(n), -1.0, 300,
                    "f32", extra={"q": q})


MIXTURE_SIGNS = np.array([[1, 1, 1, 1, 1], [-1, -1, -1, -1, -1], [1, -1, 1, -1, 1], [-1, 1, -1, 1, -1]], float)


def c5(seed: int = 5, n: int = 50_000, budget_mult: float = 8.0) -> Workload:
    """Dense-vs-sparse: n=5e4 in R^5 from a 4-component mixture (means 2*sign
    patterns MIXTURE_SIGNS, unit variance, equal weights), a=b=1/n, C/max,
    eps=0.05, 200 iterations; Spar-Sink at s = {4,8,16} n ln n."""
    d = 5

    def draw(stream):
        comp = np.minimum((uniforms(seed, stream, n) * 4).astype(np.int64), 3)
        return 2.0 * MIXTURE_SIGNS[comp] + normals(seed, stream + 10, n * d).reshape(n, d)

    x, y = draw(0), draw(1)
    a = np.full(n, 1.0 / n)
    return Workload("C5", x, y, a, a.copy(), "sqeuclid", 0.0, None, 0.05, math.inf, budget_mult * n * math.log(n),
                    -1.0, 200, "f64")


CONFIGS = {"c1": c1, "c2": c2, "c3": c3, "c4": c4, "c5": c5}


def bytes_per_iteration(n: int, nnz: int, value_bytes: int) -> int:
    """Algorithmic HBM bytes of one sparse Sinkhorn iteration:
    B_iter = 2 nnz (V + 4) + 2 (n+1) 8 + 2*4 n 8 (x gathered once, marginal,
    old scaling, new scaling, per half)."""
    return 2 * nnz * (value_bytes + 4) + 2 * (n + 1) * 8 + 64 * n
