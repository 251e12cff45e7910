"""Generate tests/golden/c4_normaliser.json: config 4's masked-grid OT
normaliser (sparsify.cpp:49-67) summed in the reference's sequential
row-major order over all 1e12 (i, j) pairs -- too slow for a test, so it is
computed once here by oracle/masked_normaliser.c and committed.

Before the C4 run the program is pinned against the compiled reference
(oracle/_ref, ot_probabilities on a dense K) at a small heavy-tailed n with
masked entries: ra_i * cb_j * inv must reproduce the reference's grid bit for
bit.

The fixture records a digest of the C4 inputs (x, y, q); the GPU test checks
the digest before comparing, so a different input generation fails loudly.

  python tests/golden/make_c4_normaliser.py [--small-only]
"""
from __future__ import annotations

import hashlib
import json
import subprocess
import sys
import tempfile
import time
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
ROOT = HERE.parent.parent
sys.path.insert(0, str(ROOT))

EXE = ROOT / "oracle" / "_build" / "masked_normaliser"


def build_exe() -> None:
    EXE.parent.mkdir(parents=True, exist_ok=True)
    subprocess.check_call(["gcc", "-std=c11", "-O2", "-ffp-contract=off", "-pthread", "-o", str(EXE),
                           str(ROOT / "oracle" / "masked_normaliser.c"), "-lm"])


def digest(x: np.ndarray, y: np.ndarray, q: float) -> str:
    h = hashlib.sha256()
    h.update(np.ascontiguousarray(x, np.float64).tobytes())
    h.update(np.ascontiguousarray(y, np.float64).tobytes())
    h.update(np.float64(q).tobytes())
    return h.hexdigest()


def run(x, y, scale, eps, a, b, threads=8) -> dict:
    with tempfile.TemporaryDirectory() as td:
        td = Path(td)
        for name, arr in (("x", x), ("y", y), ("a", a), ("b", b)):
            np.ascontiguousarray(arr, np.float64).tofile(td / f"{name}.bin")
        out = subprocess.run([str(EXE), str(td / "x.bin"), str(td / "y.bin"), str(x.shape[0]), str(x.shape[1]),
                              repr(float(scale)), repr(float(eps)), str(td / "a.bin"), str(td / "b.bin")],
                             check=True, capture_output=True, text=True, env={"NTHREADS": str(threads)})
    return json.loads(out.stdout)


def pin_small() -> None:
    from oracle import Reference
    from paper_2306_06581_b200 import workloads as W

    R = Reference()
    n = 1500
    x = W.student_t3(9, 0, 3 * n).reshape(n, 3)
    y = W.student_t3(9, 1, 3 * n).reshape(n, 3)
    a = 0.5 + W.uniforms(9, 2, n)
    a /= a.sum()
    b = 0.5 + W.uniforms(9, 3, n)
    b /= b.sum()
    scale, eps = 2.0, 0.01
    Cm, _ = R.pairwise_cost(x, y)
    Cm /= scale
    K, ratio = R.kernel_from_cost(Cm, eps)
    assert 0.0 < ratio < 1.0, ratio
    grid, fac = R.plan_probs("ot", a, b, K, ratio)
    assert not fac
    res = run(x, y, scale, eps, a, b)
    assert res["kernel_nnz"] == int(np.count_nonzero(K)), (res, np.count_nonzero(K))
    sa, sb = float.fromhex(res["sa"]), float.fromhex(res["sb"])
    ra, cb = np.sqrt(a) / sa, np.sqrt(b) / sb
    mine = np.where(K == 0.0, 0.0, ra[:, None] * cb[None, :]) * float.fromhex(res["inv"])
    assert np.array_equal(mine, grid), "normaliser does not reproduce the reference grid"
    print(f"pinned against the reference at n={n}: {res['masked_pairs']} masked pairs, grid bit-identical")


def main() -> None:
    build_exe()
    pin_small()
    if "--small-only" in sys.argv:
        return
    from paper_2306_06581_b200 import workloads as W

    w = W.c4()
    t0 = time.time()
    res = run(w.x, w.y, w.scale, w.eps, w.a, w.b)
    res.update({"config": "C4", "scale": w.scale, "eps": w.eps, "inputs_sha256": digest(w.x, w.y, w.scale),
                "seconds": time.time() - t0,
                "generator": "tests/golden/make_c4_normaliser.py (oracle/masked_normaliser.c)"})
    (HERE / "c4_normaliser.json").write_text(json.dumps(res, indent=1) + "\n")
    print(json.dumps(res))


if __name__ == "__main__":
    main()
