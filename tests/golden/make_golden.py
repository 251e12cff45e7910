"""Generate the golden fixtures in tests/golden/*.npz from the REFERENCE ITSELF.

Run in the build container (needs oracle/_ref/libsparsink_ref.so, i.e. the
unmodified reference sources under /root/reference compiled by
oracle/Makefile):

    python tests/golden/make_golden.py

Every input is drawn with the reference's own CounterRng
(proj/include/sparsink/rng.hpp) and every output comes from the reference's
public API (proj/include/sparsink/*.hpp) through oracle/ref_capi.cpp. The
fixtures pin the C restatement (oracle/spk_oracle.c) and the GPU path without
needing /root/reference at test time.
"""
from __future__ import annotations

import math
import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE.parents[1]))

from oracle import Reference  # noqa: E402


def points(R, n, d, seed):
    return R.rng_doubles(seed, 0, n * d).reshape(n, d)


def simplex(R, n, seed):
    w = 0.2 + R.rng_doubles(seed, 1, n)
    t = 0.0
    for v in w.tolist():
        t += v
    return w / t


SKETCH_CASES = [
    # name, n, d, cost, eta, eps, plan, lambda, theta, s_mult, seed
    ("ot_sqeuclid", 64, 2, "sqeuclid", 0.0, 0.05, "ot", math.inf, 0.0, 8.0, 42),
    ("ot_sqeuclid_theta", 64, 2, "sqeuclid", 0.0, 0.05, "ot", math.inf, 0.3, 8.0, 43),
    ("ot_wfr_masked", 64, 2, "wfr", 0.15, 0.05, "ot", math.inf, 0.0, 8.0, 44),
    ("uot_wfr", 64, 2, "wfr", 0.15, 0.05, "uot", 1.0, 0.0, 8.0, 45),
    ("uot_sqeuclid_theta", 64, 3, "sqeuclid", 0.0, 0.1, "uot", 0.5, 0.25, 6.0, 46),
    ("uniform_wfr_theta", 64, 2, "wfr", 0.2, 0.05, "uniform", math.inf, 0.4, 8.0, 47),
    ("uniform_sqeuclid", 64, 2, "sqeuclid", 0.0, 0.05, "uniform", math.inf, 0.0, 8.0, 48),
    ("ot_wfr_underflow", 96, 2, "wfr", 0.3, 0.01, "ot", math.inf, 0.0, 10.0, 49),
    ("ot_sqeuclid_underflow", 96, 2, "sqeuclid", 0.0, 0.002, "ot", math.inf, 0.0, 10.0, 50),
    ("uot_sqeuclid_underflow", 96, 2, "sqeuclid", 0.0, 0.002, "uot", 2.0, 0.0, 10.0, 51),
]

SOLVE_CASES = [
    # name, n, d, eps, lambda, stabilize, s_mult, seed, delta, max_iter, probs, strict
    ("spar_ot", 80, 2, 0.05, math.inf, False, 8.0, 11, 1e-9, 2000, "importance", False),
    ("spar_uot", 80, 2, 0.05, 1.0, False, 8.0, 12, 1e-9, 2000, "importance", False),
    ("spar_ot_log", 80, 2, 0.05, math.inf, True, 8.0, 13, 1e-9, 2000, "importance", False),
    ("spar_uot_log", 80, 2, 0.05, 0.7, True, 8.0, 14, 1e-9, 2000, "importance", False),
    ("spar_ot_rand", 80, 2, 0.05, math.inf, False, 8.0, 15, 1e-9, 2000, "uniform", False),
    ("spar_ot_masked", 80, 2, 0.5, math.inf, False, 240.0 / (80 * math.log(80)), 7, 1e-8, 2000, "importance",
     False),
]


def loop_search(R) -> None:
    """Hand-shaped sketches that exercise the loop's failure semantics
    (solvers.hpp:292-358): dynamic masking, divergence in either half, and
    ZeroDenominator under EmptyPolicy::Error. Found by a seeded search over
    tiny sketches with values spread over [1e-320, 1]; each fixture records
    the reference's own outcome."""
    wanted = {"dynmask": None, "diverge_u": None, "diverge_v": None, "zeroden": None, "lognan": None}
    for trial in range(20000):
        if all(v is not None for v in wanted.values()):
            break
        n = 4 + trial % 5
        u01 = R.rng_doubles(900 + trial, 0, 4 * n * n)
        mask = u01[: n * n].reshape(n, n) < 0.45
        expo = -320.0 * u01[n * n: 2 * n * n].reshape(n, n) ** 3
        vals = np.where(mask, 10.0 ** expo, 0.0)
        rp = np.zeros(n + 1, np.int64)
        ci, vv = [], []
        for i in range(n):
            for j in range(n):
                if vals[i, j] > 0:
                    ci.append(j)
                    vv.append(vals[i, j])
            rp[i + 1] = len(ci)
        if not ci:
            continue
        csr = (rp, np.array(ci, np.uint32), np.array(vv))
        wa = u01[2 * n * n: 2 * n * n + n] + 1e-3
        wb = u01[3 * n * n: 3 * n * n + n] + 1e-3
        a = wa / wa.sum()
        b = wb / wb.sum()
        uot = trial % 3 == 0
        lam = 0.8 if uot else math.inf
        for policy in ("mask", "error"):
            try:
                u, v, lu, lv, rep = R.sinkhorn(a, b, 0.1, lam, 1e-12, 400, False, policy, uot, csr=csr)
                err = 0
            except Exception as e:  # noqa: BLE001
                u = v = np.zeros(n)
                rep = {}
                err = getattr(e, "kind", 99)
            key = None
            if policy == "error" and err == 17 and wanted["zeroden"] is None:
                key = "zeroden"
            if policy == "mask" and not err:
                init_rows = int(np.sum(np.diff(rp) == 0))
                cols = np.zeros(n, bool)
                cols[np.array(ci)] = True
                if rep["diverged"] and wanted["diverge_u"] is None and not np.array_equal(v, np.where(cols, 1.0, 0.0)):
                    pass
                if rep["masked_rows"] > init_rows and not rep["diverged"] and wanted["dynmask"] is None:
                    key = "dynmask"
                elif rep["diverged"]:
                    # distinguish which half blew up by rerunning one iteration fewer
                    half = "diverge_u" if wanted["diverge_u"] is None else "diverge_v"
                    if wanted[half] is None:
                        key = half
            if key:
                wanted[key] = dict(row_ptr=rp, col_idx=np.array(ci, np.uint32), values=np.array(vv), a=a, b=b,
                                   uot=uot, lam=lam, policy=policy, eps=0.1, delta=1e-12, max_iter=400, err=err,
                                   u=u, v=v, **{f"rep_{k}": val for k, val in rep.items()})
        # log-domain: NaN residual from zero-weight unmasked atoms never converges (Appendix A)
        if wanted["lognan"] is None and trial > 50:
            a0 = a.copy()
            a0[0] = 0.0
            a0 /= a0.sum()
            try:
                u, v, lu, lv, rep = R.sinkhorn(a0, b, 0.1, 0.8, 1e-12, 50, True, "mask", True, csr=csr)
                wanted["lognan"] = dict(row_ptr=rp, col_idx=np.array(ci, np.uint32), values=np.array(vv), a=a0, b=b,
                                        uot=True, lam=0.8, policy="mask", eps=0.1, delta=1e-12, max_iter=50, err=0,
                                        u=u, v=v, lu=lu, lv=lv, stabilize=True,
                                        **{f"rep_{k}": val for k, val in rep.items()})
            except Exception:  # noqa: BLE001
                pass
    for key, case in wanted.items():
        if case is None:
            print(f"loop_{key}: not found")
            continue
        np.savez_compressed(HERE / f"loop_{key}.npz", **case)
        print(f"loop_{key}: n={len(case['a'])} err={case['err']} iters={case.get('rep_iterations')} "
              f"diverged={case.get('rep_diverged')} masked={case.get('rep_masked_rows')}/{case.get('rep_masked_cols')}")


def main() -> None:
    R = Reference()
    for name, n, d, kind, eta, eps, plan, lam, theta, smult, seed in SKETCH_CASES:
        x = points(R, n, d, seed)
        y = points(R, n, d, seed + 1000)
        a = simplex(R, n, seed + 2000)
        b = simplex(R, n, seed + 3000)
        Cm, c0 = R.pairwise_cost(x, y, kind, eta)
        K, ratio = R.kernel_from_cost(Cm, eps)
        s = smult * n * math.log(n)
        probs, fac = R.plan_probs(plan, a, b, K, ratio, lam, eps, theta)
        rp, ci, vv = R.poisson_sparsify(plan, a, b, K, ratio, s, seed, lam, eps, theta)
        np.savez_compressed(HERE / f"sketch_{name}.npz", x=x, y=y, a=a, b=b, kind=kind, eta=eta, eps=eps, plan=plan,
                            lam=lam, theta=theta, s=s, seed=seed, c0=c0, nnz_ratio=ratio, probs=probs,
                            factorized=fac, row_ptr=rp, col_idx=ci, values=vv)
        print(f"sketch_{name}: n={n} nnz={len(ci)} ratio={ratio:.4f} factorized={fac}")
    for name, n, d, eps, lam, stab, smult, seed, delta, max_iter, probs, strict in SOLVE_CASES:
        x = points(R, n, d, seed)
        y = points(R, n, d, seed + 1000)
        a = simplex(R, n, seed + 2000)
        b = simplex(R, n, seed + 3000)
        Cm, c0 = R.pairwise_cost(x, y, "sqeuclid")
        K, ratio = R.kernel_from_cost(Cm, eps)
        s = smult * n * math.log(n)
        uot = math.isfinite(lam)
        u, v, lu, lv, rep = R.spar_sink(K, ratio, Cm, a, b, eps, s, seed, lam, delta, max_iter, stab, 0.0, probs,
                                        strict, uot)
        np.savez_compressed(HERE / f"solve_{name}.npz", x=x, y=y, a=a, b=b, eps=eps, lam=lam, stabilize=stab, s=s,
                            seed=seed, delta=delta, max_iter=max_iter, probs=probs, uot=uot, u=u, v=v,
                            lu=lu if lu is not None else np.zeros(0), lv=lv if lv is not None else np.zeros(0),
                            **{f"rep_{k}": val for k, val in rep.items()})
        print(f"solve_{name}: iters={rep['iterations']} obj={rep['objective']:.12g} masked={rep['masked_rows']}"
              f"/{rep['masked_cols']} diverged={rep['diverged']}")
    loop_search(R)


if __name__ == "__main__":
    main()
