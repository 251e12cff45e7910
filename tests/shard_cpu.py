"""TEST INFRASTRUCTURE: a CPU stand-in for the CUDA shard backend, so the
multi-rank driver (paper_2306_06581_b200/sharded.py) can run over gloo on a
machine without a GPU. It restates, in numpy, what spk_shard_* do on the
device -- slab geometry, gathered layout with per-rank tails, the column
exchange and the tail-carried loop decisions -- on a row slab of a sketch the
oracle drew. It is never used by the product (which has no CPU path).
"""
from __future__ import annotations

import math

import numpy as np
import torch

T = 8  # SPK_SHARD_TAIL
POLICY_ERROR, POLICY_MASK = 0, 1


class LoopError(RuntimeError):
    pass


class CpuShard:
    def __init__(self, csr, x, y, cost_scale: float):
        """csr: the oracle's full sketch (row_ptr, col_idx, values); x, y:
        coordinates for the objective (squared Euclidean / cost_scale)."""
        self.full = csr
        self.x, self.y, self.scale = np.asarray(x), np.asarray(y), cost_scale
        self.launches = 0

    # -- plumbing ----------------------------------------------------------------
    def bind_stream(self):
        pass

    def zeros(self, n, dtype=torch.float64):
        return torch.zeros(int(n), dtype=dtype)

    def plan_rows(self, kd, a, b, plan_kind, lam, eps, world, rank, m):
        # stand-in "row sums": the full sketch's row lengths, so the driver's
        # gather must reassemble them in rank order (checked in create)
        rp = self.full[0]
        n = len(rp) - 1
        lo, hi = min(n, rank * m), min(n, rank * m + m)
        rs = torch.zeros(max(m, 1), dtype=torch.float64)
        rn = torch.zeros(max(m, 1), dtype=torch.int64)
        rs[:hi - lo] = torch.from_numpy(np.diff(rp)[lo:hi].astype(np.float64))
        rn[:hi - lo] = torch.from_numpy(np.diff(rp)[lo:hi].astype(np.int64))
        return True, rs, rn

    def create(self, kd, a, b, plan_kind, lam, eps, s, seed, opts, world, rank, rs_all, rn_all):
        rp, ci, vv = self.full
        n = len(rp) - 1
        assert np.array_equal(rn_all.numpy()[:n], np.diff(rp)), "row sums gathered out of order"
        self.n, self.W, self.r = n, world, rank
        self.m = (n + world - 1) // world
        self.lo, self.hi = min(n, rank * self.m), min(n, rank * self.m + self.m)
        self.mo = self.hi - self.lo
        self.stride = self.m + T
        a0, a1 = rp[self.lo], rp[self.hi]
        self.rp = (rp[self.lo:self.hi + 1] - a0).astype(np.int64)
        self.cols = ci[a0:a1].astype(np.int64)  # global
        self.vals = vv[a0:a1].astype(np.float64)
        self.a, self.b = np.asarray(a)[self.lo:self.hi], np.asarray(b)[self.lo:self.hi]
        self.a_tot, self.b_tot = math.fsum(a), math.fsum(b)
        self.km_part = float(self.vals.sum()) / (n * n)

    def info(self):
        return dict(n=self.n, m=self.m, stride=self.stride, lo=self.lo, hi=self.hi, row_nnz=len(self.cols),
                    col_nnz=getattr(self, "col_nnz", -1), value_bytes=8, kernel_mean_part=self.km_part,
                    kernel_nnz=0, factorized=0)

    def _gpos(self, j):
        return j + (j // self.m) * T  # global index -> gathered layout

    def export(self, world, m, row_nnz, value_bytes):
        rows_local = np.repeat(np.arange(self.mo), np.diff(self.rp))
        order = np.lexsort((rows_local, self.cols))  # by column, rows ascending
        cols = self.cols[order]
        counts = np.bincount(cols, minlength=world * m).astype(np.int64)
        sizes = [int(counts[d * m:(d + 1) * m].sum()) for d in range(world)]
        rows = (rows_local[order] + self.lo).astype(np.int32)
        return (torch.from_numpy(counts), torch.from_numpy(rows), torch.from_numpy(self.vals[order].copy()), sizes)

    def import_(self, counts, rows, vals, total):
        W, m, mo = self.W, self.m, self.mo
        cnt = counts.numpy().reshape(W, m)
        rows, vals = rows.numpy()[:total].astype(np.int64), vals.numpy()[:total]
        src_off = np.concatenate([[0], np.cumsum(cnt.reshape(-1))])[:-1].reshape(W, m)
        colrows, colvals = [], []
        for c in range(mo):
            rr, vv = [], []
            for s in range(W):
                o, k = src_off[s, c], cnt[s, c]
                rr.append(rows[o:o + k])
                vv.append(vals[o:o + k])
            colrows.append(np.concatenate(rr))
            colvals.append(np.concatenate(vv))
        self.cp = np.concatenate([[0], np.cumsum([len(x) for x in colrows])]).astype(np.int64)
        self.crows = np.concatenate(colrows) if colrows else np.zeros(0, np.int64)
        self.cvals = np.concatenate(colvals) if colvals else np.zeros(0)
        assert self.cp[-1] == total
        self.col_nnz = total

    def coverage(self):
        return int((np.diff(self.rp) == 0).sum()), int((np.diff(self.cp) == 0).sum())

    def begin(self, cfg, uot, policy, er_tot, ec_tot, u0, v0):
        if policy == POLICY_ERROR and (er_tot or ec_tot):
            raise LoopError("ZeroDenominator: kernel has empty rows or columns")
        self.f = 1.0 if not uot else cfg.lambda_ / (cfg.lambda_ + cfg.epsilon)
        self.policy, self.delta, self.max_iter = policy, cfg.delta, cfg.max_iter
        self.rne = np.diff(self.rp) > 0
        self.cne = np.diff(self.cp) > 0
        self.dyn_r = np.zeros(self.mo, np.int64)
        self.dyn_c = np.zeros(self.mo, np.int64)
        own = slice(self.r * self.stride, self.r * self.stride + self.stride)
        u0[own] = 0.0
        v0[own] = 0.0
        u0[self.r * self.stride:self.r * self.stride + self.mo] = torch.from_numpy(self.rne.astype(np.float64))
        v0[self.r * self.stride:self.r * self.stride + self.mo] = torch.from_numpy(self.cne.astype(np.float64))
        self.S = dict(t=0, it=0, stopped=False, conv=False, div=False, err=None, par=0, mr=er_tot, mc=ec_tot,
                      mu=0, eu=0.0)

    def _decide(self, half, t, x):
        S = self.S
        if S["stopped"] or (half == 0 and t == 1):
            return
        tails = x.view(self.W, self.stride)[:, self.m:].numpy()
        flagged = [q for q in range(self.W) if tails[q, 2] > 0]
        tprev, judged = (t - 1, 1) if half == 0 else (t, 0)
        if flagged:
            rs = flagged[0]
            before = sum(tails[q, 1] for q in range(rs)) + tails[rs, 3]
            S.update(stopped=True, it=tprev)
            if self.policy == POLICY_MASK:
                S.update(div=True, par=(tprev - 1) & 1)
                if judged == 0:
                    S["mr"] += int(before)
                else:
                    S["mr"] += S["mu"]
                    S["mc"] += int(before)
            else:
                S["err"] = f"ZeroDenominator at {int(tails[rs, 2]) - 1}"
            return
        if judged == 0:
            S.update(mu=int(tails[:, 1].sum()), eu=float(tails[:, 0].sum()))
            return
        S["mr"] += S["mu"]
        S["mc"] += int(tails[:, 1].sum())
        S.update(mu=0, t=tprev, it=tprev, par=tprev & 1)
        if S["mr"] == self.n or S["mc"] == self.n:
            S.update(stopped=True, err="DegenerateSketchError")
        elif tprev >= 2 and S["eu"] + float(tails[:, 0].sum()) <= self.delta:
            S.update(stopped=True, conv=True)
        elif tprev >= self.max_iter:
            S["stopped"] = True

    def half(self, h, t, x, old, out):
        self._decide(h, t, x)
        if self.S["stopped"]:
            return
        if h == 0:
            ptr, idx, val, w, ne, dyn = self.rp, self.cols, self.vals, self.a, self.rne, self.dyn_r
            idx = self._gpos(idx)
        else:
            ptr, idx, val, w, ne, dyn = self.cp, self._gpos(self.crows), self.cvals, self.b, self.cne, self.dyn_c
        base = self.r * self.stride
        xv = x.numpy()
        prod = val * xv[idx]
        tmp = np.array([prod[ptr[i]:ptr[i + 1]].sum() for i in range(self.mo)])
        o = old.numpy()[base:base + self.mo].copy()
        new = o.copy()
        err, masks, flag = 0.0, 0, -1
        for i in range(self.mo):
            if not ne[i]:
                continue
            tv = tmp[i]
            if tv <= 0.0 or not np.isfinite(tv):
                if self.policy == POLICY_MASK and tv == 0.0:
                    ne[i] = False
                    dyn[i] = t
                    new[i] = 0.0
                    masks += 1
                    err += abs(o[i])
                    continue
                flag = i if flag < 0 else flag
                continue
            q = w[i] / tv
            un = q if self.f == 1.0 else q ** self.f
            if not un <= 1e150 and self.policy == POLICY_MASK:
                flag = i if flag < 0 else flag
            new[i] = un
            err += abs(un - o[i])
        before = masks if flag < 0 else int(((dyn == t) & (np.arange(self.mo) < flag)).sum())
        ov = out.numpy()
        ov[base:base + self.mo] = new
        ov[base + self.m:base + self.m + T] = 0.0
        ov[base + self.m + 0] = err
        ov[base + self.m + 1] = masks
        ov[base + self.m + 2] = 0.0 if flag < 0 else self.lo + flag + 1
        ov[base + self.m + 3] = before

    def finish(self, t_last, v_last):
        self._decide(0, t_last + 1, v_last)

    def status(self):
        S = self.S
        if S["err"]:
            raise LoopError(S["err"])
        rep = dict(iterations=S["it"], converged=int(S["conv"]), diverged=int(S["div"]), masked_rows=S["mr"],
                   masked_cols=S["mc"], log_domain=0)
        return rep, S["stopped"], S["par"]

    def readout(self, u, v, log_domain, uot, want_obj):
        base = self.r * self.stride
        U, V = u.numpy(), v.numpy()
        uo, vo = U[base:base + self.mo], V[base:base + self.mo]
        rows_local = np.repeat(np.arange(self.mo), np.diff(self.rp))
        t = uo[rows_local] * self.vals * V[self._gpos(self.cols)]
        pos = t > 0
        row_m = np.bincount(rows_local[pos], weights=t[pos], minlength=self.mo)
        d = self.x[self.lo + rows_local] - self.y[self.cols]
        cost = (d * d).sum(axis=1) / self.scale
        c_part = float((t[pos] * cost[pos]).sum())
        h_part = float(-(t[pos] * (np.log(t[pos]) - 1.0)).sum())
        cols_local = np.repeat(np.arange(self.mo), np.diff(self.cp))
        tc = U[self._gpos(self.crows)] * self.cvals * vo[cols_local]
        pc = tc > 0
        col_m = np.bincount(cols_local[pc], weights=tc[pc], minlength=self.mo)

        def kl(x, y):
            out = np.where(x > 0, x * np.log(np.where(x > 0, x, 1.0) / y) - x + y, y)
            return float(out.sum())

        out = np.zeros(8)
        out[0] = float(np.abs(row_m - self.a).sum())
        out[1] = float(np.abs(col_m - self.b).sum())
        out[2], out[3] = c_part, h_part
        if uot:
            out[4], out[5] = kl(row_m, self.a), kl(col_m, self.b)
        return out
