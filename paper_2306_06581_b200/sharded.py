"""Row/column-sharded Spar-Sink across GPUs (one process per GPU).

SURVEY §8(e): rank r of W owns atoms [r*m, min(n,(r+1)*m)), m = ceil(n/W),
as rows of K~ (sampled locally with the reference's per-row RNG streams,
poisson_sparsify, proj/src/sparsify.cpp:184-198, so the union of the row
slabs is the single-GPU sketch bit for bit) and as columns (a CSC built once
by an all-to-all of the row slabs' entries). Each half-step of the scaling
loop (detail::scaling_loop, proj/include/sparsink/solvers.hpp:256-395) is then
local to the rank, and ONE all-gather per half completes the scaling vector
for the next half. The loop's stop/divergence/mask decisions ride in a tail
behind every rank's slab, so all ranks take them on the device from the same
gathered bits (no host round trip per iteration).

The data path is the C ABI (include/spk.h, spk_shard_*); this module is the
plumbing around it: the plan's row-sum exchange, the column exchange, the
per-iteration all-gathers and the readout's scalar reduction. Collectives go
through a `Comm`:

* TorchComm   -- torch.distributed (NCCL over NVLink on GPUs; gloo on CPU),
* ThreadComm  -- W emulated ranks as threads of one process on one GPU, with
                 host-synchronised copies (no kernel ever waits on another
                 rank's kernel), used to test the multi-rank path on one GPU.

A backend supplies the shard operations; `CudaShard` is the product (the
shared library -- no CPU fallback exists). Tests plug a CPU stand-in into the
same driver to exercise the gloo path without a GPU.
"""
from __future__ import annotations

import ctypes as C
import math
import threading
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib as L
from .api import Coords, SolverConfig, SparSinkOptions, _raise

TAIL = L.SHARD_TAIL


# ---- collectives --------------------------------------------------------------------
class Comm:
    rank: int
    world: int

    def all_gather(self, buf: torch.Tensor, chunk: int) -> None:
        """In place: buf holds world blocks of `chunk`; this rank's block is filled."""
        raise NotImplementedError

    def all_to_all(self, out: torch.Tensor, inp: torch.Tensor, out_splits: list[int], in_splits: list[int]) -> None:
        raise NotImplementedError

    def all_reduce_sum(self, t: torch.Tensor) -> None:
        raise NotImplementedError

    def barrier(self) -> None:
        raise NotImplementedError


class TorchComm(Comm):
    def __init__(self, group=None):
        import torch.distributed as dist

        self.dist = dist
        self.group = group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        self.inplace = dist.get_backend(group) == "nccl"

    def all_gather(self, buf, chunk):
        own = buf[self.rank * chunk:(self.rank + 1) * chunk]
        # NCCL gathers in place (send buffer inside the receive buffer); gloo gets a copy
        self.dist.all_gather_into_tensor(buf, own if self.inplace else own.clone(), group=self.group)

    def all_to_all(self, out, inp, out_splits, in_splits):
        self.dist.all_to_all_single(out, inp, out_splits, in_splits, group=self.group)

    def all_reduce_sum(self, t):
        self.dist.all_reduce(t, group=self.group)

    def barrier(self):
        self.dist.barrier(group=self.group)


class _ThreadWorld:
    def __init__(self, world: int):
        self.world = world
        self.bar = threading.Barrier(world)
        self.slots: list = [None] * world


class ThreadComm(Comm):
    """Rank `rank` of W threads sharing one process (and one GPU). Every
    collective synchronises the caller's stream, meets the other threads at a
    host barrier, and copies; no kernel waits on another rank's kernel."""

    def __init__(self, tw: _ThreadWorld, rank: int):
        self.tw, self.rank, self.world = tw, rank, tw.world

    @staticmethod
    def make(world: int) -> list["ThreadComm"]:
        tw = _ThreadWorld(world)
        return [ThreadComm(tw, r) for r in range(world)]

    def _sync(self, t: torch.Tensor):
        if t.is_cuda:
            torch.cuda.current_stream(t.device).synchronize()

    def _exchange(self, obj):
        self.tw.slots[self.rank] = obj
        self.tw.bar.wait()
        got = list(self.tw.slots)
        self.tw.bar.wait()
        return got

    def all_gather(self, buf, chunk):
        self._sync(buf)
        bufs = self._exchange(buf)
        for r in range(self.world):
            if r != self.rank:
                buf[r * chunk:(r + 1) * chunk].copy_(bufs[r][r * chunk:(r + 1) * chunk])
        self._sync(buf)
        self.tw.bar.wait()  # nobody overwrites its block before every copy is done

    def all_to_all(self, out, inp, out_splits, in_splits):
        self._sync(inp)
        ins = self._exchange((inp, in_splits))
        pos = 0
        for r in range(self.world):
            src, splits = ins[r]
            start = sum(splits[:self.rank])
            cnt = splits[self.rank]
            assert cnt == out_splits[r]
            out[pos:pos + cnt].copy_(src[start:start + cnt])
            pos += cnt
        self._sync(out)
        self.tw.bar.wait()

    def all_reduce_sum(self, t):
        self._sync(t)
        ts = self._exchange(t.clone())
        acc = ts[0].clone()
        for r in range(1, self.world):
            acc += ts[r]
        t.copy_(acc)
        self._sync(t)

    def barrier(self):
        self.tw.bar.wait()


# ---- the CUDA shard (product) ---------------------------------------------------------
class CudaShard:
    """spk_shard_* on one GPU; tensors are CUDA tensors on `device`."""

    def __init__(self, device: int = 0, options: dict | None = None):
        self.lib = L.load()
        self.device = torch.device("cuda", device)
        p = C.c_void_p()
        rc = self.lib.spk_ctx_create(device, C.byref(p))
        if rc != 0:
            raise RuntimeError(f"spk_ctx_create(device={device}) failed with status {rc}")
        self.ctx = p
        self.sh = None
        for k, v in (options or {}).items():  # spk_ctx_set_option keys (L.OPT_*)
            _raise(self.ctx, self.lib.spk_ctx_set_option(self.ctx, int(k), int(v)))

    def close(self):
        if self.sh:
            self.lib.spk_shard_free(self.sh)
            self.sh = None
        if self.ctx:
            self.lib.spk_ctx_destroy(self.ctx)
            self.ctx = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def bind_stream(self):
        s = torch.cuda.current_stream(self.device)
        _raise(self.ctx, self.lib.spk_ctx_set_stream(self.ctx, C.c_void_p(s.cuda_stream)))

    def zeros(self, n, dtype=torch.float64):
        return torch.zeros(int(n), dtype=dtype, device=self.device)

    @property
    def launches(self) -> int:
        return int(self.lib.spk_ctx_launch_count(self.ctx))

    def plan_rows(self, kd, a, b, plan_kind, lam, eps, world, rank, m):
        rs, rn = self.zeros(max(m, 1)), self.zeros(max(m, 1), torch.int64)
        need = C.c_int32(0)
        _raise(self.ctx, self.lib.spk_shard_plan_rows(self.ctx, C.byref(kd), L.dptr(a), L.dptr(b), plan_kind, lam, eps,
                                                      world, rank, C.c_void_p(rs.data_ptr()),
                                                      C.c_void_p(rn.data_ptr()), C.byref(need)))
        return bool(need.value), rs, rn

    def create(self, kd, a, b, plan_kind, lam, eps, s, seed, opts, world, rank, rs_all, rn_all):
        p = C.c_void_p()
        o = opts.c()
        _raise(self.ctx, self.lib.spk_shard_create(
            self.ctx, C.byref(kd), L.dptr(a), L.dptr(b), plan_kind, lam, eps, float(s),
            C.c_uint64(seed & 0xFFFFFFFFFFFFFFFF), C.byref(o), world, rank,
            C.c_void_p(rs_all.data_ptr()) if rs_all is not None else None,
            C.c_void_p(rn_all.data_ptr()) if rn_all is not None else None, C.byref(p)))
        self.sh = p

    def info(self) -> dict:
        v = [np.zeros(1, np.int64) for _ in range(7)]
        vb, fz = C.c_int32(0), C.c_int32(0)
        km, kn = np.zeros(1), np.zeros(1, np.int64)
        _raise(self.ctx, self.lib.spk_shard_info(self.sh, *[L.i64ptr(x) for x in v], C.byref(vb), L.dptr(km),
                                                 L.i64ptr(kn), C.byref(fz)))
        keys = ("n", "m", "stride", "lo", "hi", "row_nnz", "col_nnz")
        d = {k: int(x[0]) for k, x in zip(keys, v)}
        d.update(value_bytes=vb.value, kernel_mean_part=float(km[0]), kernel_nnz=int(kn[0]), factorized=fz.value)
        return d

    def export(self, world, m, row_nnz, value_bytes):
        counts = self.zeros(world * m, torch.int64)
        rows = self.zeros(max(row_nnz, 1), torch.int32)
        vals = self.zeros(max(row_nnz, 1), torch.float32 if value_bytes == 4 else torch.float64)
        sizes = np.zeros(world, np.int64)
        _raise(self.ctx, self.lib.spk_shard_export(self.sh, C.c_void_p(counts.data_ptr()), C.c_void_p(rows.data_ptr()),
                                                   C.c_void_p(vals.data_ptr()), L.i64ptr(sizes)))
        return counts, rows[:row_nnz], vals[:row_nnz], [int(x) for x in sizes]

    def import_(self, counts, rows, vals, total):
        _raise(self.ctx, self.lib.spk_shard_import(self.sh, C.c_void_p(counts.data_ptr()),
                                                   C.c_void_p(rows.data_ptr()), C.c_void_p(vals.data_ptr()),
                                                   int(total)))

    def coverage(self):
        er, ec = np.zeros(1, np.int64), np.zeros(1, np.int64)
        _raise(self.ctx, self.lib.spk_shard_coverage(self.sh, L.i64ptr(er), L.i64ptr(ec)))
        return int(er[0]), int(ec[0])

    def begin(self, cfg: SolverConfig, uot, policy, er_tot, ec_tot, u0, v0):
        c = cfg.c(policy)
        _raise(self.ctx, self.lib.spk_shard_begin(self.sh, C.byref(c), int(uot), policy, int(er_tot), int(ec_tot),
                                                  C.c_void_p(u0.data_ptr()), C.c_void_p(v0.data_ptr())))

    def half(self, h, t, x, old, out):
        _raise(self.ctx, self.lib.spk_shard_half(self.sh, h, int(t), C.c_void_p(x.data_ptr()),
                                                 C.c_void_p(old.data_ptr()), C.c_void_p(out.data_ptr())))

    def finish(self, t_last, v_last):
        _raise(self.ctx, self.lib.spk_shard_finish(self.sh, int(t_last), C.c_void_p(v_last.data_ptr())))

    def status(self):
        """-> (report dict, stopped, final parity); raises the loop's error."""
        rep, st, par = L.Report(), C.c_int32(0), C.c_int32(0)
        _raise(self.ctx, self.lib.spk_shard_status(self.sh, C.byref(rep), C.byref(st), C.byref(par)))
        return rep.as_dict(), bool(st.value), int(par.value)

    def readout(self, u, v, log_domain, uot, want_obj):
        out = np.zeros(8)
        _raise(self.ctx, self.lib.spk_shard_readout(self.sh, C.c_void_p(u.data_ptr()), C.c_void_p(v.data_ptr()),
                                                    int(log_domain), int(uot), int(want_obj), L.dptr(out)))
        return out


# ---- the driver ------------------------------------------------------------------------
@dataclass
class ShardedResult:
    u: np.ndarray
    v: np.ndarray
    log_u: np.ndarray | None
    log_v: np.ndarray | None
    report: dict = field(default_factory=dict)


def slab(n: int, world: int, rank: int) -> tuple[int, int, int]:
    """(m, lo, hi): the slab geometry shared with spk_shard_* (slab_bounds)."""
    m = (n + world - 1) // world
    lo = min(n, rank * m)
    return m, lo, min(n, lo + m)


def gathered_to_full(buf: torch.Tensor, n: int, m: int, world: int) -> np.ndarray:
    """Strip the tails: W blocks of (m + TAIL) -> the n-vector."""
    blocks = buf.view(world, m + TAIL)[:, :m]
    return blocks.reshape(-1)[:n].cpu().numpy().astype(np.float64, copy=True)


class ShardedSketch:
    """This rank's share of a sharded sketch: build_sketch (solvers.cpp:314-335)
    over W ranks -- the plan's row-sum gather, local sampling, the column
    exchange and the coverage totals. Solve it (repeatedly) with solve()."""

    def __init__(self, comm: Comm, shard, kernel: Coords, a, b, plan: str, lambda_: float, epsilon: float, s: float,
                 seed: int, opts: SparSinkOptions | None = None):
        self.comm, self.shard = comm, shard
        self.opts = opts = opts or SparSinkOptions()
        self.a = a = np.ascontiguousarray(a, dtype=np.float64)
        self.b = b = np.ascontiguousarray(b, dtype=np.float64)
        self.seed = seed
        kd, keep = kernel.desc()
        self.n, W, r = int(kd.n), comm.world, comm.rank
        self.m, self.lo, self.hi = m, _, _ = slab(self.n, W, r)
        plan_kind = L.PLAN_UNIFORM if opts.probs == "uniform" else (L.PLAN_UOT if plan == "uot" else L.PLAN_OT)
        shard.bind_stream()
        # 1. plan: support / normaliser pass over this rank's rows, gathered in rank order
        need, rs, rn = shard.plan_rows(kd, a, b, plan_kind, lambda_, epsilon, W, r, m)
        rs_all = rn_all = None
        if need:
            rs_all, rn_all = shard.zeros(W * m), shard.zeros(W * m, torch.int64)
            rs_all[r * m:(r + 1) * m].copy_(rs[:m])
            rn_all[r * m:(r + 1) * m].copy_(rn[:m])
            comm.all_gather(rs_all, m)
            comm.all_gather(rn_all, m)
        # 2. sample this rank's rows
        shard.create(kd, a, b, plan_kind, lambda_, epsilon, s, seed, opts, W, r, rs_all, rn_all)
        del rs_all, rn_all
        self.info = info = shard.info()
        self.stride = info["stride"]
        # 3. column exchange: every rank's entries of my columns, sources in rank order
        counts, rows, vals, send_sizes = shard.export(W, m, info["row_nnz"], info["value_bytes"])
        self.dev = counts.device
        send_t = torch.tensor(send_sizes, dtype=torch.int64, device=self.dev)
        recv_t = torch.zeros_like(send_t)
        comm.all_to_all(recv_t, send_t, [1] * W, [1] * W)
        recv_sizes = [int(x) for x in recv_t.cpu().tolist()]
        recv_counts = torch.zeros_like(counts)
        comm.all_to_all(recv_counts, counts, [m] * W, [m] * W)
        total = sum(recv_sizes)
        recv_rows = shard.zeros(max(total, 1), torch.int32)
        recv_vals = shard.zeros(max(total, 1), vals.dtype)
        comm.all_to_all(recv_rows[:total], rows, recv_sizes, send_sizes)
        comm.all_to_all(recv_vals[:total], vals, recv_sizes, send_sizes)
        del counts, rows, vals
        shard.import_(recv_counts, recv_rows, recv_vals, total)
        del recv_counts, recv_rows, recv_vals
        # 4. coverage totals and sketch-wide scalars
        er, ec = shard.coverage()
        tot = torch.tensor([er, ec, info["row_nnz"]], dtype=torch.int64, device=self.dev)
        comm.all_reduce_sum(tot)
        self.empty_rows, self.empty_cols, self.nnz = (int(x) for x in tot.cpu().tolist())
        km = torch.zeros(W, dtype=torch.float64, device=self.dev)
        km[r] = info["kernel_mean_part"]
        comm.all_gather(km, 1)
        self.kernel_mean = float(sum(km.cpu().tolist()))  # rank order
        if opts.strict and (self.empty_rows or self.empty_cols):  # strict check (solvers.cpp:325-333)
            from .api import ERRORS
            raise ERRORS["DegenerateSketchError"](
                f"DegenerateSketchError: sketch orphaned {self.empty_rows} rows and {self.empty_cols} columns; "
                "raise s or theta, or use a different seed")
        S = self.stride * W
        # + 2 doubles: the slab x block loop's last x tile is a 16-byte-rounded
        # TMA copy, which may read 8 bytes past the gathered vector
        self.U = [shard.zeros(S + 2)[:S], shard.zeros(S + 2)[:S]]
        self.V = [shard.zeros(S + 2)[:S], shard.zeros(S + 2)[:S]]

    def solve(self, cfg: SolverConfig, uot: bool = False, check_every: int = 0, on_loop=None,
              want_scalings: bool = True) -> ShardedResult:
        """sinkhorn_ot / sinkhorn_uot<SparseKernel> (solvers.hpp:209-232) on the
        sharded sketch, then the objective. check_every > 0 reads the loop state
        every that many iterations (a stream sync) to stop early once converged;
        0 runs max_iter iterations and decides at the end. on_loop("start"/"end")
        brackets the iteration loop (bench timing)."""
        comm, shard = self.comm, self.shard
        W, r, m, n, stride = comm.world, comm.rank, self.m, self.n, self.stride
        U, V = self.U, self.V
        policy = L.POLICY_ERROR if self.opts.strict else L.POLICY_MASK
        shard.bind_stream()
        shard.begin(cfg, uot, policy, self.empty_rows, self.empty_cols, U[0], V[0])
        comm.all_gather(V[0], stride)
        # the loop: two half-steps, two all-gathers per iteration
        if on_loop:
            on_loop("start")
        t = 0
        for t in range(1, int(cfg.max_iter) + 1):
            shard.half(0, t, V[(t - 1) & 1], U[(t - 1) & 1], U[t & 1])
            comm.all_gather(U[t & 1], stride)
            shard.half(1, t, U[t & 1], V[(t - 1) & 1], V[t & 1])
            comm.all_gather(V[t & 1], stride)
            if check_every and t % check_every == 0 and shard.status()[1]:
                break
        shard.finish(t, V[t & 1])
        if on_loop:
            on_loop("end")
        rep, _, par = shard.status()  # raises ZeroDenominator / DegenerateSketchError like the reference
        # readout partials, summed in rank order on every rank
        log_domain = bool(cfg.stabilize)
        part = torch.zeros(W * 8, dtype=torch.float64, device=self.dev)
        part[r * 8:(r + 1) * 8] = torch.from_numpy(shard.readout(U[par], V[par], log_domain, uot, True))
        comm.all_gather(part, 8)
        P = part.view(W, 8).cpu().numpy()
        res_row, res_col, cost, ent, kl_a, kl_b = (float(sum(P[q, k] for q in range(W))) for k in range(6))
        inf_rows = [int(x) - 1 for x in P[:, 6] if x > 0]
        kl_bad = [int(x) - 1 for x in P[:, 7] if x > 0]
        if inf_rows:
            from .api import ERRORS
            raise ERRORS["InfiniteCostOnSupport"](
                f"InfiniteCostOnSupport: plan mass on a blocked entry (row {min(inf_rows)})")
        if uot and kl_bad:
            from .api import SparsinkError
            raise SparsinkError("Error: KL undefined: mass off support")
        lam, eps = cfg.lambda_, cfg.epsilon
        objective = (cost + lam * kl_a + lam * kl_b - eps * ent) if uot else (cost - eps * ent)
        uf = vf = lu = lv = None
        if want_scalings:
            uf, vf = gathered_to_full(U[par], n, m, W), gathered_to_full(V[par], n, m, W)
            if log_domain:
                lu, lv = uf, vf
                uf, vf = np.exp(lu), np.exp(lv)
        rep.update(objective=objective, residual_row=res_row, residual_col=res_col, seed=self.seed,
                   kernel_mean=self.kernel_mean, world=W, sketch_nnz=self.nnz)
        return ShardedResult(uf, vf, lu, lv, rep)


def spar_sink_sharded(comm: Comm, shard, kernel: Coords, a, b, cfg: SolverConfig, s: float, seed: int,
                      opts: SparSinkOptions | None = None, uot: bool = False, check_every: int = 0,
                      on_loop=None) -> ShardedResult:
    """spar_sink_ot / spar_sink_uot (solvers.cpp:339-378) over W ranks: every
    rank passes the same inputs and returns the full u, v and the same report."""
    sk = ShardedSketch(comm, shard, kernel, a, b, "uot" if uot else "ot", cfg.lambda_, cfg.epsilon, s, seed, opts)
    return sk.solve(cfg, uot, check_every, on_loop)


def run_emulated(world: int, fn, device: int = 0, options: dict | None = None):
    """Run fn(comm, shard) for `world` emulated ranks (threads) on one GPU and
    return the per-rank results (exceptions re-raised). `options` are context
    options (L.OPT_* -> value) applied to every rank."""
    comms = ThreadComm.make(world)
    out: list = [None] * world
    err: list = [None] * world

    def body(r):
        shard = None
        try:
            torch.cuda.set_device(device)
            with torch.cuda.stream(torch.cuda.Stream(device)):
                shard = CudaShard(device, options)
                out[r] = fn(comms[r], shard)
                torch.cuda.current_stream(device).synchronize()
        except BaseException as e:  # noqa: BLE001 -- re-raised below
            err[r] = e
            comms[r].tw.bar.abort()
        finally:
            if shard is not None:
                shard.close()

    threads = [threading.Thread(target=body, args=(q,)) for q in range(world)]
    for th in threads:
        th.start()
    for th in threads:
        th.join()
    for e in err:
        if e is not None and not isinstance(e, threading.BrokenBarrierError):
            raise e
    for e in err:
        if e is not None:
            raise e
    return out


# ---- the library's own driver (include/spk.h spk_comm_* / spk_sharded_*) -----------
# The same sharded solve run entirely inside libspk_b200.so: NCCL loaded by the
# library (the CUDA-graph-captured loop) or the emulated communicator (threads
# sharing one GPU). A C / C++ caller uses exactly these entry points.
class LibComm:
    """A communicator owned by the library for `ctx` (an api.Context)."""

    def __init__(self, ctx, ptr):
        self.ctx, self.ptr, self.lib = ctx, ptr, ctx.lib

    @staticmethod
    def unique_id(lib=None) -> bytes:
        lib = lib or L.load()
        buf = C.create_string_buffer(128)
        rc = lib.spk_comm_unique_id(buf)
        if rc:
            raise RuntimeError("spk_comm_unique_id failed (NCCL unavailable?)")
        return buf.raw

    @classmethod
    def nccl(cls, ctx, uid: bytes, world: int, rank: int) -> "LibComm":
        p = C.c_void_p()
        _raise(ctx.ptr, ctx.lib.spk_comm_init(ctx.ptr, C.c_char_p(uid), world, rank, C.byref(p)))
        return cls(ctx, p)

    @classmethod
    def emulated(cls, ctx, group, rank: int) -> "LibComm":
        p = C.c_void_p()
        _raise(ctx.ptr, ctx.lib.spk_comm_init_emulated(ctx.ptr, group, rank, C.byref(p)))
        return cls(ctx, p)

    def info(self) -> dict:
        w, r, nc = C.c_int(), C.c_int(), C.c_int()
        self.lib.spk_comm_info(self.ptr, C.byref(w), C.byref(r), C.byref(nc))
        return {"world": w.value, "rank": r.value, "nccl": bool(nc.value)}

    def close(self):
        if self.ptr:
            self.lib.spk_comm_destroy(self.ptr)
            self.ptr = None


class EmulatedGroup:
    def __init__(self, world: int, lib=None):
        self.lib = lib or L.load()
        self.ptr = C.c_void_p()
        if self.lib.spk_comm_group_create(world, C.byref(self.ptr)):
            raise RuntimeError("spk_comm_group_create failed")

    def close(self):
        if self.ptr:
            self.lib.spk_comm_group_destroy(self.ptr)
            self.ptr = None


class LibShardedSketch:
    """spk_sharded_build / spk_sharded_solve: this rank's share of the sharded
    sketch, built and solved by the library's driver."""

    def __init__(self, comm: LibComm, kernel: Coords, a, b, plan: str, lambda_: float, epsilon: float, s: float,
                 seed: int, opts: SparSinkOptions | None = None):
        self.comm, self.lib = comm, comm.lib
        self.a = np.ascontiguousarray(a, dtype=np.float64)
        self.b = np.ascontiguousarray(b, dtype=np.float64)
        kd, self._keep = kernel.desc()
        o = (opts or SparSinkOptions()).c()
        kind = L.PLAN_UNIFORM if (opts and opts.probs == "uniform") else (L.PLAN_UOT if plan == "uot" else L.PLAN_OT)
        self.ptr = C.c_void_p()
        _raise(comm.ctx.ptr, self.lib.spk_sharded_build(comm.ptr, C.byref(kd), L.dptr(self.a), L.dptr(self.b), kind,
                                                        float(lambda_), float(epsilon), float(s),
                                                        C.c_uint64(seed & 0xFFFFFFFFFFFFFFFF), C.byref(o),
                                                        C.byref(self.ptr)))
        self.info = self._info()

    def _info(self) -> dict:
        v = [C.c_int64() for _ in range(6)]
        self.lib.spk_sharded_info(self.ptr, *[C.byref(x) for x in v])
        return dict(zip(("n", "nnz", "kernel_nnz", "lo", "hi", "captured_launches"), (x.value for x in v)))

    def solve(self, cfg: SolverConfig, uot: bool = False, want_scalings: bool = True) -> ShardedResult:
        n = self.info["n"]
        u, v, lu, lv = ((np.empty(n) for _ in range(4)) if want_scalings else (None,) * 4)
        rep = L.Report()
        c = cfg.c(L.POLICY_MASK)
        _raise(self.comm.ctx.ptr, self.lib.spk_sharded_solve(self.ptr, C.byref(c), int(uot), L.dptr(u), L.dptr(v),
                                                             L.dptr(lu), L.dptr(lv), C.byref(rep)))
        self.info = self._info()
        log = bool(rep.log_domain)
        return ShardedResult(u, v, lu if log else None, lv if log else None, rep.as_dict())

    def free(self):
        if self.ptr:
            self.lib.spk_sharded_free(self.ptr)
            self.ptr = None


def spar_sink_multi(devices, kernel: Coords, a, b, cfg: SolverConfig, s: float, seed: int,
                    opts: SparSinkOptions | None = None, uot: bool = False) -> ShardedResult:
    """spk_spar_sink_multi: one call from one host thread over several GPUs of
    this process (NCCL communicators and a driver thread per GPU inside)."""
    lib = L.load()
    a = np.ascontiguousarray(a, dtype=np.float64)
    b = np.ascontiguousarray(b, dtype=np.float64)
    kd, keep = kernel.desc()
    n = int(kd.n)
    u, v, lu, lv = (np.empty(n) for _ in range(4))
    rep = L.Report()
    devs = (C.c_int * len(devices))(*devices)
    o = (opts or SparSinkOptions()).c()
    c = cfg.c(L.POLICY_MASK)
    rc = lib.spk_spar_sink_multi(devs, len(devices), C.byref(kd), L.dptr(a), L.dptr(b), C.byref(c), float(s),
                                 C.c_uint64(seed & 0xFFFFFFFFFFFFFFFF), C.byref(o), int(uot), L.dptr(u), L.dptr(v),
                                 L.dptr(lu), L.dptr(lv), C.byref(rep))
    _raise(None, rc)
    log = bool(rep.log_domain)
    return ShardedResult(u, v, lu if log else None, lv if log else None, rep.as_dict())
