"""Row-sharded BD-GMRES over several ranks.

Each rank owns the nodes of a contiguous body range (shard.partition_rows):
  * matvec  : all-gather of the density shards, then bie_dlp_apply_rows on the
              rank's rows (the one exchange step of the operator);
  * BD      : body-local blocks (bie_blockdiag_factor_range) -> no communication;
  * GMRES   : Krylov vectors sharded by rows; every inner product is a local
              bie_krylov_dots followed by an all-reduce of k+1 doubles; the
              Givens/Hessenberg work (bie_krylov_givens) is replicated on every
              rank from identical all-reduced inputs.
`dist_gmres` is backend-agnostic: `GpuBackend` runs every vector operation in
libbie.so kernels with NCCL collectives; tests/test_dist_gloo.py drives the
same algorithm with a CPU/gloo test backend.
"""
from __future__ import annotations

import numpy as np

from .shard import partition_rows


def bodies_of_rows(row_begin: int, row_end: int, M: int, n_pore: int):
    """Body range [b0, b1) covering node range [row_begin, row_end) (cut at body boundaries)."""
    wall_lo = M * n_pore

    def body(node):
        return node // n_pore if node < wall_lo else M

    b0 = body(row_begin)
    b1 = body(row_end - 1) + 1
    return b0, b1


def dist_gmres(be, f_loc, tol: float = 1e-8, max_iter: int = 1000, lookahead: int = 3, fold_norms: bool = True):
    """Left-preconditioned full GMRES (reading C13) on row-sharded vectors.

    be must provide: n, zeros(len), pc(x, out), apply_pc_op(v, out), apply_op(v, out),
    dots(V, ldv, nv, w, out), axpy(V, ldv, nv, c, alpha, beta, y), scale(x, s, y),
    sqrt(inp, out, m), pythag(ss, h, m, out) (out = sqrt(ss - h[:m].h[:m]), replicated scalars),
    givens(H, ldh, cs, sn, g, h, h2, k, scal), trisolve(H, ldh, g, y, iters),
    allreduce_(t), copy_(dst, src), sub(a, b, out), host(t) -> numpy, and
    host_async(t, slot) -> handle / host_wait(handle) -> numpy (non-blocking read-back).
    Collectives per iteration: TWO all-reduces, each of k + 2 doubles -- the
    first carries V^T w and ||w||^2 (w0, the breakdown reference), the second
    V^T w' and ||w'||^2 after the first CGS pass; hk1 = ||w' - V h2|| is then
    sqrt(||w'||^2 - ||h2||^2) (V orthonormal; h2 is at the rounding level of w',
    so the difference from the direct norm is at the rounding level).  The
    convergence check of iteration k runs after iteration k + lookahead is
    enqueued (as in bie_gmres_solve): later iterations are speculative and touch
    only entries the finish does not read.  Every rank holds identical
    replicated scalars, so all ranks stop at the same iteration.
    fold_norms=False: four all-reduces per iteration with the direct norms
    ||w|| (the operation sequence of bie_gmres_solve; used to check the two
    drivers bit for bit at world size 1).
    Returns (x_loc, dict(iters, hist, res_pc, res_true, converged))."""
    n = be.n
    ldh = max_iter + 1
    V = be.zeros(ldh * n)
    H = be.zeros(ldh * max_iter)
    cs, sn, g, h, h2, tmp = (be.zeros(ldh) for _ in range(6))
    red = be.zeros(ldh + 1)  # [V^T w | w.w] of one all-reduce
    scal = be.zeros(8)
    w, t = be.zeros(n), be.zeros(n)
    x = be.zeros(n)

    def vec(k):
        return V[k * n:(k + 1) * n]

    def norm_into(v, i):  # scal[i] = ||v|| over all ranks
        be.dots(v, 0, 1, v, tmp[0:1])
        be.allreduce_(tmp[0:1])
        be.sqrt(tmp[0:1], scal[i:i + 1], 1)

    def project(k, hh):  # hh[:k+1] = V^T w and red[k+1] = w.w, one all-reduce
        be.dots(V, n, k + 1, w, red[:k + 1])
        be.dots(w, 0, 1, w, red[k + 1:k + 2])
        be.allreduce_(red[:k + 2])
        be.copy_(hh[:k + 1], red[:k + 1])

    be.pc(f_loc, w)
    norm_into(w, 0)
    beta = float(be.host(scal[0:1])[0])
    hist = [1.0]
    if beta == 0.0:
        return x, dict(iters=0, hist=np.array(hist), res_pc=0.0, res_true=0.0, converged=True)
    be.scale(w, scal[0:1], vec(0))
    be.copy_(g[0:1], scal[0:1])
    it, conv = 0, False
    pending = []

    def check():
        nonlocal it, conv
        kk, hd = pending.pop(0)
        est, brk = be.host_wait(hd)
        hist.append(float(est))
        it = kk + 1
        if est < tol or brk != 0.0:
            conv = True

    for k in range(max_iter):
        be.apply_pc_op(vec(k), w)
        if fold_norms:
            project(k, h)                                  # all-reduce 1: h, ||w||^2
            be.sqrt(red[k + 1:k + 2], scal[1:2], 1)        # w0
            be.axpy(V, n, k + 1, h, -1.0, 1.0, w)
            project(k, h2)                                 # all-reduce 2: h2, ||w'||^2
            be.axpy(V, n, k + 1, h2, -1.0, 1.0, w)
            be.pythag(red[k + 1:k + 2], h2, k + 1, scal[2:3])  # hk1 = sqrt(||w'||^2 - ||h2||^2)
        else:
            norm_into(w, 1)
            be.dots(V, n, k + 1, w, h[:k + 1])
            be.allreduce_(h[:k + 1])
            be.axpy(V, n, k + 1, h, -1.0, 1.0, w)
            be.dots(V, n, k + 1, w, h2[:k + 1])
            be.allreduce_(h2[:k + 1])
            be.axpy(V, n, k + 1, h2, -1.0, 1.0, w)
            norm_into(w, 2)
        be.givens(H, ldh, cs, sn, g, h, h2, k, scal)
        pending.append((k, be.host_async(scal[3:5], k)))
        if k + 1 < max_iter:
            be.scale(w, scal[2:3], vec(k + 1))
        if len(pending) > lookahead:
            check()
            if conv:
                break
    while pending and not conv:
        check()
    be.trisolve(H, ldh, g, tmp, it)
    be.axpy(V, n, it, tmp, 1.0, 0.0, x)
    # residual pair (P:l.678-686)
    be.apply_op(x, t)
    be.sub(f_loc, t, w)
    norm_into(w, 6)
    norm_into(f_loc, 7)
    be.pc(w, t)
    norm_into(t, 5)
    r5, r6, r7 = be.host(scal[5:8])
    return x, dict(iters=it, hist=np.array(hist), res_pc=float(r5 / beta), res_true=float(r6 / r7), converged=conv)


# Per-iteration cost model of one rank, measured on one B200 at
# config 4: the symmetric pair kernel costs C_UNIT seconds per (512-node block,
# 32-node chunk) unit; BD applies stream their inverses from HBM at HBM_BPS;
# row-local work (epilogue, CGS2 at the bench's 50-iteration depth) costs C_ROW
# per node.
C_UNIT = 22.6e-9
HBM_BPS = 6.5e12
C_ROW = 3.0e-9


def unit_split(U: int, world: int, fixed_s):
    """Slices [u_r, u_{r+1}) of the U symmetric-kernel units so that every
    rank's modelled iteration time (its units + its fixed work fixed_s[r], i.e.
    BD apply and row-local work) is equal; ranks whose fixed work alone exceeds
    the balanced time get no units."""
    fixed = np.asarray(fixed_s, dtype=np.float64)
    act = np.ones(world, dtype=bool)
    for _ in range(world):
        T = (C_UNIT * U + fixed[act].sum()) / act.sum()
        share = np.where(act, (T - fixed) / C_UNIT, 0.0)
        if np.all(share[act] >= 0):
            break
        act &= share > 0
    share = np.maximum(share, 0.0)
    cuts = np.concatenate([[0.0], np.cumsum(share)])
    cuts = np.round(cuts / cuts[-1] * U).astype(np.int64)
    return [(int(cuts[r]), int(cuts[r + 1])) for r in range(world)]


def rank_fixed_work(M: int, n_pore: int, N: int, rb: int, re: int) -> float:
    """Modelled seconds per iteration of a rank's non-pair work: streaming its
    explicit BD inverses ((2 n_b)^2 doubles per body) and its row-local work."""
    wall_lo = M * n_pore
    pores = max(0, min(re, wall_lo) - rb) // n_pore if n_pore else 0
    bd_bytes = pores * (2 * n_pore) ** 2 * 8
    if re > wall_lo:
        bd_bytes += (2 * (N - wall_lo)) ** 2 * 8
    return bd_bytes / HBM_BPS + C_ROW * (re - rb)


class GpuBackend:
    """libbie.so kernels + torch.distributed (NCCL) collectives for one rank.

    mode "sym" (default): every rank computes a slice of the symmetric kernel's
    work list into a full-size vector, the vectors are reduce-scattered to the
    row owners, and each rank adds the local terms of its rows
    (bie_dlp_pairs_partial -> reduce-scatter -> bie_dlp_epilogue_rows): the
    11-instruction pair kernel is kept at N > 1.
    mode "rows": each rank evaluates its rows one-sidedly (bie_dlp_apply_rows).
    op "slp": the paper's single-layer operator (NEXT-1) through the bie_slp_*
    counterparts (pairs_partial / epilogue_rows / apply_rows / range BD)."""

    def __init__(self, g, rank: int, world: int, group=None, mode: str = "sym", op: str = "dlp",
                 balance: bool = True):
        import torch

        from . import _bie as B

        self.torch, self.B = torch, B
        self.g, self.rank, self.world, self.group = g, rank, world, group
        # every kernel, copy and collective of this backend runs on torch's current
        # stream (one stream: no cross-stream ordering to get wrong)
        self.stream = None
        self.ranges = partition_rows(g.N, g.M, g.n_pore, world)
        self.rb, self.re = self.ranges[rank]
        self.n = 2 * (self.re - self.rb)
        b0, b1 = bodies_of_rows(self.rb, self.re, g.M, g.n_pore)
        if op not in ("dlp", "slp"):
            raise ValueError("op must be 'dlp' or 'slp'")
        self.op = op
        self.bd = B.BlockDiag(g, bodies=(b0, b1), op=op)
        assert self.bd.rows == (self.rb, self.re)
        dev = torch.device("cuda", torch.cuda.current_device())
        self.dev = dev
        self.maxlen = max(2 * (e - b) for b, e in self.ranges)
        self.pad = torch.zeros(self.maxlen, dtype=torch.float64, device=dev)
        self.gath = torch.zeros(world * self.maxlen, dtype=torch.float64, device=dev)
        self.full = torch.zeros(2 * g.N, dtype=torch.float64, device=dev)
        self.rows_out = torch.zeros(self.n, dtype=torch.float64, device=dev)
        self.mode = mode
        if mode == "sym":
            U, nblk = B.dlp_sym_info(g)
            self.blocks = (nblk * rank // world, nblk * (rank + 1) // world)
            # units weighted against each rank's fixed per-iteration work (its BD
            # apply -- the 2.15 GB Gamma_0 inverse at config 4 -- and its rows)
            fixed = [rank_fixed_work(g.M, g.n_pore, g.N, b, e) for b, e in self.ranges]
            self.unit_slices = unit_split(U, world, fixed) if balance else \
                [(U * r // world, U * (r + 1) // world) for r in range(world)]
            self.units = self.unit_slices[rank]
            self.part_full = torch.zeros(2 * g.N, dtype=torch.float64, device=dev)
            self.send = torch.zeros(world * self.maxlen, dtype=torch.float64, device=dev)
            self.recv = torch.zeros(self.maxlen, dtype=torch.float64, device=dev)

    def zeros(self, m):
        return self.torch.zeros(m, dtype=self.torch.float64, device=self.dev)

    # Collectives: NCCL on device tensors.  Other backends (gloo, used by the
    # world-size-2 correctness test on a single GPU) stage through host memory.
    def _nccl(self):
        import torch.distributed as dist

        return dist.get_backend(self.group) == "nccl"

    def _all_gather(self, out, inp):
        import torch.distributed as dist

        if self._nccl():
            dist.all_gather_into_tensor(out, inp, group=self.group)
            return
        bufs = [self.torch.empty(inp.numel(), dtype=inp.dtype) for _ in range(self.world)]
        dist.all_gather(bufs, inp.cpu(), group=self.group)
        out.copy_(self.torch.cat(bufs))

    def _reduce_scatter(self, out, inp):
        import torch.distributed as dist

        if self._nccl():
            dist.reduce_scatter_tensor(out, inp, group=self.group)
            return
        t = inp.cpu()
        dist.all_reduce(t, group=self.group)
        out.copy_(t[self.rank * out.numel():(self.rank + 1) * out.numel()])

    def _gather_full(self, v):
        if self.world == 1:
            self.full.copy_(v)
            return self.full
        self.pad[: v.numel()].copy_(v)
        self._all_gather(self.gath, self.pad)
        for r, (b, e) in enumerate(self.ranges):
            self.full[2 * b:2 * e].copy_(self.gath[r * self.maxlen: r * self.maxlen + 2 * (e - b)])
        return self.full

    def apply_op(self, v, out):
        full = self._gather_full(v)
        slp = self.op == "slp"
        if self.mode == "rows":
            if slp:
                self.B.slp_apply_rows(self.g, full, out, self.rb, self.re, stream=self.stream)
            else:
                self.B.dlp_apply_rows(self.g, full, out, self.rb, self.re, stream=self.stream)
            return
        pairs = self.B.slp_pairs_partial if slp else self.B.dlp_pairs_partial
        pairs(self.g, full, self.part_full, self.units, self.blocks, stream=self.stream)
        if self.world == 1:
            rows = self.part_full
        else:
            for r, (b, e) in enumerate(self.ranges):
                self.send[r * self.maxlen: r * self.maxlen + 2 * (e - b)].copy_(self.part_full[2 * b:2 * e])
            self._reduce_scatter(self.recv, self.send)
            rows = self.recv[: self.n]
        if slp:
            self.B.slp_epilogue_rows(self.g, full, rows, out, self.rb, self.re, stream=self.stream)
        else:
            self.B.dlp_epilogue_rows(self.g, full, rows, out, self.rb, self.re, stream=self.stream)

    def pc(self, x, out):
        self.B.blockdiag_apply(self.bd, x, out, stream=self.stream)

    def apply_pc_op(self, v, out):
        self.apply_op(v, self.rows_out)
        self.pc(self.rows_out, out)

    def dots(self, V, ldv, nv, w, out):
        self.B.Krylov.dots(V, ldv, nv, w, self.n, out, self.stream)

    def axpy(self, V, ldv, nv, c, alpha, beta, y):
        self.B.Krylov.axpy(V, ldv, nv, c, alpha, beta, y, self.n, self.stream)

    def scale(self, x, s, y):
        self.B.Krylov.scale(x, s, y, self.n, self.stream)

    def sqrt(self, inp, out, m):
        self.B.Krylov.sqrt(inp, out, m, self.stream)

    def pythag(self, ss, h, m, out):
        if not hasattr(self, "_one"):
            self._one = self.torch.ones(1, dtype=self.torch.float64, device=self.dev)
        if not hasattr(self, "_hh"):
            self._hh = self.torch.zeros(1, dtype=self.torch.float64, device=self.dev)
        self.B.Krylov.dots(h, m, 1, h, m, self._hh, self.stream)
        self.B.Krylov.axpy(self._hh, 0, 1, self._one, -1.0, 1.0, ss, 1, self.stream)
        self.B.Krylov.sqrt(ss, out, 1, self.stream)

    def givens(self, H, ldh, cs, sn, g, h, h2, k, scal):
        self.B.Krylov.givens(H, ldh, cs, sn, g, h, h2, k, scal, self.stream)

    def trisolve(self, H, ldh, g, y, iters):
        self.B.Krylov.trisolve(H, ldh, g, y, iters, self.stream)

    def allreduce_(self, t):
        if self.world > 1:
            import torch.distributed as dist

            if self._nccl():
                dist.all_reduce(t, group=self.group)
            else:
                c = t.cpu()
                dist.all_reduce(c, group=self.group)
                t.copy_(c)

    def copy_(self, dst, src):
        dst.copy_(src)

    def sub(self, a, b, out):  # out = a - b with the library's axpy kernel
        if not hasattr(self, "_one"):
            self._one = self.torch.ones(1, dtype=self.torch.float64, device=self.dev)
        out.copy_(a)
        self.B.Krylov.axpy(b, 0, 1, self._one, -1.0, 1.0, out, self.n, self.stream)

    def host(self, t):
        return t.cpu().numpy()

    def host_async(self, t, slot):
        if not hasattr(self, "_ring"):
            self._ring = self.torch.zeros((8, 2), dtype=self.torch.float64).pin_memory()
            self._evs = [self.torch.cuda.Event() for _ in range(8)]
        q = slot % 8
        self._ring[q, : t.numel()].copy_(t, non_blocking=True)
        self._evs[q].record()
        return q

    def host_wait(self, q):
        self._evs[q].synchronize()
        return self._ring[q].numpy().copy()
