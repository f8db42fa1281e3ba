"""World-size-2 gloo test of the row-sharded BD-GMRES driver (paper_1609_04484_b200.dist).

The distributed algorithm (`dist_gmres`) is the product code; the per-rank
compute here is a CPU backend on the oracle (rows of the completed operator,
body-local BD blocks, plain vector loops), so the test checks the sharding,
the all-gather of the density, the all-reduced inner products and the
replicated Givens updates against the single-process oracle solve."""
import decimal
import math
import os
import socket

import numpy as np
import torch
import torch.multiprocessing as mp

from paper_1609_04484_b200.dist import bodies_of_rows
from paper_1609_04484_b200.shard import partition_rows


class CpuBackend:
    def __init__(self, og, obd, rank, world):
        import torch.distributed as dist

        self.dist = dist
        self.og, self.obd, self.rank, self.world = og, obd, rank, world
        self.ranges = partition_rows(og.N, og.M, og.n_pore, world)
        self.rb, self.re = self.ranges[rank]
        self.n = 2 * (self.re - self.rb)
        self.maxlen = max(2 * (e - b) for b, e in self.ranges)

    def zeros(self, m):
        return torch.zeros(m, dtype=torch.float64)

    def _full(self, v):
        pad = torch.zeros(self.maxlen, dtype=torch.float64)
        pad[: v.numel()] = v
        bufs = [torch.zeros_like(pad) for _ in range(self.world)]
        self.dist.all_gather(bufs, pad)
        return torch.cat([bufs[r][: 2 * (e - b)] for r, (b, e) in enumerate(self.ranges)]).numpy()

    def apply_op(self, v, out):
        rows = np.arange(self.rb, self.re, dtype=np.int32)
        out.copy_(torch.from_numpy(self.og.apply(self._full(v), rows=rows).reshape(-1)))

    def pc(self, x, out):
        full = np.zeros(2 * self.og.N)
        full[2 * self.rb:2 * self.re] = x.numpy()
        out.copy_(torch.from_numpy(self.obd.apply(full)[2 * self.rb:2 * self.re]))

    def apply_pc_op(self, v, out):
        t = self.zeros(self.n)
        self.apply_op(v, t)
        self.pc(t, out)

    def dots(self, V, ldv, nv, w, out):
        for j in range(nv):
            out[j] = float(np.dot(V[j * ldv:j * ldv + self.n].numpy(), w.numpy()))

    def axpy(self, V, ldv, nv, c, alpha, beta, y):
        acc = np.zeros(self.n)
        for j in range(nv):
            acc += V[j * ldv:j * ldv + self.n].numpy() * float(c[j])
        y.copy_(torch.from_numpy((0.0 if beta == 0.0 else beta * y.numpy()) + alpha * acc))

    def scale(self, x, s, y):
        y.copy_(x / s[0])

    def sqrt(self, inp, out, m):
        out[:m] = torch.sqrt(inp[:m])

    def pythag(self, ss, h, m, out):
        hh = float(np.dot(h[:m].numpy(), h[:m].numpy()))
        out[0] = math.sqrt(float(ss[0]) - hh)

    def givens(self, H, ldh, cs, sn, g, h, h2, k, scal):  # same arithmetic as k_givens
        col = H[k * ldh:(k + 1) * ldh]
        for j in range(k + 1):
            col[j] = h[j] + h2[j]
        hk1 = float(scal[2])
        col[k + 1] = hk1
        for j in range(k):
            a, b = float(col[j]), float(col[j + 1])
            col[j] = float(cs[j]) * a + float(sn[j]) * b
            col[j + 1] = -float(sn[j]) * a + float(cs[j]) * b
        a, b = float(col[k]), float(col[k + 1])
        # correctly rounded sqrt(a^2 + b^2), as both GMRES implementations (reading C28)
        d = float((decimal.Decimal(a) ** 2 + decimal.Decimal(b) ** 2).sqrt(decimal.Context(prec=60)))
        cs[k], sn[k] = a / d, b / d
        col[k], col[k + 1] = d, 0.0
        g[k + 1] = -float(sn[k]) * float(g[k])
        g[k] = float(cs[k]) * float(g[k])
        scal[3] = abs(float(g[k + 1])) / float(scal[0])
        scal[4] = 1.0 if hk1 <= 1e-14 * float(scal[1]) else 0.0

    def trisolve(self, H, ldh, g, y, iters):
        for i in range(iters - 1, -1, -1):
            s = float(g[i])
            for j in range(i + 1, iters):
                s -= float(H[j * ldh + i]) * float(y[j])
            y[i] = s / float(H[i * ldh + i])

    def allreduce_(self, t):
        self.dist.all_reduce(t)

    def copy_(self, dst, src):
        dst.copy_(src)

    def sub(self, a, b, out):
        torch.sub(a, b, out=out)

    def host(self, t):
        return t.numpy().copy()

    def host_async(self, t, slot):
        return t.numpy().copy()

    def host_wait(self, h):
        return h


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import torch.distributed as dist

    import oracle
    from bie_inputs import make_problem, rhs_pipe
    from paper_1609_04484_b200.dist import dist_gmres

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        p = make_problem(2)
        og = oracle.OracleGeometry(p)
        obd = oracle.OracleBD(og)
        be = CpuBackend(og, obd, rank, world)
        f = rhs_pipe(p)
        x, res = dist_gmres(be, torch.from_numpy(f[2 * be.rb:2 * be.re].copy()), tol=1e-8, max_iter=200)
        out = [None] * world
        dist.all_gather_object(out, (x.numpy(), res))
        if rank == 0:
            q.put(out)
    finally:
        dist.destroy_process_group()


def test_bodies_of_rows():
    assert bodies_of_rows(0, 1280, 10, 128) == (0, 10)
    assert bodies_of_rows(1280, 1792, 10, 128) == (10, 11)
    assert bodies_of_rows(256, 1792, 10, 128) == (2, 11)


def test_dist_gmres_world2_gloo_matches_oracle():
    import oracle
    from bie_inputs import make_problem, rhs_pipe

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for pr in procs:
        pr.start()
    out = q.get(timeout=300)
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    p = make_problem(2)
    og = oracle.OracleGeometry(p)
    ref = oracle.gmres(og, rhs_pipe(p), oracle.OracleBD(og), tol=1e-8, max_iter=200)
    (x0, r0), (x1, r1) = out
    assert r0["iters"] == r1["iters"] == ref["iters"]
    assert np.array_equal(r0["hist"], r1["hist"])  # replicated Givens: identical on every rank
    rel = np.abs(r0["hist"] - ref["hist"]) / ref["hist"]
    assert rel.max() < 1e-10
    x = np.concatenate([x0, x1])
    assert np.abs(x - ref["x"]).max() / np.abs(ref["x"]).max() < 1e-10
    assert abs(r0["res_true"] - ref["res_true"]) < 1e-6 * ref["res_true"]
