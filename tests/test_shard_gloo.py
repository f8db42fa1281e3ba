"""World-size-2 gloo test of the row-sharded matvec logic (CPU; the per-rank
row computation is injected -- here the oracle's row subset)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

from paper_1609_04484_b200.shard import partition_rows


def test_partition_rows_bodies_and_balance():
    N, M, npore = 136192, 1000, 128
    for world in (1, 2, 4, 8):
        rs = partition_rows(N, M, npore, world)
        assert rs[0][0] == 0 and rs[-1][1] == N
        assert all(a[1] == b[0] for a, b in zip(rs, rs[1:]))
        for b, e in rs:
            assert b % npore == 0 or b == M * npore
        sizes = [e - b for b, e in rs]
        assert max(sizes) - min(sizes) <= 2 * npore or world == 1
    # wall is one body: with few bodies a rank may take it whole
    rs = partition_rows(256 + 2 * 16, 2, 16, 2)
    assert rs[0][1] in (0, 16, 32, 288)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import torch.distributed as dist

    import oracle
    from bie_inputs import density, make_problem
    from paper_1609_04484_b200.shard import partition_rows, sharded_apply

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        p = make_problem(2)
        og = oracle.OracleGeometry(p)
        ranges = partition_rows(p.N, p.M, p.n_pore, world)
        s = density(p)[0]
        b, e = ranges[rank]
        local = torch.from_numpy(s[2 * b:2 * e].copy())

        def apply_rows(full, rb, re_):
            rows = np.arange(rb, re_, dtype=np.int32)
            return torch.from_numpy(og.apply(full.numpy(), rows=rows).reshape(-1))

        y = sharded_apply(apply_rows, local, ranges, rank)
        out = [None] * world
        dist.all_gather_object(out, y.numpy())
        if rank == 0:
            q.put(np.concatenate(out))
    finally:
        dist.destroy_process_group()


def test_sharded_matvec_world2_gloo():
    import oracle
    from bie_inputs import density, make_problem

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for pr in procs:
        pr.start()
    y = q.get(timeout=120)
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    p = make_problem(2)
    ref = oracle.OracleGeometry(p).apply(density(p)[0])
    assert np.array_equal(y, ref)


def test_partition_rows_rejects_empty_ranks():
    """surplus ranks used to get empty ranges (and a wrong body range);
    now every rank owns >= 1 body or the call fails loudly."""
    import pytest

    from paper_1609_04484_b200.shard import partition_rows

    r = partition_rows(1792, 10, 128, 11)
    assert all(e > b for b, e in r) and r[0][0] == 0 and r[-1][1] == 1792
    with pytest.raises(ValueError):
        partition_rows(1792, 10, 128, 12)


def test_unit_split_balances_fixed_work():
    """dist.unit_split: units + fixed work equal across ranks (config-4 model);
    a rank whose fixed work exceeds the balanced time gets no units."""
    from paper_1609_04484_b200.dist import C_UNIT, rank_fixed_work, unit_split
    from paper_1609_04484_b200.shard import partition_rows

    N, M, n = 136192, 1000, 128
    for W in (2, 4, 8):
        ranges = partition_rows(N, M, n, W)
        fixed = [rank_fixed_work(M, n, N, b, e) for b, e in ranges]
        sl = unit_split(566000, W, fixed)
        assert sl[0][0] == 0 and sl[-1][1] == 566000
        t = [(u1 - u0) * C_UNIT + f for (u0, u1), f in zip(sl, fixed)]
        assert max(t) / min(t) < 1.001
    sl = unit_split(100, 2, [1.0, 0.0])
    assert sl == [(0, 0), (0, 100)]
