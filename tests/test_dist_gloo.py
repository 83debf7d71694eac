"""Multi-process (world_size 2, gloo, CPU) tests of the N>1 host logic:
row sharding, global mask offsets, and the single dgamma/dbeta all-reduce.

The per-shard LayerNorm backward here is the CPU oracle (the kernels need a
GPU); what is under test is that sharding rows + one all-reduce of the
dgamma/dbeta bucket reproduces the unsharded result, which is the property
bench.py relies on at --gpus N."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2210_10246_b200.dist import allreduce_ln_params, mask_offset, shard_rows


def _free_port() -> int:
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, rows, cols, out_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import oracle
    port_ = oracle.Port()
    g = np.random.default_rng(0)  # same global data on every rank
    x = g.standard_normal((rows, cols)).astype(np.float32)
    gam = (1 + 0.2 * g.standard_normal(cols)).astype(np.float32)
    bet = (0.1 * g.standard_normal(cols)).astype(np.float32)
    dy = g.standard_normal((rows, cols)).astype(np.float32)
    b, e = shard_rows(rows, rank, world)
    y, rstd, _ = port_.ln_fwd(x[b:e], gam, bet, 1e-5)
    dx, dg, db = port_.ln_bwd(dy[b:e], y, rstd, gam, bet, True)
    bucket = torch.from_numpy(np.concatenate([dg, db]).astype(np.float64))
    allreduce_ln_params(bucket)
    out_q.put((rank, b, e, dx, bucket.numpy(), mask_offset(b, cols)))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("rows", [64, 67])
def test_sharded_layernorm_backward_matches_unsharded(rows, port):
    world, cols = 2, 256
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    master_port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, master_port, rows, cols, q))
             for r in range(world)]
    for p in procs:
        p.start()
    res = sorted([q.get(timeout=120) for _ in range(world)])
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    g = np.random.default_rng(0)
    x = g.standard_normal((rows, cols)).astype(np.float32)
    gam = (1 + 0.2 * g.standard_normal(cols)).astype(np.float32)
    bet = (0.1 * g.standard_normal(cols)).astype(np.float32)
    dy = g.standard_normal((rows, cols)).astype(np.float32)
    y, rstd, _ = port.ln_fwd(x, gam, bet, 1e-5)
    dx, dg, db = port.ln_bwd(dy, y, rstd, gam, bet, True)
    # row shards: disjoint, covering, and their dx equal the unsharded rows
    assert res[0][1] == 0 and res[-1][2] == rows and res[0][2] == res[1][1]
    for _, b, e, sdx, bucket, off in res:
        assert np.array_equal(sdx, dx[b:e])
        assert off == b * cols
        # one all-reduce of the bucket == unsharded dgamma/dbeta (order only)
        np.testing.assert_allclose(bucket[:cols], dg, rtol=1e-12, atol=1e-12)
        np.testing.assert_allclose(bucket[cols:], db, rtol=1e-12, atol=1e-12)



def test_shard_rows_partition():
    for rows in (0, 1, 7, 64, 1000):
        for world in (1, 2, 3, 8):
            spans = [shard_rows(rows, r, world) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == rows
            assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
            sizes = [e - b for b, e in spans]
            assert max(sizes) - min(sizes) <= 1
    with pytest.raises(ValueError):
        shard_rows(10, 2, 2)
