"""The path's one collective -- the cross-rank sum of the LayerNorm
dgamma/dbeta -- fused into the backward's stage 2 over peer
memory (layernorm_kernels.cu: ln_param_reduce_peer_kernel).

One B200 here, so the ranks are simulated inside one process on one device:
each rank has its own inbox/flag buffers and its kernels run on its own
stream, concurrently, exactly as ranks on different GPUs would (the
kernels see plain device pointers either way; on a multi-GPU node they are
CUDA IPC mappings, ops.LnPeerRank.ipc).  Checked: the result is bit for bit
the fixed-order sum (rank 0, 1, ... of each rank's fixed-order partial sum),
identical on every rank, across consecutive epochs (inbox parity reuse), and
a sharded LayerNorm backward reproduces the unsharded one."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _local_sums(parts):
    """The kernel's local order: row group ty sums rows ty, ty+8, ... ; the 8
    group sums are then added in order (ln_param_reduce_peer_kernel)."""
    nparts, total = parts.shape
    g = np.zeros((8, total))
    for ty in range(8):
        acc = np.zeros(total)
        for c in range(ty, nparts, 8):
            acc = acc + parts[c]
        g[ty] = acc
    v = np.zeros(total)
    for k in range(8):
        v = v + g[k]
    return v


def _run_group(tops, ranks, parts, cols):
    import torch
    streams = [torch.cuda.Stream() for _ in ranks]
    outs = []
    for r, st in zip(ranks, streams):
        with torch.cuda.stream(st):
            outs.append(tops.ln_param_reduce_peer(parts[r.rank], cols, r))
    torch.cuda.synchronize()
    for r in ranks:
        r.check_status()
    return [(g.cpu().numpy(), b.cpu().numpy()) for g, b in outs]


@pytest.mark.parametrize("world,cols,nparts", [(1, 1024, 296), (2, 1024, 296), (3, 768, 37),
                                               (4, 1024, 5), (2, 37, 3), (8, 256, 64)])
def test_peer_reduce_is_the_fixed_order_sum(tops, cuda, world, cols, nparts):
    import torch
    ranks = tops.LnPeerRank.local_group(world, cols, cuda)
    g = np.random.default_rng(world * 1000 + cols)
    for epoch in range(4):  # consecutive exchanges reuse the two inbox parities
        parts = [g.standard_normal((nparts, 2 * cols)) * (1 + epoch) for _ in range(world)]
        dev = [torch.from_numpy(p).to(cuda) for p in parts]
        res = _run_group(tops, ranks, dev, cols)
        want = np.zeros(2 * cols)
        for s in range(world):
            want = want + _local_sums(parts[s])
        want = want.astype(np.float32)
        for dg, db in res:
            assert np.array_equal(dg, want[:cols]), epoch
            assert np.array_equal(db, want[cols:]), epoch


def test_peer_reduce_missing_rank_times_out(tops, cuda):
    """A rank that never arrives: the kernel gives up after the bounded wait
    (peer.timeout_ms), reports TEMPO_ERR_STATE and writes NaN -- not a
    partial sum -- to dgamma/dbeta (no hung GPU, nothing silently wrong).
    The status is sticky: later exchanges on that rank poison their outputs
    at once without waiting."""
    import time
    import torch
    ranks = tops.LnPeerRank.local_group(2, 32, cuda)
    for r in ranks:
        r.timeout_ms = 200
    parts = torch.ones((1, 64), dtype=torch.float64, device=cuda)
    dg, db = tops.ln_param_reduce_peer(parts, 32, ranks[0])  # rank 1 never runs
    torch.cuda.synchronize()
    with pytest.raises(tops.TempoError) as e:
        ranks[0].check_status()
    assert e.value.kind == "StateError"
    assert torch.isnan(dg).all() and torch.isnan(db).all()
    t0 = time.perf_counter()
    dg2, db2 = tops.ln_param_reduce_peer(parts, 32, ranks[0])  # sticky: no wait, NaN
    torch.cuda.synchronize()
    assert time.perf_counter() - t0 < 0.15
    assert torch.isnan(dg2).all() and torch.isnan(db2).all()


def test_concurrent_layernorm_backwards_on_two_streams(tops, cuda):
    """Two LayerNorm backwards of the same shape running concurrently on two
    streams with the DEFAULT workspace: each stream gets its own scratch
    (ops.ln_workspace is keyed by stream), so both equal the serial result
    bit for bit."""
    import torch
    rows, cols = 2048, 1024
    g = np.random.default_rng(11)
    mk = lambda *s: torch.from_numpy(g.standard_normal(s).astype(np.float32)).to(cuda)  # noqa: E731
    gam = (1 + 0.2 * mk(cols)).contiguous()
    bet = (0.1 * mk(cols)).contiguous()
    ins = []
    for _ in range(2):
        y, rs = tops.layernorm_ip_fwd(mk(rows, cols), gam, bet)
        ins.append((mk(rows, cols), y, rs))
    want = [tops.layernorm_ip_bwd(dy, y, rs, gam, bet) for dy, y, rs in ins]
    torch.cuda.synchronize()
    for _ in range(5):
        streams = [torch.cuda.Stream() for _ in range(2)]
        got = []
        for (dy, y, rs), st in zip(ins, streams):
            with torch.cuda.stream(st):
                got.append(tops.layernorm_ip_bwd(dy, y, rs, gam, bet))
        torch.cuda.synchronize()
        for w, o in zip(want, got):
            for a, b in zip(w, o):
                assert torch.equal(a, b)


@pytest.mark.parametrize("rows,cols", [(4096, 1024), (1024, 4096)])
def test_sharded_layernorm_backward(tops, cuda, rows, cols):
    """Row shards + the fused exchange == the unsharded backward: dx bit for
    bit, dgamma/dbeta identical on every rank and equal to the single-GPU
    values up to the summation order (fp64 partials, one float rounding).
    cols = 4096: stage 1 is the thread-block-cluster kernel (its partial rows
    = co-resident clusters) feeding the same fused exchange."""
    import torch
    world = 2
    g = np.random.default_rng(7)
    x = torch.from_numpy(g.standard_normal((rows, cols)).astype(np.float32)).to(cuda)
    gam = torch.from_numpy((1 + 0.2 * g.standard_normal(cols)).astype(np.float32)).to(cuda)
    bet = torch.from_numpy((0.1 * g.standard_normal(cols)).astype(np.float32)).to(cuda)
    dy = torch.from_numpy(g.standard_normal((rows, cols)).astype(np.float32)).to(cuda)
    y, rstd = tops.layernorm_ip_fwd(x, gam, bet)
    dx1, dg1, db1 = tops.layernorm_ip_bwd(dy, y, rstd, gam, bet)
    torch.cuda.synchronize()
    ranks = tops.LnPeerRank.local_group(world, cols, cuda)
    from paper_2210_10246_b200.dist import shard_rows
    streams = [torch.cuda.Stream() for _ in range(world)]
    outs = []
    if cols <= 2048:
        for r, st in zip(ranks, streams):
            b, e = shard_rows(rows, r.rank, world)
            with torch.cuda.stream(st):
                outs.append((b, e) + tops.layernorm_ip_bwd_peer(dy[b:e], y[b:e], rstd[b:e], gam,
                                                                 bet, r))
    else:
        # The simulated ranks share ONE GPU: a rank's exchange kernel, spinning
        # for its peer, can hold the registers the peer's 512-thread cluster
        # stage 1 needs (on separate GPUs each rank's stage 1 precedes its own
        # exchange).  So here: stage 1 of every rank (tempo_ln_ip_bwd_partials,
        # the cluster kernel), then the fused exchange of every rank on the
        # partial rows -- the same two kernels tempo_ln_ip_bwd_peer runs.
        import ctypes as C
        from paper_2210_10246_b200._capi import lib
        parts = []
        for r, st in zip(ranks, streams):
            b, e = shard_rows(rows, r.rank, world)
            nb = int(lib().tempo_ln_ip_bwd_workspace_size(e - b, cols))
            ws = torch.empty(nb, dtype=torch.uint8, device=cuda)
            dx = torch.empty(e - b, cols, device=cuda)
            npart = C.c_int64()
            with torch.cuda.stream(st):
                assert lib().tempo_ln_ip_bwd_partials(
                    dy[b:e].data_ptr(), y[b:e].data_ptr(), rstd[b:e].data_ptr(), gam.data_ptr(),
                    bet.data_ptr(), dx.data_ptr(), ws.data_ptr(), nb, e - b, cols,
                    C.byref(npart), st.cuda_stream) == 0
            parts.append((b, e, dx, ws.view(torch.float64)[: npart.value * 2 * cols]
                          .view(npart.value, 2 * cols)))
        torch.cuda.synchronize()
        for r, st, (b, e, dx, pr) in zip(ranks, streams, parts):
            with torch.cuda.stream(st):
                outs.append((b, e, dx) + tops.ln_param_reduce_peer(pr, cols, r))
    torch.cuda.synchronize()
    for r in ranks:
        r.check_status()
    for b, e, dx, dg, db in outs:
        assert torch.equal(dx, dx1[b:e])
        assert torch.equal(dg, outs[0][3]) and torch.equal(db, outs[0][4])
        assert torch.allclose(dg, dg1, rtol=1e-6, atol=1e-6)
        assert torch.allclose(db, db1, rtol=1e-6, atol=1e-6)


def _ipc_worker(rank, world, port, cols, q):
    import ctypes
    import os
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2210_10246_b200 import ops
        from paper_2210_10246_b200._capi import lib
        dev = torch.device("cuda:0")
        peer = ops.LnPeerRank.ipc(cols, dev)
        n = peer.inbox_bytes // 4                  # a pattern in this rank's inbox
        src = torch.full((n // 2,), float(rank + 1), dtype=torch.float64, device=dev)
        assert lib().tempo_tensor_scale(ctypes.c_void_p(src.data_ptr()), 1.0,
                                        ctypes.c_void_p(peer.inbox), n, None) == 0
        torch.cuda.synchronize()
        dist.barrier()
        # read every rank's inbox through the pointer this process mapped
        # (the device pointer array the exchange kernel uses), with a plain
        # device-to-device op of the C-ABI (out = a * 1.0 on float words)
        ptrs = peer._ptrs[0].cpu().tolist()
        seen = []
        for r in range(world):
            out = torch.empty(peer.inbox_bytes // 4, dtype=torch.float32, device=dev)
            rc = lib().tempo_tensor_scale(ctypes.c_void_p(ptrs[r]), 1.0,
                                          ctypes.c_void_p(out.data_ptr()), out.numel(), None)
            torch.cuda.synchronize()
            seen.append((rc, out.view(torch.float64).cpu().numpy().copy()))
        # the exchange itself across the two processes (time-sliced on one GPU)
        sums = []
        for epoch in range(3):
            parts = torch.full((5, 2 * cols), float((rank + 1) * (epoch + 1)), dtype=torch.float64,
                               device=dev)
            dist.barrier()
            dg, db = ops.ln_param_reduce_peer(parts, cols, peer)
            torch.cuda.synchronize()
            peer.check_status()
            sums.append((dg.cpu().numpy().copy(), db.cpu().numpy().copy()))
        dist.barrier()
        peer.close()
        q.put((rank, "ok", (seen, sums)))
    except Exception as ex:  # noqa: BLE001
        q.put((rank, repr(ex), None))
    dist.destroy_process_group()


def test_ipc_two_processes(cuda):
    """The multi-process path (ops.LnPeerRank.ipc: CUDA IPC handles over
    torch.distributed) with two processes on the one GPU of this box: each
    reads the other's inbox pattern through its mapped pointer, then three
    exchanges run across the processes (their kernels time-slice on one GPU,
    so the waits are longer than over NVLink, but the protocol is the same)."""
    import socket
    import torch.multiprocessing as mp
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    world, cols = 2, 64
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_ipc_worker, args=(r, world, port, cols, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = sorted([q.get(timeout=300) for _ in range(world)], key=lambda t: t[0])
    for p in procs:
        p.join(timeout=60)
    for rank, status, res in out:
        assert status == "ok", (rank, status)
        seen, sums = res
        for r, (rc, vals) in enumerate(seen):
            assert rc == 0 and np.all(vals == float(r + 1)), (rank, r)
        for epoch, (dg, db) in enumerate(sums):
            want = 5.0 * (epoch + 1) * (1 + 2)
            assert np.all(dg == want) and np.all(db == want), (rank, epoch)


@pytest.mark.gpu
def test_nccl_allreduce_ln_params_world1(tops, cuda):
    """The C-ABI NCCL fallback end to end on a one-rank communicator (the
    only NCCL group one GPU can host): unique id -> comm -> in-place sum of
    an LN backward's dgamma/dbeta bucket (identity at world 1) -> destroy."""
    import torch
    comm = tops.NcclComm(1, 0, tops.NcclComm.unique_id())
    try:
        rows, cols = 256, 1024
        g = torch.Generator(device=cuda)
        g.manual_seed(3)
        dy = torch.randn(rows, cols, device=cuda, generator=g)
        x = torch.randn(rows, cols, device=cuda, generator=g)
        gam = 1 + 0.2 * torch.randn(cols, device=cuda, generator=g)
        bet = 0.1 * torch.randn(cols, device=cuda, generator=g)
        y, rs = tops.layernorm_ip_fwd(x, gam, bet)
        bucket = torch.empty(2 * cols, device=cuda)
        tops.layernorm_ip_bwd(dy, y, rs, gam, bet, dgamma=bucket[:cols], dbeta=bucket[cols:])
        want = bucket.clone()
        comm.allreduce_ln_params(bucket)
        torch.cuda.synchronize()
        assert torch.equal(bucket, want)
    finally:
        comm.close()
