"""softmax -> dropout_recompute forward with the reference's own mask stream
(BoolMask::bernoulli_keep(shape, p, seed), tensor.cpp:186-203) generated
INSIDE the softmax kernel (tempo_softmax_dropout_fwd_refmask; generator and
consumer warps in one CTA per 2^19-output chunk, softmax_kernels.cu).

The mask must be the reference's stream bit for bit -- against the host
engine (the reference's own std::mt19937_64 + distribution) for small
streams, and against the device keep-bit generator (itself checked against
the host in test_mt_jump.py) at larger sizes and shard offsets -- and P, D
must be bitwise those of the supplied-mask forward on that mask.  Shapes
outside the fused kernel's envelope take the separate passes and must give
the same bits."""
import numpy as np
import pytest

from test_gpu_parity import to_dev, unpack

pytestmark = pytest.mark.gpu

CHUNK = 1 << 19


def _check(tops, port, cuda, rows, cols, p, seed, offset, host_ref):
    import torch
    g = np.random.default_rng(rows * cols + seed)
    z = to_dev((g.standard_normal((rows, cols)) * 3).astype(np.float32), cuda)
    n = rows * cols
    P, D, m = tops.softmax_dropout_fwd_refmask(z, p, seed, offset=offset)
    ref_bits = tops.bernoulli_keep_bits_device(n, p, seed, offset=offset)
    P2, D2, _ = tops.softmax_dropout_fwd(z, p, mask=ref_bits)
    torch.cuda.synchronize()
    assert torch.equal(m, ref_bits)
    assert torch.equal(P, P2) and torch.equal(D, D2)
    if host_ref:
        keep = port.bernoulli_keep(offset + n, p, seed)[offset:]
        assert np.array_equal(unpack(m, n), keep)
    # the fused backward reads the generated mask
    dD = to_dev(g.standard_normal((rows, cols)).astype(np.float32), cuda)
    dZ, _ = tops.attn_probs_bwd(dD, P, m, p)
    dZ2, _ = tops.attn_probs_bwd(dD, P2, ref_bits, p)
    torch.cuda.synchronize()
    assert torch.equal(dZ, dZ2)


@pytest.mark.parametrize("rows,cols", [(2048, 512), (1024, 1024), (8192, 128), (4096, 256)])
def test_refmask_fused_shapes(tops, port, cuda, rows, cols):
    """One to two chunks per shape, each row length of the fused kernel."""
    _check(tops, port, cuda, rows, cols, 0.1, 1234 + cols, 0, host_ref=True)


@pytest.mark.parametrize("offset", [CHUNK, 7 * CHUNK, 1024 * CHUNK + 3 * CHUNK])
def test_refmask_shard_offsets(tops, port, cuda, offset):
    """Row shards start at chunk-aligned global offsets (rank * 2^28 for the
    N=8 attention shards: level-2 jump digits)."""
    _check(tops, port, cuda, 4096, 512, 0.1, 99, offset, host_ref=offset < 8 * CHUNK)


def test_refmask_many_chunks(tops, port, cuda):
    """32 chunks (2^24 elements), more CTAs than one wave per SM pair."""
    _check(tops, port, cuda, 32768, 512, 0.1, 7, 0, host_ref=False)


@pytest.mark.parametrize("rows,cols,offset", [(300, 384, 64), (100, 512, 0), (64, 2048, 0),
                                              (16, 512, 32 * 5)])
def test_refmask_fallback_shapes(tops, port, cuda, rows, cols, offset):
    """Outside the fused envelope (row length, ragged chunk, unaligned offset):
    the separate generation + supplied-mask passes, the same contract."""
    _check(tops, port, cuda, rows, cols, 0.25, 5, offset, host_ref=True)


@pytest.mark.parametrize("p", [0.0, 0.5])
def test_refmask_probabilities(tops, port, cuda, p):
    _check(tops, port, cuda, 2048, 512, p, 11, 0, host_ref=True)


def test_refmask_without_d(tops, cuda):
    import torch
    z = torch.randn(2048, 512, device=cuda)
    P, D, m = tops.softmax_dropout_fwd_refmask(z, 0.1, 3, write_d=False)
    P2, _, m2 = tops.softmax_dropout_fwd_refmask(z, 0.1, 3)
    torch.cuda.synchronize()
    assert D is None and torch.equal(P, P2) and torch.equal(m, m2)


def test_refmask_argument_errors(tops, cuda):
    import torch
    z = torch.randn(64, 512, device=cuda)
    with pytest.raises(tops.TempoError):
        tops.softmax_dropout_fwd_refmask(z, 0.1, 1, offset=5)  # offset % 32
    with pytest.raises(tops.TempoError):
        tops.softmax_dropout_fwd_refmask(z, 1.0, 1)  # p >= 1
