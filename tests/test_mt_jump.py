"""The reference's mask stream (std::mt19937_64 behind BoolMask::bernoulli_keep,
tensor.cpp:186-203) reproduced by jump-ahead.

CPU: the host construction (characteristic polynomial by Berlekamp-Massey,
x^J mod P, XOR of windows) against the oracle's sequential engine
(oracle/tempo_oracle.c, itself pinned against std::mt19937_64 by
test_oracle.py) at offsets inside and across 312-word blocks and chunks.
GPU: the device generator's keep bits against the host stream
(tempo_bernoulli_keep_bits_host = the reference's own engine + distribution),
bit for bit, over several chunks, seeds, probabilities and shard offsets."""
import numpy as np
import pytest

CHUNK = 1 << 19  # kMtChunk (mt19937.h)


@pytest.mark.parametrize("seed", [5489, 42, 0xDEADBEEFCAFE])
def test_jump_ahead_matches_sequential_engine(port, seed):
    from paper_2210_10246_b200 import ops
    ref = port.mt64_stream(seed, 3 * 312 + 1_000_000 + 16)
    for steps in (0, 1, 155, 311, 312, 313, 999, 1_000_000):
        got = ops.mt_outputs_after(seed, steps, 16)
        assert np.array_equal(got, ref[steps:steps + 16]), steps


def test_jump_ahead_far(port):
    """A jump of many chunks, checked against the sequential engine."""
    from paper_2210_10246_b200 import ops
    steps = 3 * CHUNK + 77
    ref = port.mt64_stream(7, steps + 8)
    assert np.array_equal(ops.mt_outputs_after(7, steps, 8), ref[steps:])


def test_keep_bits_argument_errors():
    from paper_2210_10246_b200 import ops
    from paper_2210_10246_b200._capi import lib
    L = lib()
    assert L.tempo_bernoulli_keep_bits(10, 1.0, 1, 0, None, None, 0, None) == 3  # p >= 1
    assert L.tempo_bernoulli_keep_bits(10, 0.1, 1, 5, None, None, 0, None) == 3  # offset % 32
    assert L.tempo_bernoulli_keep_bits(0, 0.1, 1, 0, None, None, 0, None) == 0   # empty
    assert L.tempo_bernoulli_keep_bits_workspace_size(0, 100) > 0
    del ops


def _unpack(words, n):
    return np.unpackbits(np.asarray(words).view(np.uint8), bitorder="little")[:n]


@pytest.mark.gpu
@pytest.mark.parametrize("n,p,seed", [
    (1000, 0.1, 3),                 # one partial word tail, one chunk
    (CHUNK + 4096 + 17, 0.25, 11),  # two chunks, ragged end
    (5 * CHUNK, 0.1, 123456789),    # several chunks
    (40 * CHUNK + 96, 0.5, 99),     # crosses a level-1 group (32 chunks)
    (3000, 0.0, 5),                 # p = 0: all kept
])
def test_device_stream_matches_reference(tops, cuda, n, p, seed):
    import torch
    dev = tops.bernoulli_keep_bits_device(n, p, seed)
    torch.cuda.synchronize()
    host = tops.bernoulli_keep_bits(n, p, seed)
    assert np.array_equal(dev.cpu().numpy().view(np.uint32), host)


@pytest.mark.gpu
def test_device_stream_shards(tops, cuda):
    """Row shards with global offsets reproduce the unsharded stream (the
    multi-GPU layout: rank r generates its slice by jumping to its offset)."""
    import torch
    n, p, seed = 3 * CHUNK + 1000, 0.1, 2024
    full = tops.bernoulli_keep_bits(n, p, seed)
    bits = _unpack(full, n)
    for off, cnt in [(0, 64), (CHUNK - 32, 96), (CHUNK, CHUNK), (2 * CHUNK + 320, n - 2 * CHUNK - 320),
                     (37 * 32, 5000)]:
        part = tops.bernoulli_keep_bits_device(cnt, p, seed, offset=off)
        torch.cuda.synchronize()
        assert np.array_equal(_unpack(part.cpu().numpy(), cnt), bits[off:off + cnt]), (off, cnt)


@pytest.mark.gpu
def test_device_stream_feeds_the_ops(tops, port, cuda):
    """End to end: the device-generated reference mask drives the fused
    softmax+dropout forward (SUPPLIED mode) exactly like the host mask."""
    import torch
    rows, cols, p = 64, 512, 0.1
    seed = tops.mask_stream_seed(1234, 5, 0)  # encoder.cpp:168-169, site 0
    g = np.random.default_rng(3)
    z = torch.from_numpy(g.standard_normal((rows, cols)).astype(np.float32)).to(cuda)
    m_dev = tops.bernoulli_keep_bits_device(rows * cols, p, seed)
    m_host = torch.from_numpy(tops.bernoulli_keep_bits(rows * cols, p, seed).view(np.int32)).to(cuda)
    P1, D1, _ = tops.softmax_dropout_fwd(z, p, mask=m_dev)
    P2, D2, _ = tops.softmax_dropout_fwd(z, p, mask=m_host)
    assert torch.equal(D1, D2) and torch.equal(m_dev, m_host)


def test_oracle_keep_bits_at_offset(port):
    """The oracle's offset stream (engine stepped sequentially past the
    offset) agrees with its own whole-stream bernoulli_keep."""
    n, off, p, seed = 5000, 12345, 0.1, 77
    whole = port.bernoulli_keep(off + n, p, seed)
    got = _unpack(port.bernoulli_keep_bits_at(off, n, p, seed), n)
    assert np.array_equal(got, whole[off:])


ATT_SHARD = 1 << 28  # attention elements per rank at B=64 (64*16*512*512)


@pytest.mark.gpu
@pytest.mark.parametrize("rank", [2, 7])
def test_device_stream_level2_shard_offsets(tops, port, cuda, rank):
    """The N=8 attention shards start at rank * 2^28 elements = chunk
    rank * 512: ranks >= 2 take the level-2 jump digits (32^2 chunks).  The
    device stream there is checked against the engine stepped sequentially
    past the offset (not the jump construction)."""
    import torch
    off, n, p, seed = rank * ATT_SHARD, 3 * CHUNK + 96, 0.1, 4242
    dev = tops.bernoulli_keep_bits_device(n, p, seed, offset=off)
    torch.cuda.synchronize()
    assert np.array_equal(dev.cpu().numpy().view(np.uint32),
                          port.bernoulli_keep_bits_at(off, n, p, seed))


@pytest.mark.gpu
def test_device_stream_full_attention_mask(tops, cuda):
    """One whole 268,435,456-element BERT-large attention mask (512 chunks)
    against the reference's own host stream."""
    import torch
    n, p, seed = ATT_SHARD, 0.1, 1234
    dev = tops.bernoulli_keep_bits_device(n, p, seed)
    torch.cuda.synchronize()
    host = tops.bernoulli_keep_bits(n, p, seed)
    assert np.array_equal(dev.cpu().numpy().view(np.uint32), host)
