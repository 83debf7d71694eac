"""Long rows: softmax / attention-dropout rows with S > 1024 and LayerNorm
rows with H > 2048 (the paper sweeps S up to 3072; the
reference's softmax and LayerNorm take any row length,
ops_reference.cpp:47-65, 104-145).  S % 128 == 0 up to 16384 runs the
row-group kernels (W warps per row, softmax_kernels.cu), other lengths the
generic kernels; both against the CPU oracle with the tolerances of
test_gpu_parity.py (P: 1e-5*|ref| + 1e-9, dZ: 1e-5*|ref| + 1e-8, D/masks
bit-exact)."""
import numpy as np
import pytest

from test_gpu_parity import (_close_nan, _masked_scores, bits_to_dev, rel_err, to_dev,
                             unpack)

pytestmark = pytest.mark.gpu

# Forward 8 / backward 4 chunks per warp, W from {2,3,4,6,8,12,16}: 1152
# (9 chunks: W=2 fwd with 9 of 16 slots), 1536 (W=2 fwd / 3 bwd), 2176
# (17 chunks, ragged), 3072 (W=3 / 6), 6144 (W=6 / 12), 12288 (W=12 / 16x8),
# 16384 (W=16, 512-thread CTAs); 2050 and 20000: the generic kernel (not a
# multiple of 128 / longer than 16384).
LONG_COLS = [1152, 1536, 2048, 2176, 3072, 4096, 6144, 8192, 12288, 16384, 2050, 20000]


@pytest.mark.parametrize("cols", LONG_COLS)
def test_long_softmax_dropout_supplied_mask(tops, port, cuda, cols):
    import torch
    rows = 37 if cols <= 4096 else 9
    g = np.random.default_rng(cols)
    z = (g.standard_normal((rows, cols)) * 3).astype(np.float32)
    p = 0.1
    bits = tops.bernoulli_keep_bits(rows * cols, p, 4321)  # the reference's stream
    keep = port.bernoulli_keep(rows * cols, p, 4321)
    mask = bits_to_dev(bits, cuda)
    P, D, _ = tops.softmax_dropout_fwd(to_dev(z, cuda), p, mask=mask)
    Pp = tops.softmax_ip_fwd(to_dev(z, cuda))
    torch.cuda.synchronize()
    rP = port.softmax_fwd(z)
    Pg = P.cpu().numpy()
    assert np.all(np.abs(Pg - rP) <= 1e-5 * np.abs(rP) + 1e-9)
    assert np.array_equal(Pp.cpu().numpy(), Pg)  # plain == fused P, bitwise
    assert np.array_equal(D.cpu().numpy(), port.dropout_apply(Pg, keep, p).reshape(rows, cols))

    dD = g.standard_normal((rows, cols)).astype(np.float32)
    dZ, Drec = tops.attn_probs_bwd(to_dev(dD, cuda), P, mask, p, write_d=True)
    dZ2, _ = tops.attn_probs_bwd(to_dev(dD, cuda), P, mask, p, write_d=False)
    torch.cuda.synchronize()
    rdZ = port.softmax_bwd(port.dropout_apply(dD, keep, p).reshape(rows, cols), Pg)
    assert np.all(np.abs(dZ.cpu().numpy() - rdZ) <= 1e-5 * np.abs(rdZ) + 1e-8)
    assert torch.equal(Drec, D)
    assert torch.equal(dZ2, dZ)


@pytest.mark.parametrize("cols", LONG_COLS)
def test_long_plain_softmax(tops, port, cuda, cols):
    import torch
    rows = 21
    g = np.random.default_rng(cols + 1)
    z = (g.standard_normal((rows, cols)) * 4).astype(np.float32)
    P = tops.softmax_ip_fwd(to_dev(z, cuda))
    dP = g.standard_normal((rows, cols)).astype(np.float32)
    dZ = tops.softmax_ip_bwd(to_dev(dP, cuda), P)
    torch.cuda.synchronize()
    rP = port.softmax_fwd(z)
    assert np.all(np.abs(P.cpu().numpy() - rP) <= 1e-5 * np.abs(rP) + 1e-9)
    rdZ = port.softmax_bwd(dP, P.cpu().numpy())
    assert np.all(np.abs(dZ.cpu().numpy() - rdZ) <= 1e-5 * np.abs(rdZ) + 1e-8)


@pytest.mark.parametrize("cols", [2048, 3072, 2050])
def test_long_softmax_dropout_philox(tops, port, cuda, cols):
    """Philox masks on long rows: the keep rate, D from the written mask,
    the same bits run to run, and row shards with global offsets reproduce
    the unsharded mask (the generic kernel writes whole mask words, no
    per-element atomics: a word shared by two rows is written by both)."""
    import torch
    rows = 40
    g = np.random.default_rng(cols + 2)
    z = (g.standard_normal((rows, cols)) * 2).astype(np.float32)
    p = 0.25
    zt = to_dev(z, cuda)
    P, D, mask = tops.softmax_dropout_fwd(zt, p, seed=91)
    torch.cuda.synchronize()
    keep = unpack(mask, rows * cols)
    assert abs(keep.mean() - (1 - p)) < 0.01
    assert np.array_equal(D.cpu().numpy(),
                          port.dropout_apply(P.cpu().numpy(), keep, p).reshape(rows, cols))
    # the same bits as the hidden-dropout kernel's Philox stream of that length
    _, mdrop = tops.dropout_fwd(torch.zeros(rows * cols, device=cuda), p, seed=91)
    torch.cuda.synchronize()
    assert np.array_equal(unpack(mdrop, rows * cols), keep)
    # stale bits in a caller-supplied mask buffer are overwritten, not OR-ed
    junk = torch.full_like(mask, -1)
    _, _, m2 = tops.softmax_dropout_fwd(zt, p, seed=91, mask=junk, generate=True)
    torch.cuda.synchronize()
    assert np.array_equal(unpack(m2, rows * cols), keep)
    if cols % 128 == 0:
        half = rows // 2
        _, _, ma = tops.softmax_dropout_fwd(zt[:half].contiguous(), p, seed=91, offset=0)
        _, _, mb = tops.softmax_dropout_fwd(zt[half:].contiguous(), p, seed=91,
                                            offset=half * cols)
        torch.cuda.synchronize()
        assert np.array_equal(
            np.concatenate([unpack(ma, half * cols), unpack(mb, (rows - half) * cols)]), keep)


@pytest.mark.parametrize("fill", [-np.inf, float(np.finfo(np.float32).min)])
@pytest.mark.parametrize("frac", [0.5, 1.0])
@pytest.mark.parametrize("cols", [2048, 3072])
def test_long_softmax_masked_scores(tops, port, cuda, cols, fill, frac):
    import torch
    rows = 12
    z = _masked_scores(rows, cols, fill, frac, cols + int(frac * 10))
    p = 0.1
    bits = tops.bernoulli_keep_bits(rows * cols, p, 7)
    keep = port.bernoulli_keep(rows * cols, p, 7)
    mask = bits_to_dev(bits, cuda)
    P, D, _ = tops.softmax_dropout_fwd(to_dev(z, cuda), p, mask=mask)
    torch.cuda.synchronize()
    rP = port.softmax_fwd(z)
    Pg = P.cpu().numpy()
    assert _close_nan(Pg, rP, 1e-5, 1e-9)
    rD = port.dropout_apply(Pg, keep, p).reshape(rows, cols)
    assert np.array_equal(D.cpu().numpy(), rD, equal_nan=True)
    dD = np.random.default_rng(3).standard_normal((rows, cols)).astype(np.float32)
    dZ, _ = tops.attn_probs_bwd(to_dev(dD, cuda), P, mask, p)
    torch.cuda.synchronize()
    rdZ = port.softmax_bwd(port.dropout_apply(dD, keep, p).reshape(rows, cols), Pg)
    assert _close_nan(dZ.cpu().numpy(), rdZ, 1e-5, 1e-8)


def test_long_softmax_many_rows(tops, port, cuda):
    """Enough rows that every CTA of the row-group grid loops (the per-row
    parity slots of the cross-warp exchange are reused many times)."""
    import torch
    rows, cols = 6144, 2048
    g = np.random.default_rng(11)
    z = (g.standard_normal((rows, cols)) * 3).astype(np.float32)
    dD = g.standard_normal((rows, cols)).astype(np.float32)
    P, D, mask = tops.softmax_dropout_fwd(to_dev(z, cuda), 0.1, seed=5)
    dZ, _ = tops.attn_probs_bwd(to_dev(dD, cuda), P, mask, 0.1)
    torch.cuda.synchronize()
    sel = np.r_[0:64, rows - 64:rows, 1000:1100]
    rP = port.softmax_fwd(z[sel])
    Pg = P.cpu().numpy()
    assert np.all(np.abs(Pg[sel] - rP) <= 1e-5 * np.abs(rP) + 1e-9)
    keep = unpack(mask, rows * cols).reshape(rows, cols)
    rdP = port.dropout_apply(np.ascontiguousarray(dD[sel]), keep[sel].ravel(), 0.1)
    rdZ = port.softmax_bwd(rdP.reshape(len(sel), cols), np.ascontiguousarray(Pg[sel]))
    assert np.all(np.abs(dZ.cpu().numpy()[sel] - rdZ) <= 1e-5 * np.abs(rdZ) + 1e-8)


# ------------------------------------------------------------- LayerNorm
# 2052..16384: the cluster backward (K = 2..8 CTAs); 20000: generic kernels
LN_LONG_COLS = [2560, 3072, 4096, 5120, 8192, 12288, 2052, 3000, 16384, 20000]


@pytest.mark.parametrize("cols", LN_LONG_COLS)
def test_long_layernorm(tops, port, cuda, cols):
    import torch
    rows = 67
    g = np.random.default_rng(cols)
    x = (g.standard_normal((rows, cols)) * 1.5 + 0.3).astype(np.float32)
    x[5] += 300.0  # a row with |mean| >> std
    gam = (1 + 0.2 * g.standard_normal(cols)).astype(np.float32)
    bet = (0.1 * g.standard_normal(cols)).astype(np.float32)
    dy = g.standard_normal((rows, cols)).astype(np.float32)
    T = lambda a: to_dev(a, cuda)  # noqa: E731
    y, rstd = tops.layernorm_ip_fwd(T(x), T(gam), T(bet))
    dx, dg, db = tops.layernorm_ip_bwd(T(dy), y, rstd, T(gam), T(bet))
    torch.cuda.synchronize()
    ry, rrs, _ = port.ln_fwd(x, gam, bet, 1e-5)
    assert rel_err(y.cpu().numpy(), ry) <= 1e-5
    assert np.abs(rstd.cpu().numpy().astype(np.float64) / rrs - 1).max() <= 1e-6
    yg, rsg = y.cpu().numpy(), rstd.cpu().numpy()
    rdx, _, _ = port.ln_bwd(dy, yg, rsg, gam, bet, False)
    _, rdg, rdb = port.ln_bwd(dy, yg, rsg, gam, bet, True)
    assert rel_err(dx.cpu().numpy(), rdx) <= 1e-5
    assert rel_err(dg.cpu().numpy(), rdg) <= 1e-5
    assert rel_err(db.cpu().numpy(), rdb) <= 1e-5


@pytest.mark.parametrize("cols", [2048, 3072, 8192])
def test_long_softmax_special_rows(tops, port, cuda, cols):
    """NaN anywhere -> NaN row, +inf -> NaN row, one finite score among -inf
    (P = 1 there), huge logits, masked halves: as the oracle, on the
    row-group kernels (the chunk holding the special value belongs to a
    different warp of the group than the row's max)."""
    import torch
    from test_gpu_parity import _close_nan
    inf, nan, big = np.inf, np.nan, float(np.finfo(np.float32).max)
    rows = []
    r = np.zeros(cols, np.float32); r[cols - 3] = nan; rows.append(r)
    r = np.zeros(cols, np.float32); r[130] = inf; rows.append(r)
    r = np.full(cols, -inf, np.float32); r[cols // 2 + 5] = 2.0; rows.append(r)
    r = np.full(cols, -big, np.float32); r[777] = big; rows.append(r)
    r = np.linspace(-100, 0, cols).astype(np.float32); rows.append(r)
    r = np.random.default_rng(cols).standard_normal(cols).astype(np.float32); r[: cols // 2] = -inf
    rows.append(r)
    z = np.stack(rows)
    P = tops.softmax_ip_fwd(to_dev(z, cuda))
    Pd, D, m = tops.softmax_dropout_fwd(to_dev(z, cuda), 0.1, seed=2)
    torch.cuda.synchronize()
    rP = port.softmax_fwd(z)
    assert _close_nan(P.cpu().numpy(), rP, 1e-5, 1e-9)
    assert np.array_equal(Pd.cpu().numpy(), P.cpu().numpy(), equal_nan=True)


@pytest.mark.parametrize("cols", [3072, 8192])
def test_long_layernorm_special_rows(tops, port, cuda, cols):
    """A NaN in a row makes that row's y and rstd NaN (the reference's double
    sums propagate it) and leaves the other rows -- on the same row group /
    cluster tile -- untouched; a constant row has var 0 -> rstd = 1/sqrt(eps)."""
    import torch
    from test_gpu_parity import _close_nan
    g = np.random.default_rng(cols)
    x = g.standard_normal((6, cols)).astype(np.float32)
    x[1, cols // 3] = np.nan
    x[3, :] = 2.5
    gam = (1 + 0.2 * g.standard_normal(cols)).astype(np.float32)
    bet = (0.1 * g.standard_normal(cols)).astype(np.float32)
    y, rstd = tops.layernorm_ip_fwd(to_dev(x, cuda), to_dev(gam, cuda), to_dev(bet, cuda))
    torch.cuda.synchronize()
    ry, rrs, _ = port.ln_fwd(x, gam, bet, 1e-5)
    assert _close_nan(y.cpu().numpy(), ry, 1e-5, 1e-5)
    assert _close_nan(rstd.cpu().numpy(), rrs, 1e-6, 0)
