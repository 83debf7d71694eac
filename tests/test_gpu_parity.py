"""Parity of the sm_100a kernels (through the C-ABI) with the CPU oracle
(oracle/tempo_oracle.c, itself pinned bit-exact to the reference in
test_oracle.py) on identical seeded inputs.

Tolerances (the reference's rel_err = |a-b| / max(1,|a|,|b|),
gradcheck.cpp:15-17, unless stated):
  GELU   mask bits: bit-exact.  y: <= 8 ulp (bound of the fp32 fast path,
         checked on every fp32 input by tests/test_gpu_sweep.py) and
         bit-exact in the fp64 window |x - x*| < 1/64.  dx on identical (dy, y, mask):
         rel_err <= 1e-5.  fwd->bwd chain: rel_err <= 1e-5.
  LN     y, dx: rel_err <= 1e-5; rstd: rel <= 1e-6; dgamma/dbeta vs the
         reference's F64 path: rel_err <= 1e-5; run-to-run bitwise.
  softmax P: |d| <= 1e-5*|ref| + 1e-9; dZ: |d| <= 1e-5*|ref| + 1e-8.
  dropout D, dP, hidden y/dx: bit-exact; recomputed D == forward D bitwise.
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

XSTAR_D = -0.7517915246935645


def rel_err(a, b):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    both_nan = np.isnan(a) & np.isnan(b)
    d = np.abs(a - b) / np.maximum(1.0, np.maximum(np.abs(a), np.abs(b)))
    d[both_nan] = 0.0
    return float(d.max()) if d.size else 0.0


def ulp_diff(a, b):
    a = np.asarray(a, np.float32).view(np.int32).astype(np.int64)
    b = np.asarray(b, np.float32).view(np.int32).astype(np.int64)
    a = np.where(a < 0, -(a & 0x7FFFFFFF), a)
    b = np.where(b < 0, -(b & 0x7FFFFFFF), b)
    return np.abs(a - b)


def unpack(bits_t, n):
    b = bits_t.cpu().numpy().view(np.uint32)
    return np.unpackbits(b.view(np.uint8), bitorder="little")[:n]


def to_dev(a, cuda):
    import torch
    return torch.from_numpy(np.ascontiguousarray(a)).to(cuda)


def bits_to_dev(bits_np, cuda):
    import torch
    return torch.from_numpy(bits_np.view(np.int32).copy()).to(cuda)


# ------------------------------------------------------------------- GELU
def gelu_inputs(n, seed):
    g = np.random.default_rng(seed)
    x = (g.standard_normal(n) * 2.5).astype(np.float32)
    k = min(n, 64)
    x[:k] = np.linspace(-0.8, -0.7, k, dtype=np.float32)  # the minimum window
    if n > 200:
        x[100:110] = [0.0, -0.0, 13.5, -13.5, -20.0, 40.0, np.inf, -np.inf, np.nan, 1e-42]
    return x


@pytest.mark.parametrize("n,shift", [(1, 0), (31, 0), (129, 0), (4101, 0), (1024 * 3072, 0),
                                     (4101, 1), (70000, 3)])
def test_gelu_forward_exact(tops, port, table_text, cuda, n, shift):
    """The reference-exact forward (tempo_gelu_ip_fwd_exact: the reference's
    fp64 formula for every element) against the oracle (the same formula with
    glibc's erfc): <= 1 ulp, in practice bitwise (CUDA's and glibc's double
    erfc agree to ~1 double ulp); mask bit-exact; unaligned views (shift)
    take the word loop."""
    import torch
    table = tops.GeluTable(table_text)
    x = gelu_inputs(n + shift, n)
    xt = to_dev(x, cuda)[shift:]
    y, mask = tops.gelu_ip_fwd(xt, table, exact=True)
    torch.cuda.synchronize()
    xs = x[shift:]
    ry, rm = port.gelu_fwd(xs, table.info()["x_star"])
    assert np.array_equal(unpack(mask, n), rm)
    yg = y.cpu().numpy()
    assert np.array_equal(np.isnan(yg), np.isnan(ry))
    fin = np.isfinite(ry)
    d = ulp_diff(yg[fin], ry[fin])
    assert d.max(initial=0) <= 1
    assert (d > 0).mean() <= 1e-5 if d.size > 10000 else True
    # the backward of the exact forward's stash, as for the fast one
    dy = np.random.default_rng(n).standard_normal(n).astype(np.float32)
    dx = tops.gelu_ip_bwd(to_dev(dy, cuda), y, mask, table)
    torch.cuda.synchronize()
    pt = port.table(table_text)
    assert rel_err(dx.cpu().numpy(), pt.gelu_bwd(dy, ry, rm)) <= 1e-5


@pytest.mark.parametrize("n", [1, 31, 32, 127, 128, 129, 1000, 4101, 1024 * 3072])
def test_gelu_forward(tops, port, table_text, cuda, n):
    import torch
    table = tops.GeluTable(table_text)
    x = gelu_inputs(n, n)
    y, mask = tops.gelu_ip_fwd(to_dev(x, cuda), table)
    torch.cuda.synchronize()
    ry, rm = port.gelu_fwd(x, table.info()["x_star"])
    assert np.array_equal(unpack(mask, n), rm)
    yg = y.cpu().numpy()
    fin = np.isfinite(ry)
    assert np.array_equal(np.isnan(yg), np.isnan(ry))
    assert ulp_diff(yg[fin], ry[fin]).max(initial=0) <= 8
    win = np.abs(x.astype(np.float64) - XSTAR_D) < 1.0 / 64
    assert np.array_equal(yg[win], ry[win])  # fp64 window: bit-exact
    # padding bits of the last word are zero
    words = mask.cpu().numpy().view(np.uint32)
    if n % 32:
        assert words[-1] >> (n % 32) == 0


def test_gelu_forward_unaligned(tops, port, table_text, cuda):
    import torch
    table = tops.GeluTable(table_text)
    x = gelu_inputs(5001, 3)
    xt = to_dev(np.concatenate([[0.0], x]).astype(np.float32), cuda)[1:]  # 4-byte offset
    y, mask = tops.gelu_ip_fwd(xt, table)
    torch.cuda.synchronize()
    ry, rm = port.gelu_fwd(x, table.info()["x_star"])
    assert np.array_equal(unpack(mask, x.size), rm)
    fin = np.isfinite(ry)
    assert ulp_diff(y.cpu().numpy()[fin], ry[fin]).max() <= 8


@pytest.mark.parametrize("n", [1, 33, 128, 1000, 4101, 1024 * 3072])
def test_gelu_backward_identical_inputs(tops, port, table_text, cuda, n):
    import torch
    table = tops.GeluTable(table_text)
    pt = port.table(table_text)
    x = gelu_inputs(n, 7 + n)
    y, m = port.gelu_fwd(x, pt.x_star)  # the oracle's stash, fed to both
    g = np.random.default_rng(n)
    dy = g.standard_normal(n).astype(np.float32)
    bits = np.packbits(m, bitorder="little")
    bits = np.concatenate([bits, np.zeros((-bits.size) % 4, np.uint8)]).view(np.uint32)
    dx = tops.gelu_ip_bwd(to_dev(dy, cuda), to_dev(y, cuda), bits_to_dev(bits, cuda), table)
    torch.cuda.synchronize()
    rdx = pt.gelu_bwd(dy, y, m)
    assert rel_err(dx.cpu().numpy(), rdx) <= 1e-5


def test_gelu_backward_table_eval_grid(tops, port, table_text, cuda):
    """h(y, m) over a dense grid of outputs incl. clamps, seams and the tail."""
    import torch
    table = tops.GeluTable(table_text)
    pt = port.table(table_text)
    info = table.info()
    ys = np.concatenate([np.linspace(-0.3, 10.0, 200000), [info["y_min"], 0.0, -0.0, 8.0,
                                                           1.8725215943900724, 1e30, -1.0,
                                                           np.inf, -np.inf, np.nan]])
    ys = ys.astype(np.float32)
    for m in (0, 1):
        mm = np.full(ys.size, m, np.uint8)
        bits = np.packbits(mm, bitorder="little")
        bits = np.concatenate([bits, np.zeros((-bits.size) % 4, np.uint8)]).view(np.uint32)
        ones = np.ones(ys.size, np.float32)
        h = tops.gelu_ip_bwd(to_dev(ones, cuda), to_dev(ys, cuda), bits_to_dev(bits, cuda), table)
        torch.cuda.synchronize()
        assert rel_err(h.cpu().numpy(), pt.gelu_bwd(ones, ys, mm)) <= 1e-5


def _extra_tables():
    import json
    import os
    here = os.path.dirname(os.path.abspath(__file__))
    with open(os.path.join(here, "golden", "gelu_tables_extra.json")) as f:
        return json.load(f)


@pytest.mark.parametrize("name", sorted(_extra_tables()))
def test_gelu_backward_other_tables(tops, port, cuda, name):
    """Tables with more segments / other degrees (fitted by the reference):
    the device table is a kernel input, not a compiled-in constant."""
    import torch
    text = _extra_tables()[name]
    table = tops.GeluTable(text)
    pt = port.table(text)
    n = 1 << 20
    x = gelu_inputs(n, 21)
    y, m = port.gelu_fwd(x, pt.x_star)
    dy = np.random.default_rng(22).standard_normal(n).astype(np.float32)
    bits = np.packbits(m, bitorder="little")
    bits = np.concatenate([bits, np.zeros((-bits.size) % 4, np.uint8)]).view(np.uint32)
    dx = tops.gelu_ip_bwd(to_dev(dy, cuda), to_dev(y, cuda), bits_to_dev(bits, cuda), table)
    torch.cuda.synchronize()
    assert rel_err(dx.cpu().numpy(), pt.gelu_bwd(dy, y, m)) <= 1e-5
    # forward mask uses this table's x*
    yg, mg = tops.gelu_ip_fwd(to_dev(x, cuda), table)
    torch.cuda.synchronize()
    assert np.array_equal(unpack(mg, n), m)


def test_gelu_chain_forward_backward(tops, port, table_text, cuda):
    import torch
    table = tops.GeluTable(table_text)
    pt = port.table(table_text)
    n = 1 << 20
    x = gelu_inputs(n, 11)
    x[:4096] = np.linspace(-0.77, -0.73, 4096, dtype=np.float32)  # dense around x*
    dy = np.random.default_rng(5).standard_normal(n).astype(np.float32)
    y, mask = tops.gelu_ip_fwd(to_dev(x, cuda), table)
    dx = tops.gelu_ip_bwd(to_dev(dy, cuda), y, mask, table)
    torch.cuda.synchronize()
    ry, rm = port.gelu_fwd(x, pt.x_star)
    rdx = pt.gelu_bwd(dy, ry, rm)
    assert rel_err(dx.cpu().numpy(), rdx) <= 1e-5


def test_gelu_refusals(tops, table_text, cuda):
    import torch
    from paper_2210_10246_b200 import TempoError
    x = torch.randn(64, device=cuda)
    with pytest.raises(TempoError) as e:
        tops.gelu_ip_fwd(x, None)
    assert e.value.kind == "ConfigError"
    unver = tops.GeluTable(table_text.replace("max_err=7.9034905239312725e-05", "max_err=-1"))
    y, m = tops.gelu_ip_fwd(x, unver)  # forward builds
    with pytest.raises(TempoError) as e:
        tops.gelu_ip_bwd(torch.ones_like(x), y, m, unver)
    assert e.value.kind == "ConfigError" and "sweep-verified" in str(e.value)


# -------------------------------------------------------------- LayerNorm
def ln_inputs(rows, cols, seed):
    g = np.random.default_rng(seed)
    x = (g.standard_normal((rows, cols)) * 1.7 + 0.4).astype(np.float32)
    gam = (np.sign(g.standard_normal(cols)) * (1 + 0.2 * g.standard_normal(cols))).astype(np.float32)
    bet = (0.1 * g.standard_normal(cols)).astype(np.float32)
    dy = g.standard_normal((rows, cols)).astype(np.float32)
    return x, gam, bet, dy


@pytest.mark.parametrize("rows,cols", [(1, 768), (7, 1024), (333, 768), (64, 4), (5, 1000),
                                       (3, 2052), (16384, 768), (100, 256), (37, 512), (9, 1536)])
def test_layernorm_forward(tops, port, cuda, rows, cols):
    import torch
    x, gam, bet, _ = ln_inputs(rows, cols, rows * cols)
    y, rstd = tops.layernorm_ip_fwd(to_dev(x, cuda), to_dev(gam, cuda), to_dev(bet, cuda))
    torch.cuda.synchronize()
    ry, rrs, _ = port.ln_fwd(x, gam, bet, 1e-5)
    assert rel_err(y.cpu().numpy(), ry) <= 1e-5
    assert np.abs(rstd.cpu().numpy().astype(np.float64) / rrs - 1).max() <= 1e-6


@pytest.mark.parametrize("rows,cols", [(1, 768), (7, 1024), (333, 768), (64, 4), (5, 1000),
                                       (3, 2052), (16384, 768), (100, 256), (37, 512), (9, 1536)])
def test_layernorm_backward_identical_inputs(tops, port, cuda, rows, cols):
    import torch
    x, gam, bet, dy = ln_inputs(rows, cols, 3 + rows * cols)
    ry, rrs, _ = port.ln_fwd(x, gam, bet, 1e-5)
    args = [to_dev(a, cuda) for a in (dy, ry, rrs, gam, bet)]
    dx, dg, db = tops.layernorm_ip_bwd(*args)
    torch.cuda.synchronize()
    rdx, _, _ = port.ln_bwd(dy, ry, rrs, gam, bet, False)
    _, dg64, db64 = port.ln_bwd(dy, ry, rrs, gam, bet, True)
    assert rel_err(dx.cpu().numpy(), rdx) <= 1e-5
    assert rel_err(dg.cpu().numpy(), dg64) <= 1e-5
    assert rel_err(db.cpu().numpy(), db64) <= 1e-5
    dx2, dg2, db2 = tops.layernorm_ip_bwd(*args)  # fixed reduction order
    torch.cuda.synchronize()
    assert torch.equal(dx, dx2) and torch.equal(dg, dg2) and torch.equal(db, db2)


def test_layernorm_alternating_widths(tops, port, cuda):
    """Same kernels launched with different dynamic smem sizes in turn (a
    per-kernel attribute must not go stale)."""
    import torch
    for rows, cols in [(7, 1024), (5, 768), (9, 1024), (3, 512), (7, 1024)]:
        x, gam, bet, dy = ln_inputs(rows, cols, rows + cols)
        ry, rrs, _ = port.ln_fwd(x, gam, bet, 1e-5)
        y, rstd = tops.layernorm_ip_fwd(to_dev(x, cuda), to_dev(gam, cuda), to_dev(bet, cuda))
        dx, dg, db = tops.layernorm_ip_bwd(to_dev(dy, cuda), to_dev(ry, cuda), to_dev(rrs, cuda),
                                           to_dev(gam, cuda), to_dev(bet, cuda))
        torch.cuda.synchronize()
        assert rel_err(y.cpu().numpy(), ry) <= 1e-5
        rdx, _, _ = port.ln_bwd(dy, ry, rrs, gam, bet, False)
        assert rel_err(dx.cpu().numpy(), rdx) <= 1e-5


def test_layernorm_refusals(tops, cuda):
    import torch
    from paper_2210_10246_b200 import TempoError
    x = torch.randn(2, 4, device=cuda)
    gam = torch.ones(4, device=cuda)
    gam[2] = 1e-13
    with pytest.raises(TempoError) as e:
        tops.layernorm_ip_fwd(x, gam, torch.zeros(4, device=cuda))
    assert e.value.kind == "ParamError" and "gamma" in str(e.value)
    status = torch.zeros(1, dtype=torch.int32, device=cuda)
    tops.layernorm_ip_fwd(x, gam, torch.zeros(4, device=cuda), check_gamma=False,
                          dev_status=status)
    assert int(status.item()) == 3
    with pytest.raises(TempoError) as e:
        tops.layernorm_ip_fwd(x, torch.ones(4, device=cuda), torch.zeros(4, device=cuda), eps=0.0)
    assert e.value.kind == "ParamError"


@pytest.mark.parametrize("offset", [1e2, 1e3, 1e4, -3e3])
@pytest.mark.parametrize("rows,cols", [(64, 1024), (48, 768), (16, 1000), (8, 1536), (4, 2052)])
def test_layernorm_forward_large_mean(tops, port, cuda, rows, cols, offset):
    """Rows with |mean| >> std: the reference sums in fp64 and stores
    float(mean) (kernels.cpp:165-176), so the row mean must be that rounding,
    not an fp32 tree sum's (which drifts by several ulps of the mean and puts
    y 1e-4 off at |mean|/std = 1000)."""
    import torch
    g = np.random.default_rng(int(abs(offset)) + cols)
    x = (g.standard_normal((rows, cols)) + offset).astype(np.float32)
    gam = (1 + 0.2 * g.standard_normal(cols)).astype(np.float32)
    bet = (0.1 * g.standard_normal(cols)).astype(np.float32)
    y, rstd = tops.layernorm_ip_fwd(to_dev(x, cuda), to_dev(gam, cuda), to_dev(bet, cuda))
    torch.cuda.synchronize()
    ry, rrs, _ = port.ln_fwd(x, gam, bet, 1e-5)
    assert rel_err(y.cpu().numpy(), ry) <= 1e-5
    assert np.abs(rstd.cpu().numpy().astype(np.float64) / rrs - 1).max() <= 1e-6


# ------------------------------------------------- softmax + attention dropout
@pytest.mark.parametrize("rows,cols", [(1, 512), (24, 512), (7, 384), (9, 1024), (5, 100),
                                       (3, 77), (12 * 512, 512), (10, 128), (6, 256), (5, 768),
                                       (3, 1280)])
def test_softmax_dropout_supplied_mask(tops, port, cuda, rows, cols):
    import torch
    g = np.random.default_rng(rows + cols)
    z = (g.standard_normal((rows, cols)) * 3).astype(np.float32)
    p = 0.1
    bits = tops.bernoulli_keep_bits(rows * cols, p, 1234)  # the reference's stream
    keep = port.bernoulli_keep(rows * cols, p, 1234)
    mask = bits_to_dev(bits, cuda)
    P, D, mask_out = tops.softmax_dropout_fwd(to_dev(z, cuda), p, mask=mask)
    torch.cuda.synchronize()
    rP = port.softmax_fwd(z)
    Pg = P.cpu().numpy()
    assert np.all(np.abs(Pg - rP) <= 1e-5 * np.abs(rP) + 1e-9)
    assert np.array_equal(D.cpu().numpy(), port.dropout_apply(Pg, keep, p).reshape(rows, cols))
    assert np.array_equal(unpack(mask_out, rows * cols), keep)

    dD = g.standard_normal((rows, cols)).astype(np.float32)
    dZ, Drec = tops.attn_probs_bwd(to_dev(dD, cuda), P, mask, p, write_d=True)
    torch.cuda.synchronize()
    rdP = port.dropout_apply(dD, keep, p).reshape(rows, cols)
    rdZ = port.softmax_bwd(rdP, Pg)
    dZg = dZ.cpu().numpy()
    assert np.all(np.abs(dZg - rdZ) <= 1e-5 * np.abs(rdZ) + 1e-8)
    assert torch.equal(Drec, D)  # recompute == forward D, bitwise


@pytest.mark.parametrize("rows,cols", [(48, 512), (200, 100)])
def test_softmax_dropout_philox(tops, port, cuda, rows, cols):
    import torch
    g = np.random.default_rng(1)
    z = (g.standard_normal((rows, cols)) * 2).astype(np.float32)
    p = 0.25
    zt = to_dev(z, cuda)
    P, D, mask = tops.softmax_dropout_fwd(zt, p, seed=77)
    torch.cuda.synchronize()
    keep = unpack(mask, rows * cols)
    assert abs(keep.mean() - (1 - p)) < 0.015  # >= 20000 draws: 5 sigma
    assert np.array_equal(D.cpu().numpy(), port.dropout_apply(P.cpu().numpy(), keep, p).reshape(rows, cols))
    # same seed -> same mask; row shards with global offsets -> same mask
    _, _, mask2 = tops.softmax_dropout_fwd(zt, p, seed=77)
    assert torch.equal(mask, mask2)
    if cols % 128 == 0:
        half = rows // 2
        _, _, ma = tops.softmax_dropout_fwd(zt[:half].contiguous(), p, seed=77, offset=0)
        _, _, mb = tops.softmax_dropout_fwd(zt[half:].contiguous(), p, seed=77, offset=half * cols)
        torch.cuda.synchronize()
        assert np.array_equal(np.concatenate([unpack(ma, half * cols), unpack(mb, (rows - half) * cols)]), keep)


@pytest.mark.parametrize("scale", [1, 4, 16])
def test_softmax_accuracy_margin(tops, port, cuda, scale):
    """The SFU-exp forward (ex2.approx on an FMA-split exponent plus the TwoSum
    error of z - max, softmax_kernels.cu) keeps P an order of magnitude inside
    the 1e-5 contract at logit scales up to 16 (measured <= 5.1e-7)."""
    import torch
    g = np.random.default_rng(scale)
    z = (g.standard_normal((4096, 512)) * scale).astype(np.float32)
    P, _, _ = tops.softmax_dropout_fwd(to_dev(z, cuda), 0.1, seed=3)
    torch.cuda.synchronize()
    rP = port.softmax_fwd(z)
    big = rP > 1e-30
    rel = np.abs(P.cpu().numpy() - rP)[big] / rP[big]
    assert float(rel.max()) <= 1e-6, float(rel.max())


def _masked_scores(rows, cols, fill, frac, seed):
    """randn*3 scores with a fraction `frac` of each row set to `fill` (the
    attention-mask values HF / the reference's users put in: -inf,
    finfo(float32).min, -1e4); row 0 fully masked when frac == 1."""
    g = np.random.default_rng(seed)
    z = (g.standard_normal((rows, cols)) * 3).astype(np.float32)
    if frac > 0:
        k = int(round(frac * cols))
        for r in range(rows):
            z[r, g.permutation(cols)[:k]] = fill
    return z


def _close_nan(a, b, rtol, atol):
    """|a-b| <= rtol*|b| + atol where b is finite; NaN exactly where b is NaN."""
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    if not np.array_equal(np.isnan(a), np.isnan(b)):
        return False
    f = ~np.isnan(b)
    return bool(np.all(np.abs(a[f] - b[f]) <= rtol * np.abs(b[f]) + atol))


@pytest.mark.parametrize("fill", [-np.inf, float(np.finfo(np.float32).min), -1e4])
@pytest.mark.parametrize("frac", [0.0, 0.5, 1.0])
@pytest.mark.parametrize("rows,cols", [(64, 512), (9, 1024), (5, 100)])
def test_softmax_masked_scores(tops, port, cuda, rows, cols, fill, frac):
    """Masked attention scores (ops_reference.cpp:104-145): exp of a masked
    score is 0, a row of finfo.min / -1e4 is uniform, a row of -inf is NaN
    (the reference's -inf - -inf), and no NaN leaks into partly masked rows.
    P, D and dZ match the oracle with NaN exactly where it has NaN."""
    import torch
    z = _masked_scores(rows, cols, fill, frac, rows + cols + int(frac * 10))
    p = 0.1
    bits = tops.bernoulli_keep_bits(rows * cols, p, 99)
    keep = port.bernoulli_keep(rows * cols, p, 99)
    mask = bits_to_dev(bits, cuda)
    P, D, _ = tops.softmax_dropout_fwd(to_dev(z, cuda), p, mask=mask)
    Pp = tops.softmax_ip_fwd(to_dev(z, cuda))
    torch.cuda.synchronize()
    rP = port.softmax_fwd(z)
    Pg = P.cpu().numpy()
    assert _close_nan(Pg, rP, 1e-5, 1e-9)
    assert np.array_equal(Pp.cpu().numpy(), Pg, equal_nan=True)  # plain == fused P
    rD = port.dropout_apply(Pg, keep, p).reshape(rows, cols)
    assert np.array_equal(D.cpu().numpy(), rD, equal_nan=True)
    g = np.random.default_rng(5)
    dD = g.standard_normal((rows, cols)).astype(np.float32)
    dZ, Drec = tops.attn_probs_bwd(to_dev(dD, cuda), P, mask, p, write_d=True)
    torch.cuda.synchronize()
    rdZ = port.softmax_bwd(port.dropout_apply(dD, keep, p).reshape(rows, cols), Pg)
    assert _close_nan(dZ.cpu().numpy(), rdZ, 1e-5, 1e-8)
    assert np.array_equal(Drec.cpu().numpy(), D.cpu().numpy(), equal_nan=True)


def test_softmax_special_rows(tops, port, cuda):
    """Rows with NaN (anywhere -> whole row NaN), +inf (NaN row), a single
    finite score among -inf (P = 1 there), and huge logits (z - max
    overflowing): all as the oracle."""
    import torch
    cols = 512
    inf, nan, big = np.inf, np.nan, float(np.finfo(np.float32).max)
    rows = []
    r = np.zeros(cols, np.float32); r[7] = nan; rows.append(r)
    r = np.zeros(cols, np.float32); r[0] = nan; rows.append(r)
    r = np.zeros(cols, np.float32); r[3] = inf; rows.append(r)
    r = np.full(cols, -inf, np.float32); r[100] = 2.0; rows.append(r)
    r = np.full(cols, -big, np.float32); r[5] = big; rows.append(r)
    r = np.linspace(-100, 0, cols).astype(np.float32); rows.append(r)
    r = np.full(cols, 3e38, np.float32); r[::2] = -3e38; rows.append(r)
    z = np.stack(rows)
    P = tops.softmax_ip_fwd(to_dev(z, cuda))
    torch.cuda.synchronize()
    assert _close_nan(P.cpu().numpy(), port.softmax_fwd(z), 1e-5, 1e-9)
    # the generic (non-vector) kernel: 500 columns
    z2 = np.ascontiguousarray(z[:, :500])
    P2 = tops.softmax_ip_fwd(to_dev(z2, cuda))
    torch.cuda.synchronize()
    assert _close_nan(P2.cpu().numpy(), port.softmax_fwd(z2), 1e-5, 1e-9)


@pytest.mark.parametrize("rows,cols", [(4, 512), (3, 130)])
def test_plain_softmax(tops, port, cuda, rows, cols):
    import torch
    g = np.random.default_rng(2)
    z = (g.standard_normal((rows, cols)) * 4).astype(np.float32)
    P = tops.softmax_ip_fwd(to_dev(z, cuda))
    dP = g.standard_normal((rows, cols)).astype(np.float32)
    dZ = tops.softmax_ip_bwd(to_dev(dP, cuda), P)
    torch.cuda.synchronize()
    rP = port.softmax_fwd(z)
    assert np.all(np.abs(P.cpu().numpy() - rP) <= 1e-5 * np.abs(rP) + 1e-9)
    rdZ = port.softmax_bwd(dP, P.cpu().numpy())
    assert np.all(np.abs(dZ.cpu().numpy() - rdZ) <= 1e-5 * np.abs(rdZ) + 1e-8)


def test_softmax_frozen_row(tops, cuda):
    import math
    import torch
    z = torch.tensor([[math.log(1.0), math.log(3.0)]], device=cuda)
    P = tops.softmax_ip_fwd(z)
    dZ = tops.softmax_ip_bwd(torch.tensor([[1.0, 0.0]], device=cuda), P)
    torch.cuda.synchronize()
    assert P.cpu().numpy().ravel().tolist() == pytest.approx([0.25, 0.75], rel=1e-6)
    assert dZ.cpu().numpy().ravel().tolist() == pytest.approx([0.1875, -0.1875], rel=1e-5)


# ---------------------------------------------------------------- dropout
@pytest.mark.parametrize("n", [1, 33, 128, 1000, 128 * 77 + 5, 1 << 22])
def test_hidden_dropout(tops, port, cuda, n):
    import torch
    g = np.random.default_rng(n)
    x = g.standard_normal(n).astype(np.float32)
    dy = g.standard_normal(n).astype(np.float32)
    p = 0.1
    bits = tops.bernoulli_keep_bits(n, p, 99)
    keep = port.bernoulli_keep(n, p, 99)
    mask = bits_to_dev(bits, cuda)
    y, _ = tops.dropout_fwd(to_dev(x, cuda), p, mask=mask)
    dx = tops.dropout_bwd(to_dev(dy, cuda), mask, p)
    torch.cuda.synchronize()
    assert np.array_equal(y.cpu().numpy(), port.dropout_apply(x, keep, p))
    assert np.array_equal(dx.cpu().numpy(), port.dropout_apply(dy, keep, p))
    # Philox: generated mask consistent with the output, shard-invariant
    y2, m2 = tops.dropout_fwd(to_dev(x, cuda), p, seed=5)
    torch.cuda.synchronize()
    k2 = unpack(m2, n)
    assert np.array_equal(y2.cpu().numpy(), port.dropout_apply(x, k2, p))
    if n >= 256 and n % 128 == 0:
        xt = to_dev(x, cuda)
        h = (n // 2) // 128 * 128
        _, ma = tops.dropout_fwd(xt[:h], p, seed=5, offset=0)
        _, mb = tops.dropout_fwd(xt[h:], p, seed=5, offset=h)
        torch.cuda.synchronize()
        assert np.array_equal(np.concatenate([unpack(ma, h), unpack(mb, n - h)]), k2)


def test_golden_fixtures_on_gpu(tops, golden, table_text, cuda):
    """The reference-generated fixtures, end to end on the device."""
    import torch
    g = golden
    table = tops.GeluTable(table_text)
    y, m = tops.gelu_ip_fwd(to_dev(g["gelu_x"], cuda), table)
    dx = tops.gelu_ip_bwd(to_dev(g["gelu_dy"], cuda), y, m, table)
    torch.cuda.synchronize()
    assert np.array_equal(unpack(m, g["gelu_x"].size), g["gelu_mask"])
    fin = np.isfinite(g["gelu_y"])
    assert ulp_diff(y.cpu().numpy()[fin], g["gelu_y"][fin]).max() <= 8
    assert rel_err(dx.cpu().numpy(), g["gelu_dx"]) <= 1e-5
    ly, lrs = tops.layernorm_ip_fwd(to_dev(g["ln_x"], cuda), to_dev(g["ln_gamma"], cuda),
                                    to_dev(g["ln_beta"], cuda))
    ldx, ldg, ldb = tops.layernorm_ip_bwd(to_dev(g["ln_dy"], cuda), ly, lrs,
                                          to_dev(g["ln_gamma"], cuda), to_dev(g["ln_beta"], cuda))
    torch.cuda.synchronize()
    assert rel_err(ly.cpu().numpy(), g["ln_y"]) <= 1e-5
    assert rel_err(ldx.cpu().numpy(), g["ln_dx"]) <= 1e-5
    assert rel_err(ldg.cpu().numpy(), g["ln_dgamma_f64"]) <= 1e-5
    assert rel_err(ldb.cpu().numpy(), g["ln_dbeta_f64"]) <= 1e-5
    keep = g["sm_keep"].reshape(-1)
    bits = np.packbits(keep, bitorder="little")
    bits = np.concatenate([bits, np.zeros((-bits.size) % 4, np.uint8)]).view(np.uint32)
    mask = bits_to_dev(bits, cuda)
    P, D, _ = tops.softmax_dropout_fwd(to_dev(g["sm_z"], cuda), float(g["sm_p"]), mask=mask)
    dZ, _ = tops.attn_probs_bwd(to_dev(g["sm_dD"], cuda), P, mask, float(g["sm_p"]))
    torch.cuda.synchronize()
    rP = g["sm_P"]
    assert np.all(np.abs(P.cpu().numpy() - rP) <= 1e-5 * np.abs(rP) + 1e-9)
    assert np.all(np.abs(dZ.cpu().numpy() - g["sm_dZ"]) <= 1e-5 * np.abs(g["sm_dZ"]) + 1e-8)


def test_mask_pack_roundtrip(tops, cuda):
    import torch
    g = np.random.default_rng(0)
    for n in (1, 31, 32, 1000, 4097):
        b = (g.random(n) < 0.5).astype(np.uint8)
        bits = tops.pack_mask(to_dev(b, cuda))
        back = tops.unpack_mask(bits, n)
        torch.cuda.synchronize()
        assert np.array_equal(back.cpu().numpy(), b)
    st = torch.zeros(1, dtype=torch.int32, device=cuda)
    tops.pack_mask(to_dev(np.array([0, 1, 2], np.uint8), cuda), dev_status=st)
    assert int(st.item()) == 3  # BoolMask::from_bytes refuses bytes > 1


def _at_offset(t, k):
    """A copy of 1-D tensor t whose storage starts k floats past a 256-byte
    aligned allocation (k = 0: 32B-aligned -> 256-bit paths; 4: 16B-aligned ->
    float4 paths; 1: 4B-aligned -> scalar paths)."""
    import torch
    buf = torch.empty(t.numel() + 64, device=t.device, dtype=t.dtype)
    out = buf[k:k + t.numel()]
    out.copy_(t)
    return out


@pytest.mark.parametrize("n", [4096 * 37 + 77, 1 << 20])
def test_vector_paths_agree_bitwise(tops, table_text, cuda, n):
    """Every kernel path (256-bit lanes, float4 lanes, scalar) gives the same
    bits on the same data: GELU fwd (y + mask, incl. fp64-window elements),
    GELU bwd, dropout fwd (supplied mask) and bwd."""
    import torch
    table = tops.GeluTable(table_text)
    g = torch.Generator(device=cuda).manual_seed(5)
    x = torch.randn(n, device=cuda, generator=g) * 2
    x[::97] = -0.7517915  # many elements in the fp64 window around x*
    dy = torch.randn(n, device=cuda, generator=g)
    res = []
    for k in (0, 4, 1):
        xk, dyk = _at_offset(x, k), _at_offset(dy, k)
        y, m = tops.gelu_ip_fwd(xk, table)
        dx = tops.gelu_ip_bwd(dyk, _at_offset(y, k), m, table)
        keep = torch.from_numpy(tops.bernoulli_keep_bits(n, 0.1, 9).view(np.int32)).to(cuda)
        d, _ = tops.dropout_fwd(xk, 0.1, mask=keep)
        dd = tops.dropout_bwd(dyk, keep, 0.1)
        res.append((y.clone(), m.clone(), dx.clone(), d.clone(), dd.clone()))
    torch.cuda.synchronize()
    for other in res[1:]:
        for a, b in zip(res[0], other):
            assert torch.equal(a, b)


# ------------------------------------------- the split LN backward, recompute
@pytest.mark.parametrize("rows,cols", [(64, 1024), (33, 3000), (16, 4096), (7, 768)])
def test_ln_bwd_split_stages(tops, port, cuda, rows, cols):
    """tempo_ln_ip_bwd_partials + tempo_ln_param_reduce (SURVEY 8b's split
    form) equal tempo_ln_ip_bwd bitwise; partial rows of two row shards
    reduced together give the unsharded dgamma/dbeta (F64 oracle, 1e-5)."""
    import ctypes as C
    import torch
    from paper_2210_10246_b200._capi import lib
    L = lib()
    g = np.random.default_rng(rows + cols)
    x = g.standard_normal((rows, cols)).astype(np.float32)
    gam = (1 + 0.2 * g.standard_normal(cols)).astype(np.float32)
    bet = (0.1 * g.standard_normal(cols)).astype(np.float32)
    dy = g.standard_normal((rows, cols)).astype(np.float32)
    T = lambda a: to_dev(a, cuda)  # noqa: E731
    y, rs = tops.layernorm_ip_fwd(T(x), T(gam), T(bet))
    dx, dg, db = tops.layernorm_ip_bwd(T(dy), y, rs, T(gam), T(bet))
    st = torch.cuda.current_stream().cuda_stream

    def stage1(dy_t, y_t, rs_t):
        r = y_t.shape[0]
        nb = int(L.tempo_ln_ip_bwd_workspace_size(r, cols))
        ws = torch.empty(max(nb, 16), dtype=torch.uint8, device=cuda)
        dx_t = torch.empty_like(y_t)
        npart = C.c_int64(-1)
        assert L.tempo_ln_ip_bwd_partials(dy_t.data_ptr(), y_t.data_ptr(), rs_t.data_ptr(),
                                          T(gam).data_ptr(), T(bet).data_ptr(), dx_t.data_ptr(),
                                          ws.data_ptr(), nb, r, cols, C.byref(npart), st) == 0
        return dx_t, ws.view(torch.float64)[: npart.value * 2 * cols].view(npart.value, 2 * cols)

    def reduce(parts):
        dg2 = torch.empty(cols, device=cuda)
        db2 = torch.empty(cols, device=cuda)
        parts = parts.contiguous()
        assert L.tempo_ln_param_reduce(parts.data_ptr(), parts.shape[0], cols, dg2.data_ptr(),
                                       db2.data_ptr(), st) == 0
        return dg2, db2

    dy_t = T(dy)
    dx1, parts = stage1(dy_t, y, rs)
    dg1, db1 = reduce(parts)
    torch.cuda.synchronize()
    assert torch.equal(dx1, dx) and torch.equal(dg1, dg) and torch.equal(db1, db)
    # two row shards: their partial rows stacked and reduced once
    h = rows // 2
    _, pa = stage1(dy_t[:h].contiguous(), y[:h].contiguous(), rs[:h].contiguous())
    pa = pa.clone()
    _, pb = stage1(dy_t[h:].contiguous(), y[h:].contiguous(), rs[h:].contiguous())
    dg3, db3 = reduce(torch.cat([pa, pb.clone()]))
    torch.cuda.synchronize()
    _, rdg, rdb = port.ln_bwd(dy, y.cpu().numpy(), rs.cpu().numpy(), gam, bet, True)
    assert rel_err(dg3.cpu().numpy(), rdg) <= 1e-5
    assert rel_err(db3.cpu().numpy(), rdb) <= 1e-5


def test_dropout_recompute_entry(tops, cuda):
    """tempo_dropout_recompute: the recompute rule, bitwise the forward D."""
    import torch
    from paper_2210_10246_b200._capi import lib
    z = torch.randn(333, 512, device=cuda)
    P, D, m = tops.softmax_dropout_fwd(z, 0.1, seed=4)
    D2 = torch.empty_like(D)
    assert lib().tempo_dropout_recompute(P.data_ptr(), m.data_ptr(), 0.1, D2.data_ptr(), P.numel(),
                                         torch.cuda.current_stream().cuda_stream) == 0
    torch.cuda.synchronize()
    assert torch.equal(D2, D)
    assert lib().tempo_dropout_recompute(P.data_ptr(), m.data_ptr(), 1.0, D2.data_ptr(), 4,
                                         torch.cuda.current_stream().cuda_stream) == 3


@pytest.mark.parametrize("rows,cols", [(8, 1024), (8, 768), (8, 1000), (8, 2048)])
def test_layernorm_nan_row(tops, port, cuda, rows, cols):
    """A NaN in a row: that row's y and rstd are NaN as in the reference (its
    double variance propagates the NaN), the other rows are untouched."""
    import torch
    g = np.random.default_rng(cols)
    x = g.standard_normal((rows, cols)).astype(np.float32)
    x[2, 5] = np.nan
    gam = (1 + 0.2 * g.standard_normal(cols)).astype(np.float32)
    bet = (0.1 * g.standard_normal(cols)).astype(np.float32)
    y, rstd = tops.layernorm_ip_fwd(to_dev(x, cuda), to_dev(gam, cuda), to_dev(bet, cuda))
    torch.cuda.synchronize()
    ry, rrs, _ = port.ln_fwd(x, gam, bet, 1e-5)
    assert _close_nan(y.cpu().numpy(), ry, 1e-5, 1e-5)
    assert _close_nan(rstd.cpu().numpy(), rrs, 1e-6, 0)
    if cols % 32 == 0:  # the fused dropout -> add -> LN forward (cols % 32 == 0)
        yd, rsd, _ = tops.dropout_add_layernorm_fwd(to_dev(np.zeros_like(x), cuda),
                                                    to_dev(x, cuda), to_dev(gam, cuda),
                                                    to_dev(bet, cuda), 0.1, seed=1)
        torch.cuda.synchronize()
        assert _close_nan(yd.cpu().numpy(), ry, 1e-5, 1e-5)
        assert _close_nan(rsd.cpu().numpy(), rrs, 1e-6, 0)


def _reduce8_order(parts, cw=8):
    """ln_param_reduce8_kernel's fixed summation tree (layernorm_kernels.cu):
    slice ty = 0..64 sums partial rows ty, ty+64, ... in order; a warp holds
    slices 4w..4w+3 and adds them by the xor-8 then xor-16 shuffle tree; warp
    0 lane q*8+c sums warps q, q+4, q+8, q+12 in order, then the same tree."""
    nparts, total = parts.shape
    ns = 512 // cw
    sl = np.zeros((ns, total))
    for ty in range(ns):
        for c in range(ty, nparts, ns):
            sl[ty] = sl[ty] + parts[c]
    # per warp: slices 4w+t, t = 0..3 -> (s0 + s1) + (s2 + s3)
    wsum = np.array([(sl[4 * w] + sl[4 * w + 1]) + (sl[4 * w + 2] + sl[4 * w + 3])
                     for w in range(ns // 4)])
    q = [((wsum[k] + wsum[k + 4]) + wsum[k + 8]) + wsum[k + 12] for k in range(4)]
    return (q[0] + q[1]) + (q[2] + q[3])


@pytest.mark.parametrize("nparts,cols", [(1, 5), (37, 768), (296, 1024), (700, 1001),
                                         (1100, 12)])
def test_ln_param_reduce_fixed_tree(cuda, nparts, cols):
    """Stage 2 of the LN backward (tempo_ln_param_reduce, 8 columns x 64
    slices per CTA) is exactly its documented fixed-order tree, bit for bit:
    ragged column blocks (cols % 8 != 0), more partial rows than one load
    batch (nparts > 512), one partial row."""
    import torch
    from paper_2210_10246_b200._capi import lib
    g = np.random.default_rng(nparts * 7 + cols)
    parts = g.standard_normal((nparts, 2 * cols)) * np.exp(g.uniform(-8, 8, (nparts, 1)))
    dev = torch.from_numpy(parts).to(cuda)
    dg = torch.full((cols,), float("nan"), device=cuda)
    db = torch.full((cols,), float("nan"), device=cuda)
    st = torch.cuda.current_stream().cuda_stream
    assert lib().tempo_ln_param_reduce(dev.data_ptr(), nparts, cols, dg.data_ptr(),
                                       db.data_ptr(), st) == 0
    torch.cuda.synchronize()
    want = _reduce8_order(parts).astype(np.float32)
    assert np.array_equal(dg.cpu().numpy(), want[:cols])
    assert np.array_equal(db.cpu().numpy(), want[cols:])
