"""Fused hidden dropout -> residual add -> In-Place LayerNorm (forward and
backward) against the oracle composition of the reference layer
(ref_ops::dropout -> Graph::add -> tempo_ops::layernorm, encoder.cpp:180-191
and 198-210) and bitwise against the unfused kernels on the same inputs.

Tolerances: y, d_residual rel_err <= 1e-5, rstd rel <= 1e-6, dgamma/dbeta
vs the F64 oracle rel_err <= 1e-5 (as the unfused ops); mask bits and d_proj
(a product by 1/(1-p) rounded once from fp64) bit-exact."""
import numpy as np
import pytest

from test_gpu_parity import bits_to_dev, rel_err, to_dev, unpack

pytestmark = pytest.mark.gpu

# 1536 / 2048 / 3072 / 4096 / 8192 / 16384: the long-row (warp-group) kernels
SHAPES = [(64, 1024), (333, 768), (7, 512), (5, 128), (9, 1536), (3, 96), (16, 4096),
          (1, 1024), (40, 384), (9, 2048), (5, 3072), (3, 8192), (2, 16384), (3, 2080)]


def inputs(rows, cols, seed, p):
    g = np.random.default_rng(seed)
    proj = (g.standard_normal((rows, cols)) * 1.3).astype(np.float32)
    res = (g.standard_normal((rows, cols)) + 0.3).astype(np.float32)
    gam = (1 + 0.2 * g.standard_normal(cols)).astype(np.float32)
    bet = (0.1 * g.standard_normal(cols)).astype(np.float32)
    dy = g.standard_normal((rows, cols)).astype(np.float32)
    keep = (g.random(rows * cols) >= p).astype(np.uint8)
    return proj, res, gam, bet, dy, keep


def pack(keep):
    n = keep.size
    b = np.packbits(keep, bitorder="little")
    b = np.concatenate([b, np.zeros((-b.size) % 4, np.uint8)])
    return b.view(np.uint32)[:(n + 31) // 32]


@pytest.mark.parametrize("rows,cols", SHAPES)
def test_fused_forward_matches_reference_composition(tops, port, cuda, rows, cols):
    import torch
    p = 0.1
    proj, res, gam, bet, _, keep = inputs(rows, cols, rows * cols, p)
    m = bits_to_dev(pack(keep), cuda)
    y, rstd, _ = tops.dropout_add_layernorm_fwd(to_dev(proj, cuda), to_dev(res, cuda),
                                                to_dev(gam, cuda), to_dev(bet, cuda), p, mask=m)
    torch.cuda.synchronize()
    r = (res + port.dropout_apply(proj.reshape(-1), keep, p).reshape(rows, cols)).astype(np.float32)
    ry, rrs, _ = port.ln_fwd(r, gam, bet, 1e-5)
    assert rel_err(y.cpu().numpy(), ry) <= 1e-5
    assert np.abs(rstd.cpu().numpy().astype(np.float64) / rrs - 1).max() <= 1e-6
    # bitwise the unfused kernels: dropout_fwd, fp32 add, layernorm_ip_fwd
    d, _ = tops.dropout_fwd(to_dev(proj, cuda), p, mask=m)
    y2, rs2 = tops.layernorm_ip_fwd(to_dev(res, cuda) + d, to_dev(gam, cuda), to_dev(bet, cuda))
    torch.cuda.synchronize()
    if cols in (256, 512, 768, 1024):  # the same warp-per-row statistics kernel
        assert torch.equal(y, y2) and torch.equal(rstd, rs2)


@pytest.mark.parametrize("rows,cols,offset", [(64, 1024, 0), (33, 768, 4096 * 768),
                                              (8, 96, 32 * 7), (9, 1536, 128),
                                              (5, 3072, 3072 * 11), (2, 16384, 0)])
def test_fused_forward_philox_mask_is_dropouts(tops, cuda, rows, cols, offset):
    """Generated masks are the bits tempo_dropout_fwd draws for the same
    global element offsets (so row shards and the unfused path agree)."""
    import torch
    p = 0.1
    proj, res, gam, bet, _, _ = inputs(rows, cols, 7 + cols, p)
    _, _, m = tops.dropout_add_layernorm_fwd(to_dev(proj, cuda), to_dev(res, cuda),
                                             to_dev(gam, cuda), to_dev(bet, cuda), p, seed=99,
                                             offset=offset)
    _, m2 = tops.dropout_fwd(to_dev(proj, cuda), p, seed=99, offset=offset)
    torch.cuda.synchronize()
    n = rows * cols
    assert np.array_equal(unpack(m, n), unpack(m2, n))
    assert abs(unpack(m, n).mean() - (1 - p)) < 0.05


@pytest.mark.parametrize("rows,cols", [(64, 1024), (333, 768), (7, 512), (9, 1536), (3, 96),
                                       (16, 4096), (2048, 1024), (9, 2048), (5, 3072),
                                       (300, 4096), (3, 8192), (2, 16384), (3, 2080)])
def test_fused_backward_matches_reference_composition(tops, port, cuda, rows, cols):
    import torch
    p = 0.1
    proj, res, gam, bet, dy, keep = inputs(rows, cols, 5 + rows * cols, p)
    r = (res + port.dropout_apply(proj.reshape(-1), keep, p).reshape(rows, cols)).astype(np.float32)
    ry, rrs, _ = port.ln_fwd(r, gam, bet, 1e-5)
    m = bits_to_dev(pack(keep), cuda)
    args = [to_dev(a, cuda) for a in (dy, ry, rrs, gam, bet)]
    d_res, d_proj, dg, db = tops.dropout_add_layernorm_bwd(*args, m, p)
    torch.cuda.synchronize()
    rdx, _, _ = port.ln_bwd(dy, ry, rrs, gam, bet, False)
    _, dg64, db64 = port.ln_bwd(dy, ry, rrs, gam, bet, True)
    assert rel_err(d_res.cpu().numpy(), rdx) <= 1e-5
    assert rel_err(dg.cpu().numpy(), dg64) <= 1e-5
    assert rel_err(db.cpu().numpy(), db64) <= 1e-5
    # d_proj: dropout_backward of THIS d_residual, bit-exact
    want = port.dropout_apply(d_res.cpu().numpy().reshape(-1), keep, p).reshape(rows, cols)
    assert np.array_equal(d_proj.cpu().numpy(), want)
    # bitwise the unfused kernels: layernorm_ip_bwd then dropout_bwd
    dx2, dg2, db2 = tops.layernorm_ip_bwd(*args)
    dp2 = tops.dropout_bwd(dx2, m, p)
    torch.cuda.synchronize()
    assert torch.equal(d_res, dx2) and torch.equal(dg, dg2) and torch.equal(db, db2)
    assert torch.equal(d_proj, dp2)


def test_fused_refusals(tops, cuda):
    import torch
    from paper_2210_10246_b200 import TempoError
    x = torch.randn(4, 100, device=cuda)
    g, b = torch.ones(100, device=cuda), torch.zeros(100, device=cuda)
    with pytest.raises(TempoError) as e:
        tops.dropout_add_layernorm_fwd(x, x, g, b, 0.1)  # cols % 32 != 0
    assert e.value.kind == "Unsupported"
    x = torch.randn(4, 128, device=cuda)
    g, b = torch.ones(128, device=cuda), torch.zeros(128, device=cuda)
    with pytest.raises(TempoError) as e:
        tops.dropout_add_layernorm_fwd(x, x, g, b, 1.0)
    assert e.value.kind == "ParamError"
