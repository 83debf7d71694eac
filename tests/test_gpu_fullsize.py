"""Parity at BASELINE.json's full sizes.

The oracle checks a deterministic row subset (all ops are row independent
except LayerNorm's dgamma/dbeta, which is checked whole), and the full tensors
are checked through size-independent properties: recomputed D bitwise equal
to the forward D, D/P consistent with the mask everywhere, softmax rows
summing to 1, GELU masks equal to x > x*, dgamma/dbeta bitwise reproducible
run to run, and empty inputs as no-ops.
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def rel_err(a, b):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    d = np.abs(a - b) / np.maximum(1.0, np.maximum(np.abs(a), np.abs(b)))
    return float(d.max()) if d.size else 0.0


def unpack_rows(bits, rows, cols, sel):
    """Mask bits of selected rows (bit i of word i/32 = element i)."""
    words = bits.cpu().numpy().view(np.uint32)
    allbits = np.unpackbits(words.view(np.uint8), bitorder="little")
    return allbits[: rows * cols].reshape(rows, cols)[sel]


def test_cfg3_attention_full(tops, port, cuda):
    """configs[2]: dropout recompute + output-only softmax bwd on [32*12*512, 512]."""
    import torch
    rows, cols, p = 32 * 12 * 512, 512, 0.1
    g = torch.Generator(device=cuda)
    g.manual_seed(3)
    z = torch.randn(rows, cols, device=cuda, generator=g) * 2
    dD = torch.randn(rows, cols, device=cuda, generator=g)
    P, D, mask = tops.softmax_dropout_fwd(z, p, seed=11)
    dZ, Drec = tops.attn_probs_bwd(dD, P, mask, p, write_d=True)
    torch.cuda.synchronize()
    assert torch.equal(D, Drec)                       # recompute == forward, bitwise
    s = P.double().sum(dim=1)
    assert float((s - 1).abs().max()) < 1e-5          # rows of P sum to 1
    dropped = float((D == 0).double().mean())            # P > 0 everywhere here
    words = mask.view(torch.int32)
    keep_rate = float(torch.tensor([bin(int(w) & 0xffffffff).count("1") for w in
                                    words[:4096].cpu()]).sum()) / (4096 * 32)
    assert abs(keep_rate - (1 - p)) < 0.01
    # oracle on a row subset
    sel = np.sort(np.random.default_rng(0).choice(rows, 1024, replace=False))
    keep = unpack_rows(mask, rows, cols, sel)
    zs, Ps, dDs = z.cpu().numpy()[sel], P.cpu().numpy()[sel], dD.cpu().numpy()[sel]
    rP = port.softmax_fwd(zs)
    assert np.all(np.abs(Ps - rP) <= 1e-5 * np.abs(rP) + 1e-9)
    assert np.array_equal(D.cpu().numpy()[sel], port.dropout_apply(Ps, keep, p))
    rdZ = port.softmax_bwd(port.dropout_apply(dDs, keep, p), Ps)
    dZs = dZ.cpu().numpy()[sel]
    assert np.all(np.abs(dZs - rdZ) <= 1e-5 * np.abs(rdZ) + 1e-8)
    assert abs(dropped - p) < 0.002


def test_cfg4_layer_chain_full(tops, port, table_text, cuda):
    """configs[3]: the BERT-large layer op chain at B=64 (bench.Chain), checked
    on row subsets against the oracle after one full forward+backward."""
    import torch
    import bench
    chain = bench.Chain(cuda, 0, 1)
    chain.step()
    torch.cuda.synchronize()
    T, H = bench.T, bench.H
    sel = np.sort(np.random.default_rng(1).choice(T, 256, replace=False))
    # GELU forward/backward on the selected token rows
    x = chain.x_ffn1.cpu().numpy()[sel]
    pt = port.table(table_text)
    ry, rm = port.gelu_fwd(x.reshape(-1), pt.x_star)
    y = chain.y_g.cpu().numpy()[sel].reshape(-1)
    gm = unpack_rows(chain.m_g, T, 4 * H, sel).reshape(-1)
    assert np.array_equal(gm, rm)
    assert rel_err(y, ry) <= 1e-6
    rdx = pt.gelu_bwd(chain.dy_gelu.cpu().numpy()[sel].reshape(-1), y, gm)
    assert rel_err(chain.dx_g.cpu().numpy()[sel].reshape(-1), rdx) <= 1e-5
    # LayerNorm 2: forward rows + full dgamma/dbeta against the F64 oracle
    d2 = chain.d2.cpu().numpy()
    ry2, rrs2, _ = port.ln_fwd(d2, chain.g2.cpu().numpy(), chain.b2.cpu().numpy(), 1e-5)
    assert rel_err(chain.y_ln2.cpu().numpy(), ry2) <= 1e-5
    _, dg64, db64 = port.ln_bwd(chain.dy_ln2.cpu().numpy(), chain.y_ln2.cpu().numpy(),
                                chain.rs2.cpu().numpy(), chain.g2.cpu().numpy(),
                                chain.b2.cpu().numpy(), True)
    dp = chain.dparams.cpu().numpy()
    assert rel_err(dp[:H], dg64) <= 1e-5 and rel_err(dp[H:2 * H], db64) <= 1e-5
    # hidden dropout 2: y = mask ? x/(1-p) : 0 exactly, from the generated mask
    k2 = unpack_rows(chain.m2, T, H, sel)
    assert np.array_equal(chain.d2.cpu().numpy()[sel],
                          port.dropout_apply(chain.x_ffn2.cpu().numpy()[sel], k2, 0.1))
    # run-to-run: a second step with the same seeds reproduces dgamma/dbeta bitwise
    before = chain.dparams.clone()
    chain.step_idx -= 1
    chain.step()
    torch.cuda.synchronize()
    assert torch.equal(before, chain.dparams)


def test_empty_inputs_are_noops(tops, table_text, cuda):
    import torch
    e = torch.empty(0, device=cuda)
    table = tops.GeluTable(table_text)
    y, m = tops.gelu_ip_fwd(e, table)
    assert tops.gelu_ip_bwd(e, y, m, table).numel() == 0
    e2 = torch.empty(0, 768, device=cuda)
    g, b = torch.ones(768, device=cuda), torch.zeros(768, device=cuda)
    yl, rs = tops.layernorm_ip_fwd(e2, g, b)
    dx, dg, db = tops.layernorm_ip_bwd(e2, yl, rs, g, b)
    torch.cuda.synchronize()
    assert dx.numel() == 0 and float(dg.abs().sum()) == 0.0 and float(db.abs().sum()) == 0.0
    es = torch.empty(0, 512, device=cuda)
    P, D, mk = tops.softmax_dropout_fwd(es, 0.1, seed=1)
    dZ, _ = tops.attn_probs_bwd(es, P, mk, 0.1)
    yd, md = tops.dropout_fwd(e, 0.1, seed=1)
    assert tops.dropout_bwd(e, md, 0.1).numel() == 0
    torch.cuda.synchronize()


def test_cfg4_fused_layer_chain_full(tops, port, cuda):
    """configs[3] with the fused hidden dropout -> residual add -> LayerNorm
    ops (bench.py's default chain): one forward+backward at full size, the
    LN rows on a subset against the oracle composition (dropout_apply, fp32
    add, ln_fwd / ln_bwd), d_proj bit-exact from d_residual and the mask,
    dgamma/dbeta of both LNs against the F64 oracle, and bitwise run to run."""
    import torch
    import bench
    chain = bench.Chain(cuda, 0, 1, fused=True)
    chain.step()
    torch.cuda.synchronize()
    T, H, p = bench.T, bench.H, bench.P_DROP
    sel = np.sort(np.random.default_rng(2).choice(T, 256, replace=False))
    g1, b1 = chain.g1.cpu().numpy(), chain.b1.cpu().numpy()
    g2, b2 = chain.g2.cpu().numpy(), chain.b2.cpu().numpy()
    y1 = chain.y_ln1.cpu().numpy()
    for proj, res, m, g, b, y, rs in [
            (chain.x_attn_out, chain.x_res, chain.m1, g1, b1, y1, chain.rs1),
            (chain.x_ffn2, chain.y_ln1, chain.m2, g2, b2, chain.y_ln2.cpu().numpy(), chain.rs2)]:
        keep = unpack_rows(m, T, H, sel)
        r = (res.cpu().numpy()[sel] +
             port.dropout_apply(proj.cpu().numpy()[sel], keep, p)).astype(np.float32)
        ry, rrs, _ = port.ln_fwd(r, g, b, 1e-5)
        assert rel_err(y[sel], ry) <= 1e-5
        assert np.abs(rs.cpu().numpy()[sel].astype(np.float64) / rrs - 1).max() <= 1e-6
    # backward of LN1's pair: d_residual rows, d_proj bit-exact, dgamma/dbeta whole
    dp = chain.dparams.cpu().numpy()
    for dy, y, rs, g, b, m, d_res, d_proj, sl in [
            (chain.dy_ln1, y1, chain.rs1, g1, b1, chain.m1, chain.dx_res, chain.dx_d1, slice(2 * H, 4 * H)),
            (chain.dy_ln2, chain.y_ln2.cpu().numpy(), chain.rs2, g2, b2, chain.m2, chain.dx_ln2,
             chain.dx_d2, slice(0, 2 * H))]:
        dyn, rsn = dy.cpu().numpy(), rs.cpu().numpy()
        rdx, _, _ = port.ln_bwd(dyn[sel], y[sel], rsn[sel], g, b, False)
        dres = d_res.cpu().numpy()
        assert rel_err(dres[sel], rdx) <= 1e-5
        keep = unpack_rows(m, T, H, sel)
        assert np.array_equal(d_proj.cpu().numpy()[sel], port.dropout_apply(dres[sel], keep, p))
        _, dg64, db64 = port.ln_bwd(dyn, y, rsn, g, b, True)
        assert rel_err(dp[sl][:H], dg64) <= 1e-5 and rel_err(dp[sl][H:], db64) <= 1e-5
    before = chain.dparams.clone()
    chain.step_idx -= 1
    chain.step()
    torch.cuda.synchronize()
    assert torch.equal(before, chain.dparams)
