"""The dropout recompute fused into the dV GEMM (tempo_attn_dropout_dv,
tcgen05 3xTF32): dV = D^T @ dO with D = keep ? P/(1-p) : 0 rebuilt from the
stashed P and mask inside the GEMM, against the oracle composition
(port.dropout_apply -> fp64 D^T dO, rounded once).

Tolerance: rel_err (the reference's |a-b|/max(1,|a|,|b|)) <= 1e-5, and
elementwise |a-b| <= 1e-5 * (|ref| + sum_i |D_ij dO_ic|), the usual GEMM
bound -- 3xTF32 products carry ~2^-21 relative error each and the tensor
core's fp32 accumulation over K adds its own rounding (measured ~2e-6 of
sum |D dO| at K = 512)."""
import numpy as np
import pytest

from test_gpu_parity import bits_to_dev, rel_err, to_dev

pytestmark = pytest.mark.gpu


def case(heads, s_q, s_k, d, p, seed):
    g = np.random.default_rng(seed)
    z = g.standard_normal((heads, s_q, s_k)) * 2
    P = np.exp(z - z.max(-1, keepdims=True))
    P = (P / P.sum(-1, keepdims=True)).astype(np.float32)
    dO = g.standard_normal((heads, s_q, d)).astype(np.float32)
    keep = (g.random(heads * s_q * s_k) >= p).astype(np.uint8)
    return P, dO, keep


def pack(keep):
    b = np.packbits(keep, bitorder="little")
    b = np.concatenate([b, np.zeros((-b.size) % 4, np.uint8)])
    return b.view(np.uint32)[:(keep.size + 31) // 32]


@pytest.mark.parametrize("heads,s_q,s_k,d,p", [(3, 512, 512, 64, 0.1), (2, 512, 512, 32, 0.1),
                                               (2, 256, 512, 128, 0.1), (1, 32, 256, 64, 0.5),
                                               (5, 384, 256, 64, 0.0), (2, 1024, 512, 64, 0.1),
                                               # long K = s_q: the drained accumulation
                                               (1, 8192, 256, 64, 0.1), (1, 2080, 256, 32, 0.2)])
def test_dv_matches_oracle_composition(tops, port, cuda, heads, s_q, s_k, d, p):
    import torch
    P, dO, keep = case(heads, s_q, s_k, d, p, heads * s_q + d)
    dV = tops.attn_dropout_dv(to_dev(P, cuda), bits_to_dev(pack(keep), cuda), p, to_dev(dO, cuda))
    torch.cuda.synchronize()
    D = port.dropout_apply(P.reshape(-1), keep, p).reshape(P.shape).astype(np.float64)
    ref = np.einsum("hij,hic->hjc", D, dO.astype(np.float64))
    mag = np.einsum("hij,hic->hjc", np.abs(D), np.abs(dO.astype(np.float64)))
    got = dV.cpu().numpy().astype(np.float64)
    assert rel_err(got, ref.astype(np.float32)) <= 1e-5
    assert np.all(np.abs(got - ref) <= 1e-5 * (np.abs(ref) + mag))


def test_dv_equals_materialised_d_gemm(tops, cuda):
    """Against the unfused path: attn_probs_bwd's recomputed D (bitwise the
    forward D) fed to an fp32 cuBLAS GEMM (TF32 off)."""
    import torch
    heads, s, d, p = 4, 512, 64, 0.1
    g = torch.Generator(device=cuda)
    g.manual_seed(11)
    z = torch.randn(heads * s, s, device=cuda, generator=g)
    P, D, m = tops.softmax_dropout_fwd(z, p, seed=3)
    dO = torch.randn(heads, s, d, device=cuda, generator=g)
    dV = tops.attn_dropout_dv(P.view(heads, s, s), m, p, dO)
    prev = torch.backends.cuda.matmul.allow_tf32
    torch.backends.cuda.matmul.allow_tf32 = False
    try:
        ref = torch.matmul(D.view(heads, s, s).transpose(1, 2), dO)
    finally:
        torch.backends.cuda.matmul.allow_tf32 = prev
    torch.cuda.synchronize()
    assert rel_err(dV.cpu().numpy(), ref.cpu().numpy()) <= 1e-5


def test_dv_refusals(tops, cuda):
    import torch
    from paper_2210_10246_b200 import TempoError
    P = torch.rand(1, 64, 200, device=cuda)
    dO = torch.rand(1, 64, 64, device=cuda)
    m = torch.zeros(64 * 200 // 32 + 1, dtype=torch.int32, device=cuda)
    with pytest.raises(TempoError) as e:
        tops.attn_dropout_dv(P, m, 0.1, dO)  # s_k % 256 != 0
    assert e.value.kind == "Unsupported"


def test_umma_probe_layouts():
    """tests/tools/umma_probe: tcgen05 kind::tf32 on K-major SWIZZLE_128B
    operands is exact (the layout dv_gemm_kernels.cu stages), MN-major gives
    no result on this part (why the kernel transposes while staging)."""
    import os
    import subprocess
    exe = os.path.join(os.path.dirname(__file__), "tools", "_build", "umma_probe")
    out = subprocess.run([exe], capture_output=True, text=True, timeout=120).stdout
    lines = {int(l.split()[1]): l for l in out.splitlines() if l.startswith("variant")}
    assert "max|err|=0 " in lines[0]


# ------------------------------------------------ the forward consumer (ctx)
@pytest.mark.parametrize("heads,s_q,s_k,d,p", [(3, 512, 512, 64, 0.1), (2, 512, 512, 32, 0.1),
                                               (1, 128, 32, 64, 0.5), (5, 384, 256, 64, 0.0),
                                               (2, 256, 1024, 64, 0.1), (1, 128, 96, 32, 0.3),
                                               (3, 100, 64, 64, 0.1), (2, 300, 128, 32, 0.2),
                                               # long rows: the drained accumulation
                                               # (s_k > 1024), incl. a 1-slice last segment
                                               (1, 256, 2048, 64, 0.1), (1, 128, 8192, 64, 0.1),
                                               (1, 200, 4096, 32, 0.1), (2, 128, 1056, 64, 0.2)])
def test_ctx_matches_oracle_composition(tops, port, cuda, heads, s_q, s_k, d, p):
    """tempo_attn_dropout_ctx: ctx = D @ V with D rebuilt inside the tcgen05
    GEMM (P's tile staged with TMA SWIZZLE_128B = the K-major operand layout)
    against the oracle composition dropout_apply -> fp64 D @ V.  The bound
    holds at any s_k: beyond s_k = 1024 the kernel drains its TMEM
    accumulators into fp32 registers every 256 key columns, so the tensor
    core's truncating accumulation never spans more than 48 products."""
    import torch
    g = np.random.default_rng(heads * s_q + s_k + d)
    z = g.standard_normal((heads, s_q, s_k)) * 2
    P = np.exp(z - z.max(-1, keepdims=True))
    P = (P / P.sum(-1, keepdims=True)).astype(np.float32)
    V = g.standard_normal((heads, s_k, d)).astype(np.float32)
    keep = (g.random(heads * s_q * s_k) >= p).astype(np.uint8)
    ctx = tops.attn_dropout_ctx(to_dev(P, cuda), bits_to_dev(pack(keep), cuda), p, to_dev(V, cuda))
    torch.cuda.synchronize()
    D = port.dropout_apply(P.reshape(-1), keep, p).reshape(P.shape).astype(np.float64)
    ref = np.einsum("hij,hjc->hic", D, V.astype(np.float64))
    mag = np.einsum("hij,hjc->hic", np.abs(D), np.abs(V.astype(np.float64)))
    got = ctx.cpu().numpy().astype(np.float64)
    assert rel_err(got, ref.astype(np.float32)) <= 1e-5
    assert np.all(np.abs(got - ref) <= 1e-5 * (np.abs(ref) + mag))


def test_ctx_equals_materialised_d_gemm(tops, cuda):
    """The D-free forward (softmax_dropout_fwd without D + the fused ctx GEMM)
    against the materialised path (the forward's D + an fp32 cuBLAS GEMM)."""
    import torch
    heads, s, d, p = 4, 512, 64, 0.1
    g = torch.Generator(device=cuda)
    g.manual_seed(12)
    z = torch.randn(heads * s, s, device=cuda, generator=g)
    P, D, m = tops.softmax_dropout_fwd(z, p, seed=4)
    P2, none, m2 = tops.softmax_dropout_fwd(z, p, seed=4, write_d=False)
    V = torch.randn(heads, s, d, device=cuda, generator=g)
    ctx = tops.attn_dropout_ctx(P2.view(heads, s, s), m2, p, V)
    prev = torch.backends.cuda.matmul.allow_tf32
    torch.backends.cuda.matmul.allow_tf32 = False
    try:
        ref = torch.matmul(D.view(heads, s, s), V)
    finally:
        torch.backends.cuda.matmul.allow_tf32 = prev
    torch.cuda.synchronize()
    assert none is None and torch.equal(P, P2) and torch.equal(m, m2)
    assert rel_err(ctx.cpu().numpy(), ref.cpu().numpy()) <= 1e-5


def test_ctx_refusals(tops, cuda):
    import torch
    from paper_2210_10246_b200 import TempoError
    P = torch.rand(1, 100, 48, device=cuda)
    V = torch.rand(1, 48, 64, device=cuda)
    m = torch.zeros(100 * 48 // 32 + 1, dtype=torch.int32, device=cuda)
    with pytest.raises(TempoError) as e:
        tops.attn_dropout_ctx(P, m, 0.1, V)  # s_k % 32 != 0
    assert e.value.kind == "Unsupported"


@pytest.mark.parametrize("heads,s_q,s_k,d", [(300, 256, 256, 64), (200, 300, 128, 64),
                                             (333, 256, 512, 32), (500, 1, 64, 64),
                                             (160, 257, 96, 32)])
def test_persistent_many_tiles(tops, cuda, heads, s_q, s_k, d):
    """More (head, 256-row) tiles than SMs: each persistent CTA loops over
    several tiles, its slice ring and accumulator hand-off running on across
    tile boundaries (incl. ragged query blocks).  ctx and dV against the fp64
    product of the forward's D."""
    import torch
    p = 0.1
    g = torch.Generator(device=cuda)
    g.manual_seed(heads + s_q + d)
    z = torch.randn(heads * s_q, s_k, device=cuda, generator=g) * 2
    P, D, m = tops.softmax_dropout_fwd(z, p, seed=heads)
    V = torch.randn(heads, s_k, d, device=cuda, generator=g)
    dO = torch.randn(heads, s_q, d, device=cuda, generator=g)
    Dd = D.view(heads, s_q, s_k).double()
    ctx = tops.attn_dropout_ctx(P.view(heads, s_q, s_k), m, p, V)
    ref = torch.matmul(Dd, V.double())
    mag = torch.matmul(Dd.abs(), V.double().abs())
    assert bool(((ctx.double() - ref).abs() <= 1e-5 * (ref.abs() + mag)).all())
    if s_q % 32 == 0 and s_k % 256 == 0:
        dV = tops.attn_dropout_dv(P.view(heads, s_q, s_k), m, p, dO)
        refv = torch.matmul(Dd.transpose(1, 2), dO.double())
        magv = torch.matmul(Dd.abs().transpose(1, 2), dO.double().abs())
        assert bool(((dV.double() - refv).abs() <= 1e-5 * (refv.abs() + magv)).all())
