"""A/B timing of single ops at the bench shapes (not part of the contract).

  TEMPO_B200_LIB=_ab/X/libtempo_b200.so python tools/ab_time.py gelu_fwd ln_fwd ...

Prints one line per op: median device time over reps (CUDA events on the
launching stream, L2 evicted by a 512 MB read before every rep so the GPU is
busy while Python issues the launch), algorithmic GB/s, fraction of the
measured HBM peak, and a checksum of the outputs (to spot A/B differences).
"""
import hashlib
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch
    from paper_2210_10246_b200 import ops
    import bench

    dev = torch.device("cuda:0")
    peak, _ = bench.peaks()
    chain = bench.Chain(dev, 0, 1)
    chain.step()
    torch.cuda.synchronize()
    fb = torch.empty(128 * 1024 * 1024, device=dev).fill_(1.0)
    fo = torch.empty((), device=dev)
    # read-only L2 eviction (512 MB): no foreign dirty lines for the op to
    # write back (bench.py per_op does the same); FLUSH=dirty for a 1 GB fill
    if os.environ.get("FLUSH") == "dirty":
        flush = lambda: fb.fill_(0.0)  # noqa: E731
    else:
        flush = lambda: torch.sum(fb, dim=0, out=fo)  # noqa: E731
    H, T = bench.H, bench.T
    dp = chain.dparams
    o = ops
    c = chain
    calls = {
        "softmax_dropout_fwd": (lambda: o.softmax_dropout_fwd(c.z, bench.P_DROP, mask=c.m_att, generate=True, seed=7, P=c.P, D=c.D), [c.P, c.D, c.m_att]),
        "attn_probs_bwd": (lambda: o.attn_probs_bwd(c.dD, c.P, c.m_att, bench.P_DROP, write_d=True, dZ=c.dZ, D=c.Drec), [c.dZ, c.Drec]),
        "gelu_fwd": (lambda: o.gelu_ip_fwd(c.x_ffn1, c.table, y=c.y_g, mask=c.m_g), [c.y_g, c.m_g]),
        "gelu_fwd_exact": (lambda: o.gelu_ip_fwd(c.x_ffn1, c.table, y=c.y_g, mask=c.m_g, exact=True), [c.y_g, c.m_g]),
        "gelu_bwd": (lambda: o.gelu_ip_bwd(c.dy_gelu, c.y_g, c.m_g, c.table, dx=c.dx_g), [c.dx_g]),
        "ln_fwd": (lambda: o.layernorm_ip_fwd(c.d1, c.g1, c.b1, check_gamma=False, y=c.y_ln1, rstd=c.rs1), [c.y_ln1, c.rs1]),
        "ln_bwd": (lambda: o.layernorm_ip_bwd(c.dy_ln1, c.y_ln1, c.rs1, c.g1, c.b1, dx=c.dx_ln1, dgamma=dp[:H], dbeta=dp[H:2 * H], workspace=c.ws), [c.dx_ln1, dp[:2 * H]]),
        "dropout_fwd": (lambda: o.dropout_fwd(c.x_ffn2, bench.P_DROP, mask=c.m2, generate=True, seed=9, y=c.d2), [c.d2, c.m2]),
        "mt_mask": (lambda: o.bernoulli_keep_bits_device(c.z.numel(), bench.P_DROP, 7, out=c.m_att), [c.m_att]),
        "mt_mask_h": (lambda: o.bernoulli_keep_bits_device(c.x_ffn2.numel(), bench.P_DROP, 7, out=c.m2), [c.m2]),
        "copy_g": (lambda: c.y_g.copy_(c.x_ffn1), [c.y_g[:1]]),
        "copy_h": (lambda: c.d2.copy_(c.x_ffn2), [c.d2[:1]]),
        "dropout_bwd": (lambda: o.dropout_bwd(c.dx_ln2, c.m2, bench.P_DROP, dx=c.dx_d2), [c.dx_d2]),
        "dal_fwd": (lambda: o.dropout_add_layernorm_fwd(c.x_ffn2, c.y_ln1, c.g2, c.b2, bench.P_DROP, mask=c.m2, generate=True, seed=9, check_gamma=False, y=c.y_ln2, rstd=c.rs2), [c.y_ln2, c.rs2, c.m2]),
        "dal_bwd": (lambda: o.dropout_add_layernorm_bwd(c.dy_ln2, c.y_ln2, c.rs2, c.g2, c.b2, c.m2, bench.P_DROP, d_residual=c.dx_ln2, d_proj=c.dx_d2, dgamma=dp[:H], dbeta=dp[H:2 * H], workspace=c.ws), [c.dx_ln2, c.dx_d2, dp[:2 * H]]),
    }
    heads = bench.B * bench.A
    torch.manual_seed(59)  # fixed dO: the output checksums compare across builds
    dO = torch.randn(heads, bench.S, 64, device=dev)
    dV = torch.empty(heads, bench.S, 64, device=dev)
    torch.backends.cuda.matmul.allow_tf32 = False

    def dv_unfused():  # D materialised by attn_probs_bwd, then an fp32 cuBLAS GEMM
        o.attn_probs_bwd(c.dD, c.P, c.m_att, bench.P_DROP, write_d=True, dZ=c.dZ, D=c.Drec)
        torch.matmul(c.Drec.view(heads, bench.S, bench.S).transpose(1, 2), dO, out=dV)

    def dv_fused():  # no D: the tcgen05 GEMM rebuilds it from P and the mask
        o.attn_probs_bwd(c.dD, c.P, c.m_att, bench.P_DROP, write_d=False, dZ=c.dZ)
        o.attn_dropout_dv(c.P.view(heads, bench.S, bench.S), c.m_att, bench.P_DROP, dO, dV=dV)

    ctx = torch.empty(heads, bench.S, 64, device=dev)

    def ctx_unfused():  # D written by the softmax forward, then an fp32 cuBLAS GEMM
        o.softmax_dropout_fwd(c.z, bench.P_DROP, mask=c.m_att, generate=True, seed=7, P=c.P, D=c.D)
        torch.matmul(c.D.view(heads, bench.S, bench.S), dO, out=ctx)

    def ctx_fused():  # no D: P + bits, then the tcgen05 GEMM rebuilds D
        o.softmax_dropout_fwd(c.z, bench.P_DROP, mask=c.m_att, generate=True, seed=7, P=c.P,
                              write_d=False)
        o.attn_dropout_ctx(c.P.view(heads, bench.S, bench.S), c.m_att, bench.P_DROP, dO, ctx=ctx)

    calls["ctx_unfused"] = (ctx_unfused, [ctx])
    calls["ctx_fused"] = (ctx_fused, [ctx])
    calls["ctx_gemm_only"] = (lambda: o.attn_dropout_ctx(c.P.view(heads, bench.S, bench.S), c.m_att, bench.P_DROP, dO, ctx=ctx), [ctx])
    calls["dv_unfused"] = (dv_unfused, [dV])
    calls["dv_fused"] = (dv_fused, [dV])
    calls["dv_gemm_only"] = (lambda: o.attn_dropout_dv(c.P.view(heads, bench.S, bench.S), c.m_att, bench.P_DROP, dO, dV=dV), [dV])
    calls["cublas_dv_only"] = (lambda: torch.matmul(c.Drec.view(heads, bench.S, bench.S).transpose(1, 2), dO, out=dV), [dV])
    calls["attn_bwd_noD"] = (lambda: o.attn_probs_bwd(c.dD, c.P, c.m_att, bench.P_DROP, write_d=False, dZ=c.dZ), [c.dZ])
    # configs[0]: the L2-resident / launch-bound GELU pair at [1024, 3072]
    n0 = 1024 * 3072
    x0 = torch.randn(n0, device=dev) * 3
    y0, dy0, dx0 = torch.empty_like(x0), torch.randn_like(x0), torch.empty_like(x0)
    m0 = torch.empty((n0 + 31) // 32, dtype=torch.int32, device=dev)
    calls["cfg0_gelu_fwd"] = (lambda: o.gelu_ip_fwd(x0, c.table, y=y0, mask=m0), [y0, m0])
    calls["cfg0_gelu_bwd"] = (lambda: o.gelu_ip_bwd(dy0, y0, m0, c.table, dx=dx0), [dx0])
    # configs[1]: LayerNorm backward at [16384, 768] (stage 1 + the dgamma/dbeta reduction)
    r1, h1 = 16384, 768
    x1 = torch.randn(r1, h1, device=dev) + 0.4
    g1_ = 1 + 0.2 * torch.randn(h1, device=dev)
    b1_ = 0.1 * torch.randn(h1, device=dev)
    y1, rs1 = o.layernorm_ip_fwd(x1, g1_, b1_)
    dy1, dx1 = torch.randn_like(x1), torch.empty_like(x1)
    dgb1 = torch.empty(2 * h1, device=dev)
    calls["cfg1_ln_bwd"] = (lambda: o.layernorm_ip_bwd(dy1, y1, rs1, g1_, b1_, dx=dx1, dgamma=dgb1[:h1], dbeta=dgb1[h1:]), [dx1, dgb1])
    ob = bench.op_bytes()
    ob["cfg1_ln_bwd"] = r1 * h1 * 12
    ob["cfg0_gelu_fwd"] = n0 * 8.125
    ob["cfg0_gelu_bwd"] = n0 * 12.125
    n_a = c.P.numel()
    ob["dv_unfused"] = n_a * 16.125 + n_a * 4 + dO.numel() * 8
    ob["dv_fused"] = n_a * 12.125 + n_a * 4.125 + dO.numel() * 8
    ob["dv_gemm_only"] = n_a * 4.125 + dO.numel() * 8
    ob["cublas_dv_only"] = n_a * 4 + dO.numel() * 8
    ob["attn_bwd_noD"] = n_a * 12.125
    ob["ctx_unfused"] = n_a * 12.125 + n_a * 4 + dO.numel() * 8
    ob["ctx_fused"] = n_a * 8.125 + n_a * 4.125 + dO.numel() * 8
    ob["ctx_gemm_only"] = n_a * 4.125 + dO.numel() * 8
    obf = bench.op_bytes(fused=True)
    ob["dal_fwd"] = obf["dropout_add_layernorm_fwd"]
    ob["dal_bwd"] = obf["dropout_add_layernorm_bwd"]
    ob["copy_g"] = 8 * c.x_ffn1.numel()
    ob["mt_mask"] = c.z.numel() / 8
    ob["mt_mask_h"] = c.x_ffn2.numel() / 8
    ob["copy_h"] = 2 * 8 * c.x_ffn2.numel()
    names = {"ln_fwd": "layernorm_fwd", "ln_bwd": "layernorm_bwd", "gelu_fwd_exact": "gelu_fwd"}
    reps = int(os.environ.get("REPS", "20"))
    st = torch.cuda.current_stream()
    for name in sys.argv[1:]:
        fn, outs = calls[name]
        fn()
        ts = []
        for _ in range(reps):
            flush()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(st)
            fn()
            b.record(st)
            b.synchronize()
            ts.append(a.elapsed_time(b))
        t = bench.trimmed_mean(ts)
        key = names.get(name, name)
        nbytes = ob[key] / (2 if key in ("layernorm_fwd", "layernorm_bwd", "dropout_fwd", "dropout_bwd", "copy_h", "dal_fwd", "dal_bwd") else 1)
        h = hashlib.sha1()
        parts = []
        for t_ in outs:
            b_ = t_.detach().cpu().numpy().tobytes()
            h.update(b_)
            parts.append(hashlib.sha1(b_).hexdigest()[:6])
        print(json.dumps({"op": name, "lib": os.environ.get("TEMPO_B200_LIB", "default"),
                          "us": round(t * 1e3, 2), "min_us": round(min(ts) * 1e3, 2),
                          "gbs": round(nbytes / t / 1e6, 1), "frac": round(nbytes / t / 1e6 / peak, 4),
                          "sha": h.hexdigest()[:12], "parts": parts}), flush=True)


if __name__ == "__main__":
    main()
