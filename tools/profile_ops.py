"""Run one step of the (fused) bench chain, then each Tempo kernel ONCE at the
bench shapes (BERT-large layer, B=64): the fused chain's ops (softmax+dropout
fwd, attn-probs bwd, GELU fwd/bwd, dropout+add+LN fwd/bwd: 7 kernels with the
dgamma/dbeta reduce), the unfused chain's LN and dropout ops (5 kernels), and
configs[0..2] at their own shapes (7 kernels) -- the command
tools/profile_round.sh wraps in `ncu --set full -s 10 -c 19` (skip the
step's 10 launches)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch
    import bench
    dev = torch.device("cuda:0")
    chain = bench.Chain(dev, 0, 1, fused=True)
    chain.step()
    torch.cuda.synchronize()
    res = chain.per_op_timings(reps=0, flush=lambda: None)
    unf = bench.Chain(dev, 0, 1, fused=False)
    o, c, H = unf.ops, unf, bench.H
    dp = c.dparams
    o.layernorm_ip_fwd(c.d1, c.g1, c.b1, check_gamma=False, y=c.y_ln1, rstd=c.rs1)
    o.layernorm_ip_bwd(c.dy_ln1, c.y_ln1, c.rs1, c.g1, c.b1, dx=c.dx_ln1, dgamma=dp[:H],
                       dbeta=dp[H:2 * H], workspace=c.ws)
    o.dropout_fwd(c.x_ffn2, bench.P_DROP, mask=c.m2, generate=True, seed=9, y=c.d2)
    o.dropout_bwd(c.dx_ln2, c.m2, bench.P_DROP, dx=c.dx_d2)
    torch.cuda.synchronize()
    del unf, chain
    # configs[0..2] at their own shapes, one call each (no CUDA graph: ncu
    # would see the replays as more launches of the same kernels)
    g = torch.Generator(device=dev)
    g.manual_seed(77)
    rn = lambda *s_: torch.randn(*s_, device=dev, generator=g)  # noqa: E731
    table = o.GeluTable.default()
    x1 = rn(1024, 3072)
    y1, m1 = o.gelu_ip_fwd(x1, table)
    o.gelu_ip_bwd(rn(1024, 3072), y1, m1, table)
    x2 = rn(16384, 768)
    ga, be = (1 + 0.2 * rn(768)).contiguous(), (0.1 * rn(768)).contiguous()
    y2, rs2 = o.layernorm_ip_fwd(x2, ga, be, check_gamma=False)
    o.layernorm_ip_bwd(rn(16384, 768), y2, rs2, ga, be)
    z3 = rn(32 * 12 * 512, 512)
    P3, D3, m3 = o.softmax_dropout_fwd(z3, bench.P_DROP, seed=5)
    o.attn_probs_bwd(rn(32 * 12 * 512, 512), P3, m3, bench.P_DROP, write_d=True)
    torch.cuda.synchronize()
    print("ran", list(res))


if __name__ == "__main__":
    main()
