"""Error of the ctx / dV GEMMs against the fp64 product of the recomputed D, in
units of the test bound (|ref| + sum_j |D_ij V_jc|): max and mean of
|got - ref| / (|ref| + mag), for a few s_k.  Run with TEMPO_B200_LIB to compare
builds.  Prints one JSON line."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch
    from paper_2210_10246_b200 import ops
    dev = torch.device("cuda:0")
    out = {"lib": os.environ.get("TEMPO_B200_LIB", "in-tree")}
    for s_k in (512, 2048, 8192):
        heads, s_q, d, p = 4, 256, 64, 0.1
        z = torch.randn(heads * s_q, s_k, device=dev) * 3
        P, D, m = ops.softmax_dropout_fwd(z, p, seed=s_k)
        V = torch.randn(heads, s_k, d, device=dev)
        ctx = ops.attn_dropout_ctx(P.view(heads, s_q, s_k), m, p, V)
        Dd = D.view(heads, s_q, s_k).double()
        ref = torch.matmul(Dd, V.double())
        mag = torch.matmul(Dd.abs(), V.double().abs())
        e = (ctx.double() - ref).abs() / (ref.abs() + mag)
        r = {"max": float(e.max()), "mean": float(e.mean())}
        if True:
            dO = torch.randn(heads, s_q, d, device=dev)
            Pq = P.view(heads, s_q, s_k)
            if s_k % 256 == 0:
                dV = ops.attn_dropout_dv(Pq, m, p, dO)
                refv = torch.matmul(Dd.transpose(1, 2), dO.double())
                magv = torch.matmul(Dd.abs().transpose(1, 2), dO.double().abs())
                ev = (dV.double() - refv).abs() / (refv.abs() + magv)
                r["dv_max"], r["dv_mean"] = float(ev.max()), float(ev.mean())
        out[f"s_k={s_k}"] = r
    # dV's reduction runs over s_q: a long-K case for it
    heads, s_q, s_k, d, p = 1, 8192, 256, 64, 0.1
    z = torch.randn(heads * s_q, s_k, device=dev) * 3
    P, D, m = ops.softmax_dropout_fwd(z, p, seed=5)
    dO = torch.randn(heads, s_q, d, device=dev)
    dV = ops.attn_dropout_dv(P.view(heads, s_q, s_k), m, p, dO)
    Dd = D.view(heads, s_q, s_k).double()
    refv = torch.matmul(Dd.transpose(1, 2), dO.double())
    magv = torch.matmul(Dd.abs().transpose(1, 2), dO.double().abs())
    ev = (dV.double() - refv).abs() / (refv.abs() + magv)
    out["dv_s_q=8192"] = {"max": float(ev.max()), "mean": float(ev.mean())}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
