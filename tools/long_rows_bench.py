"""Device timings of the row kernels across row lengths (softmax+dropout fwd
and attn-probs bwd over S, LayerNorm fwd/bwd and the fused dropout -> add ->
LayerNorm over H) at a fixed element count, against the measured copy peak.
CUDA events, median of reps, L2 cleaned by reading a 512 MB buffer before
every rep.  Prints one JSON object.  Not part of the bench contract (bench.py
reports the same numbers in its `per_row_length` section)."""
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch
    from paper_2210_10246_b200 import ops
    dev = torch.device("cuda:0")
    peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))).get("hbm_gbs", 6532.9) \
        if os.path.exists(os.path.join(ROOT, "MEASURED_PEAKS.json")) else 6532.9
    fb = torch.empty(128 * 1024 * 1024, device=dev)
    sink = torch.empty(1, device=dev)

    def timeit(fn, reps=10):
        fn()
        ts = []
        for _ in range(reps):
            sink.copy_(fb.sum())
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            fn()
            b.record()
            b.synchronize()
            ts.append(a.elapsed_time(b))
        return statistics.median(ts)

    out = {"peak_gbs": peak, "softmax": [], "layernorm": []}
    n_attn = int(os.environ.get("N_ATTN", 1 << 27))
    for S in [int(s) for s in os.environ.get("SEQS", "512,1024,2048,3072,4096,8192").split(",")]:
        rows = n_attn // S
        n = rows * S
        z = torch.randn(rows, S, device=dev)
        P = torch.empty_like(z)
        D = torch.empty_like(z)
        m = torch.empty(ops.mask_words(n), dtype=torch.int32, device=dev)
        dD = torch.randn_like(z)
        dZ = torch.empty_like(z)
        tf = timeit(lambda: ops.softmax_dropout_fwd(z, 0.1, mask=m, seed=1, P=P, D=D, generate=True))
        tb = timeit(lambda: ops.attn_probs_bwd(dD, P, m, 0.1, dZ=dZ))
        bf, bb = n * 12.125, n * 12.125
        out["softmax"].append({"S": S, "rows": rows,
                               "fwd_ms": round(tf, 4), "fwd_frac": round(bf / tf / 1e6 / peak, 4),
                               "bwd_ms": round(tb, 4), "bwd_frac": round(bb / tb / 1e6 / peak, 4)})
        del z, P, D, m, dD, dZ
    n_ln = int(os.environ.get("N_LN", 1 << 25))
    for H in [int(h) for h in os.environ.get("HIDDENS", "1024,2048,2560,4096,8192,12288").split(",")]:
        rows = n_ln // H
        n = rows * H
        x = torch.randn(rows, H, device=dev)
        r = torch.randn_like(x)
        g = 1 + 0.1 * torch.randn(H, device=dev)
        b = 0.1 * torch.randn(H, device=dev)
        y = torch.empty_like(x)
        rs = torch.empty(rows, device=dev)
        dy = torch.randn_like(x)
        dx = torch.empty_like(x)
        dp = torch.empty_like(x)
        dg = torch.empty(H, device=dev)
        db = torch.empty(H, device=dev)
        m = torch.empty(ops.mask_words(n), dtype=torch.int32, device=dev)
        ws = ops.ln_workspace(rows, H, dev)
        tf = timeit(lambda: ops.layernorm_ip_fwd(x, g, b, y=y, rstd=rs, check_gamma=False))
        tb = timeit(lambda: ops.layernorm_ip_bwd(dy, y, rs, g, b, dx=dx, dgamma=dg, dbeta=db,
                                                 workspace=ws))
        tdf = timeit(lambda: ops.dropout_add_layernorm_fwd(x, r, g, b, 0.1, seed=3, mask=m, y=y,
                                                           rstd=rs, generate=True, check_gamma=False))
        tdb = timeit(lambda: ops.dropout_add_layernorm_bwd(dy, y, rs, g, b, m, 0.1, d_residual=dx,
                                                           d_proj=dp, dgamma=dg, dbeta=db,
                                                           workspace=ws))
        out["layernorm"].append({
            "H": H, "rows": rows,
            "fwd_ms": round(tf, 4), "fwd_frac": round(n * 8 / tf / 1e6 / peak, 4),
            "bwd_ms": round(tb, 4), "bwd_frac": round(n * 12 / tb / 1e6 / peak, 4),
            "dal_fwd_ms": round(tdf, 4), "dal_fwd_frac": round(n * 12.125 / tdf / 1e6 / peak, 4),
            "dal_bwd_ms": round(tdb, 4), "dal_bwd_frac": round(n * 16.125 / tdb / 1e6 / peak, 4)})
    print(json.dumps(out))


if __name__ == "__main__":
    main()
