"""Average board power while each op of the chain runs back to back for ~1.5 s
(nvidia-smi power.draw sampled every 50 ms) -- which kernels burn the power
budget that caps the sustained chain.  Not part of the contract."""
import os
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch
    import bench
    from paper_2210_10246_b200 import ops as o
    dev = torch.device("cuda:0")
    c = bench.Chain(dev, 0, 1)
    c.step()
    torch.cuda.synchronize()
    H = bench.H
    dp = c.dparams
    calls = {
        "softmax_dropout_fwd": lambda: o.softmax_dropout_fwd(c.z, 0.1, mask=c.m_att, generate=True, seed=7, P=c.P, D=c.D),
        "attn_probs_bwd": lambda: o.attn_probs_bwd(c.dD, c.P, c.m_att, 0.1, write_d=True, dZ=c.dZ, D=c.Drec),
        "gelu_fwd": lambda: o.gelu_ip_fwd(c.x_ffn1, c.table, y=c.y_g, mask=c.m_g),
        "gelu_bwd": lambda: o.gelu_ip_bwd(c.dy_gelu, c.y_g, c.m_g, c.table, dx=c.dx_g),
        "ln_fwd": lambda: o.layernorm_ip_fwd(c.d1, c.g1, c.b1, check_gamma=False, y=c.y_ln1, rstd=c.rs1),
        "ln_bwd": lambda: o.layernorm_ip_bwd(c.dy_ln1, c.y_ln1, c.rs1, c.g1, c.b1, dx=c.dx_ln1, dgamma=dp[:H], dbeta=dp[H:2 * H], workspace=c.ws),
        "dropout_fwd": lambda: o.dropout_fwd(c.x_ffn2, 0.1, mask=c.m2, generate=True, seed=9, y=c.d2),
        "copy_1GB": lambda: c.dZ.copy_(c.z),
    }
    only = [a for a in sys.argv[1:]]
    for name, fn in calls.items():
        if only and name not in only:
            continue
        fn()
        torch.cuda.synchronize()
        p = subprocess.Popen(["nvidia-smi", "--id=0", "--query-gpu=power.draw,clocks.sm",
                              "--format=csv,noheader,nounits", "-lms", "50"],
                             stdout=subprocess.PIPE, text=True)
        time.sleep(0.2)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        n = 0
        t0 = time.time()
        while time.time() - t0 < 1.5:
            for _ in range(20):
                fn()
            n += 20
            torch.cuda.synchronize()
        b.record()
        b.synchronize()
        p.terminate()
        out, _ = p.communicate()
        vals = [line.split(",") for line in out.strip().splitlines()]
        pw = [float(v[0]) for v in vals if len(v) > 1][4:]
        sm = [float(v[1]) for v in vals if len(v) > 1][4:]
        print(f"{name:22s} W avg {sum(pw)/max(1,len(pw)):6.1f} max {max(pw) if pw else 0:6.1f}  "
              f"sm MHz avg {sum(sm)/max(1,len(sm)):6.0f}  us/launch {a.elapsed_time(b)*1e3/n:8.1f}")


if __name__ == "__main__":
    main()
