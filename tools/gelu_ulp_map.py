"""Where does the GELU forward's fp32 fast path lose ulps?  Every fp32 input
through the shipped kernel, ulp distance to the reference formula evaluated
in fp64 (torch's CUDA erfc), histogrammed by x (sign, binade)."""
import json, math, os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2210_10246_b200 import ops


def main():
    dev = torch.device("cuda:0")
    t = ops.GeluTable.default()
    step = 1 << 28
    # key: (sign, unbiased exponent) -> [count, n>2ulp, max ulp, x at max]
    stats = {}
    for b in range(0, 1 << 32, step):
        u = torch.arange(b, b + step, device=dev, dtype=torch.int64)
        x = (u - (1 << 32) * (u >= (1 << 31))).to(torch.int32).view(torch.float32)
        y, _ = ops.gelu_ip_fwd(x, t)
        xd = x.double()
        ref = (xd * (0.5 * torch.special.erfc(-xd * math.sqrt(0.5)))).float()
        ok = ~(torch.isnan(y) | torch.isnan(ref))
        yi, ri = y.view(torch.int32).long(), ref.view(torch.int32).long()
        od = lambda i: torch.where(i < 0, -(i & 0x7fffffff), i)  # noqa: E731
        d = (od(yi) - od(ri)).abs()
        d = torch.where(ok, d, torch.zeros_like(d))
        xb = x.view(torch.int32)
        key = ((xb >> 23) & 0x1ff).long()  # sign<<8 | biased exponent
        cnt = torch.bincount(key, minlength=512)
        big = torch.bincount(key[d > 2], minlength=512)
        mx = torch.zeros(512, dtype=torch.int64, device=dev).scatter_reduce(0, key, d, "amax")
        for k in torch.nonzero(cnt).flatten().tolist():
            s = stats.setdefault(k, [0, 0, 0])
            s[0] += int(cnt[k]); s[1] += int(big[k]); s[2] = max(s[2], int(mx[k]))
    rows = []
    for k in sorted(stats):
        sign, e = k >> 8, (k & 0xff) - 127
        c, nb, m = stats[k]
        if m > 2:
            rows.append({"sign": "-" if sign else "+", "binade": f"2^{e}", "count": c, "gt2ulp": nb, "max_ulp": m})
    print(json.dumps(rows))
    os.makedirs("gpurun_out", exist_ok=True)
    json.dump(rows, open("gpurun_out/gelu_ulp_map.json", "w"), indent=1)


if __name__ == "__main__":
    main()
