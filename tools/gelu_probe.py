"""GELU forward timing vs input distribution (how much the fp64 window costs)."""
import os, sys, statistics
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))
from microbench import timeit  # noqa: E402


def main():
    import torch
    from paper_2210_10246_b200 import ops
    dev = torch.device("cuda:0")
    fb = torch.empty(64 * 1024 * 1024, device=dev)
    flush = lambda: fb.fill_(0)  # noqa: E731
    n = 32768 * 4096
    t = ops.GeluTable.default()
    y = torch.empty(n, device=dev)
    m = torch.empty(ops.mask_words(n), dtype=torch.int32, device=dev)
    for name, x in [("randn", torch.randn(n, device=dev)),
                    ("uniform[0.5,3]", torch.rand(n, device=dev) * 2.5 + 0.5),
                    ("uniform[-3,-1]", -torch.rand(n, device=dev) * 2 - 1),
                    ("all-window", torch.full((n,), -0.7517915, device=dev))]:
        ms = timeit(lambda: ops.gelu_ip_fwd(x, t, y=y, mask=m), flush)
        print(f"{name:16s} {ms:.4f} ms  {n*8.125/ms/1e6:.0f} GB/s")
        dy = torch.randn(n, device=dev)
        dx = torch.empty_like(dy)
        ops.gelu_ip_fwd(x, t, y=y, mask=m)
        ms = timeit(lambda: ops.gelu_ip_bwd(dy, y, m, t, dx=dx), flush)
        print(f"{'  bwd':16s} {ms:.4f} ms  {n*12.125/ms/1e6:.0f} GB/s")


if __name__ == "__main__":
    main()
