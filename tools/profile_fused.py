"""One fused dropout+residual+LayerNorm forward and backward at the bench
shape (32768 x 1024), after a warm-up step -- for
`ncu --set full -k regex:'dal_|ln_bwd_vec' -s 3` captures."""
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
    torch.cuda.synchronize()
    print("ran", list(res))


if __name__ == "__main__":
    main()
