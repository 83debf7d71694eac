"""Run one bench step, then each Tempo kernel of the chain ONCE at the bench
shapes (BERT-large layer, B=64) -- the command tools/profile_round.sh wraps in
`ncu --set full -s 14 -c 9` (skip the step's 14 launches, capture the 9
distinct kernels: 8 ops + the LayerNorm dgamma/dbeta reduce)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch
    import bench
    dev = torch.device("cuda:0")
    chain = bench.Chain(dev, 0, 1)
    chain.step()
    torch.cuda.synchronize()
    res = chain.per_op_timings(reps=0, flush=lambda: None)
    torch.cuda.synchronize()
    print("ran", list(res))


if __name__ == "__main__":
    main()
