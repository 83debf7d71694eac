"""Run each Tempo kernel of the bench chain a few times at the bench shapes
(BERT-large layer, B=64) -- the command ncu wraps for profiles/.

    ncu --set full -k regex:<kernel> -c 1 python tools/profile_ops.py [op ...]
"""
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
    flush_buf = torch.empty(64 * 1024 * 1024, device=dev)
    calls = chain.per_op_timings(reps=2, flush=lambda: flush_buf.fill_(0.0))
    for name, (ms, _) in calls.items():
        print(f"{name:22s} {ms:.4f} ms")


if __name__ == "__main__":
    main()
