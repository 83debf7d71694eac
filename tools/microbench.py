"""Ad-hoc device timings of single ops vs a plain copy of the same bytes
(CUDA events, L2 flushed before every rep).  Not part of the contract."""
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def timeit(fn, flush, reps=10):
    import torch
    fn()
    ts = []
    for _ in range(reps):
        flush()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        b.synchronize()
        ts.append(a.elapsed_time(b))
    return statistics.median(ts)


def main():
    import torch
    from paper_2210_10246_b200 import ops
    dev = torch.device("cuda:0")
    fb = torch.empty(64 * 1024 * 1024, device=dev)
    flush = lambda: fb.fill_(0)  # noqa: E731
    for n in (1 << 25, 1 << 27, 1 << 29):
        x = torch.randn(n, device=dev)
        y = torch.empty_like(x)
        m = torch.empty(ops.mask_words(n), dtype=torch.int32, device=dev)
        ops.dropout_fwd(x, 0.1, mask=m, generate=True, seed=1, y=y)
        gb = 8 * n / 1e9
        t_copy = timeit(lambda: y.copy_(x), flush)
        t_bwd = timeit(lambda: ops.dropout_bwd(x, m, 0.1, dx=y), flush)
        t_fwd = timeit(lambda: ops.dropout_fwd(x, 0.1, mask=m, generate=True, seed=1, y=y), flush)
        print(f"n=2^{n.bit_length()-1}: copy {gb/t_copy*1e3:.0f} GB/s  dropout_bwd "
              f"{(gb+n/8/1e9)/t_bwd*1e3:.0f}  dropout_fwd {(gb+n/8/1e9)/t_fwd*1e3:.0f}")


if __name__ == "__main__":
    main()
