"""Device time of the attention mask + softmax forward at the bench shape
(B=64, A=16, S=512: 2^28 elements) with the reference's mask stream: the
separate passes (device keep-bit generation, then the supplied-mask forward)
vs the generation inside the softmax kernel.  CUDA events, median of reps."""
import statistics
import sys
import os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch
    from paper_2210_10246_b200 import ops
    dev = torch.device("cuda:0")
    rows, S = 64 * 16 * 512, 512
    n = rows * S
    z = torch.randn(rows, S, device=dev)
    P, D = torch.empty_like(z), torch.empty_like(z)
    m = torch.empty(ops.mask_words(n), dtype=torch.int32, device=dev)
    nb = int(ops.lib().tempo_bernoulli_keep_bits_workspace_size(0, n))
    ws = torch.empty(nb, dtype=torch.uint8, device=dev)

    def t(fn, reps=7):
        fn()
        torch.cuda.synchronize()
        ts = []
        for _ in range(reps):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            fn()
            b.record()
            b.synchronize()
            ts.append(a.elapsed_time(b))
        return statistics.median(ts)

    sep_gen = t(lambda: ops.bernoulli_keep_bits_device(n, 0.1, 5, out=m))
    sep_smx = t(lambda: ops.softmax_dropout_fwd(z, 0.1, mask=m, P=P, D=D))
    fused = t(lambda: ops.softmax_dropout_fwd_refmask(z, 0.1, 5, mask=m, P=P, D=D, workspace=ws))
    print({"separate_generation_ms": round(sep_gen, 4), "separate_softmax_ms": round(sep_smx, 4),
           "fused_ms": round(fused, 4)})


if __name__ == "__main__":
    main()
