"""Exhaustive accuracy of the In-Place GELU forward value: every fp32 input,
the product's device code (fp32 fast path + fp64 window/tail paths) against
the reference's double formula (tests/tools/gelu_sweep.cu)."""
import json
import os
import subprocess

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
TOOL = os.path.join(ROOT, "tests", "tools", "_build", "gelu_sweep")


def test_gelu_forward_every_float(cuda):
    assert os.path.exists(TOOL), "build the test tools: __graft_entry__.build()"
    out = subprocess.run([TOOL], capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stdout + out.stderr
    r = json.loads(out.stdout.strip().splitlines()[-1])
    print(r)
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    with open(os.path.join(ROOT, "gpurun_out", "gelu_sweep.json"), "w") as f:
        json.dump(r, f)
    assert r["checked"] > 3_000_000_000
    assert r["nan_mismatch"] == 0
    assert r["window_mismatch"] == 0      # fp64 window: the reference's value exactly
    assert r["max_ulp"] <= 8              # fp32 fast path bound


def test_gelu_kernel_every_float(tops, cuda):
    """The shipped forward KERNEL (256-bit vector path, through the C-ABI) on
    every fp32 bit pattern, in 2^28-element batches: y against the reference
    formula evaluated in fp64 (torch's CUDA erfc), the mask bit against the
    reference's strict `x > x*` with the table's double x* (ops_tempo.cpp:77-78)."""
    import math
    import torch

    table = tops.GeluTable.default()
    xstar = table.info()["x_star"]
    step = 1 << 28
    max_ulp, win_bad, nan_bad, mask_bad, checked = 0, 0, 0, 0, 0
    hist = torch.zeros(9, dtype=torch.int64, device=cuda)
    shifts = torch.arange(32, device=cuda, dtype=torch.int32)
    for b in range(0, 1 << 32, step):
        u = torch.arange(b, b + step, device=cuda, dtype=torch.int64)
        x = (u - (1 << 32) * (u >= (1 << 31))).to(torch.int32).view(torch.float32)
        y, m = tops.gelu_ip_fwd(x, table)
        xd = x.double()
        ref = (xd * (0.5 * torch.special.erfc(-xd * math.sqrt(0.5)))).float()
        bits = ((m.view(-1, 1) >> shifts) & 1).flatten().bool()
        mask_bad += int((bits != (xd > xstar)).sum())
        yn, rn = torch.isnan(y), torch.isnan(ref)
        nan_bad += int((yn != rn).sum())
        ok = ~(yn | rn)
        yi, ri = y.view(torch.int32).long(), ref.view(torch.int32).long()
        od = lambda i: torch.where(i < 0, -(i & 0x7fffffff), i)  # noqa: E731
        d = (od(yi) - od(ri)).abs()[ok]
        checked += int(d.numel())
        max_ulp = max(max_ulp, int(d.max()))
        hist += torch.bincount(d.clamp(max=8), minlength=9)
        win = ok & ((x - (-0.751791537)).abs() < 0.015625)
        win_bad += int(((yi != ri) & win).sum())
        del u, x, y, m, xd, ref, bits
    r = {"checked": checked, "max_ulp": max_ulp, "hist": hist.tolist(), "window_mismatch": win_bad,
         "nan_mismatch": nan_bad, "mask_mismatch": mask_bad}
    print(r)
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    with open(os.path.join(ROOT, "gpurun_out", "gelu_kernel_sweep.json"), "w") as f:
        json.dump(r, f)
    assert checked > 4_000_000_000
    assert mask_bad == 0 and nan_bad == 0 and win_bad == 0
    assert max_ulp <= 8
