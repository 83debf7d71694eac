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
