"""The C++ operator API (include/tempo_b200/tempo.hpp: Graph / Tape /
StashLedger / Tensor / BoolMask / GeluPolyTable and tempo_ops::*, the
reference's proj/include/tempo interface on device buffers)."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "paper_2210_10246_b200", "_lib")


def test_host_library_links_the_c_abi():
    so = os.path.join(LIB, "libtempo_b200_host.so")
    assert os.path.exists(so)
    out = subprocess.run(["nm", "-DC", "--defined-only", so], capture_output=True, text=True,
                         check=True).stdout
    for sym in ["tempo_b200::tempo_ops::gelu(", "tempo_b200::tempo_ops::layernorm(",
                "tempo_b200::tempo_ops::softmax(", "tempo_b200::tempo_ops::dropout_recompute(",
                "tempo_b200::ref_ops::dropout(", "tempo_b200::Tape::backward(",
                "tempo_b200::StashLedger::live_by_tag"]:
        assert sym in out, sym
    deps = subprocess.run(["ldd", so], capture_output=True, text=True).stdout
    assert "libtempo_b200.so" in deps


@pytest.mark.gpu
def test_cpp_operator_api_on_gpu(cuda):
    exe = os.path.join(LIB, "test_host")
    out = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    print(out.stdout)
    assert out.returncode == 0, out.stdout + out.stderr
    assert "0 failure(s)" in out.stdout


@pytest.mark.gpu
def test_inplace_elementwise_functor_kernels(cuda):
    """include/tempo_b200/inplace_elementwise.cuh: the reference's generic
    scheme (ops_tempo.cpp:32-71) as compile-time device specs."""
    exe = os.path.join(LIB, "test_elementwise")
    out = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    print(out.stdout)
    assert out.returncode == 0, out.stdout + out.stderr
    assert "0 failure(s)" in out.stdout
