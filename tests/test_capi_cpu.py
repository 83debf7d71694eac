"""CPU-side checks of the C-ABI library (no GPU needed):

* the library loads and exports every entry point include/tempo_b200.h
  declares;
* the v1 table parser/validator accepts and rejects exactly what the
  reference's GeluPolyTable::parse does (gelu_table.cpp:227-301, :106-148),
  re-serializes bitwise (test_gelu_fit.cpp:134-151) and its host eval equals
  the reference's eval;
* argument errors map to the reference's exception classes before any GPU
  work (ops_tempo.cpp:80-83, 91-94; ops_reference.cpp:50-52, 148-151);
* the host mask stream equals BoolMask::bernoulli_keep and mask_stream_seed;
* stash accounting equals the reference memory model.
"""
import os
import re
import subprocess

import numpy as np
import pytest

from paper_2210_10246_b200 import _capi, ops
from paper_2210_10246_b200._capi import TempoError

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "tempo_b200.h")


def header_functions():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(tempo_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_header_symbol():
    names = header_functions()
    assert len(names) >= 25
    out = subprocess.run(["nm", "-D", "--defined-only", _capi.LIB_PATH], capture_output=True,
                         text=True, check=True).stdout
    exported = set(re.findall(r" T (tempo_\w+)", out))
    missing = [n for n in names if n not in exported]
    assert not missing, missing
    assert set(names) == set(_capi.SIGNATURES), "ctypes signature table out of sync with header"
    lib = _capi.lib()
    for n in names:
        assert hasattr(lib, n)


def test_library_is_sm100a():
    out = subprocess.run(["cuobjdump", "-lelf", _capi.LIB_PATH], capture_output=True, text=True)
    assert "sm_100a" in out.stdout, out.stdout + out.stderr


def test_default_table_is_the_reference_fit(table_text):
    assert _capi.lib().tempo_gelu_default_table_v1().decode() == table_text
    t = ops.GeluTable.default()
    assert t.serialize() == table_text  # bitwise round trip
    info = t.info()
    assert info["verified"] and info["n_segments"] == 6 and info["max_degree"] == 10
    assert info["x_star"] == pytest.approx(-0.75179152469356446, rel=1e-9)


@pytest.mark.parametrize("m", [0, 1])
def test_host_eval_matches_reference(golden, m):
    t = ops.GeluTable.default()
    y = golden[f"eval_y_m{m}"]
    h = t.eval_host(y, np.full(y.size, m, np.uint8))
    assert np.array_equal(h, golden[f"eval_h_m{m}"])


def _mutations(good: str):
    lines = good.splitlines(keepends=True)
    hdr = lines[0]
    yield "empty", ""
    yield "magic", "not-a-table v1\n"
    yield "version", good.replace(" v1 ", " v9 ", 1)
    yield "trailing", good.replace("\n", " 0.25\n", 2).replace(" 0.25\n", "\n", 1)
    yield "gap", hdr + "".join(lines[2:])
    yield "header_extra", hdr.rstrip("\n") + " extra=1\n" + "".join(lines[1:])
    yield "header_trunc", "gelu-poly-table v1 x_star=-0.75 y_min=-0.17\n"
    yield "bad_branch", good.replace("\n0 ", "\n2 ", 1)
    yield "bad_var", good.replace("direct-y", "cubic", 1)
    yield "bad_degree", good.replace("sqrt-shift 3", "sqrt-shift x", 1)
    yield "neg_tol", good.replace("tol=0.0001", "tol=-1", 1)
    yield "nan_coef", good.replace("0.69354245105000201", "nan", 1)
    yield "unbounded_poly", good.replace("8 inf direct-y 0 1", "8 inf direct-y 1 1 0", 1)
    yield "one_branch", "".join(l for l in lines if not l.startswith("0 "))
    yield "unverified", good.replace("max_err=7.9034905239312725e-05", "max_err=-1", 1)
    yield "shuffled", hdr + "".join(reversed(lines[1:]))
    yield "blank_lines", good.replace("\n", "\n\n")


def test_parser_matches_reference_accept_reject(ref, table_text):
    from oracle import OracleError
    for name, text in _mutations(table_text):
        try:
            ref.table_parse(text)
            ref_ok, ref_code = True, 0
        except OracleError as e:
            ref_ok, ref_code = False, e.code
        try:
            ops.GeluTable(text).close()
            ok, code = True, 0
        except TempoError as e:
            ok, code = False, e.code
        assert (ok, code) == (ref_ok, ref_code), name


def test_parser_rejections_standalone(table_text):
    # same set without the reference library: the reference's outcomes,
    # recorded from test_parser_matches_reference_accept_reject
    expect_ok = {"unverified", "shuffled", "blank_lines"}
    for name, text in _mutations(table_text):
        if name in expect_ok:
            ops.GeluTable(text).close()
        else:
            with pytest.raises(TempoError) as ei:
                ops.GeluTable(text)
            assert ei.value.kind == "ParseError", name


def test_argument_errors_before_gpu_work(table_text):
    L = _capi.lib()
    t = ops.GeluTable(table_text)
    # gelu without a table: ConfigError (ops_tempo.cpp:91-94)
    assert L.tempo_gelu_ip_fwd(None, None, None, 0, None, None) == 5
    # unverified table refuses the backward (ops_tempo.cpp:80-83)
    u = ops.GeluTable(table_text.replace("max_err=7.9034905239312725e-05", "max_err=-1"))
    assert not u.info()["verified"]
    assert L.tempo_gelu_ip_bwd(None, None, None, u.handle, None, 0, None) == 5
    assert b"sweep-verified" in L.tempo_last_error()
    # dropout p outside [0,1): ParamError (ops_reference.cpp:148-151)
    for p in (1.0, -0.1, float("nan")):
        assert L.tempo_dropout_fwd(None, p, 0, None, 0, 0, None, 0, None) == 3
        assert L.tempo_dropout_bwd(None, None, p, None, 0, None) == 3
        assert L.tempo_softmax_dropout_fwd(None, p, 0, None, 0, 0, None, None, 0, 0, None) == 3
        assert L.tempo_attn_probs_bwd(None, None, None, p, None, None, 0, 0, None) == 3
    # epsilon <= 0: ParamError (ops_reference.cpp:50-52)
    assert L.tempo_ln_ip_fwd(None, None, None, 0.0, None, None, 0, 4, None, None) == 3
    # empty last dim: DimensionError (kernels.cpp:158-161)
    assert L.tempo_ln_ip_fwd(None, None, None, 1e-5, None, None, 3, 0, None, None) == 2
    assert L.tempo_softmax_ip_fwd(None, None, 3, 0, None) == 2
    # negative sizes
    assert L.tempo_gelu_ip_fwd(None, None, None, -1, t.handle, None) == 2
    # zero-size work is a no-op that succeeds without touching a device
    assert L.tempo_gelu_ip_fwd(None, None, None, 0, t.handle, None) == 0
    assert L.tempo_dropout_fwd(None, 0.1, 1, None, 0, 0, None, 0, None) == 0
    # unknown mask mode
    assert L.tempo_dropout_fwd(None, 0.1, 7, None, 0, 0, None, 0, None) == 3


def test_host_mask_stream_is_bernoulli_keep(port, golden):
    for n, p, seed, key in [(1000, 0.1, 42, "keep_n1000_p01_s42"), (777, 0.5, 19, "keep_n777_p05_s19")]:
        bits = ops.bernoulli_keep_bits(n, p, seed)
        unpacked = np.unpackbits(bits.view(np.uint8), bitorder="little")[:n]
        assert np.array_equal(unpacked, golden[key])
    bits = ops.bernoulli_keep_bits(100003, 0.1, 7)
    unpacked = np.unpackbits(bits.view(np.uint8), bitorder="little")
    assert np.array_equal(unpacked[:100003], port.bernoulli_keep(100003, 0.1, 7))
    assert not unpacked[100003:].any()  # padding bits stay 0
    with pytest.raises(TempoError):
        ops.bernoulli_keep_bits(10, 1.0, 0)


def test_mask_stream_seed(golden):
    seeds = [ops.mask_stream_seed(s, salt, site) for s in (0, 1, 12345) for salt in (0, 1, 7)
             for site in (0, 1, 2)]
    assert np.array_equal(np.array(seeds, np.uint64), golden["stream_seeds"])


def test_stash_bytes_match_memory_model(golden):
    for s, h, a, r, o, *_ in golden["memory_model"]:
        s, h, a = int(s), int(h), int(a)
        assert ops.layer_stash_bytes_per_token(s, h, a, tempo=False, mask_bits=False) == r
        assert ops.layer_stash_bytes_per_token(s, h, a, tempo=True, mask_bits=False) == o
    # bit-packed masks: BERT-large S=512 -> 75,528 B/token
    assert ops.layer_stash_bytes_per_token(512, 1024, 16, tempo=True, mask_bits=True) == 75528


def _extra_tables():
    import json
    with open(os.path.join(ROOT, "tests", "golden", "gelu_tables_extra.json")) as f:
        return json.load(f)


@pytest.mark.parametrize("name", sorted(_extra_tables()))
def test_extra_tables_parse_roundtrip_and_eval(name, port):
    """Tables the reference fits with other tolerances / degree caps (more
    segments than the default): parsed, re-serialized bitwise, and evaluated
    on the host exactly like the reference (the C oracle is pinned to it)."""
    text = _extra_tables()[name]
    t = ops.GeluTable(text)
    assert t.serialize() == text
    info = t.info()
    assert info["verified"] and info["n_segments"] >= 9
    pt = port.table(text)
    ys = np.concatenate([np.linspace(-0.2, 9.0, 50001), [info["y_min"], 0.0, 8.0, 1e30]])
    for m in (0, 1):
        mm = np.full(ys.size, m, np.uint8)
        assert np.array_equal(t.eval_host(ys, mm), pt.eval(ys, mm))


def test_peer_exchange_sizes_and_argument_errors():
    """The fused multi-GPU dgamma/dbeta exchange: buffer sizes (two epoch
    parities x world slots of the padded 2*cols fp64 / one flag per 32-column
    block) and the argument errors raised before any GPU work."""
    import ctypes
    L = _capi.lib()
    for world, cols in [(1, 1024), (2, 1024), (8, 768), (3, 37)]:
        ncb = (2 * cols + 31) // 32
        assert L.tempo_ln_peer_inbox_bytes(world, cols) == 2 * world * ncb * 32 * 8
        assert L.tempo_ln_peer_flag_bytes(world, cols) == 2 * world * ncb * 4
    assert L.tempo_ln_peer_inbox_bytes(0, 1024) == 0
    fake = ctypes.c_void_p(16)  # never dereferenced: every case fails validation first

    def run(rank, world, epoch, arrays=True):
        st = ops._PeerStruct(rank, world, fake.value if arrays else None,
                             fake.value if arrays else None, epoch, fake.value)
        return L.tempo_ln_param_reduce_peer(fake, 1, 8, ctypes.byref(st), fake, fake, None)

    assert L.tempo_ln_param_reduce_peer(fake, 1, 8, None, fake, fake, None) == 3  # null group
    assert run(2, 2, 1) == 3      # rank outside [0, world)
    assert run(0, 0, 1) == 3      # empty world
    assert run(0, 2, 0) == 3      # epochs start at 1
    assert run(0, 2, 1, arrays=False) == 3  # missing buffer arrays
    st = ops._PeerStruct(0, 2, fake.value, fake.value, 1, fake.value)
    assert L.tempo_ln_param_reduce_peer(fake, -1, 8, ctypes.byref(st), fake, fake, None) == 2


def test_allreduce_ln_params_argument_errors():
    """tempo_allreduce_ln_params refuses bad arguments before touching NCCL
    (or a GPU); an empty bucket is a no-op."""
    L = _capi.lib()
    assert L.tempo_allreduce_ln_params(None, None, 0, None) == 0
    assert L.tempo_allreduce_ln_params(None, None, -1, None) == 2
    assert L.tempo_allreduce_ln_params(None, None, 8, None) == 3
    assert L.tempo_nccl_comm_init(2, 2, None, None) == 3
    assert L.tempo_nccl_unique_id(None) == 3
    assert L.tempo_nccl_comm_destroy(None) == 0
