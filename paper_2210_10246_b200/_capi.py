"""ctypes binding of the C-ABI boundary ``include/tempo_b200.h``.

Loads the in-tree ``paper_2210_10246_b200/_lib/libtempo_b200.so`` (built by
``__graft_entry__.build()`` / ``make -C paper_2210_10246_b200/csrc``).  There
is no fallback: if the library is missing, importing the product path raises.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
# TEMPO_B200_LIB overrides the library path (A/B builds of the same C-ABI)
LIB_PATH = os.environ.get("TEMPO_B200_LIB", os.path.join(HERE, "_lib", "libtempo_b200.so"))

# tempo_status_t (include/tempo_b200.h), mirroring proj/include/tempo/errors.hpp
STATUS_NAMES = {
    0: "OK", 1: "Error", 2: "DimensionError", 3: "ParamError", 4: "StateError",
    5: "ConfigError", 6: "LifecycleError", 7: "DomainError", 8: "ParseError", 9: "FitError",
    10: "InvariantError", 11: "AlignmentError", 20: "CudaError", 21: "Unsupported",
}

MASK_SUPPLIED = 0
MASK_PHILOX = 1


class TempoError(RuntimeError):
    """Raised for a non-zero tempo_status_t; ``kind`` names the reference's
    exception class (errors.hpp:14-61)."""

    def __init__(self, code: int, msg: str):
        self.code = code
        self.kind = STATUS_NAMES.get(code, f"status{code}")
        super().__init__(f"{self.kind}: {msg}")


_vp, _i64, _u64, _i32, _dbl, _sz = C.c_void_p, C.c_int64, C.c_uint64, C.c_int32, C.c_double, C.c_size_t

# name -> (restype, argtypes)
SIGNATURES = {
    "tempo_last_error": (C.c_char_p, []),
    "tempo_version": (C.c_char_p, []),
    "tempo_gelu_table_create": (C.c_int, [C.c_char_p, C.POINTER(_vp)]),
    "tempo_gelu_table_destroy": (C.c_int, [_vp]),
    "tempo_gelu_table_info": (C.c_int, [_vp, C.POINTER(_dbl), C.POINTER(_dbl), C.POINTER(_dbl),
                                        C.POINTER(_dbl), C.POINTER(C.c_int), C.POINTER(C.c_int),
                                        C.POINTER(C.c_int)]),
    "tempo_gelu_table_serialize": (C.c_int, [_vp, C.c_char_p, _sz, C.POINTER(_sz)]),
    "tempo_gelu_default_table_v1": (C.c_char_p, []),
    "tempo_gelu_table_eval_host": (C.c_int, [_vp, _vp, _vp, _vp, _i64]),
    "tempo_gelu_ip_fwd": (C.c_int, [_vp, _vp, _vp, _i64, _vp, _vp]),
    "tempo_gelu_ip_fwd_exact": (C.c_int, [_vp, _vp, _vp, _i64, _vp, _vp]),
    "tempo_gelu_ip_bwd": (C.c_int, [_vp, _vp, _vp, _vp, _vp, _i64, _vp]),
    "tempo_ln_ip_fwd": (C.c_int, [_vp, _vp, _vp, _dbl, _vp, _vp, _i64, _i64, _vp, _vp]),
    "tempo_ln_check_gamma": (C.c_int, [_vp, _i64, _vp]),
    "tempo_ln_ip_bwd_workspace_size": (_sz, [_i64, _i64]),
    "tempo_ln_ip_bwd": (C.c_int, [_vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _sz, _i64, _i64,
                                  _vp]),
    "tempo_ln_peer_inbox_bytes": (_sz, [C.c_int32, _i64]),
    "tempo_ln_peer_flag_bytes": (_sz, [C.c_int32, _i64]),
    "tempo_ln_ip_bwd_peer": (C.c_int, [_vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _sz, _i64,
                                       _i64, _vp, _vp]),
    "tempo_ln_param_reduce_peer": (C.c_int, [_vp, _i64, _i64, _vp, _vp, _vp, _vp]),
    "tempo_peer_alloc": (C.c_int, [_sz, C.POINTER(_vp)]),
    "tempo_allreduce_ln_params": (C.c_int, [_vp, _vp, _i64, _vp]),
    "tempo_nccl_unique_id": (C.c_int, [_vp]),
    "tempo_nccl_comm_init": (C.c_int, [C.c_int32, C.c_int32, _vp, C.POINTER(_vp)]),
    "tempo_nccl_comm_destroy": (C.c_int, [_vp]),
    "tempo_peer_free": (C.c_int, [_vp]),
    "tempo_ipc_get_handle": (C.c_int, [_vp, _vp]),
    "tempo_ipc_open_handle": (C.c_int, [_vp, C.POINTER(_vp)]),
    "tempo_ipc_close": (C.c_int, [_vp]),
    "tempo_softmax_ip_fwd": (C.c_int, [_vp, _vp, _i64, _i64, _vp]),
    "tempo_softmax_ip_bwd": (C.c_int, [_vp, _vp, _vp, _i64, _i64, _vp]),
    "tempo_softmax_dropout_fwd": (C.c_int, [_vp, _dbl, C.c_int, _vp, _u64, _u64, _vp, _vp, _i64,
                                            _i64, _vp]),
    "tempo_attn_probs_bwd": (C.c_int, [_vp, _vp, _vp, _dbl, _vp, _vp, _i64, _i64, _vp]),
    "tempo_dropout_recompute": (C.c_int, [_vp, _vp, _dbl, _vp, _i64, _vp]),
    "tempo_ln_ip_bwd_partials": (C.c_int, [_vp, _vp, _vp, _vp, _vp, _vp, _vp, _sz, _i64, _i64,
                                           _vp, _vp]),
    "tempo_ln_param_reduce": (C.c_int, [_vp, _i64, _i64, _vp, _vp, _vp]),
    "tempo_dropout_fwd": (C.c_int, [_vp, _dbl, C.c_int, _vp, _u64, _u64, _vp, _i64, _vp]),
    "tempo_attn_dropout_dv": (C.c_int, [_vp, _vp, _dbl, _vp, _vp, _i64, _i64, _i64, _i64, _vp]),
    "tempo_attn_dropout_ctx": (C.c_int, [_vp, _vp, _dbl, _vp, _vp, _i64, _i64, _i64, _i64, _vp]),
    "tempo_dropout_add_ln_fwd": (C.c_int, [_vp, _vp, _dbl, C.c_int, _vp, _u64, _u64, _vp, _vp,
                                           _dbl, _vp, _vp, _i64, _i64, _vp, _vp]),
    "tempo_dropout_add_ln_bwd": (C.c_int, [_vp, _vp, _vp, _vp, _vp, _vp, _dbl, _vp, _vp, _vp,
                                           _vp, _vp, _sz, _i64, _i64, _vp, _vp]),
    "tempo_dropout_bwd": (C.c_int, [_vp, _vp, _dbl, _vp, _i64, _vp]),
    "tempo_tensor_add": (C.c_int, [_vp, _vp, _vp, _i64, _vp]),
    "tempo_tensor_scale": (C.c_int, [_vp, _dbl, _vp, _i64, _vp]),
    "tempo_mask_pack": (C.c_int, [_vp, _vp, _i64, _vp, _vp]),
    "tempo_mask_unpack": (C.c_int, [_vp, _vp, _i64, _vp]),
    "tempo_bernoulli_keep_bits_host": (C.c_int, [_i64, _dbl, _u64, _vp]),
    "tempo_bernoulli_keep_bits_workspace_size": (_sz, [_u64, _i64]),
    "tempo_bernoulli_keep_bits": (C.c_int, [_i64, _dbl, _u64, _u64, _vp, _vp, _sz, _vp]),
    "tempo_softmax_dropout_fwd_refmask": (C.c_int, [_vp, _dbl, _u64, _u64, _vp, _vp, _vp, _i64,
                                                    _i64, _vp, _sz, _vp]),
    "tempo_mt_outputs_after_host": (C.c_int, [_u64, _u64, _i64, _vp]),
    "tempo_mask_stream_seed": (_u64, [_u64, _u64, C.c_int]),
    "tempo_layer_stash_bytes_per_token": (_i64, [_i64, _i64, _i64, C.c_int, C.c_int]),
}

_lib = None


def lib() -> C.CDLL:
    """The loaded C-ABI library (raises if it has not been built)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(
                f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; "
                f"g.build()'` (there is no CPU fallback)")
        L = C.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


def check(rc: int) -> None:
    if rc != 0:
        msg = lib().tempo_last_error()
        raise TempoError(rc, msg.decode() if msg else "")
