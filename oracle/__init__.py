"""oracle -- TEST INFRASTRUCTURE, NOT PRODUCT CODE.

Python bindings (ctypes + numpy) for the two CPU checkers of the Tempo
in-place operator path:

* ``Port``: the plain-C restatement ``oracle/tempo_oracle.c`` (each function
  cites the reference file:line it follows), built to
  ``oracle/_build/libtempo_oracle.so``.
* ``Ref``: the UNMODIFIED reference library (``/root/reference/proj/src``)
  plus ``oracle/ref_harness.cpp``'s shims, built to
  ``oracle/_ref/libtempo_ref.so`` by ``oracle/Makefile``.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline /
``--impl reference`` arm import this package, and only as the checker or the
timed reference arm.  The product package ``paper_2210_10246_b200`` never
imports it.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
PORT_SO = os.path.join(HERE, "_build", "libtempo_oracle.so")
REF_SO = os.path.join(HERE, "_ref", "libtempo_ref.so")

_f32p = np.ctypeslib.ndpointer(np.float32, flags="C_CONTIGUOUS")
_f64p = np.ctypeslib.ndpointer(np.float64, flags="C_CONTIGUOUS")
_u8p = np.ctypeslib.ndpointer(np.uint8, flags="C_CONTIGUOUS")
_u64p = np.ctypeslib.ndpointer(np.uint64, flags="C_CONTIGUOUS")
_u32p = np.ctypeslib.ndpointer(np.uint32, flags="C_CONTIGUOUS")
_i64 = C.c_int64


def build(quiet: bool = True) -> None:
    """Run oracle/Makefile (the C port always; the reference when present)."""
    out = subprocess.run(["make", "-C", HERE, "-j8"], capture_output=True, text=True)
    if out.returncode != 0:
        raise RuntimeError("oracle build failed:\n" + out.stdout + out.stderr)
    if not quiet:
        print(out.stdout)


def _f32(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float32)


def _u8(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.uint8)


class OracleError(RuntimeError):
    def __init__(self, code: int, msg: str = ""):
        super().__init__(f"code {code}: {msg}")
        self.code = code


# --------------------------------------------------------------------------
# The C restatement
# --------------------------------------------------------------------------
class Port:
    """ctypes view of oracle/tempo_oracle.c."""

    def __init__(self, path: str = PORT_SO):
        if not os.path.exists(path):
            build()
        L = C.CDLL(path)
        self.L = L
        L.orc_bernoulli_keep.argtypes = [_i64, C.c_double, C.c_uint64, _u8p]
        L.orc_mt64_stream.argtypes = [C.c_uint64, _i64, _u64p]
        L.orc_bernoulli_keep_bits_at.argtypes = [_i64, _i64, C.c_double, C.c_uint64, _u32p]
        L.orc_mt64_stream.restype = None
        L.orc_mask_stream_seed.argtypes = [C.c_uint64, C.c_uint64, C.c_int]
        L.orc_mask_stream_seed.restype = C.c_uint64
        L.orc_gelu_scalar.argtypes = [C.c_double]
        L.orc_gelu_scalar.restype = C.c_double
        L.orc_gelu_fwd.argtypes = [_f32p, _f32p, _u8p, _i64, C.c_double]
        L.orc_gelu_fwd.restype = None
        L.orc_table_parse.argtypes = [C.c_char_p]
        L.orc_table_parse.restype = C.c_void_p
        L.orc_table_free.argtypes = [C.c_void_p]
        L.orc_table_free.restype = None
        L.orc_table_x_star.argtypes = [C.c_void_p]
        L.orc_table_x_star.restype = C.c_double
        L.orc_table_y_min.argtypes = [C.c_void_p]
        L.orc_table_y_min.restype = C.c_double
        L.orc_table_eval_n.argtypes = [C.c_void_p, _f64p, _u8p, _f64p, _i64]
        L.orc_table_eval_n.restype = None
        L.orc_gelu_bwd.argtypes = [C.c_void_p, _f32p, _f32p, _u8p, _f32p, _i64]
        L.orc_gelu_bwd.restype = None
        L.orc_ln_fwd.argtypes = [_f32p, _f32p, _f32p, C.c_double, _f32p, _f32p, _f32p, _i64, _i64]
        L.orc_ln_bwd.argtypes = [_f32p, _f32p, _f32p, _f32p, _f32p, _f32p, _f64p, _f64p,
                                 _i64, _i64, C.c_int]
        L.orc_ln_bwd.restype = None
        L.orc_softmax_fwd.argtypes = [_f32p, _f32p, _i64, _i64]
        L.orc_softmax_fwd.restype = None
        L.orc_softmax_bwd.argtypes = [_f32p, _f32p, _f32p, _i64, _i64]
        L.orc_softmax_bwd.restype = None
        L.orc_dropout_apply.argtypes = [_f32p, _u8p, C.c_double, _f32p, _i64]
        L.orc_memory_model.argtypes = [_i64, _i64, _i64, C.POINTER(_i64), C.POINTER(_i64)]
        L.orc_memory_model.restype = None

    # -- masks ------------------------------------------------------------
    def bernoulli_keep(self, n: int, p: float, seed: int) -> np.ndarray:
        out = np.empty(n, np.uint8)
        rc = self.L.orc_bernoulli_keep(n, p, seed, out)
        if rc:
            raise OracleError(rc, "drop probability must lie in [0, 1)")
        return out

    def bernoulli_keep_bits_at(self, offset: int, n: int, p: float, seed: int) -> np.ndarray:
        """Packed keep bits of elements [offset, offset+n) of the sequential
        stream (the engine stepped past `offset` draws one by one)."""
        out = np.empty((n + 31) // 32, np.uint32)
        rc = self.L.orc_bernoulli_keep_bits_at(offset, n, p, seed, out)
        if rc:
            raise OracleError(rc, "drop probability must lie in [0, 1)")
        return out

    def mt64_stream(self, seed: int, n: int) -> np.ndarray:
        out = np.empty(n, np.uint64)
        self.L.orc_mt64_stream(seed, n, out)
        return out

    def mask_stream_seed(self, seed: int, salt: int, site: int) -> int:
        return int(self.L.orc_mask_stream_seed(seed, salt, site))

    # -- GELU -------------------------------------------------------------
    def gelu_scalar(self, x: float) -> float:
        return float(self.L.orc_gelu_scalar(x))

    def gelu_fwd(self, x, x_star: float):
        x = _f32(x).reshape(-1)
        y = np.empty_like(x)
        m = np.empty(x.size, np.uint8)
        self.L.orc_gelu_fwd(x, y, m, x.size, x_star)
        return y, m

    def table(self, text: str) -> "PortTable":
        return PortTable(self, text)

    # -- LayerNorm --------------------------------------------------------
    def ln_fwd(self, x, gamma, beta, eps: float):
        x = _f32(x)
        rows, cols = x.shape
        y = np.empty_like(x)
        rstd = np.empty(rows, np.float32)
        mean = np.empty(rows, np.float32)
        rc = self.L.orc_ln_fwd(x, _f32(gamma), _f32(beta), eps, y, rstd, mean, rows, cols)
        if rc:
            raise OracleError(rc, "layernorm epsilon must be positive")
        return y, rstd, mean

    def ln_bwd(self, dy, y, rstd, gamma, beta, f64: bool):
        dy = _f32(dy)
        rows, cols = dy.shape
        dx = np.empty_like(dy)
        dg = np.empty(cols, np.float64)
        db = np.empty(cols, np.float64)
        self.L.orc_ln_bwd(dy, _f32(y), _f32(rstd), _f32(gamma), _f32(beta), dx, dg, db,
                          rows, cols, int(f64))
        return dx, dg, db

    # -- softmax / dropout -------------------------------------------------
    def softmax_fwd(self, z):
        z = _f32(z)
        P = np.empty_like(z)
        self.L.orc_softmax_fwd(z, P, z.shape[0], z.shape[1])
        return P

    def softmax_bwd(self, g, y):
        g = _f32(g)
        dz = np.empty_like(g)
        self.L.orc_softmax_bwd(g, _f32(y), dz, g.shape[0], g.shape[1])
        return dz

    def dropout_apply(self, x, keep, p: float):
        x = _f32(x)
        out = np.empty_like(x)
        rc = self.L.orc_dropout_apply(x.reshape(-1), _u8(keep).reshape(-1), p,
                                      out.reshape(-1), x.size)
        if rc:
            raise OracleError(rc, "dropout p must lie in [0, 1)")
        return out

    def memory_model(self, seq: int, hidden: int, heads: int):
        a, b = _i64(), _i64()
        self.L.orc_memory_model(seq, hidden, heads, C.byref(a), C.byref(b))
        return a.value, b.value


class PortTable:
    def __init__(self, port: Port, text: str):
        self.port = port
        self.h = port.L.orc_table_parse(text.encode())
        if not self.h:
            raise OracleError(8, "unparseable table")

    def __del__(self):
        if getattr(self, "h", None):
            self.port.L.orc_table_free(self.h)
            self.h = None

    @property
    def x_star(self) -> float:
        return float(self.port.L.orc_table_x_star(self.h))

    @property
    def y_min(self) -> float:
        return float(self.port.L.orc_table_y_min(self.h))

    def eval(self, y, m) -> np.ndarray:
        y = np.ascontiguousarray(y, np.float64).reshape(-1)
        out = np.empty_like(y)
        self.port.L.orc_table_eval_n(self.h, y, _u8(m).reshape(-1), out, y.size)
        return out

    def gelu_bwd(self, dy, y, m) -> np.ndarray:
        dy = _f32(dy).reshape(-1)
        dx = np.empty_like(dy)
        self.port.L.orc_gelu_bwd(self.h, dy, _f32(y).reshape(-1), _u8(m).reshape(-1), dx, dy.size)
        return dx


# --------------------------------------------------------------------------
# The reference itself (oracle/_ref/libtempo_ref.so)
# --------------------------------------------------------------------------
class Ref:
    """ctypes view of oracle/ref_harness.cpp over the reference's sources."""

    def __init__(self, path: str = REF_SO):
        if not os.path.exists(path):
            raise FileNotFoundError(path + " (run `make -C oracle` where /root/reference exists)")
        L = C.CDLL(path)
        self.L = L
        L.ref_last_error.restype = C.c_char_p
        L.ref_fit_table_default.argtypes = [C.c_char_p, _i64, C.POINTER(_i64)]
        L.ref_fit_table.argtypes = [C.c_double, C.c_int, C.c_char_p, _i64, C.POINTER(_i64)]
        L.ref_table_eval.argtypes = [C.c_char_p, _f64p, _u8p, _f64p, _i64]
        L.ref_table_parse.argtypes = [C.c_char_p]
        L.ref_gelu_ip.argtypes = [C.c_char_p, _f32p, C.c_void_p, _i64, C.c_int, _f32p, _u8p,
                                  C.c_void_p]
        L.ref_gelu_forward.argtypes = [_f32p, _i64, _f32p]
        L.ref_layernorm_ip.argtypes = [_f32p, _f32p, _f32p, C.c_void_p, _i64, _i64, C.c_double,
                                       C.c_int, _f32p, C.c_void_p, C.c_void_p, C.c_void_p,
                                       C.c_void_p]
        L.ref_layernorm_ip_bwd.argtypes = [_f32p, _f32p, _f32p, _f32p, _f32p, _i64, _i64, C.c_int,
                                           _f32p, _f64p, _f64p]
        L.ref_softmax_dropout.argtypes = [_f32p, _u8p, C.c_double, C.c_void_p, _i64, _i64, _f32p,
                                          _f32p, C.c_void_p, C.c_void_p]
        L.ref_softmax_bwd.argtypes = [_f32p, _f32p, _i64, _i64, _f32p]
        L.ref_dropout.argtypes = [_f32p, _u8p, C.c_double, C.c_void_p, _i64, _f32p, C.c_void_p]
        L.ref_bernoulli_keep.argtypes = [_i64, C.c_double, C.c_uint64, _u8p]
        L.ref_mask_stream_seed.argtypes = [C.c_uint64, C.c_uint64, C.c_int]
        L.ref_mask_stream_seed.restype = C.c_uint64
        L.ref_memory_model.argtypes = [_i64, _i64, _i64, _i64, C.POINTER(_i64), C.POINTER(_i64),
                                       C.POINTER(_i64)]
        L.ref_ledger_bytes.argtypes = [C.c_int, _i64, _i64, C.c_char_p, C.POINTER(_i64)]
        L.ref_chain_create.argtypes = [C.c_char_p, C.c_double, _i64, _i64, _i64, _i64, C.c_uint64,
                                       C.c_int]
        L.ref_chain_create.restype = C.c_void_p
        L.ref_chain_run.argtypes = [C.c_void_p]
        L.ref_chain_destroy.argtypes = [C.c_void_p]
        L.ref_op_create.argtypes = [C.c_int, C.c_char_p, C.c_double, _i64, _i64, C.c_uint64]
        L.ref_op_create.restype = C.c_void_p
        L.ref_op_run.argtypes = [C.c_void_p]
        L.ref_op_destroy.argtypes = [C.c_void_p]

    def _check(self, rc: int) -> None:
        if rc:
            raise OracleError(rc, self.L.ref_last_error().decode())

    @staticmethod
    def _ptr(a):
        return None if a is None else a.ctypes.data_as(C.c_void_p)

    def chain_create(self, table_text: str, p: float, att_rows: int, seq: int, tokens: int,
                     hidden: int, seed: int, with_residual: bool = False):
        """bench.py's reference arm: one shard of the layer op chain with its
        inputs built once by the reference's own generators (ref_harness.cpp
        ref_chain_create).  Returns an opaque handle for chain_run."""
        h = self.L.ref_chain_create(table_text.encode(), p, att_rows, seq, tokens, hidden, seed,
                                    int(with_residual))
        if not h:
            raise OracleError(1, self.L.ref_last_error().decode())
        return h

    def op_create(self, kind: int, table_text: str, p: float, rows: int, cols: int, seed: int):
        """One op pair of BASELINE configs[0..2] (kind 0 GELU, 1 LayerNorm, 2
        softmax -> dropout_recompute) on [rows, cols], inputs built once by the
        reference's generators (ref_harness.cpp ref_op_create)."""
        h = self.L.ref_op_create(kind, table_text.encode(), p, rows, cols, seed)
        if not h:
            raise OracleError(1, self.L.ref_last_error().decode())
        return h

    def op_run(self, h) -> None:
        """Forward + Tape::backward of the op pair (the timed step)."""
        self._check(self.L.ref_op_run(h))

    def op_destroy(self, h) -> None:
        self.L.ref_op_destroy(h)

    def chain_run(self, h) -> None:
        """One forward + Tape::backward of the chain shard (the timed step)."""
        self._check(self.L.ref_chain_run(h))

    def chain_destroy(self, h) -> None:
        self.L.ref_chain_destroy(h)

    def fit_table_default(self) -> str:
        n = _i64()
        self._check(self.L.ref_fit_table_default(None, 0, C.byref(n)))
        buf = C.create_string_buffer(n.value + 1)
        self._check(self.L.ref_fit_table_default(buf, n.value + 1, C.byref(n)))
        return buf.value.decode()

    def fit_table(self, tol: float, max_degree: int) -> str:
        n = _i64()
        self._check(self.L.ref_fit_table(tol, max_degree, None, 0, C.byref(n)))
        buf = C.create_string_buffer(n.value + 1)
        self._check(self.L.ref_fit_table(tol, max_degree, buf, n.value + 1, C.byref(n)))
        return buf.value.decode()

    def table_parse(self, text: str) -> None:
        self._check(self.L.ref_table_parse(text.encode()))

    def table_eval(self, text: str, y, m) -> np.ndarray:
        y = np.ascontiguousarray(y, np.float64).reshape(-1)
        out = np.empty_like(y)
        self._check(self.L.ref_table_eval(text.encode(), y, _u8(m).reshape(-1), out, y.size))
        return out

    def gelu_ip(self, text: str, x, dy=None, f64: bool = False):
        x = _f32(x).reshape(-1)
        y = np.empty_like(x)
        m = np.empty(x.size, np.uint8)
        dyc = None if dy is None else _f32(dy).reshape(-1)
        dx = None if dy is None else np.empty_like(x)
        self._check(self.L.ref_gelu_ip(text.encode(), x, self._ptr(dyc), x.size, int(f64), y, m,
                                       self._ptr(dx)))
        return y, m, dx

    def gelu_forward(self, x):
        x = _f32(x).reshape(-1)
        y = np.empty_like(x)
        self._check(self.L.ref_gelu_forward(x, x.size, y))
        return y

    def layernorm_ip(self, x, gamma, beta, dy=None, eps: float = 1e-5, f64: bool = False):
        x = _f32(x)
        rows, cols = x.shape
        y = np.empty_like(x)
        rstd = np.empty(rows, np.float32)
        dyc = None if dy is None else _f32(dy)
        dx = None if dy is None else np.empty_like(x)
        dg = None if dy is None else np.empty(cols, np.float64)
        db = None if dy is None else np.empty(cols, np.float64)
        self._check(self.L.ref_layernorm_ip(x, _f32(gamma), _f32(beta), self._ptr(dyc), rows, cols,
                                            eps, int(f64), y, self._ptr(rstd), self._ptr(dx),
                                            self._ptr(dg), self._ptr(db)))
        return y, rstd, dx, dg, db

    def layernorm_ip_bwd(self, dy, y, rstd, gamma, beta, f64: bool = False):
        dy = _f32(dy)
        rows, cols = dy.shape
        dx = np.empty_like(dy)
        dg = np.empty(cols, np.float64)
        db = np.empty(cols, np.float64)
        self._check(self.L.ref_layernorm_ip_bwd(dy, _f32(y), _f32(rstd), _f32(gamma), _f32(beta),
                                                rows, cols, int(f64), dx, dg, db))
        return dx, dg, db

    def softmax_dropout(self, z, keep, p: float, dD=None, recompute: bool = True):
        z = _f32(z)
        rows, cols = z.shape
        P = np.empty_like(z)
        D = np.empty_like(z)
        dDc = None if dD is None else _f32(dD)
        dZ = None if dD is None else np.empty_like(z)
        Dr = np.empty_like(z) if recompute else None
        self._check(self.L.ref_softmax_dropout(z, _u8(keep).reshape(rows, cols), p,
                                               self._ptr(dDc), rows, cols, P, D, self._ptr(dZ),
                                               self._ptr(Dr)))
        return P, D, dZ, Dr

    def softmax_bwd(self, g, y):
        g = _f32(g)
        dz = np.empty_like(g)
        self._check(self.L.ref_softmax_bwd(g, _f32(y), g.shape[0], g.shape[1], dz))
        return dz

    def dropout(self, x, keep, p: float, dy=None):
        x = _f32(x).reshape(-1)
        y = np.empty_like(x)
        dyc = None if dy is None else _f32(dy).reshape(-1)
        dx = None if dy is None else np.empty_like(x)
        self._check(self.L.ref_dropout(x, _u8(keep).reshape(-1), p, self._ptr(dyc), x.size, y,
                                       self._ptr(dx)))
        return y, dx

    def bernoulli_keep(self, n: int, p: float, seed: int) -> np.ndarray:
        out = np.empty(n, np.uint8)
        self._check(self.L.ref_bernoulli_keep(n, p, seed, out))
        return out

    def mask_stream_seed(self, seed: int, salt: int, site: int) -> int:
        return int(self.L.ref_mask_stream_seed(seed, salt, site))

    def memory_model(self, batch: int, seq: int, hidden: int, heads: int):
        a, b = _i64(), _i64()
        s = (_i64 * 4)()
        self._check(self.L.ref_memory_model(batch, seq, hidden, heads, C.byref(a), C.byref(b), s))
        return a.value, b.value, [s[i] for i in range(4)]

    def ledger_bytes(self, op: int, rows: int, cols: int, table_text: str = "") -> int:
        out = _i64()
        self._check(self.L.ref_ledger_bytes(op, rows, cols, table_text.encode(), C.byref(out)))
        return out.value


def have_ref() -> bool:
    return os.path.exists(REF_SO)
