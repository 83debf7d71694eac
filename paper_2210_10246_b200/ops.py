"""Host-side mirror of the reference's operator API for the Tempo in-place path.

Each function here is the device counterpart of one reference entry point
(``proj/include/tempo/ops_tempo.hpp:33-63``, ``ops_reference.hpp:18-47``,
``gelu_table.hpp:48-91``), taking CUDA ``torch.Tensor`` buffers (fp32,
contiguous) and calling the C-ABI of ``include/tempo_b200.h`` on the current
CUDA stream.  PyTorch only provides device memory and streams; every
operator runs in this package's sm_100a kernels.  Errors surface as
:class:`TempoError` whose ``kind`` is the reference's exception class name.

Bit-packed masks are ``torch.int32`` tensors of ``ceil(n/32)`` words (bit i
of word w = element 32w+i, the reference's BoolMask order).
"""
from __future__ import annotations

import ctypes as C
import os
from typing import Optional, Tuple

import torch

from ._capi import MASK_PHILOX, MASK_SUPPLIED, TempoError, check, lib

__all__ = [
    "GeluTable", "TempoError", "gelu_ip_fwd", "gelu_ip_bwd", "layernorm_ip_fwd", "attn_dropout_ctx",
    "layernorm_ip_bwd", "ln_check_gamma", "softmax_ip_fwd", "softmax_ip_bwd",
    "softmax_dropout_fwd", "attn_probs_bwd", "dropout_fwd", "dropout_bwd", "mask_words",
    "pack_mask", "unpack_mask", "bernoulli_keep_bits", "bernoulli_keep_bits_device",
    "mt_outputs_after", "mask_stream_seed",
    "layer_stash_bytes_per_token", "MASK_SUPPLIED", "MASK_PHILOX",
]


def _ptr(t: Optional[torch.Tensor]):
    return None if t is None else C.c_void_p(t.data_ptr())


def _stream():
    return C.c_void_p(torch.cuda.current_stream().cuda_stream)


def _dev(t: torch.Tensor, name: str, dtype, device=None, numel=None, min_numel=None):
    """Validate a buffer handed to the C-ABI as a raw pointer: dtype, CUDA,
    same device as the op's primary input, contiguous (the kernels index it
    densely; no silent eager-torch copy is made), and its size."""
    if not isinstance(t, torch.Tensor):
        raise TempoError(2, f"{name}: expected a torch.Tensor")
    if t.dtype != dtype:
        raise TempoError(2, f"{name}: expected {dtype}, got {t.dtype}")
    if not t.is_cuda:
        raise TempoError(2, f"{name}: expected a CUDA tensor")
    if device is not None and t.device != device:
        raise TempoError(2, f"{name}: on {t.device}, expected {device}")
    if not t.is_contiguous():
        raise TempoError(2, f"{name}: expected a contiguous tensor")
    if numel is not None and t.numel() != numel:
        raise TempoError(2, f"{name}: has {t.numel()} elements, expected {numel}")
    if min_numel is not None and t.numel() < min_numel:
        raise TempoError(2, f"{name}: has {t.numel()} elements, needs >= {min_numel}")
    return t


def _f32(t: torch.Tensor, name: str, device=None, numel=None) -> torch.Tensor:
    return _dev(t, name, torch.float32, device, numel)


def _out(t: Optional[torch.Tensor], name: str, like: torch.Tensor) -> torch.Tensor:
    """A float32 output the size of `like`: allocated when None, else checked."""
    if t is None:
        return torch.empty_like(like)
    return _dev(t, name, torch.float32, like.device, like.numel())


def _vec_out(t: Optional[torch.Tensor], name: str, n: int, device) -> torch.Tensor:
    if t is None:
        return torch.empty(n, dtype=torch.float32, device=device)
    return _dev(t, name, torch.float32, device, n)


def _mask(t: Optional[torch.Tensor], name: str, n: int, device) -> torch.Tensor:
    """Bit-packed mask of n elements: int32 words, >= ceil(n/32) of them."""
    if t is None:
        return torch.empty(mask_words(n), dtype=torch.int32, device=device)
    return _dev(t, name, torch.int32, device, min_numel=mask_words(n))


def mask_words(n: int) -> int:
    return (int(n) + 31) // 32


def _rows_cols(t: torch.Tensor) -> Tuple[int, int]:
    if t.dim() == 0:
        raise TempoError(2, "expected rank >= 1")
    cols = t.shape[-1]
    return (t.numel() // cols if cols else 0), cols


# --------------------------------------------------------------------------
# GeluPolyTable (gelu_table.hpp:48-91)
# --------------------------------------------------------------------------
class GeluTable:
    """Parsed, validated v1 GELU derivative table (immutable, shareable)."""

    def __init__(self, v1_text: str):
        h = C.c_void_p()
        check(lib().tempo_gelu_table_create(v1_text.encode(), C.byref(h)))
        self._h = h

    @classmethod
    def default(cls) -> "GeluTable":
        """fit::fit_table() with default FitOptions (gelu_fit.cpp:331-382)."""
        return cls(lib().tempo_gelu_default_table_v1().decode())

    @property
    def handle(self) -> C.c_void_p:
        return self._h

    def info(self) -> dict:
        xs, ym, tol, me = C.c_double(), C.c_double(), C.c_double(), C.c_double()
        ver, nseg, deg = C.c_int(), C.c_int(), C.c_int()
        check(lib().tempo_gelu_table_info(self._h, C.byref(xs), C.byref(ym), C.byref(tol),
                                          C.byref(me), C.byref(ver), C.byref(nseg), C.byref(deg)))
        return {"x_star": xs.value, "y_min": ym.value, "tolerance": tol.value,
                "verified_max_error": me.value, "verified": bool(ver.value),
                "n_segments": nseg.value, "max_degree": deg.value}

    def serialize(self) -> str:
        n = C.c_size_t()
        check(lib().tempo_gelu_table_serialize(self._h, None, 0, C.byref(n)))
        buf = C.create_string_buffer(n.value + 1)
        check(lib().tempo_gelu_table_serialize(self._h, buf, n.value + 1, C.byref(n)))
        return buf.value.decode()

    def eval_host(self, y, m):
        """GeluPolyTable::eval on the host (double), for numpy arrays."""
        import numpy as np
        y = np.ascontiguousarray(y, np.float64).reshape(-1)
        m = np.ascontiguousarray(m, np.uint8).reshape(-1)
        out = np.empty_like(y)
        check(lib().tempo_gelu_table_eval_host(self._h, y.ctypes.data, m.ctypes.data,
                                               out.ctypes.data, y.size))
        return out

    def close(self) -> None:
        if getattr(self, "_h", None) is not None and self._h.value:
            lib().tempo_gelu_table_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


# --------------------------------------------------------------------------
# In-Place GELU (tempo_ops::gelu, ops_tempo.cpp:89-96)
# --------------------------------------------------------------------------
def gelu_ip_fwd(x: torch.Tensor, table: GeluTable, y: torch.Tensor = None,
                mask: torch.Tensor = None, exact: bool = False):
    """Returns (y, mask_bits).  Stash = y + mask (the input is not kept).
    exact=True: the reference formula in fp64 for every element
    (tempo_gelu_ip_fwd_exact, <= 2 ulp) instead of the fp32 fast path."""
    if table is None:
        raise TempoError(5, "in-place gelu needs a fitted table")
    x = _f32(x, "x")
    y = _out(y, "y", x)
    mask = _mask(mask, "mask", x.numel(), x.device)
    fn = lib().tempo_gelu_ip_fwd_exact if exact else lib().tempo_gelu_ip_fwd
    check(fn(_ptr(x), _ptr(y), _ptr(mask), x.numel(), table.handle, _stream()))
    return y, mask


def gelu_ip_bwd(dy: torch.Tensor, y: torch.Tensor, mask: torch.Tensor, table: GeluTable,
                dx: torch.Tensor = None) -> torch.Tensor:
    if table is None:
        raise TempoError(5, "in-place gelu needs a fitted table")
    dy, y = _f32(dy, "dy"), _f32(y, "y")
    if dy.shape != y.shape:
        raise TempoError(2, f"gelu backward shapes {tuple(dy.shape)} and {tuple(y.shape)} differ")
    y = _f32(y, "y", dy.device)
    if mask is None:
        raise TempoError(2, "mask: the forward's bit mask is required")
    mask = _mask(mask, "mask", y.numel(), y.device)
    dx = _out(dx, "dx", dy)
    check(lib().tempo_gelu_ip_bwd(_ptr(dy), _ptr(y), _ptr(mask), table.handle, _ptr(dx),
                                  y.numel(), _stream()))
    return dx


# --------------------------------------------------------------------------
# In-Place LayerNorm (tempo_ops::layernorm, ops_tempo.cpp:98-156)
# --------------------------------------------------------------------------
def ln_check_gamma(gamma: torch.Tensor) -> None:
    """ops_tempo.cpp:100-106 (synchronous)."""
    gamma = _f32(gamma, "gamma")
    check(lib().tempo_ln_check_gamma(_ptr(gamma), gamma.numel(), _stream()))


def layernorm_ip_fwd(x: torch.Tensor, gamma: torch.Tensor, beta: torch.Tensor,
                     eps: float = 1e-5, check_gamma: bool = True, y: torch.Tensor = None,
                     rstd: torch.Tensor = None, dev_status: torch.Tensor = None):
    """Returns (y, rstd).  Stash = y + rstd[row]."""
    x = _f32(x, "x")
    gamma, beta = _f32(gamma, "gamma", x.device), _f32(beta, "beta", x.device)
    rows, cols = _rows_cols(x)
    if gamma.numel() != cols or beta.numel() != cols:
        raise TempoError(2, f"layernorm affine params {tuple(gamma.shape)}, {tuple(beta.shape)} "
                            f"do not match {tuple(x.shape)}")
    if check_gamma:
        ln_check_gamma(gamma)
    y = _out(y, "y", x)
    rstd = torch.empty(x.shape[:-1], dtype=torch.float32, device=x.device) if rstd is None \
        else _f32(rstd, "rstd", x.device, rows)
    if dev_status is not None:
        _dev(dev_status, "dev_status", torch.int32, x.device, 1)
    check(lib().tempo_ln_ip_fwd(_ptr(x), _ptr(gamma), _ptr(beta), float(eps), _ptr(y), _ptr(rstd),
                                rows, cols, _ptr(dev_status), _stream()))
    return y, rstd


_ws_cache = {}


def ln_workspace(rows: int, cols: int, device, stream=None) -> torch.Tensor:
    """The LayerNorm backward's scratch (per-CTA fp64 partial rows).  Cached
    per (device, STREAM, size): two backwards of the same shape running
    concurrently on different streams must not share partial rows, while
    work on one stream is ordered, so one buffer per stream is enough."""
    nbytes = int(lib().tempo_ln_ip_bwd_workspace_size(rows, cols))
    if stream is None:
        with torch.cuda.device(device):
            stream = torch.cuda.current_stream()
    key = (str(device), int(stream.cuda_stream), nbytes)
    ws = _ws_cache.get(key)
    if ws is None:
        ws = torch.empty(max(nbytes, 16), dtype=torch.uint8, device=device)
        _ws_cache[key] = ws
    return ws


def _ln_bwd_args(dy, y, rstd, gamma, beta, dx, dgamma, dbeta, workspace):
    dy = _f32(dy, "dy")
    y = _f32(y, "y", dy.device, dy.numel())
    rows, cols = _rows_cols(y)
    rstd = _f32(rstd, "rstd", y.device, rows)
    gamma = _f32(gamma, "gamma", y.device, cols)
    beta = _f32(beta, "beta", y.device, cols)
    dx = _out(dx, "dx", dy)
    dgamma = _vec_out(dgamma, "dgamma", cols, y.device)
    dbeta = _vec_out(dbeta, "dbeta", cols, y.device)
    if workspace is None:
        ws = ln_workspace(rows, cols, y.device)
    else:
        ws = _dev(workspace, "workspace", workspace.dtype, y.device)
    nbytes = ws.numel() * ws.element_size()
    return dy, y, rstd, gamma, beta, dx, dgamma, dbeta, ws, nbytes, rows, cols


def layernorm_ip_bwd(dy: torch.Tensor, y: torch.Tensor, rstd: torch.Tensor,
                     gamma: torch.Tensor, beta: torch.Tensor, dx: torch.Tensor = None,
                     dgamma: torch.Tensor = None, dbeta: torch.Tensor = None,
                     workspace: torch.Tensor = None):
    """Returns (dx, dgamma, dbeta); dgamma/dbeta summed over all rows."""
    dy, y, rstd, gamma, beta, dx, dgamma, dbeta, ws, nbytes, rows, cols = _ln_bwd_args(
        dy, y, rstd, gamma, beta, dx, dgamma, dbeta, workspace)
    check(lib().tempo_ln_ip_bwd(_ptr(dy), _ptr(y), _ptr(rstd), _ptr(gamma), _ptr(beta), _ptr(dx),
                                _ptr(dgamma), _ptr(dbeta), _ptr(ws), nbytes, rows, cols,
                                _stream()))
    return dx, dgamma, dbeta


class _PeerStruct(C.Structure):
    """tempo_ln_peer_t (include/tempo_b200.h)."""
    _fields_ = [("rank", C.c_int32), ("world", C.c_int32),
                ("inbox", C.c_void_p), ("flags", C.c_void_p),
                ("epoch", C.c_uint32), ("status", C.c_void_p), ("timeout_ms", C.c_uint32)]


class LnPeerRank:
    """One rank's view of the fused dgamma/dbeta exchange: its own inbox and
    flag buffers plus the device arrays of every rank's buffers as mapped in
    this process.  Build with ``LnPeerRank.local_group`` (all ranks in one
    process on one device: tests) or ``LnPeerRank.ipc`` (one process per GPU:
    buffers shared by CUDA IPC handles over torch.distributed)."""

    def __init__(self, rank, world, cols, device):
        self.rank, self.world, self.cols, self.device = rank, world, cols, device
        L = lib()
        self.inbox_bytes = int(L.tempo_ln_peer_inbox_bytes(world, cols))
        self.flag_bytes = int(L.tempo_ln_peer_flag_bytes(world, cols))
        # dedicated zero-filled allocations (IPC maps whole allocations), on
        # `device`; raw device pointers
        self._owned = []
        with torch.cuda.device(device):
            self.inbox = self._alloc(self.inbox_bytes)
            self.flags = self._alloc(self.flag_bytes)
        self.status = torch.zeros(1, dtype=torch.int32, device=device)
        self.epoch = 0
        # bound on the wait for peers (0 = library default, 30 s)
        self.timeout_ms = int(os.environ.get("TEMPO_PEER_TIMEOUT_MS", "0"))
        self._ptrs = None
        self._mapped = []

    def _alloc(self, nbytes):
        p = C.c_void_p()
        check(lib().tempo_peer_alloc(nbytes, C.byref(p)))
        self._owned.append(p.value)
        return p.value

    def __del__(self):
        try:
            self.close()
            for p in self._owned:
                lib().tempo_peer_free(C.c_void_p(p))
            self._owned = []
        except Exception:  # noqa: BLE001  (interpreter shutdown)
            pass

    def _set_peers(self, inbox_ptrs, flag_ptrs):
        self._ptrs = (torch.tensor(inbox_ptrs, dtype=torch.int64, device=self.device),
                      torch.tensor(flag_ptrs, dtype=torch.int64, device=self.device))

    @classmethod
    def local_group(cls, world, cols, device):
        ranks = [cls(r, world, cols, device) for r in range(world)]
        ib = [r.inbox for r in ranks]
        fl = [r.flags for r in ranks]
        for r in ranks:
            r._set_peers(ib, fl)
        return ranks

    @classmethod
    def ipc(cls, cols, device, group=None):
        """Collective over torch.distributed: every rank maps every other
        rank's buffers through CUDA IPC handles."""
        import torch.distributed as dist
        me = cls(dist.get_rank(group), dist.get_world_size(group), cols, device)
        L = lib()
        hs = []
        for ptr in (me.inbox, me.flags):
            h = C.create_string_buffer(64)
            check(L.tempo_ipc_get_handle(C.c_void_p(ptr), h))
            hs.append(h.raw)
        allh = [None] * me.world
        dist.all_gather_object(allh, hs, group=group)
        ib, fl = [], []
        for r, (hi, hf) in enumerate(allh):
            if r == me.rank:
                ib.append(me.inbox)
                fl.append(me.flags)
                continue
            ptrs = []
            for h in (hi, hf):
                p = C.c_void_p()
                check(L.tempo_ipc_open_handle(C.create_string_buffer(h, 64), C.byref(p)))
                me._mapped.append(p.value)
                ptrs.append(p.value)
            ib.append(ptrs[0])
            fl.append(ptrs[1])
        me._set_peers(ib, fl)
        return me

    def next_struct(self):
        self.epoch += 1
        return _PeerStruct(self.rank, self.world, self._ptrs[0].data_ptr(),
                           self._ptrs[1].data_ptr(), self.epoch, self.status.data_ptr(),
                           self.timeout_ms)

    def check_status(self):
        """Raise if any exchange so far timed out (the status is sticky)."""
        if int(self.status.item()) != 0:
            raise TempoError(4, "peer exchange: a rank never arrived; dgamma/dbeta were "
                                "poisoned with NaN and the group must be rebuilt")

    def close(self):
        L = lib()
        for p in self._mapped:
            L.tempo_ipc_close(C.c_void_p(p))
        self._mapped = []


class NcclComm:
    """An NCCL communicator built through the C-ABI (tempo_nccl_comm_init),
    for tempo_allreduce_ln_params: the dgamma/dbeta sum for callers without
    P2P / IPC peers.  `uid` is the 128-byte ncclUniqueId from rank 0
    (NcclComm.unique_id()), distributed by the caller."""

    def __init__(self, world: int, rank: int, uid: bytes):
        if len(uid) != 128:
            raise TempoError(3, "nccl unique id must be 128 bytes")
        buf = C.create_string_buffer(uid, 128)
        h = C.c_void_p()
        check(lib().tempo_nccl_comm_init(int(world), int(rank), buf, C.byref(h)))
        self._h, self.world, self.rank = h, world, rank

    @staticmethod
    def unique_id() -> bytes:
        buf = C.create_string_buffer(128)
        check(lib().tempo_nccl_unique_id(buf))
        return buf.raw

    def allreduce_ln_params(self, bucket: torch.Tensor) -> None:
        """Sum the bucketed LayerNorm dgamma/dbeta over the ranks, in place."""
        _f32(bucket, "bucket")
        check(lib().tempo_allreduce_ln_params(self._h, _ptr(bucket), bucket.numel(), _stream()))

    def close(self) -> None:
        if self._h is not None and self._h.value:
            check(lib().tempo_nccl_comm_destroy(self._h))
        self._h = None


def ln_param_reduce_peer(partials: torch.Tensor, cols: int, peer: "LnPeerRank",
                         dgamma: torch.Tensor = None, dbeta: torch.Tensor = None):
    """Stage 2 on fp64 partial rows [nparts][2*cols] + the cross-rank sum."""
    dev = partials.device
    _dev(partials, "partials", torch.float64, dev)
    if partials.dim() != 2 or partials.shape[1] != 2 * cols:
        raise TempoError(2, f"partials: expected [nparts, {2 * cols}], got {tuple(partials.shape)}")
    dgamma = _vec_out(dgamma, "dgamma", cols, dev)
    dbeta = _vec_out(dbeta, "dbeta", cols, dev)
    st = peer.next_struct()
    check(lib().tempo_ln_param_reduce_peer(_ptr(partials), partials.shape[0], cols,
                                           C.byref(st), _ptr(dgamma), _ptr(dbeta), _stream()))
    return dgamma, dbeta


def layernorm_ip_bwd_peer(dy, y, rstd, gamma, beta, peer: "LnPeerRank", dx=None, dgamma=None,
                          dbeta=None, workspace=None):
    """layernorm_ip_bwd with dgamma/dbeta summed over every rank of ``peer``.
    A rank that never arrives (bounded wait, ``peer.timeout_ms``) makes
    ``peer.status`` nonzero (sticky) and the affected dgamma/dbeta NaN;
    every later exchange of this rank then poisons its outputs without
    waiting -- check ``peer.check_status()`` (bench.py checks every step)."""
    dy, y, rstd, gamma, beta, dx, dgamma, dbeta, ws, nbytes, rows, cols = _ln_bwd_args(
        dy, y, rstd, gamma, beta, dx, dgamma, dbeta, workspace)
    if cols != peer.cols:
        raise TempoError(2, f"peer exchange set up for {peer.cols} columns, got {cols}")
    st = peer.next_struct()
    check(lib().tempo_ln_ip_bwd_peer(_ptr(dy), _ptr(y), _ptr(rstd), _ptr(gamma), _ptr(beta),
                                     _ptr(dx), _ptr(dgamma), _ptr(dbeta), _ptr(ws), nbytes,
                                     rows, cols, C.byref(st), _stream()))
    return dx, dgamma, dbeta


# --------------------------------------------------------------------------
# Output-only softmax + dropout recomputation (ops_tempo.cpp:158-194)
# --------------------------------------------------------------------------
def softmax_ip_fwd(z: torch.Tensor, P: torch.Tensor = None) -> torch.Tensor:
    z = _f32(z, "z")
    rows, cols = _rows_cols(z)
    P = _out(P, "P", z)
    check(lib().tempo_softmax_ip_fwd(_ptr(z), _ptr(P), rows, cols, _stream()))
    return P


def softmax_ip_bwd(dP: torch.Tensor, P: torch.Tensor, dZ: torch.Tensor = None) -> torch.Tensor:
    P = _f32(P, "P")
    dP = _f32(dP, "dP", P.device, P.numel())
    rows, cols = _rows_cols(P)
    dZ = _out(dZ, "dZ", P)
    check(lib().tempo_softmax_ip_bwd(_ptr(dP), _ptr(P), _ptr(dZ), rows, cols, _stream()))
    return dZ


def softmax_dropout_fwd(z: torch.Tensor, p: float, mask: torch.Tensor = None,
                        seed: int = 0, offset: int = 0, P: torch.Tensor = None,
                        D: torch.Tensor = None, write_d: bool = True, generate: bool = None):
    """Fused softmax -> dropout_recompute forward.  SUPPLIED mode reads
    ``mask`` (e.g. the reference's bernoulli_keep stream); Philox mode
    (``generate``, the default when ``mask`` is None) writes a fresh mask into
    ``mask`` (allocated if None).  Returns (P, D, mask)."""
    z = _f32(z, "z")
    rows, cols = _rows_cols(z)
    if generate is None:
        generate = mask is None
    mode = MASK_PHILOX if generate else MASK_SUPPLIED
    if mask is None and not generate:
        raise TempoError(2, "mask: a supplied-mask forward needs the mask")
    mask = _mask(mask, "mask", z.numel(), z.device)
    P = _out(P, "P", z)
    D = _out(D, "D", z) if write_d else None
    check(lib().tempo_softmax_dropout_fwd(_ptr(z), float(p), mode, _ptr(mask), int(seed),
                                          int(offset), _ptr(P), _ptr(D if write_d else None),
                                          rows, cols, _stream()))
    return P, (D if write_d else None), mask


def attn_probs_bwd(dD: torch.Tensor, P: torch.Tensor, mask: torch.Tensor, p: float,
                   write_d: bool = False, dZ: torch.Tensor = None, D: torch.Tensor = None):
    """Fused dropout bwd + output-only softmax bwd (+ recomputed D).
    Returns (dZ, D or None)."""
    P = _f32(P, "P")
    dD = _f32(dD, "dD", P.device, P.numel())
    rows, cols = _rows_cols(P)
    if mask is None:
        raise TempoError(2, "mask: the forward's bit mask is required")
    mask = _mask(mask, "mask", P.numel(), P.device)
    dZ = _out(dZ, "dZ", P)
    D = _out(D, "D", P) if write_d else None
    check(lib().tempo_attn_probs_bwd(_ptr(dD), _ptr(P), _ptr(mask), float(p), _ptr(dZ),
                                     _ptr(D if write_d else None), rows, cols, _stream()))
    return dZ, (D if write_d else None)


# --------------------------------------------------------------------------
# Dropout (ops_reference.cpp:147-161, ref_ops::dropout :214-225)
# --------------------------------------------------------------------------
def dropout_fwd(x: torch.Tensor, p: float, mask: torch.Tensor = None, seed: int = 0,
                offset: int = 0, y: torch.Tensor = None, generate: bool = None):
    """y = mask ? x/(1-p) : 0.  Mask supplied (read) or generated (Philox,
    written into ``mask``; default when ``mask`` is None).  Returns (y, mask)."""
    x = _f32(x, "x")
    if generate is None:
        generate = mask is None
    mode = MASK_PHILOX if generate else MASK_SUPPLIED
    if mask is None and not generate:
        raise TempoError(2, "mask: a supplied-mask forward needs the mask")
    mask = _mask(mask, "mask", x.numel(), x.device)
    y = _out(y, "y", x)
    check(lib().tempo_dropout_fwd(_ptr(x), float(p), mode, _ptr(mask), int(seed), int(offset),
                                  _ptr(y), x.numel(), _stream()))
    return y, mask


def attn_dropout_dv(P: torch.Tensor, mask: torch.Tensor, p: float, dO: torch.Tensor,
                    dV: torch.Tensor = None) -> torch.Tensor:
    """dV = D^T @ dO per (batch, head) with the dropped-out map D = mask ?
    P/(1-p) : 0 rebuilt inside the tcgen05 GEMM from the stashed P and mask
    (the consumer of Sub-Layer Dropout Recomputation, graph.cpp:46-50 ->
    ops_tempo.cpp:17-26), D never written to HBM.  P [..., s_q, s_k],
    dO [..., s_q, d] -> dV [..., s_k, d]."""
    P = _f32(P, "P")
    if P.dim() < 2:
        raise TempoError(2, "P: expected [..., s_q, s_k]")
    s_q, s_k = P.shape[-2], P.shape[-1]
    heads = P.numel() // max(1, s_q * s_k)
    dO = _f32(dO, "dO", P.device)
    if dO.dim() != P.dim() or dO.shape[:-1] != P.shape[:-1]:
        raise TempoError(2, f"dO {tuple(dO.shape)} does not match P {tuple(P.shape)}")
    d = dO.shape[-1]
    if mask is None:
        raise TempoError(2, "mask: the forward's bit mask is required")
    mask = _mask(mask, "mask", P.numel(), P.device)
    shape = tuple(P.shape[:-2]) + (s_k, d)
    if dV is None:
        dV = torch.empty(shape, dtype=torch.float32, device=P.device)
    else:
        _f32(dV, "dV", P.device, heads * s_k * d)
    check(lib().tempo_attn_dropout_dv(_ptr(P), _ptr(mask), float(p), _ptr(dO), _ptr(dV), heads,
                                      s_q, s_k, d, _stream()))
    return dV


def attn_dropout_ctx(P: torch.Tensor, mask: torch.Tensor, p: float, V: torch.Tensor,
                     ctx: torch.Tensor = None) -> torch.Tensor:
    """ctx = D @ V per (batch, head) with D = mask ? P/(1-p) : 0 rebuilt inside
    the tcgen05 GEMM (the forward consumer of Sub-Layer Dropout
    Recomputation, tempo_ops::sdpa ops_tempo.cpp:196-210): with
    softmax_dropout_fwd(..., write_d=False) D never reaches HBM.
    P [..., s_q, s_k], V [..., s_k, d] -> ctx [..., s_q, d]."""
    P = _f32(P, "P")
    if P.dim() < 2:
        raise TempoError(2, "P: expected [..., s_q, s_k]")
    s_q, s_k = P.shape[-2], P.shape[-1]
    heads = P.numel() // max(1, s_q * s_k)
    V = _f32(V, "V", P.device)
    if V.dim() != P.dim() or V.shape[:-2] != P.shape[:-2] or V.shape[-2] != s_k:
        raise TempoError(2, f"V {tuple(V.shape)} does not match P {tuple(P.shape)}")
    d = V.shape[-1]
    if mask is None:
        raise TempoError(2, "mask: the forward's bit mask is required")
    mask = _mask(mask, "mask", P.numel(), P.device)
    shape = tuple(P.shape[:-1]) + (d,)
    if ctx is None:
        ctx = torch.empty(shape, dtype=torch.float32, device=P.device)
    else:
        _f32(ctx, "ctx", P.device, heads * s_q * d)
    check(lib().tempo_attn_dropout_ctx(_ptr(P), _ptr(mask), float(p), _ptr(V), _ptr(ctx), heads,
                                       s_q, s_k, d, _stream()))
    return ctx


def dropout_add_layernorm_fwd(proj: torch.Tensor, residual: torch.Tensor, gamma: torch.Tensor,
                              beta: torch.Tensor, p: float, mask: torch.Tensor = None,
                              seed: int = 0, offset: int = 0, generate: bool = None,
                              eps: float = 1e-5, check_gamma: bool = True, y: torch.Tensor = None,
                              rstd: torch.Tensor = None, dev_status: torch.Tensor = None):
    """The reference layer's ref_ops::dropout -> add -> tempo_ops::layernorm
    (encoder.cpp:180-191, 198-210) in one pass: y = LN(residual +
    dropout(proj)).  Returns (y, rstd, mask); stash = y + rstd + mask bits.
    generate=True (default without a mask): Philox mask by global element
    index `offset + i`, the same bits dropout_fwd would draw."""
    proj = _f32(proj, "proj")
    residual = _f32(residual, "residual", proj.device, proj.numel())
    rows, cols = _rows_cols(proj)
    gamma, beta = _f32(gamma, "gamma", proj.device, cols), _f32(beta, "beta", proj.device, cols)
    if check_gamma:
        ln_check_gamma(gamma)
    if generate is None:
        generate = mask is None
    if mask is None and not generate:
        raise TempoError(2, "mask: a supplied-mask forward needs the mask")
    mask = _mask(mask, "mask", proj.numel(), proj.device)
    y = _out(y, "y", proj)
    rstd = torch.empty(proj.shape[:-1], dtype=torch.float32, device=proj.device) if rstd is None \
        else _f32(rstd, "rstd", proj.device, rows)
    if dev_status is not None:
        _dev(dev_status, "dev_status", torch.int32, proj.device, 1)
    check(lib().tempo_dropout_add_ln_fwd(
        _ptr(proj), _ptr(residual), float(p), MASK_PHILOX if generate else MASK_SUPPLIED,
        _ptr(mask), int(seed), int(offset), _ptr(gamma), _ptr(beta), float(eps), _ptr(y),
        _ptr(rstd), rows, cols, _ptr(dev_status), _stream()))
    return y, rstd, mask


def dropout_add_layernorm_bwd(dy: torch.Tensor, y: torch.Tensor, rstd: torch.Tensor,
                              gamma: torch.Tensor, beta: torch.Tensor, mask: torch.Tensor,
                              p: float, d_residual: torch.Tensor = None,
                              d_proj: torch.Tensor = None, dgamma: torch.Tensor = None,
                              dbeta: torch.Tensor = None, workspace: torch.Tensor = None,
                              peer: "LnPeerRank" = None):
    """Backward of dropout_add_layernorm_fwd in one pass: returns (d_residual,
    d_proj, dgamma, dbeta); d_residual = the LayerNorm input gradient,
    d_proj = mask ? d_residual / (1-p) : 0.  With `peer`, dgamma/dbeta are
    summed over its ranks (as layernorm_ip_bwd_peer)."""
    dy, y, rstd, gamma, beta, d_res, dgamma, dbeta, ws, nbytes, rows, cols = _ln_bwd_args(
        dy, y, rstd, gamma, beta, d_residual, dgamma, dbeta, workspace)
    if mask is None:
        raise TempoError(2, "mask: the forward's bit mask is required")
    mask = _mask(mask, "mask", y.numel(), y.device)
    d_proj = _out(d_proj, "d_proj", dy)
    st = None
    if peer is not None:
        if cols != peer.cols:
            raise TempoError(2, f"peer exchange set up for {peer.cols} columns, got {cols}")
        st = peer.next_struct()
    check(lib().tempo_dropout_add_ln_bwd(
        _ptr(dy), _ptr(y), _ptr(rstd), _ptr(gamma), _ptr(beta), _ptr(mask), float(p),
        _ptr(d_res), _ptr(d_proj), _ptr(dgamma), _ptr(dbeta), _ptr(ws), nbytes, rows, cols,
        C.byref(st) if st is not None else None, _stream()))
    return d_res, d_proj, dgamma, dbeta


def dropout_bwd(dy: torch.Tensor, mask: torch.Tensor, p: float,
                dx: torch.Tensor = None) -> torch.Tensor:
    dy = _f32(dy, "dy")
    if mask is None:
        raise TempoError(2, "mask: the forward's bit mask is required")
    mask = _mask(mask, "mask", dy.numel(), dy.device)
    dx = _out(dx, "dx", dy)
    check(lib().tempo_dropout_bwd(_ptr(dy), _ptr(mask), float(p), _ptr(dx), dy.numel(),
                                  _stream()))
    return dx


# --------------------------------------------------------------------------
# Masks
# --------------------------------------------------------------------------
def pack_mask(bytes_: torch.Tensor, dev_status: torch.Tensor = None) -> torch.Tensor:
    """BoolMask bytes (uint8 CUDA tensor) -> packed bits."""
    b = _dev(bytes_, "bytes", torch.uint8)
    bits = torch.empty(mask_words(b.numel()), dtype=torch.int32, device=b.device)
    if dev_status is not None:
        _dev(dev_status, "dev_status", torch.int32, b.device, 1)
    check(lib().tempo_mask_pack(_ptr(b), _ptr(bits), b.numel(), _ptr(dev_status), _stream()))
    return bits


def unpack_mask(bits: torch.Tensor, n: int) -> torch.Tensor:
    bits = _mask(bits, "bits", int(n), bits.device)
    out = torch.empty(n, dtype=torch.uint8, device=bits.device)
    check(lib().tempo_mask_unpack(_ptr(bits), _ptr(out), int(n), _stream()))
    return out


def bernoulli_keep_bits(n: int, p: float, seed: int):
    """BoolMask::bernoulli_keep (tensor.cpp:186-203) on the host, packed:
    returns a numpy uint32 array of ceil(n/32) words."""
    import numpy as np
    out = np.zeros(mask_words(n), np.uint32)
    check(lib().tempo_bernoulli_keep_bits_host(int(n), float(p), int(seed), out.ctypes.data))
    return out


def bernoulli_keep_bits_device(n: int, p: float, seed: int, offset: int = 0,
                               out: Optional[torch.Tensor] = None,
                               device: Optional[torch.device] = None) -> torch.Tensor:
    """The same BoolMask::bernoulli_keep stream generated on the device (bit
    for bit, by jump-ahead): keep bits of elements [offset, offset + n) as
    ceil(n/32) int32 words.  offset must be a multiple of 32."""
    dev = device or (out.device if out is not None else torch.device("cuda", torch.cuda.current_device()))
    out = _mask(out, "out", int(n), dev)
    nbytes = int(lib().tempo_bernoulli_keep_bits_workspace_size(int(offset), int(n)))
    ws = torch.empty(max(nbytes, 1), dtype=torch.uint8, device=dev)
    check(lib().tempo_bernoulli_keep_bits(int(n), float(p), int(seed), int(offset), _ptr(out),
                                          _ptr(ws), nbytes, _stream()))
    return out


def softmax_dropout_fwd_refmask(z: torch.Tensor, p: float, seed: int, offset: int = 0,
                                mask: torch.Tensor = None, P: torch.Tensor = None,
                                D: torch.Tensor = None, write_d: bool = True,
                                workspace: torch.Tensor = None):
    """softmax_dropout_fwd with the reference's own mask stream
    (BoolMask::bernoulli_keep(shape, p, seed), elements [offset, offset + n))
    generated inside the softmax kernel; the mask is written to ``mask``.
    Returns (P, D, mask): bitwise the supplied-mask forward on
    bernoulli_keep_bits_device(n, p, seed, offset)."""
    z = _f32(z, "z")
    rows, cols = _rows_cols(z)
    mask = _mask(mask, "mask", z.numel(), z.device)
    P = _out(P, "P", z)
    D = _out(D, "D", z) if write_d else None
    nbytes = int(lib().tempo_bernoulli_keep_bits_workspace_size(int(offset), z.numel()))
    if workspace is None:
        workspace = torch.empty(max(nbytes, 1), dtype=torch.uint8, device=z.device)
    else:
        _dev(workspace, "workspace", workspace.dtype, z.device, min_numel=None)
        if workspace.numel() * workspace.element_size() < nbytes:
            raise TempoError(2, f"workspace: need {nbytes} bytes")
    check(lib().tempo_softmax_dropout_fwd_refmask(
        _ptr(z), float(p), int(seed), int(offset), _ptr(mask), _ptr(P),
        _ptr(D if write_d else None), rows, cols, _ptr(workspace),
        workspace.numel() * workspace.element_size(), _stream()))
    return P, (D if write_d else None), mask


def mt_outputs_after(seed: int, steps: int, count: int):
    """Host reference of the jump-ahead: `count` outputs of
    std::mt19937_64(seed) after discard(steps) (numpy uint64)."""
    import numpy as np
    out = np.zeros(int(count), np.uint64)
    check(lib().tempo_mt_outputs_after_host(int(seed), int(steps), int(count), out.ctypes.data))
    return out


def mask_stream_seed(seed: int, salt: int, site: int) -> int:
    return int(lib().tempo_mask_stream_seed(seed, salt, site))


def layer_stash_bytes_per_token(seq: int, hidden: int, heads: int, tempo: bool = True,
                                mask_bits: bool = True) -> int:
    return int(lib().tempo_layer_stash_bytes_per_token(seq, hidden, heads, int(tempo),
                                                       int(mask_bits)))
