"""bench.py -- Tempo in-place activation operators on B200.

One "step" = forward + backward of the Tempo activation-operator chain of one
BERT-large encoder layer (BASELINE.json configs[3]: B=64, S=512, H=1024,
A=16, p=0.1), in encoder order (proj/src/encoder.cpp:155-210):

  fwd: softmax+dropout_recompute [B*A*S, S] -> attn-out dropout [T,H] ->
       LayerNorm1 [T,H] -> GELU [T,4H] -> ffn dropout [T,H] -> LayerNorm2 [T,H]
  bwd: LN2 -> ffn dropout -> GELU -> LN1 -> attn-out dropout ->
       attn-probs (dropout bwd + softmax bwd + recomputed D for the dV GEMM)
  (+ at N>1: one NCCL all-reduce of the bucketed LN dgamma/dbeta, 4H floats)

GEMMs and residual adds are outside the path and are
replaced by synthetic fp32 buffers of the layer shapes.

N=1: configs[3] (B=64).  N>1 (`--gpus N`; run under torchrun, or bench.py
re-launches itself as N ranks): configs[4] strong scaling by default -- the
global batch of 512 sequences split by rows, 512/N per rank;
`--scaling weak` keeps B=64 per rank instead.

metric: fwd+bwd GB/s = algorithmic HBM bytes of the chain (SURVEY 8d:
GELU 8.125+12.125 B/elem, LN 8NM+4N+8M / 12NM+4N+16M, attention 12.125 +
16.125 B/elem, dropouts 8.125+8.125 B/elem) / device time, summed over ranks.

Usage: python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                       [--scaling strong|weak] [--global-batch 512] [--masks philox|reference]
       TEMPO_BENCH_BACKEND=gloo python bench.py --gpus 2   # N>1 functional run on one GPU
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

B, S, H, A, P_DROP = 64, 512, 1024, 16, 0.1
GLOBAL_B_STRONG = 512    # configs[4]: B=512 sharded by rows over the N GPUs
T = B * S                # tokens per rank
ATT_ROWS = B * A * S     # attention-probability rows per rank
METRIC = "fwd+bwd GB/s per op vs B200 HBM peak at 1/2/4/8 GPU; activation bytes/layer"
WORKLOAD = "bert-large-layer-tempo-op-chain"


# ----------------------------------------------------------------- bytes
def op_bytes(batch=B, fused=False):
    """Algorithmic HBM bytes per op, for `batch` sequences.
    fused: the hidden dropout -> residual add -> LayerNorm pairs run as one
    op each way (read proj + residual, write y + bits: 12.125 B/elem; read
    dy, y + bits, write d_residual + d_proj: 16.125 B/elem)."""
    t, ar = batch * S, batch * A * S
    n_g, n_h, n_a = t * 4 * H, t * H, ar * S
    bits = 1.0 / 8
    out = {
        "softmax_dropout_fwd": n_a * (4 + 4 + 4 + bits),     # z -> P, D, mask
        "attn_probs_bwd": n_a * (4 + 4 + bits + 4 + 4),      # dD, P, mask -> dZ, D
        "gelu_fwd": n_g * (4 + 4 + bits),
        "gelu_bwd": n_g * (4 + 4 + bits + 4),
    }
    if fused:
        out["dropout_add_layernorm_fwd"] = 2 * (n_h * (12 + bits) + 4 * t + 8 * H)
        out["dropout_add_layernorm_bwd"] = 2 * (n_h * (16 + bits) + 4 * t + 16 * H)
    else:
        out["layernorm_fwd"] = 2 * (8 * n_h + 4 * t + 8 * H)
        out["layernorm_bwd"] = 2 * (12 * n_h + 4 * t + 16 * H)
        out["dropout_fwd"] = 2 * n_h * (8 + bits)
        out["dropout_bwd"] = 2 * n_h * (8 + bits)
    return out


def unfused_equivalent_bytes(batch=B):
    """What the fused chain's work moves as separate ops, residual adds
    included (add: read 2, write 1 fp32 per element forward; its backward
    is a pass-through): the second byte model reported beside `value`."""
    t = batch * S
    n_h = t * H
    return sum(op_bytes(batch, False).values()) + 2 * 12 * n_h


def setup_peer(chain, dist, rank, world, dev, backend):
    """Map every rank's LN exchange buffers (CUDA IPC) and self-check one
    exchange against the known answer on all ranks; None -> fall back to the
    all-reduce.  Off for the gloo functional mode (ranks sharing one GPU)
    unless TEMPO_PEER=force, and with TEMPO_PEER=0."""
    import torch
    mode = os.environ.get("TEMPO_PEER", "1")  # "0": off; "force": also with gloo (tests)
    if mode == "0" or (backend != "nccl" and mode != "force"):
        return None
    peer, ok = None, 1
    try:
        peer = chain.ops.LnPeerRank.ipc(H, dev)
        parts = torch.full((3, 2 * H), float(rank + 1), dtype=torch.float64, device=dev)
        dg, db = chain.ops.ln_param_reduce_peer(parts, H, peer)
        torch.cuda.synchronize()
        peer.check_status()
        want = 3.0 * sum(r + 1 for r in range(world))
        ok = int(bool((dg == want).all()) and bool((db == want).all()))
    except Exception as ex:  # noqa: BLE001  (any failure: use the all-reduce)
        print(f"rank {rank}: peer exchange unavailable ({ex}); using all_reduce", file=sys.stderr)
        ok = 0
    flag = torch.tensor([ok], dtype=torch.int32, device=dev)
    dist.all_reduce(flag, op=dist.ReduceOp.MIN)
    if int(flag.item()) == 0:
        if peer is not None:
            peer.close()
        return None
    return peer


def trimmed_mean(ts):
    """Mean of the middle ~60 % of the samples.  CUDA event times on this
    GPU are quantised (~2.05 us steps), so for the 40-50 us ops a median
    snaps to one step; a trimmed mean of samples with random timer phase
    averages the quantisation out and still drops outliers."""
    v = sorted(ts)
    k = len(v) // 5
    v = v[k:len(v) - k] if len(v) - 2 * k > 0 else v
    return sum(v) / len(v)


def op_elements(batch=B, fused=False):
    """Elements each op processes per step (the map it streams: n for the
    elementwise ops, rows x cols for the row ops; both LNs / dropouts)."""
    t, ar = batch * S, batch * A * S
    n_g, n_h, n_a = t * 4 * H, t * H, ar * S
    out = {"softmax_dropout_fwd": n_a, "attn_probs_bwd": n_a, "gelu_fwd": n_g, "gelu_bwd": n_g}
    if fused:
        out.update({"dropout_add_layernorm_fwd": 2 * n_h, "dropout_add_layernorm_bwd": 2 * n_h})
    else:
        out.update({"layernorm_fwd": 2 * n_h, "layernorm_bwd": 2 * n_h, "dropout_fwd": 2 * n_h,
                    "dropout_bwd": 2 * n_h})
    return out


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            pk = json.load(f)
        return float(pk["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


# ------------------------------------------------------------ the chain
def _numel(shapes):
    n = 0
    for shp in shapes.values():
        k = 1
        for d in shp:
            k *= d
        n += k
    return n


class Chain:
    """Device buffers + the step of the Tempo op chain on one rank's rows.
    fused=True: each hidden dropout -> residual add -> LayerNorm pair is the
    fused op (tempo_dropout_add_ln_fwd/bwd) and the layer input is a
    residual stream; fused=False: the separate dropout and LayerNorm ops
    with no residual add (the round-1 chain)."""
    peer = None  # ops.LnPeerRank at N>1: the fused dgamma/dbeta exchange
    kernel_events = None  # list: CUDA event pairs around attn_probs_bwd in each step

    def __init__(self, dev, rank, world, seed=1234, batch=B, fused=False):
        import torch
        from paper_2210_10246_b200 import ops
        self.ops, self.torch, self.dev = ops, torch, dev
        self.rank, self.world = rank, world
        self.batch, self.fused = batch, fused
        T, ATT_ROWS = batch * S, batch * A * S  # this rank's token / attention rows
        self.T, self.ATT_ROWS = T, ATT_ROWS
        g = torch.Generator(device=dev)
        g.manual_seed(seed + rank)
        self.table = ops.GeluTable.default()
        # The per-step inputs (GEMM outputs / input-gradients in the real
        # layer: synthetic here) live in ONE contiguous buffer and the per-step
        # results in another, so the e2e measurement moves each set with one
        # copy and double-buffers with a single extra set.
        shapes_in = {"z": (ATT_ROWS, S),            # attention scores
                     "x_attn_out": (T, H),          # attention output projection
                     "x_ffn1": (T, 4 * H),          # first FFN linear output
                     "x_ffn2": (T, H),              # second FFN linear output
                     "dy_ln2": (T, H), "dy_gelu": (T, 4 * H), "dy_ln1": (T, H),
                     "dD": (ATT_ROWS, S)}
        shapes_out = {"dZ": (ATT_ROWS, S), "dx_d1": (T, H), "dx_g": (T, 4 * H),
                      "dx_d2": (T, H), "dparams": (4 * H,)}  # [dg2, db2, dg1, db1]
        if fused:
            shapes_in["x_res"] = (T, H)       # the layer input (LN1's residual)
            shapes_out["dx_res"] = (T, H)     # its gradient through LN1's residual path
        self.shapes_in, self.shapes_out = shapes_in, shapes_out
        self.in_buf = torch.empty(_numel(shapes_in), device=dev)
        self.in_buf.normal_(generator=g)
        self.out_buf = torch.zeros(_numel(shapes_out), device=dev)
        self.bind(self.in_buf, self.out_buf)
        rn = lambda *s: torch.randn(*s, device=dev, generator=g)  # noqa: E731
        self.g1 = (1 + 0.2 * rn(H)).contiguous()
        self.b1 = (0.1 * rn(H)).contiguous()
        self.g2 = (1 + 0.2 * rn(H)).contiguous()
        self.b2 = (0.1 * rn(H)).contiguous()
        # outputs / stashes, allocated once
        e = torch.empty_like
        mw = lambda n: torch.empty(ops.mask_words(n), dtype=torch.int32, device=dev)  # noqa: E731
        self.P, self.D, self.m_att = e(self.z), e(self.z), mw(self.z.numel())
        self.m1, self.m2 = mw(T * H), mw(T * H)
        self.d1 = self.d2 = None  # the unfused chain's dropout outputs
        if not fused:
            self.d1, self.d2 = e(self.x_attn_out), e(self.x_ffn2)
        self.y_ln1, self.rs1 = e(self.x_attn_out), torch.empty(T, device=dev)
        self.y_g, self.m_g = e(self.x_ffn1), mw(T * 4 * H)
        self.y_ln2, self.rs2 = e(self.x_ffn2), torch.empty(T, device=dev)
        self.dx_ln2 = e(self.x_ffn2)   # fused: LN2's residual-path gradient (to y_ln1)
        self.dx_ln1 = None if fused else e(self.x_attn_out)
        self.Drec = e(self.z)
        self.ws = ops.ln_workspace(T, H, dev)
        self.status = torch.zeros(1, dtype=torch.int32, device=dev)
        self.step_idx = 0
        self.mask_mode = "philox"  # or "reference" (bench.py --masks reference)
        # --masks reference: the attention mask generated inside the softmax
        # kernel (False: a separate generation pass, TEMPO_REFMASK_FUSED=0)
        self.refmask_fused = os.environ.get("TEMPO_REFMASK_FUSED", "1") != "0"
        # global element offsets: rank shards reproduce the unsharded masks
        self.off_att = rank * ATT_ROWS * S
        self.off_h = rank * T * H

    def bind(self, in_buf, out_buf):
        """Point the step's inputs / results at views of one input buffer and
        one result buffer."""
        for shapes, buf in ((self.shapes_in, in_buf), (self.shapes_out, out_buf)):
            o = 0
            for name, shp in shapes.items():
                n = _numel({name: shp})
                setattr(self, name, buf[o:o + n].view(shp))
                o += n

    def retained_bytes(self):
        """Bytes held between forward and backward by this chain (the stash):
        P, the three dropout masks and the GELU mask (bits), GELU y, both LN
        y + rstd.  D, the inputs and the grads are not retained."""
        ts = [self.P, self.m_att, self.m1, self.y_ln1, self.rs1, self.y_g, self.m_g, self.m2,
              self.y_ln2, self.rs2]
        return int(sum(t.numel() * t.element_size() for t in ts))

    def reference_masks(self, step):
        """The reference's own mask streams for this step, generated on the
        device bit for bit (BoolMask::bernoulli_keep with
        encoder::mask_stream_seed(run seed, salt = step, site 0/1/2),
        encoder.cpp:168-201), each rank at its global offset."""
        o, torch = self.ops, self.torch
        main = torch.cuda.current_stream()
        if not hasattr(self, "_mask_streams"):  # one stream per mask: they overlap
            self._mask_streams = [torch.cuda.Stream() for _ in range(3)]
        T, ATT_ROWS = self.T, self.ATT_ROWS
        for site, (m, n, off) in enumerate([(self.m_att, ATT_ROWS * S, self.off_att),
                                            (self.m1, T * H, self.off_h),
                                            (self.m2, T * H, self.off_h)]):
            if site == 0 and self.refmask_fused:
                continue  # generated inside the softmax forward (forward())
            s_ = self._mask_streams[site]
            s_.wait_stream(main)  # the previous step is done with this mask
            with torch.cuda.stream(s_):
                o.bernoulli_keep_bits_device(n, P_DROP, o.mask_stream_seed(1234, step, site),
                                             offset=off, out=m)
        if not self.refmask_fused:
            for s_ in self._mask_streams:
                main.wait_stream(s_)
        # else: the hidden masks' generation overlaps the attention mask's
        # jump and the fused softmax forward; each consumer waits for its own
        # mask (_mask_ready)

    def _mask_ready(self, site):
        if self.mask_mode == "reference" and self.refmask_fused:
            self.torch.cuda.current_stream().wait_stream(self._mask_streams[site])

    def forward(self, seed):
        o = self.ops
        gen = self.mask_mode != "reference"
        if not gen:
            self.reference_masks(seed)
        if not gen and self.refmask_fused:
            # the attention mask = the reference's stream, generated inside the
            # softmax kernel (tempo_softmax_dropout_fwd_refmask)
            if getattr(self, "_ws_att", None) is None:
                nb = int(o.lib().tempo_bernoulli_keep_bits_workspace_size(self.off_att,
                                                                          self.ATT_ROWS * S))
                self._ws_att = self.torch.empty(max(nb, 1), dtype=self.torch.uint8,
                                                device=self.z.device)
            o.softmax_dropout_fwd_refmask(self.z, P_DROP, o.mask_stream_seed(1234, seed, 0),
                                          offset=self.off_att, mask=self.m_att, P=self.P,
                                          D=self.D, workspace=self._ws_att)
        else:
            o.softmax_dropout_fwd(self.z, P_DROP, mask=self.m_att, generate=gen, seed=seed,
                                  offset=self.off_att, P=self.P, D=self.D)
        if self.fused:  # encoder.cpp:180-191, 198-210 as two fused passes
            self._mask_ready(1)
            o.dropout_add_layernorm_fwd(self.x_attn_out, self.x_res, self.g1, self.b1, P_DROP,
                                        mask=self.m1, generate=gen, seed=seed + 1,
                                        offset=self.off_h, check_gamma=False, y=self.y_ln1,
                                        rstd=self.rs1, dev_status=self.status)
            o.gelu_ip_fwd(self.x_ffn1, self.table, y=self.y_g, mask=self.m_g)
            self._mask_ready(2)
            o.dropout_add_layernorm_fwd(self.x_ffn2, self.y_ln1, self.g2, self.b2, P_DROP,
                                        mask=self.m2, generate=gen, seed=seed + 2,
                                        offset=self.off_h, check_gamma=False, y=self.y_ln2,
                                        rstd=self.rs2, dev_status=self.status)
            return
        self._mask_ready(1)
        o.dropout_fwd(self.x_attn_out, P_DROP, mask=self.m1, generate=gen, seed=seed + 1,
                      offset=self.off_h, y=self.d1)
        o.layernorm_ip_fwd(self.d1, self.g1, self.b1, check_gamma=False, y=self.y_ln1,
                           rstd=self.rs1, dev_status=self.status)
        o.gelu_ip_fwd(self.x_ffn1, self.table, y=self.y_g, mask=self.m_g)
        self._mask_ready(2)
        o.dropout_fwd(self.x_ffn2, P_DROP, mask=self.m2, generate=gen, seed=seed + 2,
                      offset=self.off_h, y=self.d2)
        o.layernorm_ip_fwd(self.d2, self.g2, self.b2, check_gamma=False, y=self.y_ln2,
                           rstd=self.rs2, dev_status=self.status)

    def _ln_bwd(self, dy, y, rs, g, b, dx, dg, db):
        if self.peer is not None:  # N>1: cross-rank sum fused into stage 2
            self.ops.layernorm_ip_bwd_peer(dy, y, rs, g, b, self.peer, dx=dx, dgamma=dg, dbeta=db,
                                           workspace=self.ws)
        else:
            self.ops.layernorm_ip_bwd(dy, y, rs, g, b, dx=dx, dgamma=dg, dbeta=db,
                                      workspace=self.ws)

    def _dal_bwd(self, dy, y, rs, g, b, m, d_res, d_proj, dg, db):
        self.ops.dropout_add_layernorm_bwd(dy, y, rs, g, b, m, P_DROP, d_residual=d_res,
                                           d_proj=d_proj, dgamma=dg, dbeta=db,
                                           workspace=self.ws, peer=self.peer)

    def backward(self, allreduce):
        o = self.ops
        dp = self.dparams
        if self.fused:
            self._dal_bwd(self.dy_ln2, self.y_ln2, self.rs2, self.g2, self.b2, self.m2,
                          self.dx_ln2, self.dx_d2, dp[0:H], dp[H:2 * H])
            o.gelu_ip_bwd(self.dy_gelu, self.y_g, self.m_g, self.table, dx=self.dx_g)
            self._dal_bwd(self.dy_ln1, self.y_ln1, self.rs1, self.g1, self.b1, self.m1,
                          self.dx_res, self.dx_d1, dp[2 * H:3 * H], dp[3 * H:])
            if allreduce is not None:
                allreduce(dp)
            self._attn_bwd()
            return
        self._ln_bwd(self.dy_ln2, self.y_ln2, self.rs2, self.g2, self.b2, self.dx_ln2,
                     dp[0:H], dp[H:2 * H])
        o.dropout_bwd(self.dx_ln2, self.m2, P_DROP, dx=self.dx_d2)
        o.gelu_ip_bwd(self.dy_gelu, self.y_g, self.m_g, self.table, dx=self.dx_g)
        self._ln_bwd(self.dy_ln1, self.y_ln1, self.rs1, self.g1, self.b1, self.dx_ln1,
                     dp[2 * H:3 * H], dp[3 * H:])
        if allreduce is not None:
            allreduce(dp)  # the one collective: bucketed LN dgamma/dbeta (16 KB)
        o.dropout_bwd(self.dx_ln1, self.m1, P_DROP, dx=self.dx_d1)
        self._attn_bwd()

    def _attn_bwd(self):
        o = self.ops
        ev = self.kernel_events
        if ev is not None:  # in-chain duration of the dominant kernel (roofline)
            ev.append((self.torch.cuda.Event(enable_timing=True),
                       self.torch.cuda.Event(enable_timing=True)))
            ev[-1][0].record()
        o.attn_probs_bwd(self.dD, self.P, self.m_att, P_DROP, write_d=True, dZ=self.dZ,
                         D=self.Drec)
        if ev is not None:
            ev[-1][1].record()

    def poll_peer_status(self, final=False):
        """Surface a timed-out dgamma/dbeta exchange every step without a host
        sync: the device status word (sticky: once a peer failed to arrive it
        stays nonzero and later exchanges NaN-poison their outputs) is copied
        to pinned memory on the stream each step and the host reads the last
        landed value; `final` synchronises and checks the exact value."""
        if self.peer is None:
            return
        torch = self.torch
        if not hasattr(self, "_status_host"):
            self._status_host = torch.zeros(1, dtype=torch.int32, pin_memory=True)
        if final:
            torch.cuda.synchronize()
            self.peer.check_status()
            return
        if int(self._status_host[0]) != 0:
            self.peer.check_status()
        self._status_host.copy_(self.peer.status, non_blocking=True)

    def step(self, allreduce=None):
        self.step_idx += 1
        self.forward(1000 + 3 * self.step_idx)
        self.backward(allreduce)

    # kernels launched per step (ours): softmax fwd 1, dropout fwd 2, LN fwd 2,
    # GELU fwd 1, LN bwd 2x(stage1+stage2), dropout bwd 2, GELU bwd 1, attn bwd 1;
    # fused: softmax 1, dropout+add+LN fwd 2, GELU fwd 1, its bwd 2x2, GELU bwd 1, attn 1
    LAUNCHES_PER_STEP = 14
    LAUNCHES_PER_STEP_FUSED = 10
    # --masks reference, per mask: seed, (base, jump) for each of the 2 digit
    # levels the rank-0 offsets touch, keep = 6; three masks
    REF_MASK_LAUNCHES = 18

    def per_op_timings(self, reps, flush, flush_dirty=None):
        """Per-kernel device time (CUDA events on the launching stream, L2
        flushed before every rep), for the roofline and the per-op table.
        `flush` evicts L2 by READING a buffer larger than L2 (the timed op
        starts with its inputs out of L2 and no foreign dirty lines to write
        back -- the op's own traffic, as ncu's cache-controlled replay sees
        it); `flush_dirty` (optional, reported beside it) WRITES such a
        buffer, so the op also pays the write-back of ~126 MB of dirty lines."""
        torch, o = self.torch, self.ops
        dp = self.dparams
        H_ = H
        calls = {
            "softmax_dropout_fwd": lambda: o.softmax_dropout_fwd(self.z, P_DROP, mask=self.m_att, generate=True, seed=7, P=self.P, D=self.D),
            "attn_probs_bwd": lambda: o.attn_probs_bwd(self.dD, self.P, self.m_att, P_DROP, write_d=True, dZ=self.dZ, D=self.Drec),
            "gelu_fwd": lambda: o.gelu_ip_fwd(self.x_ffn1, self.table, y=self.y_g, mask=self.m_g),
            "gelu_bwd": lambda: o.gelu_ip_bwd(self.dy_gelu, self.y_g, self.m_g, self.table, dx=self.dx_g),
        }
        if self.fused:
            calls.update({
                "dropout_add_layernorm_fwd": lambda: o.dropout_add_layernorm_fwd(self.x_ffn2, self.y_ln1, self.g2, self.b2, P_DROP, mask=self.m2, generate=True, seed=9, check_gamma=False, y=self.y_ln2, rstd=self.rs2),
                "dropout_add_layernorm_bwd": lambda: o.dropout_add_layernorm_bwd(self.dy_ln2, self.y_ln2, self.rs2, self.g2, self.b2, self.m2, P_DROP, d_residual=self.dx_ln2, d_proj=self.dx_d2, dgamma=dp[:H_], dbeta=dp[H_:2 * H_], workspace=self.ws),
            })
        else:
            calls.update({
                "layernorm_fwd": lambda: o.layernorm_ip_fwd(self.d1, self.g1, self.b1, check_gamma=False, y=self.y_ln1, rstd=self.rs1),
                "layernorm_bwd": lambda: o.layernorm_ip_bwd(self.dy_ln1, self.y_ln1, self.rs1, self.g1, self.b1, dx=self.dx_ln1, dgamma=dp[:H_], dbeta=dp[H_:2 * H_], workspace=self.ws),
                "dropout_fwd": lambda: o.dropout_fwd(self.x_ffn2, P_DROP, mask=self.m2, generate=True, seed=9, y=self.d2),
                "dropout_bwd": lambda: o.dropout_bwd(self.dx_ln2, self.m2, P_DROP, dx=self.dx_d2),
            })
        # ops that run twice per step (both LNs / both dropouts): time one
        # instance and count it twice
        mult = {"layernorm_fwd": 2, "layernorm_bwd": 2, "dropout_fwd": 2, "dropout_bwd": 2,
                "dropout_add_layernorm_fwd": 2, "dropout_add_layernorm_bwd": 2}
        out = {}
        st = torch.cuda.current_stream()
        for name, fn in calls.items():
            fn()
            if reps == 0:
                continue
            res = []
            for fl in (flush, flush_dirty):
                if fl is None:
                    res.append(None)
                    continue
                ts = []
                for _ in range(reps):
                    fl()
                    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    a.record(st)
                    fn()
                    b.record(st)
                    b.synchronize()
                    ts.append(a.elapsed_time(b))
                res.append(trimmed_mean(ts) * mult.get(name, 1))
            out[name] = (res[0], mult.get(name, 1), res[1])
        return out


# ------------------------------------------------ configs[0..2] at their shapes
def per_config_timings(dev, peak, reps=40):
    """BASELINE configs[0..2], each op pair (forward + backward) at its own
    shape, captured in ONE CUDA graph (the launch-bound small case needs it)
    and replayed with L2 cold -- a 512 MB read before every replay evicts the
    inputs without leaving dirty lines for the timed op to write back -- and
    L2 warm (back-to-back replays).  GB/s = algorithmic bytes /
    device time (CUDA events on the capture/replay stream)."""
    import torch
    from paper_2210_10246_b200 import ops
    g = torch.Generator(device=dev)
    g.manual_seed(77)
    rn = lambda *s_: torch.randn(*s_, device=dev, generator=g)  # noqa: E731
    mw = lambda n: torch.empty(ops.mask_words(n), dtype=torch.int32, device=dev)  # noqa: E731
    table = ops.GeluTable.default()
    out = []

    # configs[0]: In-Place GELU fwd+bwd, BERT-base FFN activation [8*128, 3072]
    x1, dy1 = rn(1024, 3072), rn(1024, 3072)
    y1, m1, dx1 = torch.empty_like(x1), mw(x1.numel()), torch.empty_like(x1)
    n1 = x1.numel()

    def cfg1():
        ops.gelu_ip_fwd(x1, table, y=y1, mask=m1)
        ops.gelu_ip_bwd(dy1, y1, m1, table, dx=dx1)

    # configs[1]: In-Place LayerNorm fwd+bwd incl. dgamma/dbeta, [32*512, 768]
    R2, C2 = 32 * 512, 768
    x2, dy2 = rn(R2, C2), rn(R2, C2)
    ga2, be2 = (1 + 0.2 * rn(C2)).contiguous(), (0.1 * rn(C2)).contiguous()
    y2, rs2, dx2 = torch.empty_like(x2), torch.empty(R2, device=dev), torch.empty_like(x2)
    dg2, db2 = torch.empty(C2, device=dev), torch.empty(C2, device=dev)
    ws2 = torch.empty(max(16, int(ops.lib().tempo_ln_ip_bwd_workspace_size(R2, C2))),
                      dtype=torch.uint8, device=dev)

    def cfg2():
        ops.layernorm_ip_fwd(x2, ga2, be2, check_gamma=False, y=y2, rstd=rs2)
        ops.layernorm_ip_bwd(dy2, y2, rs2, ga2, be2, dx=dx2, dgamma=dg2, dbeta=db2, workspace=ws2)

    # configs[2]: softmax + dropout recompute (p=0.1) fwd, attn-probs bwd (+D for dV)
    R3 = 32 * 12 * 512
    z3, dD3 = rn(R3, 512), rn(R3, 512)
    P3, D3, m3 = torch.empty_like(z3), torch.empty_like(z3), mw(z3.numel())
    dZ3, Dr3 = torch.empty_like(z3), torch.empty_like(z3)
    n3 = z3.numel()

    def cfg3():
        ops.softmax_dropout_fwd(z3, P_DROP, mask=m3, generate=True, seed=5, P=P3, D=D3)
        ops.attn_probs_bwd(dD3, P3, m3, P_DROP, write_d=True, dZ=dZ3, D=Dr3)

    def copy_floor1():  # the same streams with no math: x -> y, (dy, y) -> dx
        y1.copy_(x1)
        torch.add(dy1, y1, out=dx1)

    bits = 1.0 / 8
    cases = [
        ("configs[0] gelu fwd+bwd [1024,3072]", cfg1, n1 * (8 + bits + 12 + bits), n1,
         n1 * 4 * 3),
        ("floor: torch copy + add of the configs[0] streams", copy_floor1, n1 * 20, n1,
         n1 * 4 * 3),
        ("configs[1] layernorm fwd+bwd [16384,768]", cfg2,
         (8 * R2 * C2 + 4 * R2 + 8 * C2) + (12 * R2 * C2 + 4 * R2 + 16 * C2), R2 * C2,
         R2 * C2 * 4 * 2),
        ("configs[2] softmax+dropout fwd, attn-probs bwd [196608,512]", cfg3,
         n3 * (12 + bits + 16 + bits), n3, n3 * 4 * 2),
    ]
    flush_buf = torch.empty(512 * 1024 * 1024 // 4, device=dev).fill_(1.0)
    flush_out = torch.empty((), device=dev)
    st_side = torch.cuda.Stream()
    for name, fn, nbytes, nelem, in_bytes in cases:
        fn()
        torch.cuda.synchronize()
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.stream(st_side):
            with torch.cuda.graph(graph, stream=st_side):
                fn()
        torch.cuda.synchronize()
        st = torch.cuda.current_stream()
        cold, warm = [], []
        for _ in range(reps):
            torch.sum(flush_buf, dim=0, out=flush_out)  # read-only eviction of L2
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(st)
            graph.replay()
            b.record(st)
            b.synchronize()
            cold.append(a.elapsed_time(b))
        graph.replay()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(st)
        for _ in range(reps):
            graph.replay()
        b.record(st)
        b.synchronize()
        warm_ms = a.elapsed_time(b) / reps
        cold_ms = trimmed_mean(cold)
        gbs = nbytes / (cold_ms * 1e-3) / 1e9
        out.append({"config": name, "ms": round(cold_ms, 4), "bytes": int(nbytes),
                    "gbs": round(gbs, 1), "frac": round(gbs / peak, 4),
                    "gelem_per_s": round(nelem / (cold_ms * 1e-3) / 1e9, 2),
                    "l2": "cold (512 MB read before each replay)", "launches": 2,
                    "cuda_graph": True,
                    "l2_warm": {"ms": round(warm_ms, 4),
                                "gbs": round(nbytes / (warm_ms * 1e-3) / 1e9, 1),
                                "note": ("inputs L2-resident (back-to-back replays)"
                                         if in_bytes < 100e6 else "working set > L2")}})
        del graph
    return out


# ------------------------------------- the recompute fused into its consumer
def row_length_timings(dev, peak, reps=10):
    """The row kernels across row lengths at a fixed element count (outside
    the timed region): softmax+dropout fwd / attn-probs bwd over S (2^27
    elements; S <= 1024 the warp-per-row kernels, longer rows the TMA
    row-group kernels) and LayerNorm fwd/bwd over H (2^25 elements; H > 2048
    backward on a thread-block cluster).  Each op alone, L2 cleaned by a 512 MB
    read before every rep, median device time, algorithmic bytes."""
    import statistics
    import torch
    from paper_2210_10246_b200 import ops
    fb = torch.empty(128 * 1024 * 1024, device=dev).fill_(1.0)
    sink = torch.empty((), device=dev)

    def timeit(fn):
        fn()
        ts = []
        for _ in range(reps):
            torch.sum(fb, dim=0, out=sink)
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            fn()
            b.record()
            b.synchronize()
            ts.append(a.elapsed_time(b))
        return statistics.median(ts)

    def frac(nbytes, ms):
        return round(nbytes / (ms * 1e-3) / 1e9 / peak, 4)

    out = {"softmax": [], "layernorm": []}
    g = torch.Generator(device=dev)
    g.manual_seed(3)
    for S in (512, 1024, 2048, 3072, 4096):
        rows = (1 << 27) // S
        n = rows * S
        z, dD = torch.randn(rows, S, device=dev, generator=g), torch.randn(rows, S, device=dev, generator=g)
        P, D, dZ = torch.empty_like(z), torch.empty_like(z), torch.empty_like(z)
        m = torch.empty(ops.mask_words(n), dtype=torch.int32, device=dev)
        tf = timeit(lambda: ops.softmax_dropout_fwd(z, P_DROP, mask=m, seed=1, P=P, D=D, generate=True))
        tb = timeit(lambda: ops.attn_probs_bwd(dD, P, m, P_DROP, dZ=dZ))
        out["softmax"].append({"S": S, "rows": rows, "fwd_ms": round(tf, 4),
                               "fwd_frac": frac(n * 12.125, tf), "bwd_ms": round(tb, 4),
                               "bwd_frac": frac(n * 12.125, tb)})
        del z, dD, P, D, dZ, m
    for H in (1024, 2048, 4096, 8192):
        rows = (1 << 25) // H
        n = rows * H
        x, dy = torch.randn(rows, H, device=dev, generator=g), torch.randn(rows, H, device=dev, generator=g)
        ga = (1 + 0.1 * torch.randn(H, device=dev, generator=g)).contiguous()
        be = (0.1 * torch.randn(H, device=dev, generator=g)).contiguous()
        y, dx, rs = torch.empty_like(x), torch.empty_like(x), torch.empty(rows, device=dev)
        dg, db = torch.empty(H, device=dev), torch.empty(H, device=dev)
        ws = torch.empty(max(16, int(ops.lib().tempo_ln_ip_bwd_workspace_size(rows, H))),
                         dtype=torch.uint8, device=dev)
        tf = timeit(lambda: ops.layernorm_ip_fwd(x, ga, be, check_gamma=False, y=y, rstd=rs))
        tb = timeit(lambda: ops.layernorm_ip_bwd(dy, y, rs, ga, be, dx=dx, dgamma=dg, dbeta=db,
                                                 workspace=ws))
        out["layernorm"].append({"H": H, "rows": rows, "fwd_ms": round(tf, 4),
                                 "fwd_frac": frac(n * 8, tf), "bwd_ms": round(tb, 4),
                                 "bwd_frac": frac(n * 12, tb)})
        del x, dy, y, dx
    return out


def _time_cases(torch, cases, peak, reps, flush):
    """Device time of each {name: (fn, algorithmic bytes)} case: CUDA events on
    the current stream, L2 read-flushed before each rep, trimmed mean."""
    st = torch.cuda.current_stream()
    out = {}
    for name, (fn, nbytes) in cases.items():
        fn()
        ts = []
        for _ in range(reps):
            if flush is not None:
                flush()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(st)
            fn()
            b.record(st)
            b.synchronize()
            ts.append(a.elapsed_time(b))
        t_ms = trimmed_mean(ts)
        gbs = nbytes / (t_ms * 1e-3) / 1e9
        out[name] = {"ms": round(t_ms, 4), "bytes": int(nbytes), "gbs": round(gbs, 1),
                     "frac": round(gbs / peak, 4)}
    return out


def dv_consumer_timings(chain, peak, reps=11, flush=None):
    """the attention-probability backward plus the
    consumer of the dropped-out map D, the dV GEMM (dV = D^T dO per head,
    d = 64), two ways at the configs[3] shape:
      unfused: attn_probs_bwd writes the recomputed D (16.125 B/elem), then
               an fp32 cuBLAS GEMM reads it back (TF32 off);
      fused:   attn_probs_bwd without D (12.125 B/elem), then
               tempo_attn_dropout_dv rebuilds D from P + mask inside its
               tcgen05 3xTF32 GEMM (4.125 B/elem + dO + dV).
    Device time per pair (CUDA events, L2 read-flushed before each rep)."""
    torch, o = chain.torch, chain.ops
    heads, dev = chain.batch * A, chain.dev
    g = torch.Generator(device=dev)
    g.manual_seed(99)
    dO = torch.randn(heads, S, 64, device=dev, generator=g)
    dV = torch.empty(heads, S, 64, device=dev)
    P3 = chain.P.view(heads, S, S)

    def unfused():
        o.attn_probs_bwd(chain.dD, chain.P, chain.m_att, P_DROP, write_d=True, dZ=chain.dZ,
                         D=chain.Drec)
        torch.matmul(chain.Drec.view(heads, S, S).transpose(1, 2), dO, out=dV)

    def fused():
        o.attn_probs_bwd(chain.dD, chain.P, chain.m_att, P_DROP, write_d=False, dZ=chain.dZ)
        o.attn_dropout_dv(P3, chain.m_att, P_DROP, dO, dV=dV)

    def gemm_only():
        o.attn_dropout_dv(P3, chain.m_att, P_DROP, dO, dV=dV)

    n_a = chain.P.numel()
    nb_o = dO.numel() * 4
    cases = {"unfused": (unfused, n_a * (16 + 1 / 8) + n_a * 4 + 2 * nb_o),
             "fused": (fused, n_a * (12 + 1 / 8) + n_a * (4 + 1 / 8) + 2 * nb_o),
             "dv_gemm_only": (gemm_only, n_a * (4 + 1 / 8) + 2 * nb_o)}
    prev = torch.backends.cuda.matmul.allow_tf32
    torch.backends.cuda.matmul.allow_tf32 = False
    try:
        out = _time_cases(torch, cases, peak, reps, flush)
    finally:
        torch.backends.cuda.matmul.allow_tf32 = prev
    out["speedup_fused_vs_unfused"] = round(out["unfused"]["ms"] / out["fused"]["ms"], 3)
    out["what"] = ("attn_probs_bwd + dV = D^T dO (d=64): D written + fp32 cuBLAS GEMM vs "
                   "D rebuilt inside the tcgen05 3xTF32 GEMM (tempo_attn_dropout_dv)")
    return out


def ctx_consumer_timings(chain, peak, reps=11, flush=None):
    """The forward side of the same fusion: softmax + dropout forward plus the
    consumer of D, ctx = D @ V per head (d = 64), at the configs[3] shape:
      unfused: softmax_dropout_fwd writes P and D (12.125 B/elem), then an
               fp32 cuBLAS GEMM reads D (TF32 off);
      fused:   softmax_dropout_fwd without D (8.125 B/elem), then
               tempo_attn_dropout_ctx rebuilds D from P + mask inside its
               tcgen05 3xTF32 GEMM (4.125 B/elem + V + ctx).
    The mask is regenerated (Philox, seed 7) by each forward, as in the
    bench step's breakdown."""
    torch, o = chain.torch, chain.ops
    heads, dev = chain.batch * A, chain.dev
    g = torch.Generator(device=dev)
    g.manual_seed(98)
    V = torch.randn(heads, S, 64, device=dev, generator=g)
    ctx = torch.empty(heads, S, 64, device=dev)
    P3 = chain.P.view(heads, S, S)

    def unfused():
        o.softmax_dropout_fwd(chain.z, P_DROP, mask=chain.m_att, generate=True, seed=7,
                              P=chain.P, D=chain.D)
        torch.matmul(chain.D.view(heads, S, S), V, out=ctx)

    def fused():
        o.softmax_dropout_fwd(chain.z, P_DROP, mask=chain.m_att, generate=True, seed=7,
                              P=chain.P, write_d=False)
        o.attn_dropout_ctx(P3, chain.m_att, P_DROP, V, ctx=ctx)

    def gemm_only():
        o.attn_dropout_ctx(P3, chain.m_att, P_DROP, V, ctx=ctx)

    n_a = chain.P.numel()
    nb_v = V.numel() * 4
    cases = {"unfused": (unfused, n_a * (12 + 1 / 8) + n_a * 4 + 2 * nb_v),
             "fused": (fused, n_a * (8 + 1 / 8) + n_a * (4 + 1 / 8) + 2 * nb_v),
             "ctx_gemm_only": (gemm_only, n_a * (4 + 1 / 8) + 2 * nb_v)}
    prev = torch.backends.cuda.matmul.allow_tf32
    torch.backends.cuda.matmul.allow_tf32 = False
    try:
        out = _time_cases(torch, cases, peak, reps, flush)
    finally:
        torch.backends.cuda.matmul.allow_tf32 = prev
    out["speedup_fused_vs_unfused"] = round(out["unfused"]["ms"] / out["fused"]["ms"], 3)
    out["what"] = ("softmax_dropout_fwd + ctx = D V (d=64): D written + fp32 cuBLAS GEMM vs "
                   "D rebuilt inside the tcgen05 3xTF32 GEMM (tempo_attn_dropout_ctx)")
    return out


# ------------------------------------------------------------ clocks
class ClockSampler:
    def __init__(self, index=0):
        self.index, self.proc, self.path = index, None, None

    def start(self):
        q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={q}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None

    def stop(self):
        if self.proc is None:
            return None
        self.proc.terminate()
        try:
            out, _ = self.proc.communicate(timeout=5)
        except Exception:
            self.proc.kill()
            out, _ = self.proc.communicate()
        sm, mx, reasons = [], 0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in out.strip().splitlines():
            f = [x.strip() for x in line.split(",")]
            if len(f) < 7:
                continue
            try:
                sm.append(int(f[0]))
                mx = max(mx, int(f[1]))
            except ValueError:
                continue
            for nm, v in zip(names, f[3:7]):
                if v.lower() == "active":
                    reasons.add(nm)
        if not sm:
            return None
        return {"sm_mhz": int(statistics.median(sm)), "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(sm)}


# ------------------------------------------------------ CPU reference arm
def cpu_model() -> str:
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def cpu_reference_sample(frac_rows: int, threads: int, steps: int, warmup: int, batch=B,
                         fused=False):
    """The reference's own CPU implementation (oracle/_ref/libtempo_ref.so,
    compiled from /root/reference/proj/src) of the same chain: 1/frac_rows of
    one rank's rows of every op (frac_rows = 1: the whole configs[3] step),
    sharded across `threads` host threads, each running the reference's own
    Graphs / Tape::backward on its rows (distinct tapes may run concurrently,
    SPEC.md:154).  Inputs and masks are built once per thread by the
    reference's own generators outside the timed region (ref_chain_create);
    a timed step copies nothing in or out.  Returns (GB/s, s/step, sample)."""
    import oracle
    ref = oracle.Ref()
    table = open(os.path.join(ROOT, "tests", "golden", "gelu_table_default_v1.txt")).read()
    t_rows = batch * S // frac_rows        # token rows of the sample
    a_rows = batch * A * S // frac_rows    # attention rows of the sample
    handles = [None] * threads

    def create(k):
        nt = (k + 1) * t_rows // threads - k * t_rows // threads
        na = (k + 1) * a_rows // threads - k * a_rows // threads
        handles[k] = ref.chain_create(table, P_DROP, na, S, nt, H, 1000 + k, with_residual=fused)

    def run_all(fn):
        ths = [threading.Thread(target=fn, args=(k,)) for k in range(threads)]
        for t in ths:
            t.start()
        for t in ths:
            t.join()

    run_all(create)
    try:
        run = lambda k: ref.chain_run(handles[k])  # noqa: E731
        for _ in range(warmup):
            run_all(run)
        t0 = time.perf_counter()
        for _ in range(steps):
            run_all(run)
        dt = (time.perf_counter() - t0) / steps
    finally:
        for h in handles:
            if h:
                ref.chain_destroy(h)
    nbytes = sum(op_bytes(batch, fused).values()) / frac_rows
    what = ("the whole per-GPU chain" if frac_rows == 1 else f"1/{frac_rows} of the per-GPU chain rows")
    sample = (f"{what} ({t_rows} tokens, {a_rows} attention rows; {nbytes / 1e9:.3f} GB "
              f"algorithmic) per step, {threads} threads, inputs built outside the timed region")
    return nbytes / dt / 1e9, dt, sample


def cpu_reference_configs(threads: int, reps: int = 2):
    """BASELINE configs[0..2] on the reference's own CPU implementation
    (oracle/_ref: ref_op_create / ref_op_run -- the reference's builders and
    Tape::backward) at their FULL shapes, rows sharded over `threads` host
    threads (one Graph per thread), inputs built outside the
    timed region: the CPU column beside per_config (SURVEY 8d "full shapes
    for cfg1-3").  Returns {config index: {ms, gbs, threads}}."""
    import oracle
    ref = oracle.Ref()
    table = open(os.path.join(ROOT, "tests", "golden", "gelu_table_default_v1.txt")).read()
    bits = 1.0 / 8
    cfgs = [(0, 1024, 3072, 8 + bits + 12 + bits),
            (1, 32 * 512, 768, 8 + 12),
            (2, 32 * 12 * 512, 512, 12 + bits + 16 + bits)]
    out = {}
    for kind, rows, cols, bpe in cfgs:
        handles = [None] * threads

        def create(k):
            r = (k + 1) * rows // threads - k * rows // threads
            handles[k] = ref.op_create(kind, table, P_DROP, r, cols, 500 + k) if r else None

        def run_all(fn):
            ths = [threading.Thread(target=fn, args=(k,)) for k in range(threads)]
            for t in ths:
                t.start()
            for t in ths:
                t.join()

        run_all(create)
        try:
            run = lambda k: handles[k] and ref.op_run(handles[k])  # noqa: E731
            run_all(run)  # warm-up
            t0 = time.perf_counter()
            for _ in range(reps):
                run_all(run)
            dt = (time.perf_counter() - t0) / reps
        finally:
            for h in handles:
                if h:
                    ref.op_destroy(h)
        out[kind] = {"ms": round(dt * 1e3, 2), "gbs": round(rows * cols * bpe / dt / 1e9, 3),
                     "threads": threads, "kind": "reference",
                     "what": "fwd + Tape::backward of the op pair at the config's full shape"}
    return out


def reference_frac(steps: int, warmup: int, budget_steps: int = 40) -> int:
    """Row fraction of the reference arm's step: the whole chain (1) while
    steps + warmup full steps (~2.5 s each on 16 host threads) fit the time
    budget, else the smallest power of two that brings them under it."""
    f = 1
    while (steps + warmup) / f > budget_steps and f < 512:
        f *= 2
    return f


# ---------------------------------------------------------------- main
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--masks", default="philox", choices=["philox", "reference"],
                    help="dropout masks: in-kernel Philox (default) or the reference's own "
                         "std::mt19937_64 streams generated on the device every step")
    ap.add_argument("--scaling", default=None, choices=["strong", "weak"],
                    help="N>1: strong (default; configs[4], --global-batch rows split N ways) "
                         "or weak (B=64 per rank)")
    ap.add_argument("--chain", default="fused", choices=["fused", "unfused"],
                    help="fused (default): hidden dropout -> residual add -> LayerNorm as one op "
                         "each way; unfused: separate dropout / LayerNorm ops, no residual add")
    ap.add_argument("--configs-only", action="store_true",
                    help="time only BASELINE configs[0..2] at their own shapes (for ncu)")
    ap.add_argument("--global-batch", type=int, default=GLOBAL_B_STRONG,
                    help="strong scaling: global batch split across the ranks (configs[4]: 512)")
    args = ap.parse_args()

    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return relaunch(args.gpus)  # one process per GPU, as the driver's torchrun would
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.gpus != world and rank == 0:
        print(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}; measuring {world} ranks",
              file=sys.stderr)
    scaling = args.scaling or ("strong" if world > 1 else "weak")
    if scaling == "strong" and world > 1:
        if args.global_batch % world:
            raise SystemExit(f"--global-batch {args.global_batch} does not split over {world} ranks")
        batch = args.global_batch // world
    else:
        batch = B

    if args.impl == "reference":
        return main_reference(args, rank, world)

    import torch
    import torch.distributed as dist
    # TEMPO_BENCH_BACKEND=gloo: a functional check of the N>1 path on fewer
    # GPUs than ranks (ranks share devices; the numbers are then meaningless)
    backend = os.environ.get("TEMPO_BENCH_BACKEND", "nccl")
    local_dev = local % max(1, torch.cuda.device_count()) if backend == "gloo" else local
    torch.cuda.set_device(local_dev)
    dev = torch.device("cuda", local_dev)
    if world > 1:
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group(backend)
    if args.configs_only:
        print(json.dumps({"per_config": per_config_timings(dev, peaks()[0], reps=args.steps)}))
        return
    fused = args.chain == "fused"
    chain = Chain(dev, rank, world, batch=batch, fused=fused)
    chain.mask_mode = args.masks
    from paper_2210_10246_b200.dist import allreduce_ln_params
    allreduce = allreduce_ln_params if world > 1 else None
    collective = None
    if world > 1:
        # the product path: the dgamma/dbeta sum fused into each LN backward's
        # stage 2 over peer memory (CUDA IPC mappings); NCCL all-reduce only
        # if the peer setup or its self-check fails
        chain.peer = setup_peer(chain, dist, rank, world, dev, backend)
        if chain.peer is not None:
            allreduce = None
        collective = ("fused peer-memory exchange in the LN backward stage 2"
                      if chain.peer is not None else f"{backend} all_reduce of the dgamma/dbeta bucket")
    flush_buf = torch.empty(512 * 1024 * 1024 // 4, device=dev).fill_(1.0)
    flush_out = torch.empty((), device=dev)
    flush = lambda: torch.sum(flush_buf, dim=0, out=flush_out)  # noqa: E731  (read 512 MB >> L2)
    flush_dirty = lambda: flush_buf[:256 * 1024 * 1024 // 4].fill_(0.0)  # noqa: E731

    for _ in range(max(args.warmup, 3)):
        chain.step(allreduce)
    torch.cuda.synchronize()
    if int(chain.status.item()) != 0:
        raise RuntimeError("layernorm gamma refused on device")

    # ---- timed region: K steps, barrier + sync on both sides -------------
    clocks = ClockSampler(local)
    clocks.start()
    time.sleep(0.15)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    st = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    for _ in range(args.steps):
        chain.step(allreduce)
        chain.poll_peer_status()  # a timed-out exchange fails the run at the next step
    e1.record(st)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    clk = clocks.stop()
    chain.poll_peer_status(final=True)
    ms = e0.elapsed_time(e1) / args.steps
    if world > 1:
        t = torch.tensor([ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())

    per_rank_bytes = sum(op_bytes(batch, fused).values())
    value = per_rank_bytes * world / (ms * 1e-3) / 1e9
    peak, peak_kind = peaks()

    # ---- per-op device times (outside the timed region) -------------------
    per_op = chain.per_op_timings(reps=11, flush=flush, flush_dirty=flush_dirty)
    ob, oe = op_bytes(batch, fused), op_elements(batch, fused)
    per_op_rows = []
    for name, (t_ms, mult, t_dirty) in per_op.items():
        gbs = ob[name] / (t_ms * 1e-3) / 1e9
        per_op_rows.append({"op": name, "ms": round(t_ms, 4), "bytes": int(ob[name]),
                            "gbs": round(gbs, 1), "frac": round(gbs / peak, 4),
                            "elements": int(oe[name]),
                            "gelem_per_s": round(oe[name] / (t_ms * 1e-3) / 1e9, 2),
                            "launches": mult, "l2": "cold, clean (512 MB read before each rep)",
                            "after_dirty_flush": {
                                "ms": round(t_dirty, 4),
                                "frac": round(ob[name] / (t_dirty * 1e-3) / 1e9 / peak, 4),
                                "l2": "256 MB written before each rep: the op also writes back "
                                      "~126 MB of foreign dirty lines"}})
    # the dominant kernel's duration inside the running chain: the timed
    # steps again with CUDA events around attn_probs_bwd on its stream (a
    # separate pass, so the events cannot perturb the headline region)
    chain.kernel_events = []
    for _ in range(args.steps):
        chain.step(allreduce)
    torch.cuda.synchronize()
    in_chain = [a.elapsed_time(b) for a, b in chain.kernel_events]
    chain.kernel_events = None
    k_ms = sum(in_chain) / len(in_chain)
    k_bytes = op_bytes(batch)["attn_probs_bwd"]
    k_gbs = k_bytes / (k_ms * 1e-3) / 1e9
    roofline = {"bound": "hbm", "kernel": "attn_probs_bwd", "achieved": round(k_gbs, 1),
                "peak": peak, "unit": "GB/s", "frac": round(k_gbs / peak, 4), "traffic": None,
                "peak_kind": f"{peak_kind} copy bandwidth (MEASURED_PEAKS.json hbm_gbs)",
                "bytes_per_launch": int(k_bytes), "ms_per_launch": round(k_ms, 4),
                "timing": f"CUDA events around the kernel in each of {len(in_chain)} chain steps",
                "share_of_step": round(k_ms / ms, 4),
                "isolated": {"ms": next(r["ms"] for r in per_op_rows if r["op"] == "attn_probs_bwd"),
                             "frac": next(r["frac"] for r in per_op_rows if r["op"] == "attn_probs_bwd")},
                "per_unit": "16.125 B/element: dD, P (4+4) + mask bit + dZ, D (4+4); SURVEY 8d",
                # also against the 8 TB/s HBM3e specification
                "frac_of_hbm_spec": round(k_gbs / 8000.0, 4)}
    prof_traffic = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(prof_traffic) and batch == B:  # captured at the configs[3] shapes
        try:
            tr = json.load(open(prof_traffic)).get("attn_probs_bwd")
            if tr:
                roofline["traffic"] = tr
        except Exception:
            pass

    # ---- configs[0..2] at their own shapes (outside the timed region) -------
    per_config = per_config_timings(dev, peak) if rank == 0 else None
    if per_config and world == 1 and not args.no_cpu_baseline:
        try:  # the reference's CPU path beside each config
            cpu_cfg = cpu_reference_configs(len(os.sched_getaffinity(0)))
            for c in per_config:
                for i in range(3):
                    if c["config"].startswith(f"configs[{i}]"):
                        c["cpu_reference"] = cpu_cfg[i]
                        c["gpu_vs_cpu_reference"] = round(c["ms"] and cpu_cfg[i]["ms"] / c["ms"], 1)
        except Exception as ex:  # noqa: BLE001  (report, do not fail the bench)
            per_config.append({"cpu_reference": f"unavailable: {str(ex)[:160]}"})
    per_row_length = None
    if rank == 0:
        try:
            per_row_length = row_length_timings(dev, peak)
        except Exception as ex:  # noqa: BLE001  (report, do not fail the bench)
            per_row_length = {"unavailable": str(ex)[:200]}
    # ---- the dropout recompute fused into the dV GEMM ----
    dv_consumer = None
    if rank == 0:
        try:
            dv_consumer = dv_consumer_timings(chain, peak, flush=flush)
        except Exception as ex:  # noqa: BLE001  (report, do not fail the bench)
            dv_consumer = {"unavailable": str(ex)[:200]}
    ctx_consumer = None
    if rank == 0:
        try:
            ctx_consumer = ctx_consumer_timings(chain, peak, flush=flush)
        except Exception as ex:  # noqa: BLE001  (report, do not fail the bench)
            ctx_consumer = {"unavailable": str(ex)[:200]}

    # ---- the reference mask stream on the device (outside the timed region) --
    ref_mask = None
    if rank == 0:
        n_att = chain.ATT_ROWS * S
        chain.ops.bernoulli_keep_bits_device(n_att, P_DROP, 7, out=chain.m_att)  # tables + warm-up
        ts = []
        for _ in range(3):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(st)
            chain.ops.bernoulli_keep_bits_device(n_att, P_DROP, 8, out=chain.m_att)
            b.record(st)
            b.synchronize()
            ts.append(a.elapsed_time(b))
        t_ms = min(ts)
        ref_mask = {"what": "BoolMask::bernoulli_keep stream (std::mt19937_64) of the attention "
                            "mask, bit-exact, device jump-ahead", "elements": n_att,
                    "ms": round(t_ms, 3), "gelem_per_s": round(n_att / t_ms / 1e6, 1)}

    # ---- the same chain through the C++ operator API (Graph/Tape) ---------
    cpp_api = None
    exe = os.path.join(ROOT, "paper_2210_10246_b200", "_lib", "bench_graph")
    if rank == 0 and world == 1 and os.path.exists(exe):
        try:
            r = subprocess.run([exe, "20", "3"], capture_output=True, text=True, timeout=300)
            cpp_api = json.loads(r.stdout.strip().splitlines()[-1])
            # the same with Tape::backward(..., synchronize = false)
            r = subprocess.run([exe, "20", "3", "async"], capture_output=True, text=True,
                               timeout=300)
            cpp_api["async_backward"] = json.loads(r.stdout.strip().splitlines()[-1])
        except Exception as ex:
            cpp_api = {"unavailable": str(ex)[:200]}

    # ---- e2e: the public API with host buffers -----------------------------
    e2e = None
    if not args.no_e2e:
        if world > 1:
            dist.barrier()  # rank 0's extra measurements above: realign before the exchanges
        e2e = e2e_measure(chain, args, world, allreduce, dist if world > 1 else None)
    if chain.peer is not None:
        torch.cuda.synchronize()
        chain.peer.check_status()  # no exchange may have timed out (results would be partial)

    # ---- CPU baseline (reference library on host cores, rank 0, N=1) -------
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            threads = len(os.sched_getaffinity(0))
            v, dt, sample = cpu_reference_sample(frac_rows=1, threads=threads, steps=2, warmup=1,
                                                 fused=fused)
            v1, dt1, _ = cpu_reference_sample(frac_rows=512, threads=1, steps=1, warmup=0,
                                              fused=fused)
            cpu = {"value": round(v, 4), "unit": "GB/s", "cores": threads, "kind": "reference",
                   "sample": sample, "s_per_step": round(dt, 3), "cpu_model": cpu_model(),
                   "one_thread": {"value": round(v1, 4), "unit": "GB/s",
                                  "sample": "1/512 of the per-GPU chain rows, 1 thread"}}
        except Exception as ex:  # the reference library is prebuilt here; report if absent
            cpu = {"value": None, "unit": "GB/s", "cores": 0, "kind": "reference",
                   "sample": f"unavailable: {ex}"}

    if rank == 0:
        line = {
            "metric": METRIC, "value": round(value, 2), "unit": "GB/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms, 4),
            "higher_is_better": True, "scaling": scaling, "vs_baseline": None, "dtype": "f32",
            "data": ("synthetic (torch.randn inputs of the layer shapes; " +
                     ("Philox dropout masks)" if args.masks == "philox" else
                      "the reference's mt19937_64 dropout masks, generated on the device "
                      "every step)")),
            "config": {"workload": WORKLOAD, "batch_per_gpu": batch, "global_batch": batch * world,
                       "seq_len": S, "hidden": H, "heads": A, "dropout_p": P_DROP,
                       "parallelism": f"rows{world}", "collective": collective,
                       "chain": ("fused: hidden dropout -> residual add -> LayerNorm as one op "
                                 "each way (tempo_dropout_add_ln_fwd/bwd)" if fused else
                                 "unfused: separate dropout and LayerNorm ops, no residual add"),
                       "bytes_per_step_per_gpu": int(per_rank_bytes),
                       "l2": f"working set {per_rank_bytes / 1e9:.1f} GB/step per GPU >> 126 MB L2",
                       "baseline_config": ("configs[3] (B=64, one GPU)" if world == 1 else
                                           f"configs[4]: global B={batch * world} row-sharded "
                                           f"over {world} GPUs" if scaling == "strong" else
                                           f"weak: B={batch} per GPU")},
            "roofline": roofline,
            "cpu_baseline": cpu,
            "e2e": e2e,
            "gpu_launches": ((Chain.LAUNCHES_PER_STEP_FUSED if fused else Chain.LAUNCHES_PER_STEP) +
                             (Chain.REF_MASK_LAUNCHES if args.masks == "reference" else 0)) * args.steps,
            "mask_stream": args.masks,
            "reference_mask_generation": ref_mask,
            "cpp_api": cpp_api,
            "clocks": clk,
            "per_op": per_op_rows,
            "per_config": per_config,
            "per_row_length": per_row_length,
            "dv_consumer": dv_consumer,
            "ctx_consumer": ctx_consumer,
            "frac_of_peak": round(value / world / peak, 4),
            "unfused_equivalent": ({
                "what": "the same step's work as separate ops incl. the residual adds "
                        "(dropout 8.125 + add 12 + LN 8 B/elem fwd, LN 12 + dropout 8.125 bwd)",
                "bytes_per_step_per_gpu": int(unfused_equivalent_bytes(batch)),
                "gbs": round(unfused_equivalent_bytes(batch) * world / (ms * 1e-3) / 1e9, 2)}
                if fused else None),
            "elements_per_s": {"value": round(sum(op_elements(batch, fused).values()) * world / (ms * 1e-3) / 1e9, 2),
                               "unit": "Gelem/s", "what": "elements streamed by all ops of the chain"},
            "stash": stash_report(chain),
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def free_port() -> int:
    import socket
    s_ = socket.socket()
    s_.bind(("127.0.0.1", 0))
    p = s_.getsockname()[1]
    s_.close()
    return p


def relaunch(n):
    """`bench.py --gpus N` outside torchrun: re-run this command as N ranks
    (torch.distributed.run, one process per GPU, rendezvous on 127.0.0.1);
    rank 0 prints the JSON line."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={n}", "--master-addr=127.0.0.1", f"--master-port={free_port()}",
           os.path.abspath(__file__)] + sys.argv[1:]
    r = subprocess.run(cmd)
    sys.exit(r.returncode)


def stash_report(chain):
    from paper_2210_10246_b200 import ops
    ref_tok = ops.layer_stash_bytes_per_token(S, H, A, tempo=False, mask_bits=False)
    tmp1_tok = ops.layer_stash_bytes_per_token(S, H, A, tempo=True, mask_bits=False)
    ours_tok = ops.layer_stash_bytes_per_token(S, H, A, tempo=True, mask_bits=True)
    # in-path retained buffers, measured from the device allocations
    measured = chain.retained_bytes()
    # what the reference keeps for the SAME ops (memory_model.cpp:31-65): scores,
    # probs, dropped-out map + 1-byte mask; both LN inputs + outputs; GELU input
    # + output; 1-byte hidden dropout masks
    T, ATT_ROWS = chain.T, chain.ATT_ROWS
    ref_same = (3 * 4 + 1) * ATT_ROWS * S + 4 * (4 * T * H) + 2 * 4 * T * 4 * H + 2 * T * H
    return {"unit": "bytes/layer", "tokens": T,
            "reference_layer": ref_tok * T, "tempo_1byte_masks_layer": tmp1_tok * T,
            "tempo_b200_layer": ours_tok * T,
            "in_path_retained_measured": measured, "in_path_reference": ref_same,
            "saving_vs_reference": round(1 - ours_tok / ref_tok, 4)}


def e2e_measure(chain, args, world, allreduce, dist):
    """Same metric through the public API with HOST buffers: every step
    copies its inputs from pinned host memory (H2D) and reads every result
    back (D2H) inside the timed region.  Inputs and results each live in ONE
    contiguous pinned host buffer and ONE contiguous device buffer per set
    (Chain.bind views), so a step is one H2D and one D2H copy; both are
    double-buffered (set 0 = the chain's own buffers, set 1 one extra pair):
    step i+1's inputs upload while step i computes and step i-1's results
    download, so the step costs about the PCIe time of its copies (full
    duplex) rather than their sum plus compute."""
    torch = chain.torch
    n_in, n_out = chain.in_buf.numel(), chain.out_buf.numel()
    d_in = [chain.in_buf, torch.empty(n_in, device=chain.dev)]
    d_out = [chain.out_buf, torch.empty(n_out, device=chain.dev)]
    h_in = torch.empty(n_in, dtype=torch.float32, pin_memory=True)
    h_in.copy_(chain.in_buf)
    h_out = [torch.empty(n_out, dtype=torch.float32, pin_memory=True) for _ in range(2)]
    bi, bo = n_in * 4, n_out * 4
    comp = torch.cuda.current_stream()
    s_in, s_out = torch.cuda.Stream(), torch.cuda.Stream()
    ev_in = [torch.cuda.Event(), torch.cuda.Event()]    # input set j uploaded
    ev_used = [torch.cuda.Event(), torch.cuda.Event()]  # input set j consumed by compute
    ev_done = [torch.cuda.Event(), torch.cuda.Event()]  # output set j computed
    ev_out = [torch.cuda.Event(), torch.cuda.Event()]   # output set j downloaded
    for j in range(2):
        ev_used[j].record(comp)
        ev_out[j].record(s_out)

    def upload(j):
        with torch.cuda.stream(s_in):
            s_in.wait_event(ev_used[j])
            d_in[j].copy_(h_in, non_blocking=True)
            ev_in[j].record(s_in)

    def step(i, upload_next=True):
        j = i % 2
        comp.wait_event(ev_in[j])
        comp.wait_event(ev_out[j])  # results of step i-2 (same output set) downloaded
        chain.bind(d_in[j], d_out[j])
        chain.step(allreduce)
        ev_used[j].record(comp)
        ev_done[j].record(comp)
        if upload_next:
            upload(1 - j)  # next step's inputs, overlapped
        with torch.cuda.stream(s_out):
            s_out.wait_event(ev_done[j])
            h_out[j].copy_(d_out[j], non_blocking=True)
            ev_out[j].record(s_out)

    k = max(1, min(args.steps, 20))  # steady state: the one undrained D2H amortised over k
    upload(0)
    step(0, upload_next=False)  # warm-up
    torch.cuda.synchronize()
    if dist is not None:
        dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(comp)
    s_in.wait_event(e0)
    upload(1)                   # step 1's inputs: inside the timed region
    for i in range(1, k + 1):
        step(i, upload_next=i < k)
    for j in range(2):
        comp.wait_event(ev_out[j])
    e1.record(comp)
    torch.cuda.synchronize()
    chain.bind(chain.in_buf, chain.out_buf)  # back to the chain's own buffers
    del d_in, d_out
    ms = e0.elapsed_time(e1) / k
    if dist is not None:
        t = torch.tensor([ms], device=chain.dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    v = sum(op_bytes(chain.batch, chain.fused).values()) * world / (ms * 1e-3) / 1e9
    return {"value": round(v, 2), "unit": "GB/s", "h2d_bytes_per_step": int(bi),
            "d2h_bytes_per_step": int(bo), "ms_per_step": round(ms, 3), "steps": k,
            "overlap": "one H2D (step i+1) || compute (step i) || one D2H (step i-1); "
                       "inputs and results double-buffered"}


def main_reference(args, rank, world):
    """--impl reference: the reference's own CPU implementation of the path
    (oracle/_ref, compiled from /root/reference/proj/src) on the host cores,
    same metric/config/unit.  Each step is the whole per-GPU chain when
    steps + warmup full steps fit a few minutes (reference_frac), else a
    stated row fraction.  Under torchrun only rank 0 runs."""
    if rank != 0:
        return
    scaling = args.scaling or ("strong" if world > 1 else "weak")
    batch = args.global_batch // world if (scaling == "strong" and world > 1) else B
    threads = len(os.sched_getaffinity(0))
    frac = reference_frac(args.steps, args.warmup)
    fused = args.chain == "fused"
    v, dt, sample = cpu_reference_sample(frac_rows=frac, threads=threads, steps=args.steps,
                                         warmup=args.warmup, batch=batch, fused=fused)
    line = {
        "metric": METRIC, "value": round(v, 4), "unit": "GB/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(dt * 1e3, 2),
        "higher_is_better": True, "scaling": scaling, "vs_baseline": None, "dtype": "f32",
        "data": "synthetic (the reference's Tensor::randn inputs, BoolMask::bernoulli_keep masks)",
        "impl": "reference", "same_config": frac == 1,
        "config": {"workload": WORKLOAD, "batch_per_gpu": batch, "global_batch": batch * world,
                   "seq_len": S, "hidden": H, "heads": A, "dropout_p": P_DROP,
                   "parallelism": f"rows{world}",
                   "chain": ("hidden dropout -> residual add (Graph::add) -> LayerNorm, as the "
                             "reference layer composes them" if fused else
                             "dropout and LayerNorm, no residual add"),
                   "sample_rows": f"1/{frac} of one GPU's rows" if frac > 1 else "all of one GPU's rows"},
        "cpu_baseline": {"value": round(v, 4), "unit": "GB/s", "cores": threads,
                         "kind": "reference", "sample": sample, "cpu_model": cpu_model()},
        "e2e": {"value": round(v, 4), "unit": "GB/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
