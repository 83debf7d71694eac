"""Generate the golden fixtures in tests/golden/ from the REFERENCE itself.

Runs the unmodified reference library (oracle/_ref/libtempo_ref.so, built by
``make -C oracle`` from /root/reference/proj/src) through its own operator
builders and Tape::backward, on seeded inputs, and stores inputs + outputs.
Only needed where /root/reference exists; the committed fixtures travel.

    python tests/golden/make_golden.py
"""
from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

import oracle  # noqa: E402


def special_x() -> np.ndarray:
    xs = [0.0, -0.0, 1.0, -1.0, -2.0, 2.0, 8.0, -8.0, 13.0, -13.0, -13.5, -20.0, 30.0,
          -0.75179152469399924, -0.7517915, -0.7517916, -0.751791537, -0.751791477,
          1e-30, -1e-30, 1e-45, -1e-45, 3.4e38, -3.4e38, float("inf"), float("-inf")]
    x32 = np.array(xs, np.float32)
    # dense walk across the minimum window and the tail threshold
    near = np.linspace(-0.80, -0.70, 257, dtype=np.float32)
    tail = np.linspace(-14.0, -12.0, 65, dtype=np.float32)
    return np.concatenate([x32, near, tail])


def main() -> None:
    ref = oracle.Ref()
    table = ref.fit_table_default()
    with open(os.path.join(HERE, "gelu_table_default_v1.txt"), "w") as f:
        f.write(table)

    # tables fitted with other options (more segments / other degrees), for the
    # generic device paths (gelu_fit.hpp:32-46)
    import json
    extra = {}
    for tol, deg in [(1e-5, 13), (1e-6, 13), (1e-4, 4), (3e-6, 8)]:
        extra[f"tol{tol:g}_deg{deg}"] = ref.fit_table(tol, deg)
    with open(os.path.join(HERE, "gelu_tables_extra.json"), "w") as f:
        json.dump(extra, f, indent=1)

    g = np.random.default_rng(20221019)
    out = {}

    # ---- GELU: forward + backward through Tape::backward -------------------
    x = np.concatenate([special_x(), g.standard_normal(4096).astype(np.float32) * 2.0])
    dy = g.standard_normal(x.size).astype(np.float32)
    y, m, dx = ref.gelu_ip(table, x, dy)
    out.update(gelu_x=x, gelu_dy=dy, gelu_y=y, gelu_mask=m, gelu_dx=dx)
    # table.eval at chosen outputs (gelu_table.cpp:172-188)
    ys = np.concatenate([np.linspace(-0.2, 9.0, 2001), [0.0, -0.16997120747990366, -1.0,
                                                         8.0, 1e300, -0.5]])
    for mm in (0, 1):
        out[f"eval_y_m{mm}"] = ys
        out[f"eval_h_m{mm}"] = ref.table_eval(table, ys, np.full(ys.size, mm, np.uint8))

    # ---- LayerNorm (F32 path, and the F64 path for dgamma/dbeta) -----------
    rows, cols = 12, 768
    lx = (g.standard_normal((rows, cols)) * 1.5 + 0.3).astype(np.float32)
    gam = (np.sign(g.standard_normal(cols)) * (1 + 0.2 * g.standard_normal(cols))).astype(np.float32)
    bet = (0.1 * g.standard_normal(cols)).astype(np.float32)
    ldy = g.standard_normal((rows, cols)).astype(np.float32)
    ly, lrs, ldx, ldg, ldb = ref.layernorm_ip(lx, gam, bet, ldy)
    ldx64, ldg64, ldb64 = ref.layernorm_ip_bwd(ldy, ly, lrs, gam, bet, f64=True)
    out.update(ln_x=lx, ln_gamma=gam, ln_beta=bet, ln_dy=ldy, ln_y=ly, ln_rstd=lrs, ln_dx=ldx,
               ln_dgamma=ldg, ln_dbeta=ldb, ln_dgamma_f64=ldg64, ln_dbeta_f64=ldb64)
    # frozen row of test_ops_reference.cpp:35-49
    fy, frs, _, _, _ = ref.layernorm_ip(np.array([[1.0, 3.0]], np.float32),
                                        np.ones(2, np.float32), np.zeros(2, np.float32))
    out.update(ln_frozen_y=fy, ln_frozen_rstd=frs)

    # ---- softmax + dropout_recompute + backward ------------------------------
    srows, scols, p = 24, 512, 0.1
    z = (g.standard_normal((srows, scols)) * 3.0).astype(np.float32)
    keep = ref.bernoulli_keep(srows * scols, p, 7).reshape(srows, scols)
    dD = g.standard_normal((srows, scols)).astype(np.float32)
    P, D, dZ, Dr = ref.softmax_dropout(z, keep, p, dD)
    out.update(sm_z=z, sm_keep=keep, sm_dD=dD, sm_P=P, sm_D=D, sm_dZ=dZ, sm_Drec=Dr, sm_p=p)

    # ---- hidden dropout ------------------------------------------------------
    hx = g.standard_normal(1000).astype(np.float32)
    hk = ref.bernoulli_keep(1000, 0.1, 11)
    hdy = g.standard_normal(1000).astype(np.float32)
    hy, hdx = ref.dropout(hx, hk, 0.1, hdy)
    out.update(do_x=hx, do_keep=hk, do_dy=hdy, do_y=hy, do_dx=hdx)

    # ---- masks / seeds / memory model -----------------------------------------
    out["keep_n1000_p01_s42"] = ref.bernoulli_keep(1000, 0.1, 42)
    out["keep_n777_p05_s19"] = ref.bernoulli_keep(777, 0.5, 19)
    out["stream_seeds"] = np.array([ref.mask_stream_seed(s, salt, site)
                                    for s in (0, 1, 12345) for salt in (0, 1, 7)
                                    for site in (0, 1, 2)], np.uint64)
    mm = []
    for (b, s, h, a) in [(1, 128, 768, 12), (1, 512, 768, 12), (1, 2048, 768, 12),
                         (64, 512, 1024, 16)]:
        r, o, sv = ref.memory_model(b, s, h, a)
        mm.append([s, h, a, r, o] + sv)
    out["memory_model"] = np.array(mm, np.int64)

    np.savez_compressed(os.path.join(HERE, "golden.npz"), **out)
    print("wrote", os.path.join(HERE, "golden.npz"), sorted(out))


if __name__ == "__main__":
    main()
