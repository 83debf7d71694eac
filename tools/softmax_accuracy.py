import sys, numpy as np, torch
sys.path.insert(0, '.')
import oracle
from paper_2210_10246_b200 import ops
port = oracle.Port()
g = np.random.default_rng(0)
for scale in (1, 4, 16):
    z = (g.standard_normal((4096, 512)) * scale).astype(np.float32)
    P, D, m = ops.softmax_dropout_fwd(torch.from_numpy(z).cuda(), 0.1, seed=3)
    rP = port.softmax_fwd(z)
    Pg = P.cpu().numpy()
    rel = np.abs(Pg - rP) / np.maximum(np.abs(rP), 1e-30)
    big = rP > 1e-30
    print(scale, "max rel err P", float(rel[big].max()), "max abs", float(np.abs(Pg - rP).max()))
