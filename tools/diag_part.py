"""Localise a per-partition gradient discrepancy (GPU vs oracle) to matrix rows/cols.

    python tools/diag_part.py [dropedge 0|1] [gemm]
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]
from cpu_libs import oracle  # noqa: E402
from paper_2308_03209_b200 import sagecut as sc  # noqa: E402

de = bool(int(sys.argv[1])) if len(sys.argv) > 1 else True
gemm = sys.argv[2] if len(sys.argv) > 2 else "simt"
C, n, m = 47, 20000, 200000
O = oracle()
rng = np.random.default_rng(C)
og = O.graph_build(n, rng.integers(0, n, size=(m, 2), dtype=np.int32))
lab = rng.integers(0, C, size=n).astype(np.int32)
f = rng.standard_normal((n, 100)).astype(np.float32)
f[np.arange(n), lab % 100] += 1.0
perm = rng.permutation(n)
tr, va, te = (np.zeros(n, np.uint8) for _ in range(3))
tr[perm[:n * 6 // 10]], va[perm[n * 6 // 10:n * 8 // 10]], te[perm[n * 8 // 10:]] = 1, 1, 1
og.set_data(f, lab, C, tr, va, te)
g, _ = sc.build_graph(n, og.edges())
g.set_data(og.features(100).astype(np.float32), lab, C, tr, va, te)
gp = sc.partition_random(g, 4, 1)
op = og.partition("random", 4, 1)
H = [64, 64]
t = sc.CoFreeTrainer(g, gp, sc.TrainConfig(layers=2, hidden=H, learning_rate=0.01, use_dropedge=de, seed=3, gemm=gemm))
to = op.trainer(H, lr=0.01, dropedge=de, seed=3, f32=True)
t.step(0)
to.step(0)
shapes = [("W0", 64, 100), ("U0", 64, 164), ("W1", 64, 64), ("U1", 64, 128), ("head", C, 64)]
for i in range(4):
    a, b = t.part_grads(i).astype(np.float64), to.part_grads(i)
    k = 0
    msg = []
    for nm, r, c in shapes:
        x, y = a[k:k + r * c].reshape(r, c), b[k:k + r * c].reshape(r, c)
        k += r * c
        d = np.abs(x - y)
        rows = d.sum(1)
        top = np.argsort(-rows)[:3]
        msg.append(f"{nm}: rel {np.linalg.norm(x - y) / np.linalg.norm(y):.1e} top rows {list(top)} "
                   f"({[f'{rows[j] / max(np.abs(y[j]).sum(), 1e-30):.1e}' for j in top]})")
    print(f"part {i} (mask {t.part_mask(i)} vs {to.part_mask(i)}):\n   " + "\n   ".join(msg))
