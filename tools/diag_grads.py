"""Per-matrix gradient error of the CUDA path vs the oracle (diagnostics for tolerance failures).

    python tools/diag_grads.py C [gemm] [n] [m]
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]
from cpu_libs import oracle  # noqa: E402
from paper_2308_03209_b200 import sagecut as sc  # noqa: E402

C = int(sys.argv[1])
gemm = sys.argv[2] if len(sys.argv) > 2 else "auto"
n = int(sys.argv[3]) if len(sys.argv) > 3 else 3000
m = int(sys.argv[4]) if len(sys.argv) > 4 else 10 * n
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
t = sc.CoFreeTrainer(g, gp, sc.TrainConfig(layers=2, hidden=H, learning_rate=0.01, use_dropedge=True, seed=3,
                                           gemm=gemm))
to = op.trainer(H, lr=0.01, dropedge=True, seed=3, f32=True)
names, sizes, inp = [], [], 100
for l, h in enumerate(H):
    names += [f"W{l}", f"U{l}"]
    sizes += [h * inp, h * (h + inp)]
    inp = h
names.append("head")
sizes.append(C * inp)
for e in range(3):
    t.step(e)
    to.step(e)
    lg = np.concatenate([t.part_logits(i).ravel() for i in range(4)])
    olg = np.concatenate([to.part_logits(i, C).ravel() for i in range(4)])
    print(f"  logits rel {np.linalg.norm(lg - olg) / np.linalg.norm(olg):.2e}  params rel "
          f"{np.linalg.norm(t.params() - to.params()) / np.linalg.norm(to.params()):.2e}")
    a, b = t.grads().astype(np.float64), to.gathered()
    k = 0
    row = []
    for nm, sz in zip(names, sizes):
        x, y = a[k:k + sz], b[k:k + sz]
        row.append(f"{nm}:{np.linalg.norm(x - y) / np.linalg.norm(y):.1e}(|{np.linalg.norm(y):.1e}|)")
        k += sz
    tot = np.linalg.norm(a - b) / np.linalg.norm(b)
    parts = [np.linalg.norm(t.part_grads(i) - to.part_grads(i)) / np.linalg.norm(to.part_grads(i)) for i in range(4)]
    print(f"C={C} {gemm} step {e}: total {tot:.2e} parts {[f'{p:.1e}' for p in parts]} ", " ".join(row))
