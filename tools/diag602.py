import os, sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]
from paper_2308_03209_b200 import sagecut as sc
from cpu_libs import oracle
rng = np.random.default_rng(0)
def rel(a, b):
    return float(np.linalg.norm(np.asarray(a, np.float64) - b) / np.linalg.norm(b))
M = 5000
for K in (100, 600, 602, 604):
    A = np.zeros((M, (K + 3) // 4 * 4), np.float32)
    A[:, :K] = rng.standard_normal((M, K))
    B = rng.standard_normal((32, K)).astype(np.float32)
    ref = A[:, :K].astype(np.float64) @ B.T.astype(np.float64)
    print("NT K", K, "tc", rel(sc.debug_gemm(A, B), ref), "simt", rel(sc.debug_gemm(A, B, simt=True), ref))
    A2 = rng.standard_normal((M, 32)).astype(np.float32)
    B2 = rng.standard_normal((32, 32)).astype(np.float32)
    ref2 = A2.astype(np.float64) @ B2.T + ref
    print("  dual", rel(sc.debug_gemm(A2, B2, A2=A, B2=B), ref2))
    C1 = sc.debug_gemm_tn(A2, A2, A[:, :K].copy() if K % 4 else A)
    r1 = A2.T.astype(np.float64) @ np.concatenate([A2, A[:, :K]], 1).astype(np.float64)
    print("  tn", rel(C1[:, :32 + K], r1) if C1.shape[1] >= 32 + K else "shape", C1.shape)
O = oracle()
d = 602
n = 2000
og = O.graph_build(n, rng.integers(0, n, size=(16000, 2), dtype=np.int32))
lab = rng.integers(0, 5, size=n).astype(np.int32)
f = rng.standard_normal((n, d)).astype(np.float32)
f[np.arange(n), lab] += 1.0
tr = (rng.random(n) < 0.6).astype(np.uint8); va = ((1 - tr) * (rng.random(n) < 0.5)).astype(np.uint8); te = (1 - tr - va).astype(np.uint8)
og.set_data(f, lab, 5, tr, va, te)
for gm in ("simt", "auto"):
    g, _ = sc.build_graph(n, og.edges())
    g.set_data(og.features(d).astype(np.float32), lab, 5, tr, va, te)
    t = sc.CoFreeTrainer(g, sc.partition_random(g, 4, 1), sc.TrainConfig(layers=2, hidden=[32, 32], use_dropedge=True, seed=2, gemm=gm))
    to = og.partition("random", 4, 1).trainer([32, 32], lr=0.01, dropedge=True, seed=2, f32=True)
    for e in range(2):
        l, _ = t.step(e); ol, _ = to.step(e)
        lg = np.concatenate([t.part_logits(i).ravel() for i in range(4)]); olg = np.concatenate([to.part_logits(i, 5).ravel() for i in range(4)])
        print(gm, e, "loss", abs(l - ol) / ol, "logits", rel(lg, olg), "grads", rel(t.grads(), to.gathered()))
