"""The composed top layer (sc_trainer::fuse_top, the tensor-core default): the last layer's update
and the head are both linear (nn.hpp:233-234, 240: no activation after the update), so the trainer
computes logits = mean Z_L^T + h Z_R^T with Z = head U_{L-1}, and in backward Xp = G^T [mean | h],
dHead = Xp U^T, dU_{L-1} = head^T Xp, dmean = inv (G Z_L), dh = G Z_R + dz W (nn.hpp:259-290
re-associated). Same mathematics as the reference's order; the rounding differs at the level of one
fp32 GEMM. Checked here against the unfused tensor-core path (SC_FUSE_TOP=0) on one step with the
same inputs (teacher-forced), and over free-running steps; test_gpu_parity checks the default
(fused) path against the oracle / the reference's goldens."""
import os

import numpy as np
import pytest

from cpu_libs import oracle
from test_gpu_parity import gpu_graph

pytestmark = pytest.mark.gpu


def rel(a, b):
    return float(np.linalg.norm(np.asarray(a, np.float64) - b) / max(np.linalg.norm(np.asarray(b, np.float64)), 1e-30))


def trainer(sc, og, hidden, fuse, pta="1", dropedge=True, compact="0"):
    env = {"SC_FUSE_TOP": "1" if fuse else "0", "SC_PTA": pta, "SC_COMPACT_ACTS": compact}
    old = {k: os.environ.get(k) for k in env}
    os.environ.update(env)
    try:
        g = gpu_graph(sc, og, 24)
        part = sc.partition_random(g, 4, 3)
        return sc.CoFreeTrainer(g, part, sc.TrainConfig(layers=len(hidden), hidden=hidden, use_dropedge=dropedge,
                                                        seed=1, learning_rate=1e-2))
    finally:
        for k, v in old.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v


# pta = "1": with 2 Cp <= H (here C = 6 -> Cp = 8) the top layer also aggregates projected rows
# (logits = h Z_R^T + A_norm (msg Z_L^T); backward Ghat = A^T (inv G), Xp = [Ghat^T msg | G^T h],
# dz = 1[msg > 0] (Ghat Z_L)); compact = "1": the ReLU decisions come from sign bits
@pytest.mark.parametrize("hidden,pta,compact", [([32], "1", "0"), ([64, 64], "1", "0"), ([48, 48, 48], "1", "0"),
                                                ([64, 64], "0", "0"), ([64, 64], "1", "1")])
def test_composed_top_layer_matches_unfused(hidden, pta, compact):
    from paper_2308_03209_b200 import sagecut as sc
    og = oracle().graph_sbm(400, 6, 0.1, 0.01, 24, 0.3, 7)
    a = trainer(sc, og, hidden, True, pta, compact=compact)
    b = trainer(sc, og, hidden, False)
    la, lb = a.step(0), b.step(0)
    assert abs(la[0] - lb[0]) <= 1e-6 * abs(lb[0])
    for i in range(4):
        assert rel(a.part_logits(i), b.part_logits(i)) <= 2e-6
        assert rel(a.part_grads(i), b.part_grads(i)) <= 1e-5
    assert rel(a.grads(), b.grads()) <= 1e-5
    # free-running: same trajectory within the fp32 parity bar
    for e in range(1, 5):
        la, lb = a.step(e), b.step(e)
        assert abs(la[0] - lb[0]) <= 1e-5 * abs(lb[0])
    assert rel(a.params(), b.params()) <= 1e-4


def test_composed_top_layer_evaluate():
    """Full-graph evaluation runs the same composed forward (trainer_evaluate)."""
    from paper_2308_03209_b200 import sagecut as sc
    og = oracle().graph_sbm(400, 6, 0.1, 0.01, 24, 0.3, 7)
    a = trainer(sc, og, [32, 32], True)
    b = trainer(sc, og, [32, 32], False)
    b.set_params(a.params())
    ea, eb = a.evaluate(), b.evaluate()
    assert ea == eb  # argmax accuracy: identical unless a logit tie is decided by 1 ulp
