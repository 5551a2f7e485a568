"""Memory modes for large graphs (R-MAT 20M / 1B at p = 16): the per-partition x0 row cache and
logits buffers replaced by shared buffers (SC_SHARED_X0 / SC_SHARED_LOGITS, chosen automatically
when they would exceed their budget). Same arithmetic: parameters bitwise equal to the cached mode."""
import os

import numpy as np
import pytest

from cpu_libs import oracle
from test_gpu_parity import gpu_graph

pytestmark = pytest.mark.gpu


def run(sc, og, env):
    old = {k: os.environ.get(k) for k in env}
    os.environ.update(env)
    try:
        g = gpu_graph(sc, og, 8)
        part = sc.partition_random(g, 6, 3)
        t = sc.CoFreeTrainer(g, part, sc.TrainConfig(layers=2, hidden=[16, 16], use_dropedge=True, seed=1))
        losses = [t.step(e)[0] for e in range(3)]
        return t, losses
    finally:
        for k, v in old.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v


def test_shared_buffers_same_bits():
    from paper_2308_03209_b200 import sagecut as sc
    og = oracle().graph_sbm(200, 4, 0.15, 0.01, 8, 0.3, 7)
    a, la = run(sc, og, {"SC_SHARED_X0": "0", "SC_SHARED_LOGITS": "0"})
    b, lb = run(sc, og, {"SC_SHARED_X0": "1", "SC_SHARED_LOGITS": "1"})
    assert la == lb
    np.testing.assert_array_equal(a.params(), b.params())
    np.testing.assert_array_equal(a.part_logits(5), b.part_logits(5))  # the last trained partition
    with pytest.raises(ValueError, match="not kept"):
        b.part_logits(0)


@pytest.mark.parametrize("hidden", [[64, 64, 64], [40, 40]])
def test_compact_activations_same_bits(hidden):
    """Compact activations (SC_COMPACT_ACTS=1, chosen automatically when the per-layer set would
    not fit, e.g. R-MAT 20M / 1B at p = 16): one msg buffer shared by the layers and the ReLU
    decisions kept as sign bits for the transposed aggregation. The decision bit is the same
    comparison the msg row gives, so every step, gradient and eval metric is bitwise the same."""
    from paper_2308_03209_b200 import sagecut as sc
    og = oracle().graph_sbm(300, 4, 0.15, 0.01, 8, 0.3, 7)
    out = []
    for compact in ("0", "1"):
        old = os.environ.get("SC_COMPACT_ACTS")
        os.environ["SC_COMPACT_ACTS"] = compact
        try:
            g = gpu_graph(sc, og, 8)
            part = sc.partition_random(g, 4, 3)
            t = sc.CoFreeTrainer(g, part, sc.TrainConfig(layers=len(hidden), hidden=hidden, use_dropedge=True,
                                                         seed=1))
            steps = [t.step(e) for e in range(3)]
            out.append((steps, t.params(), t.grads(), t.evaluate()))
        finally:
            if old is None:
                os.environ.pop("SC_COMPACT_ACTS", None)
            else:
                os.environ["SC_COMPACT_ACTS"] = old
    (sa, pa, ga, ea), (sb, pb, gb, eb) = out
    assert sa == sb
    np.testing.assert_array_equal(pa, pb)
    np.testing.assert_array_equal(ga, gb)
    assert ea == eb


def test_tn_dual_launch_matches_two_launches():
    """SC_TN_DUAL=1 (opt-in): a layer's dU and dW in one split-K launch over A = [dh | dz]. Same
    products, different split-K partition of the rows, so gradients agree to fp32 rounding."""
    from paper_2308_03209_b200 import sagecut as sc
    og = oracle().graph_sbm(300, 4, 0.15, 0.01, 8, 0.3, 7)
    out = []
    for dual in ("0", "1"):
        old = os.environ.get("SC_TN_DUAL")
        os.environ["SC_TN_DUAL"] = dual
        try:
            # TcGemm reads SC_TN_DUAL when the trainer is created
            g = gpu_graph(sc, og, 8)
            part = sc.partition_random(g, 2, 3)
            t = sc.CoFreeTrainer(g, part, sc.TrainConfig(layers=2, hidden=[256, 256], use_dropedge=True, seed=1))
            t.step(0)
            out.append(t.grads())
        finally:
            if old is None:
                os.environ.pop("SC_TN_DUAL", None)
            else:
                os.environ["SC_TN_DUAL"] = old
    a, b = out
    assert np.linalg.norm(a - b) <= 2e-6 * np.linalg.norm(a)
