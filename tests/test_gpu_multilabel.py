"""Multi-label training and evaluation through the CUDA path (C ABI) against
the oracle and the reference's goldens (tests/golden/make_golden_multilabel.py).

bce against Graph::multilabels (nn.hpp:348-378; graph.cpp:91-98 label_targets),
micro-F1 evaluate_splits (trainer.cpp:72-87), the single-split evaluate of the
trainer's model and of a given model (trainer.cpp:101-112), the comm audit
(trainer.hpp:61-76) and the no-silent-fallback counter. Same bar as
test_gpu_parity.py: logits / gradients / parameters <= 1e-4 relative, loss
<= 1e-5 over 5 free-running steps.
"""
import numpy as np
import pytest

from cpu_libs import oracle
from test_gpu_parity import REL, gpu_graph, rel

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def sc():
    from paper_2308_03209_b200 import sagecut
    return sagecut


@pytest.fixture(scope="module")
def O():
    return oracle()


def ml_graphs(sc, O, Y):
    og = O.graph_sbm(200, 4, 0.15, 0.01, 8, 0.3, 7)
    g = gpu_graph(sc, og, 8)
    og.set_multilabels(Y)
    g.set_multilabels(Y)
    return og, g


@pytest.mark.parametrize("gemm", ["auto", "simt"])
def test_multilabel_trajectory(sc, O, golden, gemm):
    z = golden("multilabel")
    og, g = ml_graphs(sc, O, z["Y"])
    gp = sc.partition_random(g, 8, 3)
    op = og.partition("random", 8, 3)
    cfg = sc.TrainConfig(layers=2, hidden=[16, 16], learning_rate=0.01, loss="bce", use_dropedge=True, seed=1,
                         gemm=gemm)
    t = sc.CoFreeTrainer(g, gp, cfg)
    to = op.trainer([16, 16], lr=0.01, loss="bce", dropedge=True, seed=1, f32=True)
    for e in range(5):
        loss, gn = t.step(e)
        ol, _ = to.step(e)
        assert abs(loss - ol) <= 1e-5 * abs(ol)
        assert abs(loss - z["traj_loss"][e]) <= 1e-5 * abs(z["traj_loss"][e])
        lg = np.concatenate([t.part_logits(i).ravel() for i in range(8)])
        olg = np.concatenate([to.part_logits(i, 5).ravel() for i in range(8)])
        assert rel(lg, olg) <= REL
        assert rel(t.grads(), to.gathered()) <= REL
        assert rel(t.grads(), z["traj_grads"][e]) <= REL
        assert rel(t.params(), z["traj_params"][e]) <= REL
    # micro-F1 per split: the reference's numbers up to a prediction flipping on a
    # logit within fp32 noise of 0 (one flip moves F1 by < 0.01 at these sizes)
    np.testing.assert_allclose(t.evaluate(), z["traj_eval"], atol=0.01)
    tr, va, te = og.masks()
    for name, m in (("train", tr), ("val", va), ("test", te)):
        assert abs(t.evaluate_mask(m) - float(z[f"eval_model_{name}"])) <= 0.01
    assert t.comm_audit() == (8 * t.param_count, 0)
    if gemm == "auto":
        # layer 0's dU ([mean | h_in]: the 16 mean columns are not a multiple of the 32-column TMA box)
        # runs on the SIMT kernel, counted: 8 partitions x 5 steps. The top layer is composed with the
        # head (trainer.hpp fuse_top / pta): its products Ghat^T msg and G^T h have one B source each
        # and run on the tensor cores.
        assert t.fallback_count() == 1 * 8 * 5


def test_multilabel_errors(sc, O, golden):
    z = golden("multilabel")
    og, g = ml_graphs(sc, O, z["Y"])
    gp = sc.partition_random(g, 2, 3)
    with pytest.raises(ValueError, match="softmax_ce requires multi-class labels"):
        sc.CoFreeTrainer(g, gp, sc.TrainConfig(layers=1, hidden=[4], loss="softmax_ce"))
    bad = z["Y"].copy()
    bad[3, 2] = 0.5
    with pytest.raises(ValueError, match="bce targets must be 0 or 1"):
        g.set_multilabels(bad)


@pytest.mark.parametrize("p", [1, 8])
def test_evaluate_given_model(sc, O, golden, p):
    """evaluate(model, g, mask) (trainer.cpp:101-112) on the multi-class graph: the
    standalone forward-only engine and a trainer's evaluate_mask (p = 1 reuses the
    training activations, p = 8 runs on the forward-only buffers) agree with the
    reference's f64 evaluate."""
    z = golden("multilabel")
    og = O.graph_sbm(200, 4, 0.15, 0.01, 8, 0.3, 7)
    g = gpu_graph(sc, og, 8)
    init = z["mc_init"].astype(np.float32)
    masks = og.masks()
    gp = sc.partition_random(g, p, 3)
    t = sc.CoFreeTrainer(g, gp, sc.TrainConfig(layers=2, hidden=[16, 16], seed=1))
    np.testing.assert_array_equal(t.params(), init)
    for name, m in zip(("train", "val", "test"), masks):
        ref = float(z[f"mc_eval_{name}"])
        assert abs(sc.evaluate(init, g, m, [16, 16]) - ref) <= 0.01
        assert abs(t.evaluate_mask(m) - ref) <= 0.01
    with pytest.raises(ValueError, match="evaluate: empty mask"):
        sc.evaluate(init, g, np.zeros(200, np.uint8), [16, 16])
