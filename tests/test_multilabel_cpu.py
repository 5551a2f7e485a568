"""Multi-label path and the reference's analytic helpers on CPU: the oracle
restatement and the product library's host-only entry points against golden
vectors from the real reference (tests/golden/make_golden_multilabel.py).

* bce against Graph::multilabels (nn.hpp:348-378, graph.cpp:91-98) over a
  5-step DropEdge trajectory, micro-F1 evaluation (trainer.cpp:72-87), the
  reference's single-split evaluate (trainer.cpp:101-112);
* comm_volume (trainer.cpp:38-49), expected_rf_random / imbalance_lower_bound
  (partition.cpp:344-362), TrainResult::audit.
"""
import ctypes as C

import numpy as np
import pytest

from cpu_libs import oracle


@pytest.fixture(scope="module")
def O():
    return oracle()


def sbm_multilabel(O, Y):
    og = O.graph_sbm(200, 4, 0.15, 0.01, 8, 0.3, 7)
    og.set_multilabels(Y)
    return og


def test_oracle_multilabel_trajectory(O, golden):
    z = golden("multilabel")
    og = sbm_multilabel(O, z["Y"])
    part = og.partition("random", 8, 3)
    t = part.trainer([16, 16], lr=0.01, loss="bce", dropedge=True, seed=1, f32=True)
    np.testing.assert_array_equal(t.params(), z["traj_init"])
    for e in range(5):
        loss, gn = t.step(e)
        assert abs(loss - z["traj_loss"][e]) <= 1e-12 * abs(z["traj_loss"][e])
        assert abs(gn - z["traj_gnorm"][e]) <= 1e-12 * abs(z["traj_gnorm"][e])
        np.testing.assert_allclose(t.params(), z["traj_params"][e], rtol=1e-12, atol=0)
        np.testing.assert_allclose(t.gathered(), z["traj_grads"][e], rtol=1e-10, atol=1e-14)
    # micro-F1 of the final model on each split (evaluate_splits, trainer.hpp:132-140)
    np.testing.assert_array_equal(np.array(t.eval()), z["traj_eval"])


def test_oracle_evaluate(O, golden):
    z = golden("multilabel")
    og = sbm_multilabel(O, z["Y"])
    theta = z["traj_params"][-1]
    for name, m in zip(("train", "val", "test"), og.masks()):
        assert og.evaluate(theta, [16, 16], m) == float(z[f"eval_model_{name}"])
    gm = O.graph_sbm(200, 4, 0.15, 0.01, 8, 0.3, 7)
    for name, m in zip(("train", "val", "test"), gm.masks()):
        assert gm.evaluate(z["mc_init"], [16, 16], m) == float(z[f"mc_eval_{name}"])
    with pytest.raises(ValueError, match="evaluate: empty mask"):
        gm.evaluate(z["mc_init"], [16, 16], np.zeros(200, np.uint8))


def test_oracle_softmax_rejects_multilabel(O, golden):
    og = sbm_multilabel(O, golden("multilabel")["Y"])
    part = og.partition("random", 2, 3)
    with pytest.raises(ValueError, match="softmax_ce requires multi-class labels"):
        part.trainer([4], loss="softmax_ce")


def test_analytic_helpers_oracle_and_library(O, golden):
    z = golden("multilabel")
    from paper_2308_03209_b200 import sagecut as sc  # host-only entry points: no GPU needed
    for args, out in zip(z["comm_args"], z["comm_out"]):
        mode = "cofree" if args[0] == 0 else "halo_sync_model"
        a = [int(x) for x in args[1:]]
        assert O.comm_volume(mode, *a) == [int(x) for x in out]
        r = sc.comm_volume(mode, *a)
        assert [r.floats_per_iteration, r.gradient_floats, r.embedding_floats] == [int(x) for x in out]
    for (p, d), out in zip(z["erf_args"], z["erf_out"]):
        assert O.expected_rf_random(int(p), int(d)) == out
        assert sc.expected_rf_random(int(p), int(d)) == out
    for (p, mx, mn), out in zip(z["ilb_args"], z["ilb_out"]):
        assert O.imbalance_lower_bound(int(p), int(mx), int(mn)) == out
        assert sc.imbalance_lower_bound(int(p), int(mx), int(mn)) == out
    # the reference's error cases (test_partition.cpp:285, trainer.cpp:40)
    for f in (lambda m: m.imbalance_lower_bound(2, 3, 0), lambda m: m.expected_rf_random(0, 3),
              lambda m: m.comm_volume("cofree", 0, 10, 1, 1, 0)):
        with pytest.raises(ValueError):
            f(O)
        with pytest.raises(ValueError):
            f(sc)
    assert z["audit"].tolist() == [8 * int(z["audit_params"])] * 3 + [0]
