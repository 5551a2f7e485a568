"""The fp64 torch checker (tests/torch_ref.py) pinned to the oracle restatement's
f64 mode (itself pinned to the reference's goldens) on sbm200 partitions, so it
can stand in for the oracle at the headline shapes (tests/test_gpu_scale_parity.py)."""
import numpy as np
import pytest

from cpu_libs import oracle
from torch_ref import partition_step


@pytest.mark.parametrize("loss,de", [("softmax_ce", True), ("softmax_ce", False), ("bce", True)])
def test_torch_ref_matches_oracle_f64(loss, de):
    O = oracle()
    og = O.graph_sbm(200, 4, 0.15, 0.01, 8, 0.3, 7)
    part = og.partition("random", 4, 3)
    t = part.trainer([16, 12], lr=0.01, loss=loss, dropedge=de, seed=1, f32=False)
    theta = t.params()
    t.step(0)
    feats = og.features(8)
    labels = og.labels()
    tr = og.masks()[0]
    w_all = part.weights("dar")
    normalizer = float(tr.sum())
    for i in range(4):
        a = part.part(i)
        mask = None
        if de:
            k = t.part_mask(i)
            mask = O.precompute_masks(len(a.edges), 10, 0.5, O.substream(1, "dropedge", i))[k]
        w = np.where(tr[a.nodes] != 0, w_all[i], 0.0)
        targets = np.eye(4)[labels[a.nodes]] if loss == "bce" else None
        r = partition_step(theta, 8, [16, 12], 4, a.offsets, a.nbrs, a.eids, mask, feats[a.nodes], w, normalizer,
                           labels=labels[a.nodes], targets=targets, loss=loss)
        np.testing.assert_allclose(r["logits"].numpy(), t.part_logits(i, 4), rtol=1e-12, atol=1e-12)
        assert abs(r["loss"] - t.part_loss(i)) <= 1e-12 * abs(t.part_loss(i))
        g = t.part_grads(i)
        assert np.linalg.norm(r["grads"] - g) <= 1e-12 * np.linalg.norm(g)
