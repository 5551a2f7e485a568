"""The oracle restatement (oracle/liboracle.so) against golden vectors dumped
from the real reference (tests/golden/make_golden.py, oracle/_ref).

Bit-exact for every integer / RNG / index output; the f32/f64 training
trajectories agree to the last ulp on these sizes, checked at 1e-12 relative.
"""
import hashlib

import numpy as np
import pytest

from cpu_libs import oracle


@pytest.fixture(scope="module")
def O():
    return oracle()


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def test_rng_known_answers(O, golden):
    g = golden("rng")
    tags = [str(t) for t in g["tags"]]
    assert [O.substream(0, t) for t in tags] == [int(x) for x in g["substream0"]]
    assert [O.substream(7, t) for t in tags] == [int(x) for x in g["substream_seed7"]]
    assert [O.substream(1, "dropedge", i) for i in range(8)] == [int(x) for x in g["substream_1idx"]]
    assert [[O.substream(1, "dropedge.select", i, e) for e in range(6)] for i in range(8)] == \
        g["substream_2idx"].astype(object).tolist()
    assert [O.mix64(int(x)) for x in g["mix64_in"]] == [int(x) for x in g["mix64_out"]]
    np.testing.assert_array_equal(O.rng_draws(12345, 0, 64), g["u64_seed12345"])
    for n in (2, 3, 7, 8, 10, 1000003, 2**33 + 5):
        np.testing.assert_array_equal(O.rng_draws(99, 1, 256, n), g[f"below_{n}"])
    np.testing.assert_array_equal(O.rng_draws(3, 2, 64), g["double_seed3"])
    np.testing.assert_array_equal(O.rng_draws(31, 3, 64), g["gauss_seed31"])
    # SURVEY Appendix A probe: substream(0,"init") and its first next_double
    assert O.substream(0, "init") == 0x99FBAF5308475366
    assert O.rng_draws(0x99FBAF5308475366, 2, 1)[0] == 0.40312434338362879


def _check_partition(gr, part, g, prefix, full):
    np.testing.assert_array_equal(part.assignment(), g[prefix + "assign"])
    st = part.stats()
    np.testing.assert_array_equal(st["per_node_rf"], g[prefix + "per_node_rf"])
    np.testing.assert_array_equal(
        np.array([st["rf"], st["edge_balance"], st["node_balance"], st["duplicated_nodes"]]), g[prefix + "stats"])
    for s in ("dar", "vanilla_inv", "none"):
        np.testing.assert_array_equal(np.concatenate(part.weights(s)), g[prefix + "w_" + s])
    if full:
        for i in range(part.p):
            a = part.part(i)
            for f in ("nodes", "edges", "edge_gids", "local_deg", "offsets", "nbrs", "eids", "g2l"):
                np.testing.assert_array_equal(getattr(a, f), g[f"{prefix}p{i}_{f}"], err_msg=f"part {i} {f}")


def test_karate(O, golden):
    g = golden("karate")
    gr = O.graph_build(int(g["n"]), g["edges"])
    np.testing.assert_array_equal(gr.edges(), g["edges"])
    for a, name in zip(gr.csr(), ("offsets", "nbrs", "eids", "degrees")):
        np.testing.assert_array_equal(a, g[name])
    for p in (1, 2, 4, 8):
        _check_partition(gr, gr.partition("random", p, 0), g, f"random_p{p}_", True)
    _check_partition(gr, gr.partition("dbh", 4, 0), g, "dbh_p4_", True)
    pk = gr.partition("random", 4, 0)
    e0 = pk.sizes(0)[1]
    np.testing.assert_array_equal(O.precompute_masks(e0, 3, 0.5, O.substream(0, "dropedge", 0)), g["masks_p0_k3"])
    # karate random p=8 seed 0, rf 3.235294, dup 76
    assert g["random_p8_assign"][:16].tolist() == [3, 3, 5, 3, 3, 7, 4, 0, 2, 6, 6, 2, 3, 5, 4, 1]
    assert "".join(map(str, g["masks_p0_k3"][0])) == "110000111011100010001110"


@pytest.fixture(scope="module")
def sbm(O):
    return O.graph_sbm(200, 4, 0.15, 0.01, 8, 0.3, 7)


def test_sbm200_graph(sbm, golden):
    g = golden("sbm200")
    np.testing.assert_array_equal(sbm.edges(), g["edges"])
    np.testing.assert_array_equal(sbm.features(8), g["features"])
    np.testing.assert_array_equal(sbm.labels(), g["labels"])
    for a, name in zip(sbm.masks(), ("train", "val", "test")):
        np.testing.assert_array_equal(a, g[name])


@pytest.mark.parametrize("algo", ["random", "dbh"])
@pytest.mark.parametrize("p", [1, 2, 4, 8])
def test_sbm200_partitions(sbm, golden, algo, p):
    _check_partition(sbm, sbm.partition(algo, p, 3), golden("sbm200"), f"{algo}_p{p}_", algo == "random" and p == 8)


def test_sbm200_masks_select_init(O, sbm, golden):
    g = golden("sbm200")
    part = sbm.partition("random", 8, 3)
    for i in range(8):
        np.testing.assert_array_equal(O.precompute_masks(part.sizes(i)[1], 10, 0.5, O.substream(1, "dropedge", i)),
                                      g[f"masks_p{i}"])
    np.testing.assert_array_equal(O.precompute_masks(100, 10, 0.5, 3), g["masks_100_10_05_3"])
    assert [[O.select_mask(1, i, e, 10) for e in range(20)] for i in range(8)] == g["select_seed1"].tolist()
    np.testing.assert_array_equal(O.init_params(8, [16, 16], 4, 1, f32=False), g["init_8_16_16_4_seed1_f64"])
    np.testing.assert_array_equal(O.init_params(8, [16, 16], 4, 1, f32=True), g["init_8_16_16_4_seed1_f32"])


def _check_traj(part, g, prefix, classes, **cfg):
    t = part.trainer(**cfg)
    np.testing.assert_array_equal(t.params(), g[prefix + "init"])
    for e in range(5):
        loss, gn = t.step(e)
        np.testing.assert_allclose(loss, g[prefix + "loss"][e], rtol=1e-12)
        np.testing.assert_allclose(gn, g[prefix + "gnorm"][e], rtol=1e-12)
        assert [t.part_mask(i) for i in range(part.p)] == g[prefix + "masks"][e].tolist()
        np.testing.assert_allclose(t.gathered(), g[prefix + "grads"][e], rtol=1e-12, atol=1e-15)
        np.testing.assert_allclose(t.params(), g[prefix + "params"][e], rtol=1e-12, atol=1e-15)
        if prefix + "logits" in g:
            lg = np.concatenate([t.part_logits(i, classes).reshape(-1) for i in range(part.p)])
            np.testing.assert_allclose(lg, g[prefix + "logits"][e], rtol=1e-12, atol=1e-14)
    np.testing.assert_allclose(t.eval(), g[prefix + "eval"], rtol=0, atol=0)


@pytest.mark.parametrize("prec", ["f32", "f64"])
@pytest.mark.parametrize("de", ["plain", "de"])
def test_sbm200_trajectories(sbm, golden, prec, de):
    part = sbm.partition("random", 8, 3)
    _check_traj(part, golden("sbm200"), f"traj_{prec}_{de}_", 4, hidden=[16, 16], lr=0.01, dropedge=(de == "de"),
                seed=1, f32=(prec == "f32"))


def test_sbm200_bce_vanilla_dbh(sbm, golden):
    g = golden("sbm200")
    part = sbm.partition("random", 8, 3)
    _check_traj(part, g, "traj_f32_bce_", 4, hidden=[16, 16], lr=0.01, loss="bce", seed=1, f32=True)
    _check_traj(part, g, "traj_f32_vanilla_", 4, hidden=[16, 16], lr=0.01, reweight="vanilla_inv", seed=1, f32=True)
    _check_traj(sbm.partition("dbh", 4, 3), g, "traj_f32_dbh4_", 4, hidden=[16, 16, 16], lr=0.02, dropedge=True, k=4,
                ratio=0.3, seed=5, f32=True)


def test_er10k_config0(O, golden):
    """configs[0]: ER 10k / 200k, 64 feats, 2 x 32, 4 vertex-cut partitions."""
    g = golden("er10k")
    ge = O.graph_sbm(10000, 4, 0.004, 0.004, 64, 1.0, 0)
    assert ge.m == int(g["m"])
    assert sha(ge.edges()) == str(g["edges_sha"])
    assert sha(ge.features(64)) == str(g["features_sha"])
    pe = ge.partition("random", 4, 0)
    assert sha(pe.assignment()) == str(g["assign_sha"])
    st = pe.stats()
    np.testing.assert_array_equal(
        np.array([st["rf"], st["edge_balance"], st["node_balance"], st["duplicated_nodes"]]), g["stats"])
    assert sha(st["per_node_rf"]) == str(g["per_node_rf_sha"])
    np.testing.assert_allclose([w.sum() for w in pe.weights("dar")], g["w_dar_sum"], rtol=1e-15)
    for i in range(4):
        a = pe.part(i)
        assert [len(a.nodes), len(a.edges)] == g[f"p{i}_sizes"].tolist()
        assert sha(np.concatenate([a.offsets, a.nbrs, a.eids])) == str(g[f"p{i}_csr_sha"])
        assert sha(O.precompute_masks(len(a.edges), 10, 0.5, O.substream(0, "dropedge", i))) == str(g[f"p{i}_mask_sha"])
    _check_traj(pe, g, "traj_", 4, hidden=[32, 32], lr=0.01, dropedge=True, seed=0, f32=True)


def test_input_validation(O):
    with pytest.raises(ValueError):
        O.precompute_masks(10, 0, 0.5, 1)
    with pytest.raises(ValueError):
        O.precompute_masks(10, 3, 1.0, 1)
    gr = O.graph_build(3, np.array([[0, 1], [1, 2]], np.int32))
    with pytest.raises(ValueError):
        gr.build_vertex_cut(2, np.array([0, 2], np.int32))
    with pytest.raises(ValueError):
        gr.partition("random", 0, 1)
