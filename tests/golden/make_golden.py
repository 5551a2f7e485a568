"""Generate the golden fixtures under tests/golden/ from the REAL reference.

Run here (the reference tree only exists in this container):

    make -C oracle && python tests/golden/make_golden.py

Every value is produced by oracle/_ref/libsagecut_ref.so, i.e. the unmodified
reference sources (/root/reference/proj/src + header-only nn.hpp/trainer.hpp)
compiled behind oracle/eigen_shim. The shim itself is validated by running the
reference's own unit suites against it (`make -C oracle ref-tests`: 98/98 pass).

Fixtures:
  rng.npz      substream / draw / next_below / next_gaussian known answers
  karate.npz   karate club (proj/tests/fixtures/karate.edges via load_graph):
               canonical edges, random/dbh assignments, per-part CSR, stats,
               DAR weights, masks (the survey's Appendix A probe values)
  sbm200.npz   SbmSpec{200,4,0.15,0.01,8,0.3,7} (proj/tests/support.hpp:33-37):
               graph + data, partitions, weights, masks, selections, init, and
               5-step train_cofree trajectories (f32 / f64, DropEdge on/off, CE/BCE)
  er10k.npz    configs[0]: ER 10k nodes / ~200k edges, 64 feats, 4 classes,
               2 x 32, p=4 random vertex cut; 5-step trajectories
"""
from __future__ import annotations

import hashlib
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
# Goldens use the shim's plain loop GEMM (k-ascending sums, no BLAS blocking) so
# the oracle restatement can be pinned to them at ~1 ulp.
os.environ["SAGECUT_REF_NO_BLAS"] = "1"
sys.path.insert(0, os.path.dirname(HERE))
from cpu_libs import reference  # noqa: E402

KARATE = "/root/reference/proj/tests/fixtures/karate.edges"


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def rng_fixture(R):
    out = {}
    tags = ["init", "partition.random", "dropedge", "dropedge.mask", "dropedge.select", "split", "sbm.edges"]
    out["tags"] = np.array(tags)
    out["substream0"] = np.array([R.substream(0, t) for t in tags], np.uint64)
    out["substream_seed7"] = np.array([R.substream(7, t) for t in tags], np.uint64)
    out["substream_1idx"] = np.array([R.substream(1, "dropedge", i) for i in range(8)], np.uint64)
    out["substream_2idx"] = np.array([[R.substream(1, "dropedge.select", i, e) for e in range(6)] for i in range(8)],
                                     np.uint64)
    out["mix64_in"] = np.array([0, 1, 2, 0xDEADBEEF, 2**63, 2**64 - 1], np.uint64)
    out["mix64_out"] = np.array([R.mix64(int(x)) for x in out["mix64_in"]], np.uint64)
    out["u64_seed12345"] = R.rng_draws(12345, 0, 64)
    for n in (2, 3, 7, 8, 10, 1000003, 2**33 + 5):
        out[f"below_{n}"] = R.rng_draws(99, 1, 256, n)
    out["double_seed3"] = R.rng_draws(3, 2, 64)
    out["gauss_seed31"] = R.rng_draws(31, 3, 64)
    return out


def graph_arrays(g, prefix, d=None):
    out = {f"{prefix}n": np.int64(g.n), f"{prefix}edges": g.edges()}
    off, nb, ei, dg = g.csr()
    out.update({f"{prefix}offsets": off, f"{prefix}nbrs": nb, f"{prefix}eids": ei, f"{prefix}degrees": dg})
    if d:
        out[f"{prefix}features"] = g.features(d)
        out[f"{prefix}labels"] = g.labels()
        tr, va, te = g.masks()
        out.update({f"{prefix}train": tr, f"{prefix}val": va, f"{prefix}test": te})
    return out


def partition_arrays(part, prefix, full=True):
    out = {f"{prefix}assign": part.assignment()}
    st = part.stats()
    out[f"{prefix}per_node_rf"] = st["per_node_rf"]
    out[f"{prefix}stats"] = np.array([st["rf"], st["edge_balance"], st["node_balance"], st["duplicated_nodes"]])
    for s in ("dar", "vanilla_inv", "none"):
        out[f"{prefix}w_{s}"] = np.concatenate(part.weights(s))
    if full:
        for i in range(part.p):
            a = part.part(i)
            for f in ("nodes", "edges", "edge_gids", "local_deg", "offsets", "nbrs", "eids", "g2l"):
                out[f"{prefix}p{i}_{f}"] = getattr(a, f)
    return out


def trajectory(part, prefix, classes, steps=5, **cfg):
    t = part.trainer(**cfg)
    out = {f"{prefix}init": t.params()}
    loss, gn, params, grads, masks, plosses, logits = [], [], [], [], [], [], []
    for e in range(steps):
        l, g = t.step(e)
        loss.append(l)
        gn.append(g)
        params.append(t.params())
        grads.append(t.gathered())
        masks.append([t.part_mask(i) for i in range(part.p)])
        plosses.append([t.part_loss(i) for i in range(part.p)])
        logits.append(np.concatenate([t.part_logits(i, classes).reshape(-1) for i in range(part.p)]))
    out[f"{prefix}loss"] = np.array(loss)
    out[f"{prefix}gnorm"] = np.array(gn)
    out[f"{prefix}params"] = np.stack(params)
    out[f"{prefix}grads"] = np.stack(grads)
    out[f"{prefix}masks"] = np.array(masks)
    out[f"{prefix}part_loss"] = np.array(plosses)
    out[f"{prefix}logits"] = np.stack(logits)
    out[f"{prefix}eval"] = np.array(t.eval())
    return out


def main():
    R = reference()
    np.savez_compressed(os.path.join(HERE, "rng.npz"), **rng_fixture(R))

    # ---- karate ----
    # load_graph (graph_io.cpp:41-80) = parse "u v" lines, n = max id + 1, then
    # build_graph; parsed here because the reference's iostream parser crashes
    # when loaded into a process that already imported numpy.
    raw = np.array([[int(t) for t in ln.split()] for ln in open(KARATE) if ln.strip() and not ln.startswith("#")],
                   np.int32)
    gk = R.graph_build(int(raw.max()) + 1, raw)
    kar = graph_arrays(gk, "")
    for p in (1, 2, 4, 8):
        kar.update(partition_arrays(gk.partition("random", p, 0), f"random_p{p}_"))
    kar.update(partition_arrays(gk.partition("dbh", 4, 0), "dbh_p4_"))
    pk = gk.partition("random", 4, 0)
    e0 = pk.sizes(0)[1]
    kar["masks_p0_k3"] = R.precompute_masks(e0, 3, 0.5, R.substream(0, "dropedge", 0))
    np.savez_compressed(os.path.join(HERE, "karate.npz"), **kar)

    # ---- sbm200 ----
    gs = R.graph_sbm(200, 4, 0.15, 0.01, 8, 0.3, 7)
    sb = graph_arrays(gs, "", d=8)
    for p in (1, 2, 4, 8):
        sb.update(partition_arrays(gs.partition("random", p, 3), f"random_p{p}_", full=(p == 8)))
        sb.update(partition_arrays(gs.partition("dbh", p, 3), f"dbh_p{p}_", full=False))
    part = gs.partition("random", 8, 3)
    for i in range(8):
        ne = part.sizes(i)[1]
        sb[f"masks_p{i}"] = R.precompute_masks(ne, 10, 0.5, R.substream(1, "dropedge", i))
    sb["masks_100_10_05_3"] = R.precompute_masks(100, 10, 0.5, 3)
    sb["select_seed1"] = np.array([[R.select_mask(1, i, e, 10) for e in range(20)] for i in range(8)])
    sb["init_8_16_16_4_seed1_f64"] = R.init_params(8, [16, 16], 4, 1, f32=False)
    sb["init_8_16_16_4_seed1_f32"] = R.init_params(8, [16, 16], 4, 1, f32=True)
    for f32 in (True, False):
        for de in (False, True):
            pre = f"traj_{'f32' if f32 else 'f64'}_{'de' if de else 'plain'}_"
            sb.update(trajectory(part, pre, 4, hidden=[16, 16], lr=0.01, dropedge=de, seed=1, f32=f32))
    sb.update(trajectory(part, "traj_f32_bce_", 4, hidden=[16, 16], lr=0.01, loss="bce", seed=1, f32=True))
    sb.update(trajectory(part, "traj_f32_vanilla_", 4, hidden=[16, 16], lr=0.01, reweight="vanilla_inv", seed=1,
                         f32=True))
    part_dbh = gs.partition("dbh", 4, 3)
    sb.update(trajectory(part_dbh, "traj_f32_dbh4_", 4, hidden=[16, 16, 16], lr=0.02, dropedge=True, k=4,
                         ratio=0.3, seed=5, f32=True))
    np.savez_compressed(os.path.join(HERE, "sbm200.npz"), **sb)

    # ---- ER 10k (configs[0]) ----
    ge = R.graph_sbm(10000, 4, 0.004, 0.004, 64, 1.0, 0)
    er = {"n": np.int64(ge.n), "m": np.int64(ge.m), "edges_sha": np.array(sha(ge.edges())),
          "features_sha": np.array(sha(ge.features(64)))}
    pe = ge.partition("random", 4, 0)
    er["assign_sha"] = np.array(sha(pe.assignment()))
    st = pe.stats()
    er["stats"] = np.array([st["rf"], st["edge_balance"], st["node_balance"], st["duplicated_nodes"]])
    er["per_node_rf_sha"] = np.array(sha(st["per_node_rf"]))
    er["w_dar_sum"] = np.array([w.sum() for w in pe.weights("dar")])
    for i in range(4):
        a = pe.part(i)
        er[f"p{i}_sizes"] = np.array([len(a.nodes), len(a.edges)])
        er[f"p{i}_csr_sha"] = np.array(sha(np.concatenate([a.offsets, a.nbrs, a.eids])))
        er[f"p{i}_mask_sha"] = np.array(sha(R.precompute_masks(len(a.edges), 10, 0.5, R.substream(0, "dropedge", i))))
    t = trajectory(pe, "traj_", 4, hidden=[32, 32], lr=0.01, dropedge=True, seed=0, f32=True)
    t.pop("traj_logits")  # 40k x 4 x 5 doubles: keep the fixture small
    er.update(t)
    np.savez_compressed(os.path.join(HERE, "er10k.npz"), **er)
    for f in sorted(os.listdir(HERE)):
        if f.endswith(".npz"):
            print(f, os.path.getsize(os.path.join(HERE, f)))


if __name__ == "__main__":
    main()
