"""Free-running multi-step parity at a headline shape (run on the GPU box):

    python tools/scale_parity.py [--config products|reddit] [--steps 5] [--out profiles/r02_scale_free.json]

Three trainers start from the same init (seed 1) on the same graph / vertex cut /
DropEdge masks and run `steps` epochs free (each on its own parameters):
  tc    the library (tcgen05 fp16x3 GEMMs)                      [fp32]
  simt  the library with the fp32 SIMT GEMMs (gemm = "simt")     [fp32 control]
  f64   the fp64 restatement of train_cofree_impl (tests/torch_ref.py per partition,
        ascending-partition gather, Adam of nn.hpp:400-432 in double)
Per epoch it records the loss, grad norm, and the relative L2 distance of the
gathered gradients and of the parameters between every pair. The reference's
own f32 mode is one more fp32 implementation: its distance to f64 is of the
same kind as tc's and simt's (the C oracle cannot run these sizes).
"""
import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))


def rel(a, b):
    a, b = np.asarray(a, np.float64).ravel(), np.asarray(b, np.float64).ravel()
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="products")
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--out", default=None)
    args = ap.parse_args()
    import torch

    import bench
    from paper_2308_03209_b200 import sagecut as sc
    from torch_ref import partition_step

    cfg = bench.CONFIGS[args.config]
    n, uv, feats, labels, tr, va, te = bench.synth_host(cfg, seed=0)
    g, _ = sc.build_graph(n, uv)
    del uv
    g.set_data(feats, labels, cfg["classes"], tr, va, te)
    part = sc.partition_random(g, cfg["parts"], 0)
    p, L, H = cfg["parts"], cfg["layers"], cfg["hidden"]
    hidden = [H] * L
    runs = {}
    for gemm in ("auto", "simt"):
        t = sc.CoFreeTrainer(g, part, sc.TrainConfig(layers=L, hidden=[H], learning_rate=cfg["lr"],
                                                     use_dropedge=cfg["dropedge"], dropedge_k=cfg["k"],
                                                     drop_ratio=cfg["ratio"], seed=1, gemm=gemm))
        r = {"theta0": t.params(), "loss": [], "gnorm": [], "grads": [], "params": [], "masks": []}
        t0 = time.perf_counter()
        for e in range(args.steps):
            loss, gn = t.step(e)
            r["loss"].append(loss)
            r["gnorm"].append(gn)
            r["grads"].append(t.grads().astype(np.float64))
            r["params"].append(t.params().astype(np.float64))
            r["masks"].append([t.part_mask(i) for i in range(p)])
        r["seconds"] = time.perf_counter() - t0
        t.close()
        torch.cuda.empty_cache()
        runs["tc" if gemm == "auto" else "simt"] = r
    # fp64 restatement of train_cofree_impl
    w_all = sc.compute_weights("dar", g, part).per_part
    normalizer = float((tr != 0).sum())
    parts = [part.part(i) for i in range(p)]
    masksets = [sc.precompute_masks(len(a.edges), cfg["k"], cfg["ratio"], sc.substream(1, "dropedge", i)).masks
                if cfg["dropedge"] else None for i, a in enumerate(parts)]
    theta = runs["tc"]["theta0"].astype(np.float64)
    m1, m2 = np.zeros_like(theta), np.zeros_like(theta)
    f = {"loss": [], "gnorm": [], "grads": [], "params": []}
    t0 = time.perf_counter()
    for e in range(args.steps):
        gathered, total = None, 0.0
        for i, a in enumerate(parts):
            mask = None
            if cfg["dropedge"]:
                mask = masksets[i][sc.select_mask(1, i, e, cfg["k"])]
            w = w_all[i] * (tr[a.nodes] != 0)
            r = partition_step(theta, cfg["feats"], hidden, cfg["classes"], a.adj_offsets, a.adj_neighbors, a.adj_edge_ids, mask,
                               feats[a.nodes], w, normalizer, labels=labels[a.nodes], device="cuda")
            gathered = r["grads"] if gathered is None else gathered + r["grads"]
            total += r["loss"]
            del r
            torch.cuda.empty_cache()
        step = e + 1  # adam_step (nn.hpp:400-432) in double
        m1 = 0.9 * m1 + 0.1 * gathered
        m2 = 0.999 * m2 + 0.001 * gathered * gathered
        theta = theta - cfg["lr"] * (m1 / (1 - 0.9 ** step)) / (np.sqrt(m2 / (1 - 0.999 ** step)) + 1e-8)
        f["loss"].append(total)
        f["gnorm"].append(float(np.linalg.norm(gathered)))
        f["grads"].append(gathered)
        f["params"].append(theta.copy())
    f["seconds"] = time.perf_counter() - t0
    runs["f64"] = f
    out = {"config": args.config, "partitions": p, "layers": L, "hidden": H, "steps": args.steps,
           "nodes": n, "edges": g.num_edges(), "seconds": {k: v["seconds"] for k, v in runs.items()},
           "loss": {k: v["loss"] for k, v in runs.items()}, "gnorm": {k: v["gnorm"] for k, v in runs.items()},
           "same_masks": runs["tc"]["masks"] == runs["simt"]["masks"], "per_step": []}
    for e in range(args.steps):
        row = {"epoch": e}
        for a_, b_ in (("tc", "f64"), ("simt", "f64"), ("tc", "simt")):
            row[f"grads_{a_}_vs_{b_}"] = rel(runs[a_]["grads"][e], runs[b_]["grads"][e])
            row[f"params_{a_}_vs_{b_}"] = rel(runs[a_]["params"][e], runs[b_]["params"][e])
            row[f"loss_{a_}_vs_{b_}"] = abs(runs[a_]["loss"][e] - runs[b_]["loss"][e]) / abs(runs[b_]["loss"][e])
        out["per_step"].append(row)
    s = json.dumps(out, indent=1)
    print(s)
    if args.out:
        open(args.out, "w").write(s + "\n")


if __name__ == "__main__":
    main()
