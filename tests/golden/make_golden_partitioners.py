"""Golden fixtures for the greedy partitioners, from the REAL reference.

    make -C oracle && python tests/golden/make_golden_partitioners.py

Every value comes from oracle/_ref/libsagecut_ref.so (the unmodified reference
sources, see make_golden.py): partition_ne (partition.cpp:116-201) with its
overshoot warnings, partition_edge_cut_greedy (:233-278),
edge_cut_from_assignment (:203-231) and edge_cut_to_vertex_cut (:280-308).

partitioners.npz keys, per graph G in {karate, sbm200, star, er10k}:
  G_edges                       canonical edges (er10k: sha only)
  G_ne_p{p}[_s{slack}]_assign   NE edge assignment, and ..._warnings (newline-joined)
  G_ec_p{p}_s{seed}_nodes       greedy edge-cut node assignment
  G_ec_p{p}_s{seed}_kept|cut|halo_counts|halo_nodes
  G_ec2vc_p{p}_s{seed}_assign   vertex cut converted from that edge cut
"""
from __future__ import annotations

import hashlib
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
from cpu_libs import reference  # noqa: E402

KARATE = "/root/reference/proj/tests/fixtures/karate.edges"


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def star_edges():
    """Hub 0 with 60 leaves, a 40-node path, a triangle, and isolated nodes 110..119."""
    e = [(0, i) for i in range(1, 61)]
    e += [(61 + i, 62 + i) for i in range(39)]
    e += [(101, 102), (102, 103), (101, 103), (5, 70)]
    return 120, np.array(e, np.int32)


def dump(out, name, g, cases_ne, cases_ec, full=True):
    if full:
        out[f"{name}_edges"] = g.edges()
    else:
        out[f"{name}_edges_sha"] = np.array(sha(g.edges()))
    for p, slack in cases_ne:
        part, warn = g.partition_ne(p, 0, slack)
        key = f"{name}_ne_p{p}" + ("" if slack == 1.1 else f"_s{slack}")
        a = part.assignment()
        if full:
            out[key + "_assign"] = a
        else:
            out[key + "_assign_sha"] = np.array(sha(a))
        out[key + "_warnings"] = np.array("\n".join(warn))
    for p, seed in cases_ec:
        na = g.edge_cut_greedy(p, seed)
        kept, cut, halo = g.edge_cut(p, na)
        key = f"{name}_ec_p{p}_s{seed}"
        a = g.edge_cut_to_vertex_cut(p, na, seed).assignment()
        if full:
            out[key + "_nodes"] = na
            out[key + "_cut"] = cut
            out[key + "_halo_nodes"] = np.concatenate(halo) if halo else np.zeros(0, np.int32)
            out[f"{name}_ec2vc_p{p}_s{seed}_assign"] = a
        else:
            out[key + "_nodes_sha"] = np.array(sha(na))
            out[key + "_cut_sha"] = np.array(sha(cut))
            out[key + "_halo_sha"] = np.array(sha(np.concatenate(halo)))
            out[f"{name}_ec2vc_p{p}_s{seed}_assign_sha"] = np.array(sha(a))
        out[key + "_kept"] = kept
        out[key + "_halo_counts"] = np.array([len(h) for h in halo], np.int64)


def main():
    R = reference()
    out = {}
    raw = np.array([[int(t) for t in ln.split()] for ln in open(KARATE) if ln.strip() and not ln.startswith("#")],
                   np.int32)
    gk = R.graph_build(int(raw.max()) + 1, raw)
    dump(out, "karate", gk, [(1, 1.1), (2, 1.1), (4, 1.1), (8, 1.1), (8, 1.0), (3, 1.0)],
         [(1, 0), (2, 0), (4, 0), (4, 1), (8, 3)])
    gs = R.graph_sbm(200, 4, 0.15, 0.01, 8, 0.3, 7)
    dump(out, "sbm200", gs, [(2, 1.1), (4, 1.1), (8, 1.1), (5, 1.0)], [(4, 3), (8, 3), (3, 11)])
    n, e = star_edges()
    gst = R.graph_build(n, e)
    dump(out, "star", gst, [(2, 1.1), (3, 1.1), (4, 1.0), (7, 1.5)], [(2, 0), (3, 5), (6, 2)])
    ge = R.graph_sbm(10000, 4, 0.004, 0.004, 64, 1.0, 0)
    dump(out, "er10k", ge, [(4, 1.1), (8, 1.1)], [(4, 0)], full=False)
    np.savez_compressed(os.path.join(HERE, "partitioners.npz"), **out)
    print(f"wrote {len(out)} arrays; warnings:",
          {k: str(v) for k, v in out.items() if k.endswith("_warnings") and str(v)})


if __name__ == "__main__":
    main()
