"""Greedy partitioners: NE, greedy edge cut, edge cut ->
vertex cut, edge_cut_from_assignment (proj/src/partition.cpp:116-308).

CPU: the oracle restatement against tests/golden/partitioners.npz (dumped from
the compiled reference by tests/golden/make_golden_partitioners.py) and against
oracle/_ref on seeded random graphs. GPU (-m gpu): libsagecut_cuda.so through
its C ABI against the same goldens and the oracle, bit-exact (assignments,
warnings, kept/cut lists, halo sets), plus the reference's error behaviour.
"""
import hashlib
import os

import numpy as np
import pytest

from cpu_libs import REF_SO, oracle, reference

HERE = os.path.dirname(os.path.abspath(__file__))


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


@pytest.fixture(scope="module")
def G():
    return dict(np.load(os.path.join(HERE, "golden", "partitioners.npz")))


def _cases(G):
    """(graph, ne cases [(p, slack, key)], ec cases [(p, seed, key)], full) from the fixture keys."""
    out = {}
    for k in G:
        name = k.split("_")[0]
        out.setdefault(name, ([], []))
        if k.endswith("_warnings"):
            rest = k[len(name) + len("_ne_p"):-len("_warnings")]
            p, _, s = rest.partition("_s")
            out[name][0].append((int(p), float(s) if s else 1.1, k[:-len("_warnings")]))
        elif k.endswith("_kept"):
            rest = k[len(name) + len("_ec_p"):-len("_kept")]
            p, _, s = rest.partition("_s")
            out[name][1].append((int(p), int(s), k[:-len("_kept")]))
    return out


def _check_lib(G, name, g_edges_fn, ne_fn, ec_fn, stats_fn, ec2vc_fn):
    ne_cases, ec_cases = _cases(G)[name]
    full = f"{name}_edges" in G
    for p, slack, key in ne_cases:
        assign, warn = ne_fn(p, slack)
        if full:
            np.testing.assert_array_equal(assign, G[key + "_assign"], err_msg=key)
        else:
            assert sha(assign) == str(G[key + "_assign_sha"]), key
        assert "\n".join(warn) == str(G[key + "_warnings"]), key
    for p, seed, key in ec_cases:
        na = ec_fn(p, seed)
        kept, cut, halo = stats_fn(p, na)
        np.testing.assert_array_equal(kept, G[key + "_kept"], err_msg=key)
        np.testing.assert_array_equal([len(h) for h in halo], G[key + "_halo_counts"], err_msg=key)
        vc = ec2vc_fn(p, na, seed)
        ec_key = key.replace("_ec_", "_ec2vc_")
        if full:
            np.testing.assert_array_equal(na, G[key + "_nodes"], err_msg=key)
            np.testing.assert_array_equal(cut, G[key + "_cut"], err_msg=key)
            np.testing.assert_array_equal(np.concatenate(halo), G[key + "_halo_nodes"], err_msg=key)
            np.testing.assert_array_equal(vc, G[ec_key + "_assign"], err_msg=key)
        else:
            assert sha(na) == str(G[key + "_nodes_sha"]) and sha(cut) == str(G[key + "_cut_sha"]), key
            assert sha(np.concatenate(halo)) == str(G[key + "_halo_sha"]), key
            assert sha(vc) == str(G[ec_key + "_assign_sha"]), key


def _oracle_graph(O, G, name):
    if name == "sbm200":
        return O.graph_sbm(200, 4, 0.15, 0.01, 8, 0.3, 7)
    if name == "er10k":
        return O.graph_sbm(10000, 4, 0.004, 0.004, 64, 1.0, 0)
    e = G[f"{name}_edges"]
    n = 120 if name == "star" else int(e.max()) + 1
    return O.graph_build(n, e)


@pytest.mark.parametrize("name", ["karate", "sbm200", "star", "er10k"])
def test_oracle_partitioners_vs_golden(G, name):
    O = oracle()
    g = _oracle_graph(O, G, name)
    if f"{name}_edges" in G:
        np.testing.assert_array_equal(g.edges(), G[f"{name}_edges"])
    else:
        assert sha(g.edges()) == str(G[f"{name}_edges_sha"])

    def ne(p, s):
        part, w = g.partition_ne(p, 0, s)
        return part.assignment(), w
    _check_lib(G, name, None, ne, g.edge_cut_greedy, g.edge_cut,
               lambda p, na, seed: g.edge_cut_to_vertex_cut(p, na, seed).assignment())


@pytest.mark.skipif(not os.path.exists(REF_SO), reason="oracle/_ref not built")
@pytest.mark.parametrize("seed", [0, 1, 2])
def test_oracle_matches_reference_on_random_graphs(seed):
    """Seeded random graphs with isolated nodes, skewed degrees and odd p."""
    O, R = oracle(), reference()
    rng = np.random.default_rng(seed)
    n = 3000
    hubs = rng.integers(0, 20, size=(4000, 1))
    e = np.concatenate([np.concatenate([hubs, rng.integers(0, n - 50, size=(4000, 1))], 1),
                        rng.integers(0, n - 50, size=(6000, 2))]).astype(np.int32)  # nodes >= n-50 isolated
    go, gr = O.graph_build(n, e), R.graph_build(n, e)
    for p in (3, 5, 8):
        (a, wa), (b, wb) = go.partition_ne(p, 0, 1.05), gr.partition_ne(p, 0, 1.05)
        np.testing.assert_array_equal(a.assignment(), b.assignment())
        assert wa == wb
        na, nb = go.edge_cut_greedy(p, seed), gr.edge_cut_greedy(p, seed)
        np.testing.assert_array_equal(na, nb)
        np.testing.assert_array_equal(go.edge_cut_to_vertex_cut(p, na, 7).assignment(),
                                      gr.edge_cut_to_vertex_cut(p, nb, 7).assignment())


# ---------------------------------------------------------------------------- GPU
@pytest.fixture(scope="module")
def sc():
    from paper_2308_03209_b200 import sagecut
    return sagecut


def _gpu_fns(sc, g):
    def ne(p, s):
        vc = sc.partition_ne(g, p, 0, s)
        return vc.edge_assignment, vc.warnings

    def ec(p, seed):
        return sc.partition_edge_cut_greedy(g, p, seed).node_assignment

    def stats(p, na):
        e = sc.edge_cut_from_assignment(g, p, na)
        return np.array([len(k) for k in e.kept_edges]), e.cut_edges, e.halo_sets

    def ec2vc(p, na, seed):
        return sc.edge_cut_to_vertex_cut(g, sc.edge_cut_from_assignment(g, p, na), seed).edge_assignment
    return ne, ec, stats, ec2vc


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["karate", "sbm200", "star", "er10k"])
def test_gpu_partitioners_vs_golden(sc, G, name):
    og = _oracle_graph(oracle(), G, name)
    g, _ = sc.build_graph(og.n, og.edges())
    _check_lib(G, name, None, *_gpu_fns(sc, g))


@pytest.mark.gpu
@pytest.mark.parametrize("seed", [0, 1])
def test_gpu_partitioners_vs_oracle_random(sc, seed):
    """Larger seeded graphs (skewed + isolated nodes): every output bit-exact, incl. the vertex cuts' parts."""
    O = oracle()
    rng = np.random.default_rng(100 + seed)
    n = 40000
    hubs = rng.integers(0, 64, size=(60000, 1))
    e = np.concatenate([np.concatenate([hubs, rng.integers(0, n - 100, size=(60000, 1))], 1),
                        rng.integers(0, n - 100, size=(140000, 2))]).astype(np.int32)
    og = O.graph_build(n, e)
    g, _ = sc.build_graph(n, e)
    for p in (4, 7):
        vc = sc.partition_ne(g, p, 0, 1.02)
        ov, ow = og.partition_ne(p, 0, 1.02)
        np.testing.assert_array_equal(vc.edge_assignment, ov.assignment())
        assert vc.warnings == ow
        for i in range(p):
            a, b = vc.part(i), ov.part(i)
            np.testing.assert_array_equal(a.nodes, b.nodes)
            np.testing.assert_array_equal(a.adj_neighbors, b.nbrs)
        ec = sc.partition_edge_cut_greedy(g, p, seed)
        na = og.edge_cut_greedy(p, seed)
        np.testing.assert_array_equal(ec.node_assignment, na)
        kept, cut, halo = og.edge_cut(p, na)
        np.testing.assert_array_equal([len(k) for k in ec.kept_edges], kept)
        np.testing.assert_array_equal(ec.cut_edges, cut)
        for a, b in zip(ec.halo_sets, halo):
            np.testing.assert_array_equal(a, b)
        edges = g.edges()
        for i, k in enumerate(ec.kept_edges):  # kept lists: ascending ids, both endpoints in part i
            assert (np.diff(k) > 0).all() and (na[edges[k, 0]] == i).all() and (na[edges[k, 1]] == i).all()
        np.testing.assert_array_equal(sc.edge_cut_to_vertex_cut(g, ec, 9).edge_assignment,
                                      og.edge_cut_to_vertex_cut(p, na, 9).assignment())


@pytest.mark.gpu
def test_gpu_partitioner_errors(sc):
    g, _ = sc.build_graph(4, np.array([[0, 1], [1, 2]], np.int32))
    with pytest.raises(ValueError, match="balance_slack must be >= 1"):
        sc.partition_ne(g, 2, 0, 0.5)
    with pytest.raises(ValueError, match="num_parts must be >= 1"):
        sc.partition_ne(g, 0, 0)
    with pytest.raises(ValueError, match="node assignment references an invalid part"):
        sc.edge_cut_from_assignment(g, 2, np.array([0, 1, 2, 0], np.int32))
    with pytest.raises(ValueError, match="node assignment length does not match node count"):
        sc.edge_cut_from_assignment(g, 2, np.array([0, 1], np.int32))
    # p = 1: everything in part 0, no cut; p > edges: NE leaves trailing parts empty of edges
    assert (sc.partition_ne(g, 1, 0).edge_assignment == 0).all()
    vc = sc.partition_ne(g, 5, 0)
    assert vc.num_parts == 5
