"""The C++ drop-in facade (include/sagecut_b200.hpp) driven by a compiled
program, checked against the oracle: same API shape as the reference's
sagecut:: functions, same results, same exception types."""
import os
import subprocess

import numpy as np
import pytest

from cpu_libs import oracle

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
EXE = os.path.join(ROOT, "tests", "cpp", "facade_main")


def test_cpp_facade_matches_oracle(tmp_path):
    assert os.path.exists(EXE), "build with __graft_entry__.build() (make -C paper_2308_03209_b200/csrc facade)"
    O = oracle()
    og = O.graph_sbm(200, 4, 0.15, 0.01, 8, 0.3, 7)
    n, e, f = og.n, og.edges(), og.features(8).astype(np.float32)
    lab = og.labels()
    tr, va, te = og.masks()
    p, seed, epochs = 4, 1, 3
    path = tmp_path / "in.txt"
    with open(path, "w") as fh:
        fh.write(f"{n} {len(e)} 8 4 {p} {seed} {epochs}\n")
        fh.write("\n".join(f"{u} {v}" for u, v in e) + "\n")
        fh.write("\n".join(" ".join(repr(float(x)) for x in row) for row in f) + "\n")
        for arr in (lab, tr, va, te):
            fh.write(" ".join(str(int(x)) for x in arr) + "\n")
    out = subprocess.run([EXE, str(path), str(tmp_path)], capture_output=True, text=True, timeout=300)
    assert out.returncode == 0, out.stderr
    res = {ln.split(" ", 1)[0]: ln.split(" ", 1)[1] if " " in ln else "" for ln in out.stdout.strip().split("\n")}
    op = og.partition("random", p, 3)
    assert int(res["edges"]) == og.m
    assert [int(x) for x in res["assign"].split()] == op.assignment().tolist()
    st = op.stats()
    assert float(res["rf"]) == st["rf"] and int(res["dup"]) == st["duplicated_nodes"]
    np.testing.assert_array_equal(np.array(res["w0"].split(), float), op.weights("dar")[0])
    m0 = op.sizes(0)[1]
    np.testing.assert_array_equal(np.array(res["mask0"].split(), np.uint8), O.precompute_masks(m0, 3, 0.5, 17)[0])
    t = op.trainer([16, 16], lr=0.01, dropedge=True, seed=seed, f32=True)
    ref_loss = [t.step(ep)[0] for ep in range(epochs)]
    np.testing.assert_allclose(np.array(res["loss"].split(), float), ref_loss, rtol=1e-5)
    theta = np.array(res["params"].split(), float)
    assert np.linalg.norm(theta - t.params()) / np.linalg.norm(t.params()) <= 1e-4
    ne, warn = og.partition_ne(p, 0, 1.0)
    assert [int(x) for x in res["ne"].split()] == ne.assignment().tolist()
    assert int(res["ne_warnings"]) == len(warn)
    na = og.edge_cut_greedy(p, 5)
    assert [int(x) for x in res["ec_nodes"].split()] == na.tolist()
    kept, cut, halo = og.edge_cut(p, na)
    assert int(res["ec_cut"]) == len(cut) and int(res["ec_halo"]) == sum(len(h) for h in halo)
    assert [int(x) for x in res["ec2vc"].split()] == og.edge_cut_to_vertex_cut(p, na, 5).assignment().tolist()
    assert res["reload_same"] == "1" and res["ckpt_same"] == "1"
    assert (tmp_path / "model.ckpt").read_bytes()[:4] == b"CFCK"
    assert len((tmp_path / "metrics.jsonl").read_text().splitlines()) == epochs
    assert '"weight_scheme": "dar"' in (tmp_path / "part.json").read_text()
    assert res["error"].startswith("invalid_argument num_parts must be >= 1")
    # evaluate of the trained model, CommAudit, comm_volume, expected_rf / imbalance bound
    assert abs(float(res["eval_test"]) - O.graph_sbm(200, 4, 0.15, 0.01, 8, 0.3, 7).evaluate(
        theta, [16, 16], te)) <= 0.02
    P = len(theta)
    assert [int(x) for x in res["audit"].split()] == [p * P] * epochs + [0]
    assert [int(x) for x in res["comm"].split()] == O.comm_volume("halo_sync_model", p, P, 2, 16, 100)
    assert float(res["erf"]) == O.expected_rf_random(p, 13)
    assert float(res["ilb"]) == O.imbalance_lower_bound(p, 9, 2)
