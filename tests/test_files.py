"""The reference's file formats, byte for byte against the reference's
own writers (oracle/_ref: proj/src/partition_io.cpp, checkpoint.cpp, trainer.cpp:126-140):
partition JSON (with / without embedded loss weights), edge-cut JSON, CFCK checkpoints and
metrics JSONL; plus load round trips and the reference's error behaviour."""
import ctypes as C
import os

import numpy as np
import pytest

from cpu_libs import REF_SO, oracle, reference

needs_ref = pytest.mark.skipif(not os.path.exists(REF_SO), reason="oracle/_ref not built")


def _ref_fns(R):
    L = R.lib
    L.ref_save_partition.argtypes = [C.c_void_p, C.c_void_p, C.c_char_p, C.c_int]
    L.ref_load_partition.restype = C.c_void_p
    L.ref_load_partition.argtypes = [C.c_void_p, C.c_char_p]
    L.ref_save_edge_cut.argtypes = [C.c_void_p, C.c_int, C.c_void_p, C.c_char_p]
    L.ref_save_checkpoint_f32.argtypes = [C.c_void_p, C.c_int, C.c_void_p, C.c_int, C.c_int, C.c_char_p]
    L.ref_load_checkpoint.restype = C.c_int64
    L.ref_load_checkpoint.argtypes = [C.c_char_p, C.c_void_p]
    L.ref_write_metrics.argtypes = [C.c_char_p, C.c_int, C.c_void_p, C.c_void_p]
    return L


def _metrics_rows():
    rng = np.random.default_rng(0)
    return [dict(epoch=e, train_loss=float(rng.random() * 3), train_metric=float(rng.random()),
                 val_metric=float(rng.random()), test_metric=1.0 / 3.0, grad_norm=float(rng.random() * 1e-3),
                 comm_floats=8 * 521984) for e in range(4)]


@needs_ref
def test_reference_writers_run(tmp_path):
    """CPU: the reference writers behind the harness produce what the GPU tests compare against."""
    R = reference()
    L = _ref_fns(R)
    g = R.graph_sbm(200, 4, 0.15, 0.01, 8, 0.3, 7)
    part = g.partition("random", 4, 3)
    assert L.ref_save_partition(g.h, part.h, str(tmp_path / "p.json").encode(), 0) == 0
    assert (tmp_path / "p.json").read_text().startswith("{\n  \"edge_assignment\": [")
    rows = _metrics_rows()
    ep = np.array([r["epoch"] for r in rows], np.int32)
    vals = np.array([[r[k] for k in ("train_loss", "train_metric", "val_metric", "test_metric", "grad_norm",
                                     "comm_floats")] for r in rows], np.float64)
    assert L.ref_write_metrics(str(tmp_path / "m.jsonl").encode(), len(rows), ep.ctypes.data, vals.ctypes.data) == 0
    assert len((tmp_path / "m.jsonl").read_text().splitlines()) == 4


@pytest.fixture(scope="module")
def sc():
    from paper_2308_03209_b200 import sagecut
    return sagecut


def _graphs(sc):
    O, R = oracle(), reference()
    og = O.graph_sbm(200, 4, 0.15, 0.01, 8, 0.3, 7)
    rg = R.graph_sbm(200, 4, 0.15, 0.01, 8, 0.3, 7)
    g, _ = sc.build_graph(og.n, og.edges())
    tr, va, te = og.masks()
    g.set_data(og.features(8).astype(np.float32), og.labels(), 4, tr, va, te)
    return og, rg, g


@pytest.mark.gpu
@needs_ref
def test_partition_json_bytes_and_round_trip(sc, tmp_path):
    og, rg, g = _graphs(sc)
    L = _ref_fns(reference())
    for algo, p, seed in (("random", 4, 3), ("ne", 5, 0)):
        part = sc.partition_random(g, p, seed) if algo == "random" else sc.partition_ne(g, p, seed)
        rpart = rg.partition(algo, p, seed)
        for scheme, code in ((None, -1), ("dar", 0), ("vanilla_inv", 1), ("none", 2)):
            mine, ref = tmp_path / f"{algo}{scheme}.json", tmp_path / f"{algo}{scheme}.ref.json"
            sc.save_partition(part, str(mine), weights=scheme)
            assert L.ref_save_partition(rg.h, rpart.h, str(ref).encode(), code) == 0
            assert mine.read_bytes() == ref.read_bytes(), (algo, scheme)
        back = sc.load_partition(str(mine), g)  # our loader on the reference's file
        np.testing.assert_array_equal(back.edge_assignment, part.edge_assignment)
        for i in range(p):
            np.testing.assert_array_equal(back.part(i).nodes, part.part(i).nodes)
    other, _ = sc.build_graph(50, np.array([[0, 1], [1, 2]], np.int32))
    with pytest.raises(RuntimeError, match="partition was built for"):
        sc.load_partition(str(mine), other)
    with pytest.raises(RuntimeError, match="cannot open partition file"):
        sc.load_partition(str(tmp_path / "missing.json"), g)


@pytest.mark.gpu
@needs_ref
def test_edge_cut_json_bytes(sc, tmp_path):
    og, rg, g = _graphs(sc)
    L = _ref_fns(reference())
    for p, seed in ((3, 1), (6, 4)):
        ec = sc.partition_edge_cut_greedy(g, p, seed)
        mine, ref = tmp_path / f"ec{p}.json", tmp_path / f"ec{p}.ref.json"
        sc.save_edge_cut(g, ec, str(mine))
        na = np.ascontiguousarray(ec.node_assignment, np.int32)
        assert L.ref_save_edge_cut(rg.h, p, na.ctypes.data, str(ref).encode()) == 0
        assert mine.read_bytes() == ref.read_bytes()


@pytest.mark.gpu
@needs_ref
def test_checkpoint_and_metrics_bytes(sc, tmp_path):
    og, rg, g = _graphs(sc)
    L = _ref_fns(reference())
    hidden = [16, 16]
    t = sc.CoFreeTrainer(g, sc.partition_random(g, 4, 3), sc.TrainConfig(layers=2, hidden=hidden, seed=1))
    for e in range(2):
        t.step(e)
    mine, ref = tmp_path / "m.ckpt", tmp_path / "r.ckpt"
    t.save_checkpoint(str(mine))
    theta = t.params().astype(np.float32)
    h = np.array(hidden, np.int32)
    assert L.ref_save_checkpoint_f32(theta.ctypes.data, 8, h.ctypes.data, 2, 4, str(ref).encode()) == 0
    assert mine.read_bytes() == ref.read_bytes()
    assert mine.read_bytes()[:4] == b"CFCK"
    t2 = sc.CoFreeTrainer(g, sc.partition_random(g, 4, 3), sc.TrainConfig(layers=2, hidden=hidden, seed=9))
    t2.load_checkpoint(str(ref))  # the reference's checkpoint into our trainer
    np.testing.assert_array_equal(t2.params(), theta)
    (tmp_path / "bad.ckpt").write_bytes(b"XXXX" + mine.read_bytes()[4:])
    with pytest.raises(RuntimeError, match="bad magic"):
        t2.load_checkpoint(str(tmp_path / "bad.ckpt"))
    t3 = sc.CoFreeTrainer(g, sc.partition_random(g, 4, 3), sc.TrainConfig(layers=1, hidden=[16], seed=1))
    with pytest.raises(ValueError, match="does not match the model"):
        t3.load_checkpoint(str(mine))
    rows = _metrics_rows()
    sc.write_metrics_jsonl(rows, str(tmp_path / "m.jsonl"))
    ep = np.array([r["epoch"] for r in rows], np.int32)
    vals = np.array([[r[k] for k in ("train_loss", "train_metric", "val_metric", "test_metric", "grad_norm",
                                     "comm_floats")] for r in rows], np.float64)
    assert L.ref_write_metrics(str(tmp_path / "r.jsonl").encode(), len(rows), ep.ctypes.data, vals.ctypes.data) == 0
    assert (tmp_path / "m.jsonl").read_bytes() == (tmp_path / "r.jsonl").read_bytes()
