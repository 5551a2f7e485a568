"""The library's own world > 1 training path, executed (the GPU
analogue of the reference's worker-count invariance, test_trainer.cpp:129-142).

2 or 3 processes share the one GPU, each a rank of trainer.cu's multi-GPU
protocol (partition i on rank i % world in exchange round i / world, padding
rounds when p % world != 0, bucket-major gradient slots, ordered gather, the
same Adam step on every rank), holding only its own partitions
(sc_graph_set_part_ownership). The exchange moves the same bytes as NCCL's
all-gather through a gloo host transport (sc_trainer_set_exchange). Losses,
grad norms, gathered gradients and parameters must equal world 1 BITWISE.
"""
import os
import socket
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
WORKER = os.path.join(ROOT, "tests", "mr_worker.py")


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def run(case, world, tmp_path):
    port = free_port()
    outs = [str(tmp_path / f"{case}_w{world}_r{r}.npz") for r in range(world)]
    procs = [subprocess.Popen([sys.executable, WORKER, str(r), str(world), str(port), case, outs[r]],
                              stdout=subprocess.PIPE, stderr=subprocess.STDOUT, text=True) for r in range(world)]
    logs = [p.communicate(timeout=600)[0] for p in procs]
    for p, log in zip(procs, logs):
        assert p.returncode == 0, log[-3000:]
    return [dict(np.load(o)) for o in outs]


@pytest.mark.parametrize("case,world", [("sbm_p8", 2), ("sbm_p7", 3), ("er_p4", 3)])
def test_world_invariance(case, world, tmp_path):
    ref = run(case, 1, tmp_path)[0]
    ranks = run(case, world, tmp_path)
    p = {"sbm_p8": 8, "sbm_p7": 7, "er_p4": 4}[case]
    P = ref["params"].size
    for r, z in enumerate(ranks):
        for k in ("losses", "gnorms", "params", "grads"):
            np.testing.assert_array_equal(z[k], ref[k], err_msg=f"rank {r} {k}")
        assert z["local"].tolist() == list(range(r, p, world))
        assert int(z["audit"][0]) == len(z["local"]) * P and int(z["audit"][1]) == 0
    assert int(ref["audit"][0]) == p * P


def test_emulated_rank_matches_its_share():
    """sc_trainer_emulate_rank (the bench's configs[4] run: rank 0 of an 8-GPU job on one GPU): the
    rank holds and trains exactly its partitions (i % world == rank), each partition's gradient and
    loss are bitwise those of the full world-1 run, and with the exchange skipped the gathered
    gradient is the ordered sum of this rank's partitions only (the others' slots stay zero)."""
    from cpu_libs import oracle
    from paper_2308_03209_b200 import sagecut as sc
    from test_gpu_parity import gpu_graph
    og = oracle().graph_sbm(200, 4, 0.15, 0.01, 8, 0.3, 7)
    cfg = sc.TrainConfig(layers=2, hidden=[16, 16], use_dropedge=True, seed=1)
    g1 = gpu_graph(sc, og, 8)
    t1 = sc.CoFreeTrainer(g1, sc.partition_random(g1, 8, 3), cfg)
    t1.step(0)
    world, rank = 4, 0
    g2 = gpu_graph(sc, og, 8)
    g2.set_part_ownership(rank, world)
    part2 = sc.partition_random(g2, 8, 3)
    assert [part2.part_held(i) for i in range(8)] == [i % world == rank for i in range(8)]
    t2 = sc.CoFreeTrainer(g2, part2, cfg, rank=rank, world=world, _defer_comm=True)
    t2.emulate_rank()
    t2.step(0)
    mine = list(range(rank, 8, world))
    expect = np.zeros(t1.param_count, np.float32)
    for i in mine:
        np.testing.assert_array_equal(t2.part_grads(i), t1.part_grads(i))
        assert t2.part_loss(i) == t1.part_loss(i)
        expect = expect + t1.part_grads(i)  # float32, ascending partition order
    np.testing.assert_array_equal(t2.grads(), expect)


def test_feature_rows_fill_same_bits():
    """set_data(features=None, dim) + set_feature_rows in chunks (host and device sources; the bench's
    device-side synthesis for configs[4]) trains bitwise like set_data with the whole matrix."""
    import torch
    from cpu_libs import oracle
    from paper_2308_03209_b200 import sagecut as sc
    from test_gpu_parity import gpu_graph
    og = oracle().graph_sbm(200, 4, 0.15, 0.01, 8, 0.3, 7)
    cfg = sc.TrainConfig(layers=2, hidden=[16, 16], use_dropedge=True, seed=1)
    ga = gpu_graph(sc, og, 8)
    ta = sc.CoFreeTrainer(ga, sc.partition_random(ga, 4, 3), cfg)
    la = [ta.step(e)[0] for e in range(3)]
    feats = og.features(8).astype(np.float32)
    gb, _ = sc.build_graph(og.n, og.edges())
    tr, va, te = og.masks()
    gb.set_data(None, og.labels(), int(og.labels().max()) + 1, tr, va, te, dim=8)
    gb.set_feature_rows(0, feats[:70])                      # host rows
    dev = torch.from_numpy(feats[70:]).cuda()
    torch.cuda.synchronize()
    gb.set_feature_rows(70, device_ptr=dev.data_ptr(), num_rows=dev.shape[0])  # device rows
    tb = sc.CoFreeTrainer(gb, sc.partition_random(gb, 4, 3), cfg)
    lb = [tb.step(e)[0] for e in range(3)]
    assert la == lb
    np.testing.assert_array_equal(ta.params(), tb.params())
    with pytest.raises(Exception, match="out of range"):
        gb.set_feature_rows(og.n - 1, feats[:2])
