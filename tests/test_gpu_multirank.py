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
