"""Multi-rank protocol on CPU (gloo, world_size 2).

libsagecut_cuda.so trains partition i on rank i % world, writes each
partition's gradient into its own slot of a [p x |theta|] buffer (other ranks'
slots zero), all-reduces the slots (NCCL sum) and sums them in ascending
partition order on every rank (trainer.cu:trainer_step_async). Because each
slot has exactly one non-zero contributor, the all-reduce is exact and the
result is bitwise the reference's single-process gather (trainer.hpp:79-94)
for any GPU count. This test runs that protocol with the oracle's
per-partition gradients over gloo and checks bitwise equality, plus bench.py's
reference arm under torchrun (rank 0 prints, rank 1 exits 0).
"""
import json
import os
import subprocess
import sys

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _worker(rank, world, port, out):
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    from cpu_libs import oracle
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    O = oracle()
    g = O.graph_sbm(200, 4, 0.15, 0.01, 8, 0.3, 7)
    part = g.partition("random", 8, 3)
    t = part.trainer([16, 16], lr=0.01, dropedge=True, seed=1, f32=True)
    t.step(0)  # computes every partition's gradient (single-process reference)
    P = t.nparam
    slots = torch.zeros(8, P, dtype=torch.float32)
    losses = torch.zeros(8, dtype=torch.float64)
    for i in range(rank, 8, world):  # this rank's partitions
        slots[i] = torch.from_numpy(t.part_grads(i).astype(np.float32))
        losses[i] = t.part_loss(i)
    dist.all_reduce(slots)
    dist.all_reduce(losses)
    gathered = slots[0].clone()
    for i in range(1, 8):  # ascending partition order
        gathered += slots[i]
    ref = torch.from_numpy(t.gathered().astype(np.float32))
    total = float(sum(losses[i].item() for i in range(8)))
    ok = bool(torch.equal(gathered, ref))
    ref_total = float(sum(t.part_loss(i) for i in range(8)))
    out[rank] = (ok, total == ref_total)
    dist.destroy_process_group()


def test_slot_allreduce_reproduces_ordered_gather_bitwise():
    mgr = mp.Manager()
    out = mgr.dict()
    port = 29500 + os.getpid() % 1000
    mp.start_processes(_worker, args=(2, port, out), nprocs=2, join=True, start_method="spawn")
    assert out[0] == (True, True) and out[1] == (True, True)


@pytest.mark.skipif(not os.path.exists(os.path.join(ROOT, "oracle", "_ref", "libsagecut_ref.so")) and
                    not os.path.exists(os.path.join(ROOT, "oracle", "liboracle.so")), reason="no CPU reference")
def test_bench_reference_arm_under_torchrun():
    port = 29700 + os.getpid() % 200
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2", "--master-addr",
           "127.0.0.1", "--master-port", str(port), os.path.join(ROOT, "bench.py"), "--impl", "reference", "--gpus",
           "2", "--steps", "1", "--warmup", "1", "--config", "er10k"]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout  # rank 0 only
    d = json.loads(lines[0])
    assert d["impl"] == "reference" and d["value"] > 0 and d["cpu_baseline"]["kind"] in ("reference", "port")
    assert d["e2e"]["h2d_bytes_per_step"] == 0
