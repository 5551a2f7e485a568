"""Multi-rank protocol on CPU (gloo, world_size 2 and 3).

libsagecut_cuda.so trains partition i on rank i % world (exchange round
i // world) and writes its gradient into its own slot. Slots are bucket-major
(trainer.hpp: one bucket per parameter matrix in for_each_matrix order, holding
pp = ceil(p / world) * world per-partition copies), so the copies of one round
are contiguous. As soon as backward finishes a bucket (head, then U_l, W_l for
l = L-1 .. 0) the rank all-gathers that round's range on a comm stream
(trainer.cu:exchange_bucket); the partition loss goes first. A rank without a
partition in the last round (p % world != 0) issues the same sequence on its
zero padding slot. Every slot has one writer, so after the exchange each rank
sums the slots in ascending partition order and gets bitwise the reference's
single-process gather (trainer.hpp:79-94). This test runs that protocol with
the oracle's per-partition gradients over gloo and checks bitwise equality,
plus bench.py's reference arm under torchrun (rank 0 prints, rank 1 exits 0).
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


def _buckets(d, hidden, C):
    """for_each_matrix offsets: W_l (H x in), U_l (H x (H + in)), ..., head (C x E); last = |theta|."""
    off, b, inp = 0, [], d
    for H in hidden:
        b.append(off)
        off += H * inp
        b.append(off)
        off += H * (H + inp)
        inp = H
    b.append(off)
    off += C * inp
    b.append(off)
    return b


def _worker(rank, world, port, out):
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    from cpu_libs import oracle
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    O = oracle()
    g = O.graph_sbm(200, 4, 0.15, 0.01, 8, 0.3, 7)
    p = 8
    part = g.partition("random", p, 3)
    t = part.trainer([16, 16], lr=0.01, dropedge=True, seed=1, f32=True)
    t.step(0)  # computes every partition's gradient (single-process reference)
    P = t.nparam
    b_off = _buckets(8, [16, 16], 4)
    assert b_off[-1] == P
    nb = len(b_off) - 1
    pp = -(-p // world) * world
    slots = torch.zeros(P * pp, dtype=torch.float32)
    losses = torch.zeros(pp, dtype=torch.float64)

    def slot(b, i):
        ln = b_off[b + 1] - b_off[b]
        return slots[b_off[b] * pp + i * ln: b_off[b] * pp + (i + 1) * ln]

    def exchange(b, j):  # all-gather round j's contiguous range of bucket b (or the losses, b = -1)
        if b < 0:
            chunk = losses[j * world: (j + 1) * world]
        else:
            ln = b_off[b + 1] - b_off[b]
            chunk = slots[b_off[b] * pp + j * world * ln: b_off[b] * pp + (j + 1) * world * ln]
        parts = list(chunk.chunk(world))
        mine = parts[rank].clone()
        dist.all_gather(parts, mine)  # gloo: list form, written in place into the views

    for j in range(pp // world):
        i = j * world + rank
        if i < p:  # forward + loss, then backward emits buckets head, U_{L-1}, W_{L-1}, ..., W_0
            losses[i] = t.part_loss(i)
            exchange(-1, j)
            g_i = torch.from_numpy(t.part_grads(i).astype(np.float32))
            for b in range(nb - 1, -1, -1):
                slot(b, i).copy_(g_i[b_off[b]:b_off[b + 1]])
                exchange(b, j)
        else:  # idle rank: same collective sequence on its padding slot
            exchange(-1, j)
            for b in range(nb - 1, -1, -1):
                exchange(b, j)
    gathered = torch.empty(P, dtype=torch.float32)
    for b in range(nb):
        acc = slot(b, 0).clone()
        for i in range(1, p):  # ascending partition order
            acc += slot(b, i)
        gathered[b_off[b]:b_off[b + 1]] = acc
    ref = torch.from_numpy(t.gathered().astype(np.float32))
    total = float(sum(losses[i].item() for i in range(p)))
    ok = bool(torch.equal(gathered, ref))
    ref_total = float(sum(t.part_loss(i) for i in range(p)))
    out[rank] = (ok, total == ref_total)
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_bucketed_allgather_reproduces_ordered_gather_bitwise(world):
    mgr = mp.Manager()
    out = mgr.dict()
    port = 29500 + (os.getpid() * 7 + world) % 1000
    mp.start_processes(_worker, args=(world, port, out), nprocs=world, join=True, start_method="spawn")
    assert all(out[r] == (True, True) for r in range(world)), dict(out)


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
