"""One rank of a multi-process CoFree run on a shared GPU (tests/test_gpu_multirank.py).

    python tests/mr_worker.py RANK WORLD PORT CASE OUT.npz

Every rank builds the same graph, holds only its own partitions
(sc_graph_set_part_ownership), creates its trainer with (rank, world) and runs
the library's world > 1 exchange path (trainer.cu: exchange rounds, padding
rounds, bucket-major slots, ordered gather) with a gloo all-gather as the host
transport (sc_trainer_set_exchange) in place of NCCL. World 1 runs with no
exchange at all. Writes per-epoch losses / grad norms and the final parameters.
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

CASES = {
    # name: (graph args, d, p, hidden, dropedge, epochs, seed)
    "sbm_p8": ((200, 4, 0.15, 0.01, 8, 0.3, 7), 8, 8, [16, 16], True, 4, 1),
    "sbm_p7": ((200, 4, 0.15, 0.01, 8, 0.3, 7), 8, 7, [16, 16], True, 4, 1),
    "er_p4": ((10000, 4, 0.004, 0.004, 64, 1.0, 0), 64, 4, [32, 32], True, 3, 0),
}


def main():
    rank, world, port, case, out = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3]), sys.argv[4], sys.argv[5]
    gargs, d, p, hidden, de, epochs, seed = CASES[case]
    from cpu_libs import oracle
    from paper_2308_03209_b200 import sagecut as sc

    og = oracle().graph_sbm(*gargs)
    g, _ = sc.build_graph(og.n, og.edges())
    tr, va, te = og.masks()
    g.set_data(og.features(d).astype(np.float32), og.labels(), int(og.labels().max()) + 1, tr, va, te)
    g.set_part_ownership(rank, world)
    part = sc.partition_random(g, p, 3)
    held = [part.part_held(i) for i in range(p)]
    assert held == [i % world == rank for i in range(p)], held
    cfg = sc.TrainConfig(layers=len(hidden), hidden=hidden, learning_rate=0.01, use_dropedge=de, seed=seed)
    t = sc.CoFreeTrainer(g, part, cfg, rank=rank, world=world) if world == 1 else None
    if world > 1:
        import torch
        import torch.distributed as dist

        dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)

        def allgather(kind, rnd, bucket, send):
            x = torch.frombuffer(bytearray(send), dtype=torch.uint8)
            outs = [torch.empty_like(x) for _ in range(world)]
            dist.all_gather(outs, x)
            return b"".join(o.numpy().tobytes() for o in outs)

        # world > 1 without an NCCL id: the exchange goes through the gloo transport below
        t = sc.CoFreeTrainer(g, part, cfg, rank=rank, world=world, nccl_id=None, _defer_comm=True)
        t.set_exchange(allgather)
    losses, gnorms = [], []
    for e in range(epochs):
        loss, gn = t.step(e)
        losses.append(loss)
        gnorms.append(gn)
    audit = t.comm_audit()
    np.savez(out, losses=np.array(losses), gnorms=np.array(gnorms), params=t.params(), grads=t.grads(),
             audit=np.array(audit, np.uint64), local=np.array([i for i in range(p) if i % world == rank]))
    if world > 1:
        import torch.distributed as dist
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
