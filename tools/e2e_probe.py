"""Probe the e2e overhead: device-resident steps vs host-fed steps (sync set_features vs staged).

    python tools/e2e_probe.py [steps]
"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2308_03209_b200 import sagecut as sc  # noqa: E402

K = int(sys.argv[1]) if len(sys.argv) > 1 else 4
cfg = bench.CONFIGS["products"]
ctx = sc.Context(0)
n, uv, feats, labels, tr, va, te = bench.synth_host(cfg, seed=0)
g, _ = sc.build_graph(n, uv, ctx)
g.set_data(feats, labels, cfg["classes"], tr, va, te)
part = sc.partition_random(g, cfg["parts"], 0)
t = sc.CoFreeTrainer(g, part, sc.TrainConfig(layers=3, hidden=[256], learning_rate=3e-3, use_dropedge=True,
                                             dropedge_k=10, drop_ratio=0.5, seed=1))
pinned = torch.from_numpy(feats).pin_memory()
print("pinned:", pinned.is_pinned())
ep = 0
for _ in range(2):
    t.step(ep)
    ep += 1


def run(name, body):
    global ep
    ctx.sync()
    w0 = time.perf_counter()
    ctx.timer_start()
    body()
    ms = ctx.timer_stop()
    print(f"{name}: {ms / K:.1f} ms/step device, {(time.perf_counter() - w0) * 1e3 / K:.1f} ms/step wall", flush=True)


def resident():
    global ep
    for _ in range(K):
        t.step(ep)
        ep += 1


def sync_feed():
    global ep
    for _ in range(K):
        g.set_features(None, host_ptr=pinned.data_ptr())
        t.step(ep)
        ep += 1


def staged():
    global ep
    t.stage_features(host_ptr=pinned.data_ptr())
    for k in range(K):
        t.step_async(ep)
        if k + 1 < K:
            t.stage_features(host_ptr=pinned.data_ptr())
        t.last()
        ep += 1


def copy_only():
    for _ in range(K):
        g.set_features(None, host_ptr=pinned.data_ptr())
    ctx.sync()


for name, body in (("resident", resident), ("sync_feed", sync_feed), ("staged", staged), ("copy_only", copy_only),
                   ("resident", resident), ("staged", staged), ("sync_feed", sync_feed)):
    run(name, body)
