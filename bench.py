#!/usr/bin/env python
"""Benchmark: one CoFree-GNN training epoch (all p vertex-cut partitions:
forward, weighted loss, backward, gradient exchange, Adam) on B200s.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]
                    [--config products|reddit|er10k]
    torchrun --nproc-per-node N bench.py --gpus N ...

Metric (BASELINE.json): epoch time and aggregated edges/s,
    edges/s = L * sum_i kept_CSR_entries_i / epoch_time
(forward directed edge traversals; with DropEdge only kept entries count),
plus the aggregation (SpMM) kernel's fraction of the measured HBM roofline.

Scaling: the partition count p is FIXED (8 for the products/reddit shapes)
and the p partitions are spread over the N GPUs (partition i on rank i % N),
so total work is constant as N grows ("strong"). The only cross-GPU traffic is
the per-epoch gradient all-reduce (NCCL) inside libsagecut_cuda.so.

--impl reference times the reference's own CPU implementation
(oracle/_ref = the unmodified reference sources built behind the Eigen shim;
falls back to the oracle port) on a bounded sample of the same workload.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CONFIGS = {
    # configs[2]: the headline (products-shaped, 3-layer GraphSAGE 256, DropEdge p=0.5)
    "products": dict(workload="ogbn-products-shaped synthetic (BASELINE configs[2])", nodes=2_449_029,
                     pairs=62_000_000, feats=100, classes=47, layers=3, hidden=256, parts=8, dropedge=True, k=10,
                     ratio=0.5, lr=3e-3),
    # configs[1]: Reddit-shaped; 114.6M directed = 57.3M undirected edges; SAGE (no GCN in the reference)
    "reddit": dict(workload="Reddit-shaped synthetic (BASELINE configs[1])", nodes=232_965, pairs=57_400_000,
                   feats=602, classes=41, layers=2, hidden=256, parts=8, dropedge=False, k=10, ratio=0.5, lr=1e-2),
    # configs[3]: power-law R-MAT (a,b,c,d) = (0.57,0.19,0.19,0.05), 20M nodes / 1B edge samples, 128 feats,
    # 3 x 256 SAGE (47 classes: the survey's choice). Full size needs > 180 GB at N = 1 (activations of
    # ~7.5M-row partitions plus the 1B-edge graph); --scale 0.25 (5M / 250M) is the default single-GPU size.
    "rmat": dict(workload="power-law R-MAT synthetic (BASELINE configs[3])", nodes=20_000_000, pairs=1_000_000_000,
                 feats=128, classes=47, layers=3, hidden=256, parts=8, dropedge=False, k=10, ratio=0.5, lr=3e-3,
                 rmat=(0.57, 0.19, 0.19, 0.05), default_scale=0.25),
    # configs[3] at FULL size (20M nodes / 1B samples) on one GPU: p = 16 partitions time-multiplexed
    # (the layout 8 GPUs would run as two partitions each); activations switch to the compact set
    # (shared msg buffer + ReLU sign bits) automatically when the per-layer set would not fit.
    "rmat_full": dict(workload="power-law R-MAT synthetic (BASELINE configs[3]), full size, p = 16",
                      nodes=20_000_000, pairs=1_000_000_000, feats=128, classes=47, layers=3, hidden=256, parts=16,
                      dropedge=False, k=10, ratio=0.5, lr=3e-3, rmat=(0.57, 0.19, 0.19, 0.05), default_scale=1.0),
    # configs[4]: ogbn-papers100M-shaped (111M nodes / 1.6B edges, 128 feats, 172 classes, 3 layers, hidden
    # 128 = the paper's; SAGE: no GCN in the reference). One vertex-cut partition per GPU (p = 8) is
    # memory-infeasible: a random cut puts ~98 % of the nodes in every partition (55 GB per activation
    # matrix). The job runs p = 1024 partitions over 8 GPUs (128 per rank, time-multiplexed); on this
    # 1-GPU box the bench runs rank 0's share of that job (sc_trainer_emulate_rank: the rank holds only
    # its partitions, exchanges skipped). Graph, features and labels are generated on the device.
    "papers": dict(workload="ogbn-papers100M-shaped synthetic (BASELINE configs[4]), p = 1024 over 8 GPUs: "
                            "rank 0's share on one B200", nodes=111_059_956, pairs=1_615_685_872, feats=128,
                   classes=172, layers=3, hidden=128, parts=1024, dropedge=False, k=10, ratio=0.5, lr=3e-3,
                   device_gen=True, emulate_world=8, full_graph_eval=False, e2e=False),
    # configs[0]: ER 10k / 200k, 64 feats, 2 layers (reference default hidden 32), p = 4
    "er10k": dict(workload="Erdos-Renyi 10k/200k (BASELINE configs[0])", nodes=10_000, pairs=200_000, feats=64,
                  classes=4, layers=2, hidden=32, parts=4, dropedge=False, k=10, ratio=0.5, lr=1e-2),
}


def dist_env():
    return int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)), int(os.environ.get("LOCAL_RANK", 0))


# ---------------------------------------------------------------------------- data
def synth_host(cfg, seed=0, scale=1.0):
    """O(E) seeded synthetic graph of the config's shape (never the reference's O(n^2) generators).
    Uniform random endpoint pairs (canonicalised/deduped by build_graph), labels uniform, features
    one-hot(label) + N(0, 1) (synth.cpp:91-97 convention), 60/20/20 split."""
    rng = np.random.default_rng(seed)
    n = max(int(cfg["nodes"] * scale), 16)
    m = max(int(cfg["pairs"] * scale), 16)
    if "rmat" in cfg:
        feats, labels, tr, va, te = synth_data(n, cfg, seed)
        return n, rmat_edges(n, m, cfg["rmat"], seed).numpy(), feats, labels, tr, va, te
    uv = rng.integers(0, n, size=(m, 2), dtype=np.int32)
    labels = rng.integers(0, cfg["classes"], size=n, dtype=np.int32)
    feats = rng.standard_normal((n, cfg["feats"]), dtype=np.float32)
    feats[np.arange(n), labels % cfg["feats"]] += 1.0
    perm = rng.permutation(n)
    tr = np.zeros(n, np.uint8)
    va = np.zeros(n, np.uint8)
    te = np.zeros(n, np.uint8)
    n_tr, n_va = n * 6 // 10, n * 2 // 10
    tr[perm[:n_tr]] = 1
    va[perm[n_tr:n_tr + n_va]] = 1
    te[perm[n_tr + n_va:]] = 1
    return n, uv, feats, labels, tr, va, te


def rmat_edges(n, m, abcd, seed=0, device=None):
    """R-MAT edge samples (Chakrabarti et al.): each endpoint bit picks a quadrant with probabilities
    (a, b, c, d) over 2^L >= n ids, ids folded into [0, n) and randomly relabelled (hubs spread out).
    O(m log n); generated on the GPU with torch when `device` is given (input synthesis only)."""
    import torch
    a, b, c, _ = abcd
    L = max(1, int(math.ceil(math.log2(n))))
    gen = torch.Generator(device=device or "cpu").manual_seed(seed)
    perm = torch.randperm(n, generator=gen, device=device or "cpu").to(torch.int64)
    out = torch.empty((m, 2), dtype=torch.int32, device=device or "cpu")
    chunk = 1 << 25
    for s0 in range(0, m, chunk):
        k = min(chunk, m - s0)
        u = torch.zeros(k, dtype=torch.int64, device=device or "cpu")
        v = torch.zeros_like(u)
        for _ in range(L):
            r = torch.rand(k, generator=gen, device=device or "cpu")
            ub = r >= a + b                              # quadrants c, d: row bit 1
            vb = ((r >= a) & (r < a + b)) | (r >= a + b + c)  # quadrants b, d: column bit 1
            u = (u << 1) | ub.to(torch.int64)
            v = (v << 1) | vb.to(torch.int64)
        out[s0:s0 + k, 0] = perm[u % n].to(torch.int32)
        out[s0:s0 + k, 1] = perm[v % n].to(torch.int32)
    return out


def synth_data(n, cfg, seed=0):
    """labels uniform, features one-hot(label) + N(0, 1), 60/20/20 split (synth.cpp:91-97 convention)."""
    rng = np.random.default_rng(seed + 1)
    labels = rng.integers(0, cfg["classes"], size=n, dtype=np.int32)
    feats = rng.standard_normal((n, cfg["feats"]), dtype=np.float32)
    feats[np.arange(n), labels % cfg["feats"]] += 1.0
    perm = rng.permutation(n)
    tr, va, te = (np.zeros(n, np.uint8) for _ in range(3))
    n_tr, n_va = n * 6 // 10, n * 2 // 10
    tr[perm[:n_tr]] = 1
    va[perm[n_tr:n_tr + n_va]] = 1
    te[perm[n_tr + n_va:]] = 1
    return feats, labels, tr, va, te


def synth_device(cfg, scale, device):
    """Device-side synthesis for graphs too large for host numpy (configs[4]): uniform random endpoint
    pairs (canonicalised / deduped by build_graph), labels uniform, 60/20/20 split; features are filled
    afterwards by fill_features_device (same convention as synth_data). Returns (n, uv_dev, labels,
    train, val, test) with uv_dev an int32 [m, 2] device tensor."""
    import torch
    n = max(int(cfg["nodes"] * scale), 16)
    m = max(int(cfg["pairs"] * scale), 16)
    gen = torch.Generator(device=device).manual_seed(0)
    uv = torch.empty((m, 2), dtype=torch.int32, device=device)
    chunk = 1 << 27
    for s0 in range(0, m, chunk):
        k = min(chunk, m - s0)
        uv[s0:s0 + k] = torch.randint(0, n, (k, 2), generator=gen, device=device, dtype=torch.int32)
    labels = torch.randint(0, cfg["classes"], (n,), generator=gen, device=device, dtype=torch.int32)
    perm = torch.randperm(n, generator=gen, device=device)
    split = torch.zeros(n, dtype=torch.uint8, device=device)
    n_tr, n_va = n * 6 // 10, n * 2 // 10
    split[perm[n_tr:n_tr + n_va]] = 1
    split[perm[n_tr + n_va:]] = 2
    del perm
    sp = split.cpu().numpy()
    tr, va, te = ((sp == c).astype(np.uint8) for c in range(3))
    torch.cuda.synchronize(device)
    return n, uv, labels, tr, va, te


def fill_features_device(g, labels_dev, cfg, device, rows_per_chunk=1 << 22):
    """features = N(0, 1) + one-hot(label mod d), written chunk by chunk into the library's zero
    feature matrix (sc_graph_set_feature_rows) so no second n x d copy exists."""
    import torch
    gen = torch.Generator(device=device).manual_seed(1)
    n, d = labels_dev.shape[0], cfg["feats"]
    for r0 in range(0, n, rows_per_chunk):
        k = min(rows_per_chunk, n - r0)
        x = torch.randn((k, d), generator=gen, device=device, dtype=torch.float32)
        x[torch.arange(k, device=device), (labels_dev[r0:r0 + k] % d).long()] += 1.0
        torch.cuda.synchronize(device)
        g.set_feature_rows(r0, device_ptr=x.data_ptr(), num_rows=k)
        del x


def kept_entries(sizes_m, cfg):
    """sum_i CSR entries kept per epoch: every DropEdge mask keeps exactly ceil((1-r) m_i) edges."""
    if cfg["dropedge"]:
        return sum(2 * math.ceil((1.0 - cfg["ratio"]) * m) for m in sizes_m)
    return sum(2 * m for m in sizes_m)


# ---------------------------------------------------------------------------- clocks
class ClockSampler:
    def __init__(self, gpu_index=0):
        self.samples, self.proc, self.gpu = [], None, gpu_index

    def __enter__(self):
        q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={q}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except FileNotFoundError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            parts = [x.strip() for x in line.split(",")]
            if len(parts) >= 8:
                self.samples.append(parts)

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except Exception:
                self.proc.kill()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4) if s[4 + i].lower() == "active"})
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.samples)}


def measured_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def measured_tensor_peak():
    """Sustained dense bf16 TF/s (a GEMM timed inside a long step), per the profiling recipe."""
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p.get("bf16_tflops_sustained") or p["bf16_tflops"]), "measured (sustained)"
    except Exception:
        return 2250.0, "fallback (nominal dense bf16)"


def ncu_traffic(config, scale):
    """Per-launch DRAM bytes (dram__bytes_read.sum + dram__bytes_write.sum) of the aggregation kernels
    for THIS config and scale, from the committed ncu capture (profiles/ncu_traffic.json, written by
    tools/ncu_traffic.py), or None when that config was not captured."""
    path = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    try:
        with open(path) as f:
            entry = json.load(f).get(f"{config}@{scale:g}")
        return entry if isinstance(entry, dict) else None
    except Exception:
        return None


def host_info():
    """CPU model, host threads and RAM of the machine the CPU baseline runs on."""
    model, mem_gb = None, None
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    model = line.split(":", 1)[1].strip()
                    break
        with open("/proc/meminfo") as f:
            for line in f:
                if line.startswith("MemTotal"):
                    mem_gb = round(int(line.split()[1]) / 1e6, 1)
                    break
    except OSError:
        pass
    return {"cpu_model": model, "host_threads": os.cpu_count(), "ram_gb": mem_gb}


# ---------------------------------------------------------------------------- CPU reference
def cpu_reference_sample(cfg, steps, warmup, scale=None):
    """The reference's own training epoch (train_cofree_impl minus the per-epoch eval) on a bounded
    sample of the same workload shape, all host threads (workers = min(p, nproc))."""
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    import cpu_libs

    kind = "reference"
    try:
        lib = cpu_libs.reference()
    except (FileNotFoundError, OSError):
        lib, kind = cpu_libs.oracle(), "port"
    if scale is None:
        scale = min(1.0, 50_000 / cfg["nodes"])
    n, uv, feats, labels, tr, va, te = synth_host(cfg, seed=0, scale=scale)
    g = lib.graph_build(n, uv)
    g.set_data(feats, labels, cfg["classes"], tr, va, te)
    part = g.partition("random", cfg["parts"], 0)
    cores = min(cfg["parts"], os.cpu_count() or 1)
    t = part.trainer([cfg["hidden"]] * cfg["layers"], lr=cfg["lr"], dropedge=cfg["dropedge"], k=cfg["k"],
                     ratio=cfg["ratio"], seed=1, f32=True, workers=cores)
    kept = kept_entries([part.sizes(i)[1] for i in range(cfg["parts"])], cfg)
    for e in range(warmup):
        t.step(e)
    t0 = time.perf_counter()
    for e in range(steps):
        t.step(warmup + e)
    sec = (time.perf_counter() - t0) / max(steps, 1)
    value = cfg["layers"] * kept / sec
    sample = (f"{n} nodes / {g.m} edges (scale {scale:.4f} of the config, same avg degree, feats, layers, hidden, "
              f"p, DropEdge), {steps} epoch(s) after {warmup} warm-up, no per-epoch eval")
    blas = None
    if kind == "reference":
        try:
            blas = bool(lib.lib.ref_blas_active())
        except Exception:
            pass
    return dict(value=value, unit="edges/s", cores=cores, kind=kind, sample=sample, epoch_s=sec, host=host_info(),
                gemm_backend=("OpenBLAS sgemm, 1 thread/worker" if blas else "shim loop GEMM") if kind == "reference"
                else "oracle loops")


def full_scale_reference():
    """The committed full-scale measurement of the reference: one products partition's
    training step timed at full size on the GPU box's host, extrapolated x p (profiles/, written by
    `bench.py --cpu-full-partition`), or None."""
    path = os.path.join(ROOT, "profiles", "r02_reference_full_partition.json")
    try:
        with open(path) as f:
            return json.load(f)
    except Exception:
        return None


def cpu_full_partition(cfg, part_index=0):
    """the reference's per-partition training step (forward + loss + backward of
    train_cofree_impl's worker, 1 thread) on ONE partition of the FULL-size workload, timed once, then
    extrapolated to an epoch: x p with one worker, x ceil(p / workers) with `workers` threads (the
    reference runs min(workers, p) partitions at a time; memory permitting)."""
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    import cpu_libs

    lib = cpu_libs.reference()
    t0 = time.perf_counter()
    n, uv, feats, labels, tr, va, te = synth_host(cfg, seed=0)
    g = lib.graph_build(n, uv)
    del uv
    g.set_data(feats, labels, cfg["classes"], tr, va, te)
    part = g.partition("random", cfg["parts"], 0)
    t = part.trainer([cfg["hidden"]] * cfg["layers"], lr=cfg["lr"], dropedge=cfg["dropedge"], k=cfg["k"],
                     ratio=cfg["ratio"], seed=1, f32=True, workers=1)
    setup = time.perf_counter() - t0
    sec = t.time_part_step(part_index, 0, 1)
    p = cfg["parts"]
    kept = kept_entries([part.sizes(i)[1] for i in range(p)], cfg)
    workers = min(p, os.cpu_count() or 1)
    epoch1 = sec * p
    epochw = sec * math.ceil(p / workers)
    return {"kind": "reference", "what": "one full-scale partition's step (1 thread), extrapolated",
            "partition": part_index, "partition_step_s": sec, "setup_s": setup,
            "epoch_s_1_worker": epoch1, "edges_per_s_1_worker": cfg["layers"] * kept / epoch1,
            "workers": workers, "epoch_s_workers": epochw, "edges_per_s_workers": cfg["layers"] * kept / epochw,
            "host": host_info(), "workload": cfg["workload"]}


def run_reference_arm(args, cfg):
    rank, world, _ = dist_env()
    if rank != 0:
        return
    res = cpu_reference_sample(cfg, args.steps, args.warmup)
    line = {"impl": "reference", "metric": "aggregated_edges_per_s", "value": res["value"], "unit": "edges/s",
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup, "ms_per_step": res["epoch_s"] * 1e3,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": {"workload": cfg["workload"] + " [bounded CPU sample]", "partitions": cfg["parts"],
                       "layers": cfg["layers"], "hidden": cfg["hidden"], "feats": cfg["feats"],
                       "classes": cfg["classes"], "dropedge": cfg["dropedge"]},
            "cpu_baseline": {"value": res["value"], "unit": "edges/s", "cores": res["cores"], "kind": res["kind"],
                             "sample": res["sample"], "gemm": res["gemm_backend"], "host": res["host"],
                             "full_scale_extrapolated": full_scale_reference()},
            "e2e": {"value": res["value"], "unit": "edges/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------- GPU arm
def run_gpu_arm(args, cfg):
    rank, world, local = dist_env()
    import torch

    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("gloo")
    from paper_2308_03209_b200 import sagecut as sc

    ctx = sc.Context(local)
    t_setup = time.perf_counter()
    # identical seeded synthetic inputs on every rank (generated once per rank)
    scale = args.scale if args.scale is not None else cfg.get("default_scale", 1.0)
    emu = cfg.get("emulate_world", 0) if world == 1 else 0  # one rank of a larger job on this GPU
    feats = None
    if cfg.get("device_gen"):  # too large for host synthesis: edges, labels and features on the device
        n, uv_dev, labels_dev, tr, va, te = synth_device(cfg, scale, f"cuda:{local}")
        g, rep = sc.build_graph_device(n, uv_dev.data_ptr(), uv_dev.shape[0], ctx)
        del uv_dev
        torch.cuda.empty_cache()
        g.set_data(None, labels_dev.cpu().numpy(), cfg["classes"], tr, va, te, dim=cfg["feats"])
        fill_features_device(g, labels_dev, cfg, f"cuda:{local}")
        del labels_dev
        torch.cuda.empty_cache()
    elif "rmat" in cfg:  # R-MAT edges are sampled on the device and handed over as a device edge list
        n = max(int(cfg["nodes"] * scale), 16)
        uv_dev = rmat_edges(n, max(int(cfg["pairs"] * scale), 16), cfg["rmat"], seed=0, device=f"cuda:{local}")
        torch.cuda.synchronize()  # generated on torch's stream; the library reads it on its own
        feats, labels, tr, va, te = synth_data(n, cfg, 0)
        g, rep = sc.build_graph_device(n, uv_dev.data_ptr(), uv_dev.shape[0], ctx)
        del uv_dev
        torch.cuda.empty_cache()
    else:
        n, uv, feats, labels, tr, va, te = synth_host(cfg, seed=0, scale=scale)
        g, rep = sc.build_graph(n, uv, ctx)
    if feats is not None:
        g.set_data(feats, labels, cfg["classes"], tr, va, te)
    if emu:
        g.set_part_ownership(0, emu)  # rank 0 holds (and trains) partitions i % emu == 0 only
    partitioner = getattr(args, "partitioner", "random")
    part = {"random": sc.partition_random, "dbh": sc.partition_dbh,
            "ne": sc.partition_ne}[partitioner](g, cfg["parts"], 0)
    sizes_all = [part.part_sizes(i)[1] for i in range(cfg["parts"])]
    mine = range(rank, cfg["parts"], world) if not emu else range(0, cfg["parts"], emu)
    sizes_m = [sizes_all[i] for i in mine] if emu else sizes_all
    deg = g.degrees()
    degree_stats = {"max": int(deg.max()), "mean": float(deg.mean()), "p99": float(np.percentile(deg, 99)),
                    "isolated": int((deg == 0).sum())}
    del deg
    kept = kept_entries(sizes_m, cfg)
    kept_spread = 0.0
    if emu:
        per_rank = [kept_entries(sizes_all[r::emu], cfg) for r in range(emu)]
        kept_spread = (max(per_rank) - min(per_rank)) / max(per_rank)
    nccl_id = None
    if world > 1:
        obj = [sc.CoFreeTrainer.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        nccl_id = obj[0]
    tcfg = sc.TrainConfig(layers=cfg["layers"], hidden=[cfg["hidden"]], learning_rate=cfg["lr"],
                          use_dropedge=cfg["dropedge"], dropedge_k=cfg["k"], drop_ratio=cfg["ratio"], seed=1,
                          gemm=args.gemm)
    if emu:
        trainer = sc.CoFreeTrainer(g, part, tcfg, rank=0, world=emu, _defer_comm=True)
        trainer.emulate_rank()
    else:
        trainer = sc.CoFreeTrainer(g, part, tcfg, rank=rank, world=world, nccl_id=nccl_id)
    setup_s = time.perf_counter() - t_setup

    def barrier():
        if dist:
            dist.barrier()

    def max_over_ranks(x):
        if not dist:
            return x
        t = torch.tensor([x], dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    epoch = 0
    for _ in range(args.warmup):
        trainer.step(epoch)
        epoch += 1
    # ---- timed region (the headline value): K epochs, no profiling events, device time on the
    # library's stream between a barrier + sync on both sides
    trainer.profile(False)
    barrier()
    ctx.sync()
    launches0 = ctx.launch_count()
    def fallback_count():
        try:
            return trainer.fallback_count()
        except AttributeError:  # an older library build under SC_LIB (A/B runs)
            return -1

    fallbacks0 = fallback_count()
    losses = []
    with ClockSampler(local) as clocks:
        ctx.timer_start()
        for _ in range(args.steps):
            losses.append(trainer.step(epoch)[0])
            epoch += 1
        ms = ctx.timer_stop()
    launches = ctx.launch_count() - launches0
    fallbacks = fallback_count() - fallbacks0
    free_b, total_b = torch.cuda.mem_get_info(local)  # device memory in use (graph, partitions, trainer)
    try:
        mem_mode = trainer.memory_mode()
    except AttributeError:  # an older library build under SC_LIB (A/B runs)
        mem_mode = None
    barrier()
    ms_step = max_over_ranks(ms / args.steps)
    value = cfg["layers"] * kept / (ms_step / 1e3)

    # ---- breakdown pass (separate, not part of `value`): the same K epochs with CUDA events around
    # every kernel group on the stream it runs on; the roofline objects come from here
    trainer.profile(True)
    prof, flops = {}, {}
    barrier()
    ctx.sync()
    ctx.timer_start()
    for _ in range(args.steps):
        trainer.step(epoch)
        fl = trainer.kernel_flops()
        for k, (kms, by) in trainer.kernel_times().items():
            flops[k] = flops.get(k, 0.0) + fl.get(k, 0.0)
            a = prof.setdefault(k, [0.0, 0.0])
            a[0] += kms
            a[1] += by
        epoch += 1
    prof_ms = ctx.timer_stop() / args.steps
    trainer.profile(False)

    # ---- full-graph evaluation (evaluate_splits, trainer.hpp:306), timed apart from the epoch
    eval_metrics, eval_ms = None, None
    if cfg.get("full_graph_eval", True):
        ctx.sync()
        ctx.timer_start()
        eval_metrics = trainer.evaluate()
        eval_ms = ctx.timer_stop()

    # ---- e2e: the public API with host buffers: every step's input (the feature matrix, from pinned
    # host memory) is copied host -> device inside the timed region and the loss, grad-norm (f64) and
    # non-finite flag (i32) read back (20 bytes).
    # Step k+1's copy (and its partitions' layer-0 row gathers) is staged on the library's copy
    # stream while step k computes; step 0's copy is exposed.
    e2e = None
    if cfg.get("e2e", True):
        pinned = torch.from_numpy(feats).pin_memory()
        barrier()
        ctx.sync()
        ctx.timer_start()
        trainer.stage_features(host_ptr=pinned.data_ptr())
        for k in range(args.steps):
            trainer.step_async(epoch)  # commits the staged features
            if k + 1 < args.steps:
                trainer.stage_features(host_ptr=pinned.data_ptr())
            trainer.last()
            epoch += 1
        e2e_ms = max_over_ranks(ctx.timer_stop() / args.steps)
        e2e = {"value": cfg["layers"] * kept / (e2e_ms / 1e3), "unit": "edges/s", "ms_per_step": e2e_ms,
               "h2d_bytes_per_step": int(feats.nbytes), "d2h_bytes_per_step": 20}

    if rank != 0:
        if dist:
            dist.destroy_process_group()
        return
    peak, peak_kind = measured_peaks()
    # aggregation groups: H-wide layers, and (projected top layer) the Cp-wide top-layer aggregations
    spmm_groups = ("spmm_fwd", "spmm_bwd", "spmm_fwd_top", "spmm_bwd_top")
    spmm_ms = sum(prof.get(k, [0, 0])[0] for k in spmm_groups)
    spmm_bytes = sum(prof.get(k, [0, 0])[1] for k in spmm_groups)
    launches_dir = cfg["layers"] * len(mine) * args.steps  # per direction
    launches_spmm = 2 * launches_dir
    achieved = spmm_bytes / (spmm_ms / 1e3) / 1e9 if spmm_ms > 0 else 0.0
    # DRAM-measured view (ncu, this config): what the kernel actually moved. When the algorithmic
    # bytes exceed it (L2-resident message rows, e.g. Reddit's 239 MB msg matrix), the algorithmic
    # fraction can pass 1; the DRAM fraction stays a true roofline fraction.
    traffic = ncu_traffic(args.config, scale)
    dram = None
    if traffic and spmm_ms > 0 and "spmm_fwd" in traffic and "spmm_bwd" in traffic:
        dram_bytes = launches_dir * (traffic["spmm_fwd"] + traffic["spmm_bwd"])
        dram = {"GB_per_s": dram_bytes / (spmm_ms / 1e3) / 1e9, "frac": dram_bytes / (spmm_ms / 1e3) / 1e9 / peak,
                "bytes_per_launch_fwd": traffic["spmm_fwd"], "bytes_per_launch_bwd": traffic["spmm_bwd"],
                "source": traffic.get("source")}
    props = torch.cuda.get_device_properties(local)
    l2_bytes = getattr(props, "L2_cache_size", None)
    max_rows = max(part.part_sizes(i)[0] for i in range(cfg["parts"]))
    act_bytes = max_rows * cfg["hidden"] * 4
    total_prof = sum(v[0] for v in prof.values())
    tpeak_all, _ = measured_tensor_peak()

    def bound_frac(k, v):
        """lower-bound time of the group (its algorithmic bytes at the HBM peak, its executed fp16x3 MMA
        flops at the measured dense tensor peak — whichever is larger) over its measured time"""
        if v[0] <= 0 or not peak:
            return None
        t_hbm = v[1] / (peak * 1e9)
        t_tc = 3 * flops.get(k, 0.0) / (tpeak_all * 1e12) if tpeak_all else 0.0
        return max(t_hbm, t_tc) / (v[0] / 1e3)

    kernels = {k: {"ms_per_step": v[0] / args.steps, "share": v[0] / total_prof if total_prof else None,
                   "GB_per_s": (v[1] / (v[0] / 1e3) / 1e9) if v[0] > 0 and v[1] > 0 else None,
                   "TFLOP_per_s_fp16x3": (3 * flops[k] / (v[0] / 1e3) / 1e12) if flops.get(k) and v[0] > 0 else None,
                   "frac_of_bound": bound_frac(k, v)}
               for k, v in sorted(prof.items(), key=lambda kv: -kv[1][0])}
    dominant = max(prof.items(), key=lambda kv: kv[1][0])[0] if prof else None
    # tensor roofline of the dominant GEMM group: fp16x3 issues three fp16 MMAs per fp32-equivalent
    # product, so the tensor pipe executes 3x the algorithmic 2MNK flops
    gemm_groups = [k for k in prof if flops.get(k, 0) > 0]
    gdom = max(gemm_groups, key=lambda k: prof[k][0]) if gemm_groups else None
    tpeak, tpeak_kind = measured_tensor_peak()
    roofline_gemm = None
    if gdom:
        alg = flops[gdom] / (prof[gdom][0] / 1e3) / 1e12
        roofline_gemm = {"kernel": f"{gdom} (tcgen05 fp16x3)", "bound": "tensor", "achieved": 3 * alg,
                         "algorithmic_tflops": alg, "peak": tpeak, "peak_kind": tpeak_kind, "unit": "TFLOP/s",
                         "frac": 3 * alg / tpeak, "hbm_GB_per_s": prof[gdom][1] / (prof[gdom][0] / 1e3) / 1e9,
                         "note": "achieved = executed fp16 MMA flops (3 x 2MNK) / measured kernel time; the SM "
                                 "clock sits at the power cap (see clocks)"}
    cpu = None
    if world == 1 and not args.no_cpu_baseline:
        try:
            cpu = cpu_reference_sample(cfg, steps=1, warmup=0)
            cpu = {k: cpu[k] for k in ("value", "unit", "cores", "kind", "sample", "host")}
            cpu["full_scale_extrapolated"] = full_scale_reference()
        except Exception as e:  # the baseline must not sink the GPU line
            cpu = {"value": None, "unit": "edges/s", "cores": 0, "kind": "unavailable", "sample": str(e)}
    line = {
        "metric": "aggregated_edges_per_s", "value": value, "unit": "edges/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": {"workload": cfg["workload"] + (f" [scale {scale}]" if scale != 1.0 else ""),
                   "nodes": g.num_nodes, "edges": g.num_edges(),
                   "feats": cfg["feats"], "classes": cfg["classes"], "layers": cfg["layers"],
                   "hidden": cfg["hidden"], "partitions": cfg["parts"],
                   "partitioner": {"random": "random vertex cut", "dbh": "DBH vertex cut",
                                   "ne": "neighbour-expansion vertex cut"}[partitioner],
                   "dropedge": f"p={cfg['ratio']} K={cfg['k']}" if cfg["dropedge"] else None,
                   "degrees": degree_stats, "rf": sc.replication_stats(part, g).rf,
                   "kept_csr_entries_per_epoch": kept, "parallelism": f"dp{world} over {cfg['parts']} fixed partitions",
                   "gemm": args.gemm,
                   "l2": {"l2_bytes": l2_bytes, "activation_matrix_bytes": act_bytes,
                          "inputs_exceed_l2": bool(l2_bytes and act_bytes > l2_bytes),
                          "note": "no L2 flush between steps: every step streams activation matrices of "
                                  f"{act_bytes / 1e9:.2f} GB (largest partition x hidden x 4 B) "
                                  + ("> L2" if l2_bytes and act_bytes > l2_bytes else "<= L2 (partly L2-resident)")}},
        "epoch_ms": ms_step,
        "timing": "value: unprofiled timed region; kernels / roofline: a separate profiled pass of the same K "
                  f"epochs ({prof_ms:.2f} ms/epoch with events)",
        "roofline": {"kernel": "spmm (masked mean aggregation fwd + transposed bwd)", "bound": "hbm",
                     "achieved": achieved, "peak": peak, "peak_kind": peak_kind, "unit": "GB/s",
                     "frac": achieved / peak if peak else None,
                     "traffic": ((traffic["spmm_fwd"] + traffic["spmm_bwd"]) / 2 if dram else None),
                     "launches": launches_spmm,
                     "bytes_per_launch": spmm_bytes / max(launches_spmm, 1),
                     "share_of_step": spmm_ms / total_prof if total_prof else None,
                     "by_group": {k: {"ms_per_step": prof[k][0] / args.steps,
                                      "GB_per_s": prof[k][1] / (prof[k][0] / 1e3) / 1e9,
                                      "frac": prof[k][1] / (prof[k][0] / 1e3) / 1e9 / peak if peak else None}
                                  for k in spmm_groups if k in prof and prof[k][0] > 0},
                     "dram_measured": dram},
        "dominant_kernel": dominant,
        "roofline_gemm": roofline_gemm,
        "kernels": kernels,
        "cpu_baseline": cpu,
        "e2e": e2e if e2e else {"value": None, "note": "not measured for this config: staging the next step's "
                                                       "n x d features needs a second feature matrix on the device"},
        "gpu_launches": launches,
        "simt_fallbacks": fallbacks,
        "eval": ({"ms": eval_ms, "train_val_test": list(eval_metrics),
                  "note": "full-graph evaluate_splits (trainer.hpp:306), not in the epoch time"} if eval_metrics
                 else {"ms": None, "note": "full-graph evaluation not run for this config: its forward-only "
                                           "buffers (4 x n x hidden fp32) exceed one GPU"}),
        "clocks": clocks.summary(),
        "setup_s": setup_s,
        "hbm_used_gb": round((total_b - free_b) / 1e9, 1),
        "memory_mode": mem_mode,
        "emulated_rank": ({"world": emu, "rank": 0, "partitions_held": len(mine),
                           "kept_csr_entries_all_ranks": kept_entries(sizes_all, cfg),
                           "projected_job_edges_per_s": cfg["layers"] * kept_entries(sizes_all, cfg) / (ms_step / 1e3),
                           "note": f"rank 0 of a {emu}-GPU job on one GPU: it holds and trains only its partitions "
                                   "(i % world == 0); the gradient all-gathers are skipped (no peers), so the "
                                   "projection assumes the exchange stays hidden behind backward as at N <= 8 and "
                                   "equal per-rank work (random cut: per-rank kept entries within "
                                   f"{kept_spread:.2%})"} if emu else None),
        "loss_first_last": [losses[0], losses[-1]] if losses else None,
    }
    print(json.dumps(line), flush=True)
    if dist:
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--config", default="products", choices=sorted(CONFIGS))
    ap.add_argument("--gemm", default="auto", choices=["auto", "simt"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-full-partition", action="store_true",
                    help="time the reference on one FULL-size partition (minutes of CPU; BASELINE.md §3) and write "
                         "profiles/r02_reference_full_partition.json")
    ap.add_argument("--parts", type=int, default=None, help="override the config's partition count p")
    ap.add_argument("--partitioner", default="random", choices=["random", "dbh", "ne"],
                    help="vertex-cut partitioner (partition.cpp:92-201); the headline uses random")
    ap.add_argument("--scale", type=float, default=None,
                    help="scale nodes and edges of the config (default 1; rmat: 0.25, see CONFIGS)")
    args = ap.parse_args()
    cfg = dict(CONFIGS[args.config])
    if args.parts:
        cfg["parts"] = args.parts
    if args.cpu_full_partition:
        res = cpu_full_partition(cfg)
        print(json.dumps(res), flush=True)
        with open(os.path.join(ROOT, "profiles", "r02_reference_full_partition.json"), "w") as f:
            json.dump(res, f, indent=1)
        return
    if args.impl == "reference":
        run_reference_arm(args, cfg)
    else:
        run_gpu_arm(args, cfg)


if __name__ == "__main__":
    main()
