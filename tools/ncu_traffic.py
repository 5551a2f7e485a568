"""Per-config DRAM traffic of the aggregation kernels (run on the GPU box; ncu replays every
captured launch, so this is never a timing run):

    python tools/ncu_traffic.py --config products [--scale 1]   (appends to profiles/ncu_traffic.json)

ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum --cache-control none --clock-control none on
the first forward and backward aggregation launches (spmm_kernel, and spmm_narrow_kernel for the
projected top layer's 48-wide rows) of `bench.py --steps 1 --warmup 0`; with
--cache-control none the L2 keeps whatever the previous kernels left, as in the real step, so for an
L2-resident message matrix (Reddit) the DRAM bytes come out below the algorithmic bytes. Written as
{"<config>@<scale>": {"spmm_fwd": bytes/launch, "spmm_bwd": bytes/launch, "source": ...}}; bench.py
reads it for roofline.traffic and roofline.dram_measured.
"""
import argparse
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="products")
    ap.add_argument("--scale", type=float, default=None)
    ap.add_argument("--count", type=int, default=12)
    args = ap.parse_args()
    sys.path.insert(0, ROOT)
    import bench
    scale = args.scale if args.scale is not None else bench.CONFIGS[args.config].get("default_scale", 1.0)
    cmd = ["ncu", "--metrics", "dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum",
           "--cache-control", "none", "--clock-control", "none", "-k", "regex:spmm_(kernel|narrow_kernel)", "-c", str(args.count),
           "--csv", sys.executable, os.path.join(ROOT, "bench.py"), "--steps", "1", "--warmup", "0",
           "--no-cpu-baseline", "--config", args.config, "--scale", str(scale)]
    out = subprocess.run(cmd, capture_output=True, text=True, cwd=ROOT).stdout
    rows = list(csv.reader(io.StringIO(out[out.index('"ID"'):])))
    hdr = rows[0]
    ki, mi, vi, ii = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value"), hdr.index("ID")
    per = {}
    for r in rows[1:]:
        if len(r) <= vi:
            continue
        d = per.setdefault(r[ii], {"name": r[ki]})
        d[r[mi]] = float(r[vi].replace(",", ""))
    def backward(name):  # spmm_kernel<NCH, kBwd, ...> / spmm_narrow_kernel<LPR, CPL, kBwd, ...>: ncu prints 0/1 or false/true
        args_ = name.split("(")[0]
        args_ = args_[args_.index("<") + 1:args_.rindex(">")].split(",")
        return args_[2 if "narrow" in name else 1].strip() in ("1", "true")  # narrow: <LPR, CPL, kBwd, ...>

    fwd = [d for d in per.values() if not backward(d["name"])]
    bwd = [d for d in per.values() if backward(d["name"])]

    def avg(ds):
        return sum(d["dram__bytes_read.sum"] + d["dram__bytes_write.sum"] for d in ds) / len(ds) if ds else None

    path = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    data = json.load(open(path)) if os.path.exists(path) else {}
    data = {k: v for k, v in data.items() if isinstance(v, dict)}
    data[f"{args.config}@{scale:g}"] = {
        "spmm_fwd": avg(fwd), "spmm_bwd": avg(bwd), "launches": {"fwd": len(fwd), "bwd": len(bwd)},
        "source": "ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum --cache-control none, "
                  f"first {args.count} aggregation launches (spmm_kernel, spmm_narrow_kernel) of bench.py --config {args.config} --scale {scale:g}"}
    json.dump(data, open(path, "w"), indent=1, sort_keys=True)
    print(json.dumps(data[f"{args.config}@{scale:g}"]))


if __name__ == "__main__":
    main()
