"""Time the partitioners on the bench's products-shaped graph (2.45M nodes / 62M edges).

    python tools/time_partitioners.py [scale]

Prints one JSON line: seconds for build_graph, partition_random / dbh (device),
partition_ne (host heap + device vertex-cut build), the greedy edge cut (host BFS)
and edge_cut_to_vertex_cut (device), plus the replication factors.
"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2308_03209_b200 import sagecut as sc  # noqa: E402

scale = float(sys.argv[1]) if len(sys.argv) > 1 else 1.0
n, uv, *_ = bench.synth_host(bench.CONFIGS["products"], seed=0, scale=scale)
ctx = sc.default_context()
out = {"nodes": n}


def timed(name, f):
    ctx.sync()
    t0 = time.perf_counter()
    r = f()
    ctx.sync()
    out[name + "_s"] = round(time.perf_counter() - t0, 3)
    return r


g, _ = timed("build_graph", lambda: sc.build_graph(n, uv, ctx))
out["edges"] = g.num_edges()
for name, f in (("random", lambda: sc.partition_random(g, 8, 0)), ("dbh", lambda: sc.partition_dbh(g, 8, 0)),
                ("ne", lambda: sc.partition_ne(g, 8, 0))):
    vc = timed("partition_" + name, f)
    out["rf_" + name] = round(sc.replication_stats(vc, g).rf, 4)
    del vc
ec = timed("edge_cut_greedy", lambda: sc.partition_edge_cut_greedy(g, 8, 0))
out["ec_cut_edges"] = len(ec.cut_edges)
vc = timed("ec2vc", lambda: sc.edge_cut_to_vertex_cut(g, ec, 0))
out["rf_ec2vc"] = round(sc.replication_stats(vc, g).rf, 4)
print(json.dumps(out))
