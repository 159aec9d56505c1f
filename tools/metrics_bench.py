"""Partition metrics at scale: compute_metrics on the
device for C4 with Low-NN depth 1-3, against the oracle restatement (the
reference's algorithm, 1 thread) on the same graph and assignment.

  python tools/metrics_bench.py [--config C4]
"""
import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import torch  # noqa: E402,F401  (NCCL soname order)
from paper_2507_03840_b200 import esg  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="C4")
    args = ap.parse_args()
    import oracle as O
    ctx = esg.Context(0)
    s, r, _, _ = esg.config_structure(args.config)
    g = esg.build_graph(ctx, s, r)
    gx = g.export()
    deg = g.in_degrees()
    rows = []
    for depth in (1, 2, 3):
        P = 1 << depth
        part = esg.lownn_partition(s, deg, depth, r)
        esg.partition_metrics(g, part, P)  # warm-up
        t = time.perf_counter()
        m = esg.partition_metrics(g, part, P)
        gpu_s = time.perf_counter() - t
        t = time.perf_counter()
        parts, d, i = O.compute_metrics(s.n_atoms, gx["src"], gx["dst"], part, P)
        cpu_s = time.perf_counter() - t
        same = bool(np.array_equal(m.parts, parts) and (m.node_imbalance, m.edge_imbalance, m.mean_neighbors) == tuple(d)
                    and (m.max_neighbors, m.total_recv, m.cut_edges) == tuple(i))
        rows.append({"depth": depth, "gpu_s": gpu_s, "cpu_s": cpu_s, "speedup": cpu_s / gpu_s, "identical": same,
                     "cut_edges": m.cut_edges, "total_recv": m.total_recv, "mean_neighbors": m.mean_neighbors,
                     "edges_per_s_gpu": g.n_edges / gpu_s})
    print(json.dumps({"config": args.config, "atoms": s.n_atoms, "edges": g.n_edges, "rows": rows}), flush=True)


if __name__ == "__main__":
    main()
