"""Times Low-NN on C4 (192k atoms): host restatement vs the device path."""
import json, time, sys
import numpy as np
sys.path.insert(0, ".")
from paper_2507_03840_b200 import esg

ctx = esg.Context(0)
s, r, _, _ = esg.config_structure("C4")
deg = esg.build_graph(ctx, s, r).in_degrees()
out = {"workload": "C4", "n_atoms": s.n_atoms}
for depth in (1, 2, 3):
    esg.lownn_partition_gpu(ctx, s, deg, depth, r)  # warm-up (allocations, cub)
    t = []
    for _ in range(5):
        t0 = time.perf_counter(); g = esg.lownn_partition_gpu(ctx, s, deg, depth, r); t.append(time.perf_counter() - t0)
    th = []
    for _ in range(3):
        t0 = time.perf_counter(); h = esg.lownn_partition(s, deg, depth, r); th.append(time.perf_counter() - t0)
    assert np.array_equal(g, h)
    out[f"depth{depth}"] = {"gpu_ms": 1e3 * min(t), "host_ms": 1e3 * min(th)}
print(json.dumps(out))
