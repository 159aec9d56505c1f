"""Training-step timing (config 5 shape): forward (fp32 path, inputs saved),
masked loss, reverse pass, rank-ordered gradient sums and the Adam step,
through the C ABI.  Targets are seeded head-space values (half masked).

  python tools/train_bench.py [--config C2] [--steps 3]
"""
import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2507_03840_b200 import esg  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="C2")
    ap.add_argument("--steps", type=int, default=3)
    args = ap.parse_args()
    ctx = esg.Context(0)
    s, r, layers, basis = esg.config_structure(args.config)
    g = esg.build_graph(ctx, s, r)
    cfg = esg.ModelConfig(l_max=4, e_width=16, layers=layers, n_radial=32, r_cut=r, seed=1,
                          linear_precision=esg.LINEAR_FP32)
    net = esg.Network(ctx, cfg, basis)
    net.init_params()
    net.prepare(g, s.species)
    rng = np.random.default_rng(7)
    ol = net.out_len
    nt = (rng.standard_normal((net.n_owned, ol)) * 0.1).astype(np.float32)
    et = (rng.standard_normal((net.n_edges, ol)) * 0.1).astype(np.float32)
    nm = (rng.random((net.n_owned, ol)) < 0.5).astype(np.uint8)
    em = (rng.random((net.n_edges, ol)) < 0.5).astype(np.uint8)
    net.set_targets(nt, nm, et, em)
    n_total = int(nm.sum() + em.sum())
    opt = esg.Adam(net)
    net.train_step(opt, n_total)  # warm-up (allocations)
    t0 = time.perf_counter()
    res = [net.train_step(opt, n_total) for _ in range(args.steps)]
    wall = (time.perf_counter() - t0) / args.steps
    fwd = float(np.mean([x[1] for x in res]))
    bwd = float(np.mean([x[2] for x in res]))
    t1 = time.perf_counter()
    net.loss_grad(n_total)
    t_lg = time.perf_counter() - t1
    t1 = time.perf_counter()
    net.set_params(net.params())
    t_up = time.perf_counter() - t1
    t1 = time.perf_counter()
    net.forward(copy_out=False)
    t_fwd = time.perf_counter() - t1
    print(json.dumps({"loss_grad_wall_s": t_lg, "param_upload_s": t_up, "forward_wall_s": t_fwd}))
    print(json.dumps({"config": args.config, "edges": net.n_edges, "steps": args.steps,
                      "step_s": wall, "forward_ms": fwd, "backward_ms": bwd,
                      "train_edges_per_s": net.n_edges / wall, "losses": [x[0] for x in res]}))


if __name__ == "__main__":
    main()
