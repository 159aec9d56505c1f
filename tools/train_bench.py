"""Training-step timing (config 5): forward (fp32 path, block inputs kept),
masked loss, reverse pass, rank-ordered gradient sums (NCCL allgather) and
the Adam step, through the C ABI.  Targets are seeded head-space values
(half masked).  Max over ranks of the step wall time.

  python tools/train_bench.py [--config C2|C5] [--steps 2]
  torchrun --nproc-per-node P --master-addr 127.0.0.1 tools/train_bench.py --config C5

C5 is SURVEY §8's weak-scaling set: tile(C2, {2,2,2} / {4,2,2} / {4,4,2} /
{4,4,4}) on 1 / 2 / 4 / 8 GPUs, r_cut 12 A, about 24k atoms per GPU.
"""
import argparse
import json
import math
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2507_03840_b200 import esg  # noqa: E402

C5_REPS = {1: (2, 2, 2), 2: (4, 2, 2), 4: (4, 4, 2), 8: (4, 4, 4)}


def structure(config, world):
    if config == "C5":
        s, r, layers, basis = esg.config_structure("C2")
        return esg.tile(s, C5_REPS[world]), 12.0, layers, basis
    return esg.config_structure(config)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="C2")
    ap.add_argument("--steps", type=int, default=2)
    args = ap.parse_args()
    rank, world = int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1))
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("gloo")
        ids = [esg.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(ids, src=0)
        ctx = esg.Context(local, rank, world, ids[0])
    else:
        ctx = esg.Context(0)
    s, r, layers, basis = structure(args.config, world)
    g = esg.build_graph(ctx, s, r)
    plan = None
    if world > 1:
        part = esg.lownn_partition(s, g.in_degrees(), int(round(math.log2(world))), r)
        plan = esg.build_comm_plan(g, s.species, part, world, rank)
    cfg = esg.ModelConfig(l_max=4, e_width=16, layers=layers, n_radial=32, r_cut=r, seed=1,
                          linear_precision=esg.LINEAR_FP32)
    net = esg.Network(ctx, cfg, basis)
    net.init_params()
    net.prepare(g, s.species, plan)
    # seeded targets for the whole graph, sliced to this rank's view
    rng = np.random.default_rng(7)
    ol = net.out_len
    nt = (rng.standard_normal((s.n_atoms, ol)) * 0.1).astype(np.float32)
    nm = (rng.random((s.n_atoms, ol)) < 0.5).astype(np.uint8)
    et = (rng.standard_normal((g.n_edges, ol)) * 0.1).astype(np.float32)
    em = (rng.random((g.n_edges, ol)) < 0.5).astype(np.uint8)
    n_total = int(nm.sum() + em.sum())
    if plan is not None:
        pe = plan.export()
        owned, ei = pe["row_global"][:plan.n_owned], pe["edge_index"]
        net.set_targets(nt[owned], nm[owned], et[ei], em[ei])
    else:
        net.set_targets(nt, nm, et, em)
    del nt, nm, et, em
    opt = esg.Adam(net)
    net.train_step(opt, n_total)  # warm-up (allocations, NCCL setup)
    torch.cuda.synchronize()
    if dist is not None:
        dist.barrier()
    t0 = time.perf_counter()
    res = [net.train_step(opt, n_total) for _ in range(args.steps)]
    torch.cuda.synchronize()
    step = (time.perf_counter() - t0) / args.steps
    if dist is not None:
        t = torch.tensor([step], dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        step = float(t.item())
    if rank == 0:
        print(json.dumps({"config": args.config, "world": world, "atoms": s.n_atoms, "edges": g.n_edges,
                          "edges_per_gpu": net.n_edges, "steps": args.steps, "step_s": step,
                          "forward_ms_rank0": float(np.mean([x[1] for x in res])),
                          "backward_ms_rank0": float(np.mean([x[2] for x in res])),
                          "train_edges_per_s": g.n_edges / step, "losses": [x[0] for x in res]}), flush=True)
    if dist is not None:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
