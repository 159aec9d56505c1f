"""P-GPU training step (Low-NN partition, NCCL halo and halo backward, rank-
ordered gradient sums inside libesg_b200) versus the 1-GPU serial step on the
same graph and targets (test_runtime.cpp:330-388): loss and gradients agree
to fp32 round-off (rank partial sums reorder the reductions), and the
replicas stay in lockstep through Adam steps (esg_train_step's hash checks).

  torchrun --nproc-per-node P --master-addr 127.0.0.1 tools/multi_gpu_train_check.py
"""
import math
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2507_03840_b200 import esg  # noqa: E402


def targets(n, n_edges, out_len, seed=7):
    """Seeded head-space targets for the whole graph (node rows, edge rows)."""
    rng = np.random.default_rng(seed)
    nt = rng.standard_normal((n, out_len)).astype(np.float32) * 0.1
    et = rng.standard_normal((n_edges, out_len)).astype(np.float32) * 0.1
    nm = (rng.random((n, out_len)) < 0.5).astype(np.uint8)
    em = (rng.random((n_edges, out_len)) < 0.5).astype(np.uint8)
    return nt, nm, et, em


def main():
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dist.init_process_group("gloo")
    ids = [esg.nccl_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(ids, src=0)
    ctx = esg.Context(local, rank, world, ids[0])
    s, r, layers = esg.make_jittered_lattice(300, 2.2, 0.45, [72, 8, 8], 5), 5.0, 2
    cfg = esg.ModelConfig(l_max=4, e_width=16, layers=layers, n_radial=32, r_cut=r, seed=1,
                          linear_precision=esg.LINEAR_FP32)
    g = esg.build_graph(ctx, s, r)
    part = esg.lownn_partition(s, g.in_degrees(), int(round(math.log2(world))), r)
    plan = esg.build_comm_plan(g, s.species, part, world, rank)
    net = esg.Network(ctx, cfg, esg.BASIS_HFO2)
    net.init_params()
    net.prepare(g, s.species, plan)
    nt, nm, et, em = targets(s.n_atoms, g.n_edges, net.out_len)
    pe = plan.export()
    owned = pe["row_global"][:plan.n_owned]
    ei = pe["edge_index"]
    net.set_targets(nt[owned], nm[owned], et[ei], em[ei])
    n_total = int(nm.sum() + em.sum())
    loss, partials, grads = net.loss_grad(n_total)
    opt = esg.Adam(net)
    step_losses = [net.train_step(opt, n_total)[0] for _ in range(3)]  # raises on replica divergence
    hashes = [None] * world
    dist.all_gather_object(hashes, net.param_hash())
    ok = len(set(hashes)) == 1
    if rank == 0:
        ctx1 = esg.Context(local, 0, 1)
        net1 = esg.Network(ctx1, cfg, esg.BASIS_HFO2)
        net1.init_params()
        g1 = esg.build_graph(ctx1, s, r)
        net1.prepare(g1, s.species)
        net1.set_targets(nt, nm, et, em)
        sloss, _, sgrads = net1.loss_grad(n_total)
        rel = float(np.linalg.norm(grads.astype(np.float64) - sgrads) / np.linalg.norm(sgrads))
        dl = abs(loss - sloss) / abs(sloss)
        print(f"world {world}: loss {loss:.9g} serial {sloss:.9g} rel {dl:.2e}; grad relL2 {rel:.2e}; "
              f"replica hashes equal {ok}; step losses {[round(x, 6) for x in step_losses]}")
        ok &= dl <= 1e-6 and rel <= 1e-5 and step_losses[-1] < step_losses[0]
        print(f"train lockstep {ok}")
    flag = torch.tensor([int(ok)])
    dist.broadcast(flag, 0)
    dist.destroy_process_group()
    sys.exit(0 if flag.item() else 1)


if __name__ == "__main__":
    main()
