"""P-GPU forward (Low-NN partition, NCCL halo inside libesg_b200) versus the
1-GPU serial forward of the same graph: every per-destination reduction is
segment-local with a fixed order, so the outputs must agree bit for bit
(the reference pins the same property: test_runtime.cpp:235-271).

  torchrun --nproc-per-node P --master-addr 127.0.0.1 tools/multi_gpu_check.py [--config C3] [--oracle]
"""
import argparse
import math
import os
import shutil
import sys
import tempfile

import numpy as np
import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2507_03840_b200 import esg  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="small")
    ap.add_argument("--precision", default="fp32")
    ap.add_argument("--oracle", action="store_true", help="rank 0 also checks the serial heads against the oracle")
    ap.add_argument("--golden", action="store_true",
                    help="C3: every rank checks its partitioned heads against tests/golden/c3_heads_sample.npz")
    args = ap.parse_args()
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dist.init_process_group("gloo")
    ids = [esg.nccl_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(ids, src=0)
    ctx = esg.Context(local, rank, world, ids[0])
    if args.config == "small":
        s, r, layers, basis = esg.make_jittered_lattice(600, 2.2, 0.45, [72, 8, 8], 5), 6.0, 2, esg.BASIS_HFO2
    else:
        s, r, layers, basis = esg.config_structure(args.config)
    prec = esg.LINEAR_BF16 if args.precision == "bf16" else esg.LINEAR_FP32
    cfg = esg.ModelConfig(l_max=4, e_width=16, layers=layers, n_radial=32, r_cut=r, seed=1, linear_precision=prec)
    g = esg.build_graph(ctx, s, r)
    part = esg.lownn_partition(s, g.in_degrees(), int(round(math.log2(world))), r)
    plan = esg.build_comm_plan(g, s.species, part, world, rank)
    net = esg.Network(ctx, cfg, basis)
    net.init_params()
    net.prepare(g, s.species, plan)
    no, eo, tm = net.forward()
    pe = plan.export()
    owned = pe["row_global"][:plan.n_owned]
    ok = tm.exchanges == 2 * layers
    if args.golden:
        # the committed float-oracle heads of C3 on a fixed sample
        # (tools/make_c3_golden.py): this rank's sampled rows, fp32 bar
        gd = np.load(os.path.join(ROOT, "tests", "golden", "c3_heads_sample.npz"))
        assert args.config == "C3" and int(gd["n_edges"]) == g.n_edges
        loc_n = {int(v): i for i, v in enumerate(owned)}
        loc_e = {int(v): i for i, v in enumerate(pe["edge_index"])}
        pairs = [(no[loc_n[int(v)]], gd["node_heads"][i]) for i, v in enumerate(gd["node_index"]) if int(v) in loc_n]
        pairs += [(eo[loc_e[int(v)]], gd["edge_heads"][i]) for i, v in enumerate(gd["edge_index"]) if int(v) in loc_e]
        d2 = sum(float(np.sum((a.astype(np.float64) - b) ** 2)) for a, b in pairs)
        r2 = sum(float(np.sum(b.astype(np.float64) ** 2)) for a, b in pairs)
        mx = max([float(np.abs(a.astype(np.float64) - b).max()) for a, b in pairs] or [0.0])
        got = [None] * world
        dist.all_gather_object(got, (len(pairs), d2, r2, mx))
        if rank == 0:
            n = sum(x[0] for x in got)
            scale = max(float(gd["node_max"]), float(gd["edge_max"]))
            mxr = max(x[3] for x in got) / scale
            rl2 = (sum(x[1] for x in got) / sum(x[2] for x in got)) ** 0.5
            passed = n == len(gd["node_index"]) + len(gd["edge_index"]) and mxr < 2e-4 and rl2 < 2e-5
            print(f"partitioned heads vs C3 float-oracle sample ({n} rows over {world} ranks): "
                  f"max-abs/max {mxr:.3e} rel-L2 {rl2:.3e} pass {passed}")
            ok &= passed
    if args.config != "small":
        # large configs: every rank runs the serial forward of the same graph on
        # its own GPU and compares its slice locally (no multi-GB gathers)
        ctx1 = esg.Context(local, 0, 1)
        net1 = esg.Network(ctx1, cfg, basis)
        net1.init_params()
        g1 = esg.build_graph(ctx1, s, r)
        net1.prepare(g1, s.species)
        sno, seo, stm = net1.forward()
        same = np.array_equal(no, sno[owned]) and np.array_equal(eo, seo[pe["edge_index"]])
        diff = max(float(np.abs(no - sno[owned]).max()), float(np.abs(eo - seo[pe["edge_index"]]).max()))
        res = [None] * world
        dist.all_gather_object(res, (rank, same, diff, tm.exchanges, tm.halo_ms, tm.halo_bytes, tm.forward_ms,
                                     stm.forward_ms, len(pe["edge_index"])))
        if rank == 0:
            for x in res:
                print(f"rank {x[0]}: bit-exact {x[1]} max|diff| {x[2]} exchanges {x[3]} halo {x[4]:.3f} ms "
                      f"({x[5] / 1e6:.1f} MB) forward {x[6]:.1f} ms (serial {x[7]:.1f} ms), {x[8]} edges")
            allsame = all(x[1] for x in res)
            print(f"world {world} {args.config} {args.precision}: bit-exact {allsame}")
            ok &= allsame
            if args.oracle:
                sys.path.insert(0, os.path.join(ROOT, "tests"))
                import oracle as O
                import time
                t0 = time.time()
                ref = O.build_graph(s.positions, s.cell, np.ones(3, np.uint8), r)
                om = O.Model(4, 16, layers, 32, r, 1, basis)
                rno, reo = om.forward(O.serial_view(s.n_atoms, s.species, ref), np.float32)
                for nm, got, want in (("nodes", sno, rno), ("edges", seo, reo)):
                    mx = float(np.abs(got - want).max() / np.abs(want).max())
                    rl2 = float(np.linalg.norm(got - want) / np.linalg.norm(want))
                    passed = mx < 2e-4 and rl2 < 2e-5
                    print(f"heads vs float oracle ({nm}): max-abs/max {mx:.3e} rel-L2 {rl2:.3e} pass {passed} "
                          f"[oracle {time.time() - t0:.0f} s, {O.num_threads()} threads]")
                    ok &= passed
        net1.close()
        g1.close()
    else:
        outs = [None] * world
        dist.all_gather_object(outs, (owned, pe["edge_index"], no, eo, tm.exchanges, tm.halo_ms))
        # per-rank block shards into a directory rank 0 picks
        d = [tempfile.mkdtemp(prefix="esg_blk_") if rank == 0 else None]
        dist.broadcast_object_list(d, src=0)
        shard = os.path.join(d[0], f"rank{rank}.blk")
        net.write_block_shard(shard, esg.BLOCKS_UNCOUPLED)
        dist.barrier()
        if rank == 0:
            ctx1 = esg.Context(local, 0, 1)
            net1 = esg.Network(ctx1, cfg, basis)
            net1.init_params()
            g1 = esg.build_graph(ctx1, s, r)
            net1.prepare(g1, s.species)
            sno, seo, _ = net1.forward()
            gno = np.zeros_like(sno)
            geo = np.zeros_like(seo)
            for o, ei, a, b, ex, hm in outs:
                gno[o] = a
                geo[ei] = b
                ok &= ex == 2 * layers
            same = np.array_equal(gno, sno) and np.array_equal(geo, seo)
            print(f"world {world}: exchanges/forward {outs[0][4]}, halo ms {[round(x[5], 3) for x in outs]}, "
                  f"bit-exact {same}, max|diff| {max(np.abs(gno - sno).max(), np.abs(geo - seo).max())}")
            ok &= same
            # rank 0's gathered text from the shards == the 1-GPU text file
            merged, serial = os.path.join(d[0], "merged.txt"), os.path.join(d[0], "serial.txt")
            esg.merge_block_shards_to_text([os.path.join(d[0], f"rank{r}.blk") for r in range(world)], merged)
            net1.write_blocks_text(serial, esg.BLOCKS_UNCOUPLED)
            with open(merged, "rb") as a, open(serial, "rb") as b:
                same_txt = a.read() == b.read()
            print(f"blocks text identical {same_txt} ({os.path.getsize(serial)} bytes)")
            ok &= same_txt
            shutil.rmtree(d[0], ignore_errors=True)
    ok_t = torch.tensor([int(ok)])
    dist.all_reduce(ok_t, op=dist.ReduceOp.MIN)
    ok = bool(ok_t.item())
    dist.destroy_process_group()
    sys.exit(0 if ok else 1)


if __name__ == "__main__":
    main()
