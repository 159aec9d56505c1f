#!/usr/bin/env python
"""Benchmark: eGNN forward edges/s on B200 (BASELINE.json metric) + halo ms.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config C4] [--impl ours|reference]

N = 1 runs the 190k-atom workload C4 (tile(C2, {4,4,4}),
192,000 atoms, r_cut 10 Å, l_max 4, E 16, M = 3).  For N > 1 the driver
launches one process per GPU with torchrun; every rank builds the same graph,
the Low-NN partition assigns nodes, each rank runs its view and exchanges
halos through NCCL inside libesg_b200.so (strong scaling on the same graph).
`value` is whole-job edges/s from device time (CUDA events, max over ranks);
`e2e` is the same metric through the public API with host buffers
(H2D of the atom positions, graph build + prepare + forward, D2H of every
Hamiltonian head output).  `--impl reference` times the reference's own CPU
forward (oracle/_ref: the unmodified reference sources built by oracle/ref.mk;
the oracle/ restatement when that was not built) on all host threads, on a
bounded sample of the same workload.
"""
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

METRIC = "eGNN forward edges/sec at 1/2/4/8 B200 (190k-atom graph); halo-exchange ms"
CONFIG_DESC = {
    "C1": "C1: jittered Si lattice 512 atoms, r_cut 8 A, 1 layer, DZVP-like basis",
    "C2": "C2: jittered HfO2 3000 atoms (375 vacancies), r_cut 12 A, 3 layers, SZV basis",
    "C3": "C3: jittered HfO2 20000 atoms, r_cut 12 A, 3 layers, SZV basis",
    "C4": "C4: tile(C2,{4,4,4}) 192000 atoms, r_cut 10 A, 3 layers, SZV basis",
}
# per-edge compulsory HBM bytes of each kernel category
H, E = 25, 16
ROW = H * E * 4  # 1600 B fp32 feature row
PROF_NAMES = ["init", "rotate_in", "so2_linears", "rotate_out_edge", "node_update", "heads", "halo", "copy"]
# fp32 (the headline): rotate_in writes the fp16x3 split image of A1 (1216
# K slots x hi|lo fp16 = 4,864 B per edge), the fp16x3 chain reads it and
# writes fp32 Y (1,600 B) and the attention logit
A1_F16S = 1216 * 4
BYTES_PER_EDGE_FP32 = {
    "rotate_in": ROW + 12 + 8 + A1_F16S,         # edge row + dir + indices + A1 write
    "so2_linears": A1_F16S + ROW + 4,             # A1 read + Y write + logit
    "rotate_out_edge": ROW + 12 + 2 * ROW,        # Y read + dir + edge row RMW
    "node_update": ROW + 12 + 4,                  # Y read + dir + logit (+ node rows, amortised)
}
A1_BF16 = 1280 * 2  # bf16 order-major operand, m-blocks padded to 64
Y_BF16 = H * E * 2
BYTES_PER_EDGE_BF16 = {
    "rotate_in": ROW + 12 + 8 + A1_BF16,
    "so2_linears": A1_BF16 + Y_BF16,
    "rotate_out_edge": Y_BF16 + 12 + 2 * ROW,
    "node_update": Y_BF16 + 12,
}
# SO(2) linear FLOPs per edge-block (lin1 445,440 + lin2 148,480)
SO2_FLOPS_PER_EDGE = 593920
# fused-minimum bytes per edge-layer and per node-layer
ALG_EDGE_LAYER, ALG_NODE_LAYER = 4832, 4800


def measured_traffic(name, prec):
    """ncu dram__bytes_read.sum + dram__bytes_write.sum per edge of a kernel
    category in one precision mode, from the committed capture summary
    (profiles/traffic.json), or None when that kernel has not been captured."""
    try:
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as f:
            return json.load(f).get(prec, {}).get(name)
    except (OSError, ValueError):
        return None


def env_int(k, d):
    try:
        return int(os.environ.get(k, d))
    except ValueError:
        return d


class Clocks:
    """nvidia-smi sampler for the timed region (B200_PROFILING.md clocks line)."""

    def __init__(self, device):
        self.device = device
        self.proc = None

    def __enter__(self):
        q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.device), f"--query-gpu={q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None
        return self

    def __exit__(self, *a):
        self.lines = []
        if self.proc is not None:
            time.sleep(0.25)
            self.proc.terminate()
            try:
                out, _ = self.proc.communicate(timeout=5)
                self.lines = [l for l in out.splitlines() if l.strip()]
            except Exception:
                pass

    def summary(self):
        sm, mx, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for l in getattr(self, "lines", []):
            f = [x.strip() for x in l.split(",")]
            if len(f) < 7:
                continue
            try:
                sm.append(float(f[0]))
                mx = max(mx, float(f[1]))
            except ValueError:
                continue
            for n, v in zip(names, f[3:7]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        loaded = [x for x in sm if x > 0.5 * max(sm)] or sm
        return {"sm_mhz": float(np.median(loaded)), "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def tensor_peak():
    """Sustained dense fp16/bf16 TFLOP/s (kind::f16, the fp16x3 chain's MMA kind)."""
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["bf16_tflops_sustained"]), "measured (cuBLAS bf16, sustained)"
    except Exception:
        return 1400.0, "fallback (B200_PROFILING.md sustained)"


# ------------------------------------------------------------------ CPU leg
CPU_SAMPLE_DST = 128  # destinations in the CPU sample (both arms: the same workload slice)


def cpu_sample(s, r, layers, basis, k=CPU_SAMPLE_DST, g=None, reps=1, warmup=0):
    """Times the reference's CPU forward on a fixed sample of the workload:
    all incoming edges of the first k destinations, the full M-layer forward
    + heads in float32 (the reference's --precision single path), on all host
    threads.  kind "reference": the reference's own code (oracle/_ref, its
    Network<float>::build_forward per thread on a destination group; prepare
    -- edge rotations and radial features -- is not timed); kind "port": the
    CPU restatement (oracle/) when the reference was not built.  Returns
    (edges/s, threads, sample text, kind).  g: the graph arrays (the oracle
    builds them when None; the GPU arm passes its bit-identical export)."""
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    import oracle as O
    import ref as R

    threads = os.cpu_count() or 1
    O.set_threads(threads)
    if g is None:
        g = O.build_graph(s.positions, s.cell, np.ones(3, np.uint8), r)
    deg = np.bincount(g["dst"], minlength=s.n_atoms)
    off = np.concatenate([[0], np.cumsum(deg)])
    k = min(k, s.n_atoms)
    e1 = int(off[k])
    src = g["src"][:e1]
    rows = np.unique(np.concatenate([np.arange(k), src]))
    # owned rows first (0..k-1 are the destinations), then the other sources
    order = np.concatenate([np.arange(k), np.setdiff1d(rows, np.arange(k))])
    pos_of = np.full(s.n_atoms, -1, np.int64)
    pos_of[order] = np.arange(len(order))
    v = dict(n_rows=len(order), n_owned=k, row_species=s.species[order], src_row=pos_of[src].astype(np.int32),
             dst_row=g["dst"][:e1].astype(np.int32), disp=g["disp"][:e1], dist=g["dist"][:e1])
    kind = "reference" if R.available() else "port"
    if kind == "port":
        om = O.Model(4, 16, layers, 32, r, 1, basis)

    def once():
        if kind == "reference":
            return R.forward_view_timed(v, basis, layers, r, threads)[1]
        t0 = time.perf_counter()
        om.forward(v, np.float32)
        return time.perf_counter() - t0

    for _ in range(warmup):
        once()
    dt = float(np.median([once() for _ in range(max(1, reps))]))
    what = ("the reference's Network<float>::build_forward (oracle/_ref, unmodified reference sources), "
            f"destinations split over {threads} threads" if kind == "reference" else
            f"the CPU restatement (oracle/), {threads} threads")
    return e1 / dt, threads, (f"all incoming edges of the first {k} destinations ({e1} edges), {layers}-layer "
                              f"forward + heads, float32, {what}, median of {max(1, reps)}"), kind


def config_dict(name, atoms, edges, r, layers, world, prec):
    return {"workload": CONFIG_DESC[name], "atoms": atoms, "edges": edges, "r_cut": r, "layers": layers, "l_max": 4,
            "e_width": 16,
            "linears": ("tcgen05 kind::f16 fp16x3 split (hi.hi + hi.lo + lo.hi, power-of-two scales), fp32 accumulate"
                        if prec == "fp32" else "tcgen05 bf16, fp32 accumulate"),
            "parallelism": f"graph-partition dp{world} (Low-NN, NCCL halo)",
            "l2": "inputs larger than L2 (edge table %.0f GB)" % (edges * ROW / 1e9)}


def run_reference(args):
    from paper_2507_03840_b200 import esg

    rank = env_int("RANK", 0)
    if rank != 0:
        return 0
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    import oracle as O

    # inputs from the oracle's own generators (synthetic.cpp:17-41, structure.cpp:40-63)
    spec = {"C1": (512, 2.71, 0.30, [14], 1, None, 8.0, 1, esg.BASIS_SI),
            "C2": (3000, 2.20, 0.45, [72, 8, 8], 2, None, 12.0, 3, esg.BASIS_HFO2),
            "C3": (20000, 2.20, 0.45, [72, 8, 8], 3, None, 12.0, 3, esg.BASIS_HFO2),
            "C4": (3000, 2.20, 0.45, [72, 8, 8], 2, [4, 4, 4], 10.0, 3, esg.BASIS_HFO2)}[args.config]
    pos, cell, sp = O.jittered_lattice(*spec[:5])
    if spec[5]:
        pos, cell, sp = O.tile(pos, cell, np.ones(3, np.uint8), sp, spec[5])
    r, layers, basis = spec[6], spec[7], spec[8]
    s = esg.AtomicStructure(pos, sp, cell, np.ones(3, bool))
    g = O.build_graph(s.positions, s.cell, np.ones(3, np.uint8), r)
    # one timed sample forward per step after the warm-up ones: the same
    # destination sample as the GPU arm's cpu_baseline
    val, cores, sample, kind = cpu_sample(s, r, layers, basis, g=g, reps=max(1, args.steps), warmup=args.warmup)
    info = (cores, sample)
    line = {"metric": METRIC, "value": val, "unit": "edges/s", "n_gpus": args.gpus, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": None, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "fp32", "data": "synthetic", "impl": "reference",
            "config": config_dict(args.config, s.n_atoms, len(g["src"]), r, layers, 1, "fp32"),
            "cpu_baseline": {"value": val, "unit": "edges/s", "cores": info[0], "kind": kind, "sample": info[1]},
            "e2e": {"value": val, "unit": "edges/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


# ------------------------------------------------------------------ GPU leg
def run_ours(args):
    import torch
    from paper_2507_03840_b200 import esg

    rank, world = env_int("RANK", 0), env_int("WORLD_SIZE", 1)
    local = env_int("LOCAL_RANK", rank)
    if world != args.gpus:
        args.gpus = world
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("gloo", init_method="env://")
    ids = [esg.nccl_unique_id() if rank == 0 else None]
    if world > 1:
        dist.broadcast_object_list(ids, src=0)
    ctx = esg.Context(local, rank, world, ids[0] if world > 1 else None)

    s, r, layers, basis = esg.config_structure(args.config)
    prec = esg.LINEAR_BF16 if args.precision == "bf16" else esg.LINEAR_FP32
    cfg = esg.ModelConfig(l_max=4, e_width=16, layers=layers, n_radial=32, r_cut=r, seed=1, linear_precision=prec)
    t0 = time.perf_counter()
    g = esg.build_graph(ctx, s, r)
    t_graph = time.perf_counter() - t0
    def lownn(ctx, s, deg, depth, r):  # ESG_LOWNN_HOST=1: the host restatement (A/B only)
        if os.environ.get("ESG_LOWNN_HOST") == "1":
            return esg.lownn_partition(s, deg, depth, r)
        return esg.lownn_partition_gpu(ctx, s, deg, depth, r)

    t0 = time.perf_counter()
    plan = None
    if world > 1:
        depth = int(round(math.log2(world)))
        part = lownn(ctx, s, g.in_degrees(), depth, r)
        plan = esg.build_comm_plan(g, s.species, part, world, rank)
    t_part = time.perf_counter() - t0
    net = esg.Network(ctx, cfg, basis)
    net.init_params()
    t0 = time.perf_counter()
    net.prepare(g, s.species, plan)
    t_prep = time.perf_counter() - t0

    def barrier():
        if dist is not None:
            dist.barrier()

    def allmax(x):
        if dist is None:
            return x
        t = torch.tensor([x], dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    def allsum(x):
        if dist is None:
            return x
        t = torch.tensor([x], dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.SUM)
        return float(t.item())

    for _ in range(args.warmup):
        net.forward(copy_out=False)
    lib = esg.lib()
    import ctypes as C
    ms_cat = np.zeros(8)
    n_cat = np.zeros(8, np.int64)
    lib.esg_profile(net._h, C.c_int(1), None, None)
    barrier()
    torch.cuda.synchronize()
    fwd_ms, msg_ms, halo_ms, launches = [], [], [], 0
    halo_skew, halo_xch, halo_bytes = [], [], []
    with Clocks(local) as clk:
        w0 = time.perf_counter()
        for _ in range(args.steps):
            _, _, tm = net.forward(copy_out=False)
            fwd_ms.append(tm.forward_ms)
            msg_ms.append(tm.message_ms)
            halo_ms.append(tm.halo_ms)
            halo_skew.append(tm.halo_skew_ms)
            halo_xch.append(tm.halo_exchange_ms)
            halo_bytes.append(tm.halo_bytes)
            launches += tm.gpu_launches
        torch.cuda.synchronize()
        wall = time.perf_counter() - w0
    barrier()
    lib.esg_profile(net._h, C.c_int(0), ms_cat.ctypes.data_as(C.c_void_p), n_cat.ctypes.data_as(C.c_void_p))
    clocks = clk.summary()
    ms_step = allmax(float(np.mean(fwd_ms)))
    halo_step = allmax(float(np.mean(halo_ms)))
    halo = None
    if world > 1:
        # per forward, max over ranks: the 2M exchanges' total, the part spent
        # waiting for the slowest rank (a one-float allreduce lines the ranks
        # up before each exchange while profiling) and the exchange proper
        # (pack start -> last recv); NVLink GB/s = this rank's sent + received
        # bytes over its exchange time
        xch = float(np.mean(halo_xch))
        gbs = float(np.mean(halo_bytes)) / (xch / 1e3) / 1e9 if xch > 0 else None
        halo = {"ms_per_forward": halo_step, "exchanges_per_forward": 2 * layers,
                "ms_per_exchange": halo_step / (2 * layers),
                "skew_ms_per_forward": allmax(float(np.mean(halo_skew))),
                "exchange_ms_per_forward": allmax(xch),
                "bytes_per_forward_max_rank": allmax(float(np.mean(halo_bytes))),
                "nvlink_gbs_min_over_ranks": -allmax(-gbs) if gbs else None,
                "method": "CUDA events around each exchange, no host sync inside the forward; max over ranks"}
    msg_step = allmax(float(np.mean(msg_ms)))
    total_edges = g.n_edges
    value = total_edges / (ms_step / 1e3)

    # roofline of the dominant kernel category (this rank's live CUDA events)
    prec_name = "fp32" if prec == esg.LINEAR_FP32 else "bf16"
    bytes_tab = BYTES_PER_EDGE_FP32 if prec == esg.LINEAR_FP32 else BYTES_PER_EDGE_BF16
    dom = int(np.argmax(ms_cat[:6]))
    name = PROF_NAMES[dom]
    roof = None
    hbm, peak_kind = peaks()
    tpk, tpk_kind = tensor_peak()
    if name in bytes_tab and ms_cat[dom] > 0:
        # node_update runs in the M node blocks, rotate_out_edge in the M edge
        # blocks, rotate_in / so2_linears in all 2M blocks
        blocks = layers if name in ("node_update", "rotate_out_edge") else 2 * layers
        alg_bytes = bytes_tab[name] * net.n_edges * blocks * args.steps
        achieved = alg_bytes / (ms_cat[dom] / 1e3) / 1e9
        launches_dom = max(int(n_cat[dom]), 1)
        edges_per_launch = net.n_edges * blocks * args.steps / launches_dom
        tr = measured_traffic(name, prec_name)
        roof = {"bound": "hbm", "achieved": achieved, "peak": hbm, "unit": "GB/s", "frac": achieved / hbm,
                "traffic": (tr["dram_bytes_per_edge"] * edges_per_launch) if tr else None,
                "kernel": name, "peak_source": peak_kind,
                "bytes_per_edge": bytes_tab[name], "edges_per_launch": edges_per_launch,
                "traffic_source": tr.get("source") if tr else None,
                "launches": int(n_cat[dom]), "avg_launch_ms": float(ms_cat[dom] / launches_dom)}
        if name == "so2_linears":
            # the same launches against the tensor pipe: algorithmic fp32 FLOPs
            # of lin1 + lin2; the fp16x3 split issues 3 kind::f16 products per
            # fp32 one, so its ceiling is a third of the dense fp16 rate
            alg_tf = SO2_FLOPS_PER_EDGE * net.n_edges * 2 * layers * args.steps / (ms_cat[dom] / 1e3) / 1e12
            ceil = tpk / 3 if prec == esg.LINEAR_FP32 else tpk
            roof["tensor"] = {"achieved": alg_tf, "peak": ceil, "unit": "TFLOP/s (algorithmic fp32)"
                              if prec == esg.LINEAR_FP32 else "TFLOP/s", "frac": alg_tf / ceil,
                              "peak_source": tpk_kind + (" / 3 (three products per fp32 product)"
                                                         if prec == esg.LINEAR_FP32 else "")}
    # the whole message-passing path against SURVEY §8(d)'s fused minimum
    path = {"bytes": (ALG_EDGE_LAYER * net.n_edges + ALG_NODE_LAYER * net.n_owned) * layers,
            "t_mp_ms": msg_step}
    path["achieved_gbs"] = path["bytes"] / (msg_step / 1e3) / 1e9 if msg_step > 0 else None
    path["frac"] = path["achieved_gbs"] / hbm if path["achieved_gbs"] else None

    # e2e through the public API with host buffers
    e2e = None
    if args.e2e_steps > 0:
        node_out = np.empty((net.n_owned, net.out_len), np.float32)
        edge_out = np.empty((net.n_edges, net.out_len), np.float32)
        try:
            node_out = torch.empty((net.n_owned, net.out_len), dtype=torch.float32, pin_memory=True).numpy()
            edge_out = torch.empty((net.n_edges, net.out_len), dtype=torch.float32, pin_memory=True).numpy()
        except Exception:
            pass
        barrier()
        torch.cuda.synchronize()
        # graph (+ plan), prepare, forward (its outputs' D2H runs on a copy
        # stream into pinned memory and overlaps the next step), teardown,
        # and the final wait for the last step's copies
        phases = np.zeros(5)
        t0 = time.perf_counter()
        for _ in range(args.e2e_steps):
            ta = time.perf_counter()
            g2 = esg.build_graph(ctx, s, r)  # H2D of the positions
            plan2 = None
            if world > 1:
                part2 = lownn(ctx, s, g2.in_degrees(), int(round(math.log2(world))), r)
                plan2 = esg.build_comm_plan(g2, s.species, part2, world, rank)
            tb = time.perf_counter()
            net.prepare(g2, s.species, plan2)
            tc = time.perf_counter()
            net.forward_into_async(node_out, edge_out, timing=False)  # queued; D2H of every head output queued
            td = time.perf_counter()
            g2.close()
            te = time.perf_counter()
            phases[:4] += [tb - ta, tc - tb, td - tc, te - td]
        tf = time.perf_counter()
        net.wait_outputs()  # every step's outputs are on the host
        phases[4] += time.perf_counter() - tf
        torch.cuda.synchronize()
        e2e_s = allmax((time.perf_counter() - t0) / args.e2e_steps)
        d2h = int(allsum(node_out.nbytes + edge_out.nbytes))
        e2e = {"value": total_edges / e2e_s, "unit": "edges/s",
               "h2d_bytes_per_step": int(s.positions.nbytes),
               "d2h_bytes_per_step": d2h, "step_s": e2e_s,
               "phases_s_max_over_ranks": {k: allmax(float(phases[i] / args.e2e_steps)) for i, k in
                                           enumerate(("graph_and_plan", "prepare", "forward", "teardown",
                                                      "d2h_drain"))},
               "d2h_overlap": "outputs stream to pinned host memory on a copy stream while the last edge block "
                              "and the next step run (esg_forward_async / esg_forward_wait)",
               "pinned_host_outputs": bool(getattr(torch.from_numpy(edge_out), "is_pinned", lambda: False)())}

    # bf16 tensor-core linears on the same graph (throughput side key): time
    # and the measured deviation of its heads from this run's fp32 heads
    # (the fp32 path is within rel-L2 2e-5 of the float oracle, test_gpu_parity)
    bf16_mode = None
    if args.bf16_steps > 0 and prec == esg.LINEAR_FP32 and world == 1:
        n_cmp = min(net.n_edges, 2_000_000)
        ref_n, ref_e = net.outputs_host(n_cmp)
        net.set_precision(esg.LINEAR_BF16)
        net.forward(copy_out=False)
        torch.cuda.synchronize()
        b16 = [net.forward(copy_out=False)[2].forward_ms for _ in range(args.bf16_steps)]
        got_n, got_e = net.outputs_host(n_cmp)
        ms16 = float(np.mean(b16))
        def dev(a, b):
            return {"rel_l2": float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-30)),
                    "max_abs_over_max": float(np.abs(a - b).max() / max(np.abs(b).max(), 1e-30))}
        bf16_mode = {"value": total_edges / (ms16 / 1e3), "unit": "edges/s", "ms_per_step": ms16,
                     "steps": args.bf16_steps, "dtype": "bf16",
                     "linears": "tcgen05 kind::f16 bf16 operands, fp32 accumulate",
                     "deviation_vs_fp32_heads": {"nodes": dev(got_n, ref_n),
                                                 "edges_first_%d" % n_cmp: dev(got_e, ref_e)},
                     "tolerance": "bf16 bar: rel-L2 <= 2e-2, max-abs <= 5e-2 x max (fp32 bar 2e-5 / 2e-4)"}
        net.set_precision(prec)

    cpu = None
    if rank == 0 and world == 1 and args.cpu_seconds > 0:
        v, cores, sample, kind = cpu_sample(s, r, layers, basis, g=g.export())
        cpu = {"value": v, "unit": "edges/s", "cores": cores, "kind": kind, "sample": sample}
    line = {"metric": METRIC, "value": value, "unit": "edges/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": prec_name, "data": "synthetic",
            "config": config_dict(args.config, s.n_atoms, total_edges, r, layers, world, prec_name),
            "e2e": e2e, "roofline": roof, "path_roofline": path, "cpu_baseline": cpu, "clocks": clocks,
            "bf16_mode": bf16_mode, "gpu_launches": int(allsum(launches)),
            "halo_ms_per_forward": halo_step, "halo_exchanges_per_forward": 2 * layers if world > 1 else 0,
            "halo": halo,
            "message_ms_per_forward": msg_step,
            "kernel_ms_per_forward": {PROF_NAMES[i]: float(ms_cat[i] / args.steps) for i in range(8)},
            "setup_s": {"graph": t_graph, "partition_plan": t_part, "prepare": t_prep},
            "wall_ms_per_step": 1e3 * wall / args.steps}
    if world == 1 and args.train_steps > 0:
        # config 5's training step, measured on C2 after the
        # C4 tables are released: forward (fp32 path, inputs kept), masked
        # loss, reverse pass, gradient sums and the Adam step
        net.close()
        g.close()
        node_out = edge_out = None  # noqa: F841  (the e2e pinned host buffers)
        import gc
        gc.collect()
        line["train"] = train_measure(ctx, args.train_steps)
    if rank == 0:
        print(json.dumps(line), flush=True)
    if dist is not None:
        dist.barrier()
        dist.destroy_process_group()
    return 0


def train_measure(ctx, steps, config="C2"):
    import torch
    from paper_2507_03840_b200 import esg
    s, r, layers, basis = esg.config_structure(config)
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
    net.train_step(opt, n_total)  # warm-up
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    res = [net.train_step(opt, n_total) for _ in range(steps)]
    torch.cuda.synchronize()
    step_s = (time.perf_counter() - t0) / steps
    out = {"workload": CONFIG_DESC[config] + ", training step (fp32 linears)", "edges": net.n_edges,
           "steps": steps, "step_ms": 1e3 * step_s, "forward_ms": float(np.mean([x[1] for x in res])),
           "backward_ms": float(np.mean([x[2] for x in res])), "edges_per_s": net.n_edges / step_s,
           "loss_first_last": [res[0][0], res[-1][0]], "targets": "seeded head-space values, half masked"}
    opt.close()
    net.close()
    g.close()
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="C4", choices=["C1", "C2", "C3", "C4"])
    ap.add_argument("--precision", default="fp32", choices=["bf16", "fp32"],
                    help="fp32: the fp32-faithful linears (the headline); bf16: throughput mode")
    ap.add_argument("--e2e-steps", type=int, default=10)
    ap.add_argument("--cpu-seconds", type=float, default=15.0, help="0 skips the CPU baseline sample")
    ap.add_argument("--train-steps", type=int, default=2, help="C2 training steps after the forward (0: skip)")
    ap.add_argument("--bf16-steps", type=int, default=3, help="forwards timed in the bf16 side mode (0: skip)")
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
