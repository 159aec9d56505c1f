"""Block export measurement on one GPU.

After one forward of --config (default C3, HfO2, about 12M edges):
  * device export: the uncoupled value kernel (fp64) and the key kernel into
    HBM, CUDA-event times from inside the library; algorithmic bytes per item
    = head row read (out_len x 4 B) + block values written (n_orb_a x n_orb_b
    x 8 B) + key record (24 B, key kernel)
  * shard write through the pinned pipeline: to /dev/null (pipeline and D2H
    only) and to a file under --dir (adds the file system)
  * CPU baseline: the reference's output stage for one rank (coupled map,
    text, blocks_to_uncoupled, text; oracle_export_text) on the first
    --cpu-items items, 1 thread

  python tools/blocks_bench.py [--config C3] [--dir /tmp] [--cpu-items 100000]
"""
import argparse
import json
import os
import sys
import tempfile
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
from paper_2507_03840_b200 import esg  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="C3")
    ap.add_argument("--dir", default=tempfile.gettempdir())
    ap.add_argument("--cpu-items", type=int, default=100000)
    ap.add_argument("--reps", type=int, default=5)
    args = ap.parse_args()
    torch.cuda.set_device(0)
    ctx = esg.Context(0)
    s, r, layers, basis = esg.config_structure(args.config)
    cfg = esg.ModelConfig(l_max=4, e_width=16, layers=layers, n_radial=32, r_cut=r, seed=1,
                          linear_precision=esg.LINEAR_BF16)
    net = esg.Network(ctx, cfg, basis)
    net.init_params()
    g = esg.build_graph(ctx, s, r)
    net.prepare(g, s.species)
    net.forward(copy_out=False)
    nb, nv = net.blocks_count()
    ol = net.out_len
    with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
        peak = json.load(f)["hbm_gbs"]

    dk = torch.empty(nb * 24, dtype=torch.uint8, device="cuda:0")
    dv = torch.empty(nv, dtype=torch.float64, device="cuda:0")
    net.blocks_to_device(0, dv.data_ptr())  # warm-up (tables, offsets)
    vals_ms = min(net.blocks_to_device(0, dv.data_ptr()) for _ in range(args.reps))
    keys_ms = min(net.blocks_to_device(dk.data_ptr(), 0) for _ in range(args.reps))
    v_bytes = nb * ol * 4 + nv * 8
    k_bytes = nb * 24
    del dk, dv
    torch.cuda.empty_cache()

    # the pipeline's ceiling: pinned device -> host bandwidth (1 GiB, best of 3)
    src = torch.empty(1 << 30, dtype=torch.uint8, device="cuda:0")
    dst = torch.empty(1 << 30, dtype=torch.uint8, pin_memory=True)
    d2h = []
    for _ in range(3):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        dst.copy_(src, non_blocking=True)
        e1.record()
        torch.cuda.synchronize()
        d2h.append((1 << 30) / e0.elapsed_time(e1) / 1e6)
    d2h_gbs = max(d2h)
    del src, dst

    file_bytes = 64 + nb * 24 + nv * 8
    net.write_block_shard("/dev/null", esg.BLOCKS_UNCOUPLED)  # warm-up: pinned staging buffers
    null_s = []
    for _ in range(3):
        t = time.perf_counter()
        net.write_block_shard("/dev/null", esg.BLOCKS_UNCOUPLED)
        null_s.append(time.perf_counter() - t)
    null_s = min(null_s)
    path = os.path.join(args.dir, "esg_blocks_bench.blk")
    disk_s = None
    try:
        st = os.statvfs(args.dir)
        if st.f_bavail * st.f_frsize > 2 * file_bytes:
            t = time.perf_counter()
            net.write_block_shard(path, esg.BLOCKS_UNCOUPLED)
            disk_s = time.perf_counter() - t
    finally:
        if os.path.exists(path):
            os.remove(path)

    # CPU baseline: the reference's output stage on a sample of items
    import oracle as O
    ni = min(args.cpu_items, nb)
    keys, shapes, off, _ = net.blocks(esg.BLOCKS_COUPLED)
    no, eo, _ = net.forward()
    rows = np.concatenate([no, eo])[:ni]
    om = O.Model(4, 16, layers, 32, r, 1, basis)
    d = tempfile.mkdtemp()
    t = time.perf_counter()
    om.export_text(keys[:ni], rows, s.species, os.path.join(d, "c.txt"), os.path.join(d, "u.txt"))
    cpu_s = time.perf_counter() - t
    text_bytes = os.path.getsize(os.path.join(d, "c.txt")) + os.path.getsize(os.path.join(d, "u.txt"))
    for fn in ("c.txt", "u.txt"):
        os.remove(os.path.join(d, fn))
    os.rmdir(d)

    out = {
        "config": args.config, "items": nb, "atoms": s.n_atoms, "edges": g.n_edges, "values": nv,
        "value_kernel": {"ms": vals_ms, "bytes": v_bytes, "gbs": v_bytes / vals_ms / 1e6,
                         "frac_hbm": v_bytes / vals_ms / 1e6 / peak, "items_per_s": nb / vals_ms * 1e3},
        "key_kernel": {"ms": keys_ms, "bytes": k_bytes, "gbs": k_bytes / keys_ms / 1e6},
        "shard": {"bytes": file_bytes, "devnull_s": null_s, "devnull_gbs": file_bytes / null_s / 1e9,
                  "disk_s": disk_s, "disk_gbs": file_bytes / disk_s / 1e9 if disk_s else None,
                  "dir": args.dir, "items_per_s_devnull": nb / null_s, "pinned_d2h_gbs": d2h_gbs,
                  "frac_d2h": file_bytes / null_s / 1e9 / d2h_gbs},
        "cpu_baseline": {"items": int(ni), "s": cpu_s, "items_per_s": ni / cpu_s, "cores": 1,
                         "text_bytes": text_bytes, "kind": "port",
                         "what": "coupled map + text + blocks_to_uncoupled + text (model_run.cpp:141-153)"},
        "hbm_peak_gbs": peak,
    }
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
