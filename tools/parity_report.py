"""Parity report: GPU forward (fp32 CUDA-core linears and bf16 tcgen05
linears) against the CPU oracle in float32 and float64, on C1 and C2.
Prints one JSON line per (config, mode) with max-abs / relative errors of
the node and edge Hamiltonian heads and of the uncoupled blocks.

  python tools/parity_report.py [C1 C2] > profiles/parity_r01.jsonl
"""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import oracle as O  # noqa: E402
from paper_2507_03840_b200 import esg  # noqa: E402


def errs(got, want):
    d = np.abs(got.astype(np.float64) - want.astype(np.float64))
    scale = float(np.abs(want).max())
    return {"max_abs": float(d.max()), "max_abs_over_max_ref": float(d.max() / scale),
            "rel_l2": float(np.linalg.norm(d) / np.linalg.norm(want)), "ref_max": scale}


def main():
    names = sys.argv[1:] or ["C1", "C2"]
    ctx = esg.Context(0)
    for name in names:
        s, r, layers, basis = esg.config_structure(name)
        g = esg.build_graph(ctx, s, r)
        gx = g.export()
        view = O.serial_view(s.n_atoms, s.species, gx)
        om = O.Model(4, 16, layers, 32, r, 1, basis)
        t0 = time.time()
        rno32, reo32 = om.forward(view, np.float32)
        t32 = time.time() - t0
        t0 = time.time()
        rno64, reo64 = om.forward(view, np.float64)
        t64 = time.time() - t0
        oracle_gap = {"node": errs(rno32, rno64), "edge": errs(reo32, reo64)}
        print(json.dumps({"config": name, "mode": "oracle_f32_vs_f64", "edges": g.n_edges, "oracle_s": [t32, t64],
                          **oracle_gap}), flush=True)
        for mode, prec in (("gpu_fp32", esg.LINEAR_FP32), ("gpu_bf16_tcgen05", esg.LINEAR_BF16)):
            cfg = esg.ModelConfig(l_max=4, e_width=16, layers=layers, n_radial=32, r_cut=r, seed=1,
                                  linear_precision=prec)
            net = esg.Network(ctx, cfg, basis)
            net.init_params()
            net.prepare(g, s.species)
            no, eo, tm = net.forward()
            blocks = net.blocks_uncoupled()
            line = {"config": name, "mode": mode, "edges": g.n_edges, "forward_ms": tm.forward_ms,
                    "vs_oracle_f32": {"node": errs(no, rno32), "edge": errs(eo, reo32)},
                    "vs_oracle_f64": {"node": errs(no, rno64), "edge": errs(eo, reo64)},
                    "blocks_values": int(blocks.size), "blocks_finite": bool(np.isfinite(blocks).all())}
            print(json.dumps(line), flush=True)
            net.close()


if __name__ == "__main__":
    main()
