"""fp32 forward (fp16x3 chain) on one GPU: the same graph with the default
edge chunking, with small chunks, and on the tf32 path.  Chunking must not
change a bit (the table scales are whole-table maxima); tf32 vs fp16x3 must
agree to fp32 rounding.

  python tools/f3_chunk_check.py [--config C3]
"""
import argparse
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2507_03840_b200 import esg  # noqa: E402


def run(ctx, g, s, cfg, basis, env):
    old = {k: os.environ.get(k) for k in env}
    os.environ.update(env)
    try:
        net = esg.Network(ctx, cfg, basis)
        net.init_params()
        net.prepare(g, s.species)
        no, eo, tm = net.forward()
        net.close()
    finally:
        for k, v in old.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v
    return no, eo


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="C3")
    a = ap.parse_args()
    s, r, layers, basis = esg.config_structure(a.config)
    ctx = esg.Context(0, 0, 1)
    cfg = esg.ModelConfig(l_max=4, e_width=16, layers=layers, n_radial=32, r_cut=r, seed=1,
                          linear_precision=esg.LINEAR_FP32)
    g = esg.build_graph(ctx, s, r)
    print(a.config, "edges", g.n_edges, flush=True)
    base = run(ctx, g, s, cfg, basis, {})
    runs = [("default again", {}), ("chunk 700k", {"ESG_CHUNK_EDGES": "700000"}),
            ("chunk 1M", {"ESG_CHUNK_EDGES": "1048576"}), ("chunk 4M", {"ESG_CHUNK_EDGES": "4194304"}),
            ("chunk 64k", {"ESG_CHUNK_EDGES": "65536"}), ("tf32", {"ESG_F16X3": "0"}),
            ("tf32 64k", {"ESG_F16X3": "0", "ESG_CHUNK_EDGES": "65536"})]
    for name, env in runs:
        o = run(ctx, g, s, cfg, basis, env)
        for nm, x, y in (("nodes", o[0], base[0]), ("edges", o[1], base[1])):
            d = np.abs(x - y)
            i = np.unravel_index(np.argmax(d), d.shape)
            print(f"{name:10s} {nm}: bit-exact {np.array_equal(x, y)} max|diff| {d.max():.3e} at {i} "
                  f"(|y| max {np.abs(y).max():.3e}, rel-L2 {np.linalg.norm(x - y) / np.linalg.norm(y):.3e}, "
                  f"rows differing {int((d.reshape(d.shape[0], -1).max(1) > 0).sum())})", flush=True)


if __name__ == "__main__":
    main()
