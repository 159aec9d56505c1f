"""Golden head samples of BASELINE config 3 (20,000-atom HfO2, 12 A, 3
layers, 12.8M edges) from the float oracle (oracle/oracle.cpp, the CPU
restatement pinned to the reference build by tests/test_ref_pin.py).  The
full oracle forward takes ~15 min on 8 cores, too long for a GPU-box test, so
its heads on a fixed sample are committed: 512 nodes and 4,096 edges (seeded
choice, global indices), float32.

  python tools/make_c3_golden.py   # -> tests/golden/c3_heads_sample.npz
"""
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import oracle as O  # noqa: E402
from paper_2507_03840_b200 import esg  # noqa: E402


def main():
    s, r, layers, basis = esg.config_structure("C3")
    t0 = time.time()
    g = O.build_graph(s.positions, s.cell, np.ones(3, np.uint8), r)
    om = O.Model(4, 16, layers, 32, r, 1, basis)
    no, eo = om.forward(O.serial_view(s.n_atoms, s.species, g), np.float32)
    rng = np.random.default_rng(2026)
    ni = np.sort(rng.choice(s.n_atoms, 512, replace=False))
    ei = np.sort(rng.choice(len(g["src"]), 4096, replace=False))
    np.savez_compressed(os.path.join(ROOT, "tests", "golden", "c3_heads_sample.npz"), node_index=ni,
                        node_heads=no[ni], edge_index=ei, edge_heads=eo[ei], n_edges=len(g["src"]),
                        node_max=np.abs(no).max(), edge_max=np.abs(eo).max(),
                        node_l2=np.linalg.norm(no.astype(np.float64)), edge_l2=np.linalg.norm(eo.astype(np.float64)))
    print(f"C3 oracle forward {time.time() - t0:.0f} s, {O.num_threads()} threads, {len(g['src'])} edges")


if __name__ == "__main__":
    main()
