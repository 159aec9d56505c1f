import os, sys
import numpy as np
sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/tests')
from paper_2507_03840_b200 import esg
import oracle as O
ctx = esg.Context(0)
s = esg.make_jittered_lattice(64, 2.2, 0.45, [esg.HF, esg.O, esg.O], 2)
r = 5.0
g = esg.build_graph(ctx, s, r)
ref = O.build_graph(s.positions, s.cell, np.ones(3, np.uint8), r)
cfg = esg.ModelConfig(l_max=4, e_width=16, layers=2, n_radial=32, r_cut=r, seed=1)
om = O.Model(4, 16, 2, 32, r, 1, esg.BASIS_HFO2)
nt, nm, et, em, nt64, et64 = om.toy_targets(s.n_atoms, s.species, ref)
n_total = int(nm.sum() + em.sum())
(sa, sq, _), rg = O.loss_grad(om, O.serial_view(s.n_atoms, s.species, ref), (nt64, nm, et64, em), n_total, np.float64)
for f3 in ("1", "0"):
    os.environ["ESG_F16X3"] = f3
    net = esg.Network(ctx, cfg, esg.BASIS_HFO2)
    net.init_params()
    net.prepare(g, s.species)
    net.set_targets(nt, nm, et, em)
    loss, _, grads = net.loss_grad(n_total)
    gerr = float(np.linalg.norm(grads - rg) / np.linalg.norm(rg))
    print("F16X3", f3, "loss", loss, (sa + sq) / n_total, "gerr", gerr, "edges", g.n_edges)
    worst = []
    for name, rows, cols, off in om.entries():
        a = grads[off:off + rows * cols].astype(np.float64); b = rg[off:off + rows * cols]
        worst.append((float(np.linalg.norm(a - b)), float(np.linalg.norm(b)), name))
    worst.sort(reverse=True)
    for w in worst[:8]: print("   ", w)
    net.close()
