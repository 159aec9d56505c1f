import sys, os
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np
import oracle as O
from paper_2507_03840_b200 import esg
ctx = esg.Context(0)
s = esg.make_jittered_lattice(40, 2.2, 0.45, [72, 8, 8], 4)
cfg = esg.ModelConfig(l_max=4, e_width=16, layers=2, n_radial=32, r_cut=4.5, seed=1)
net = esg.Network(ctx, cfg, esg.BASIS_HFO2); net.init_params()
g = esg.build_graph(ctx, s, 4.5); net.prepare(g, s.species)
no, eo, _ = net.forward()
flat = net.blocks_uncoupled()
om = O.Model(4, 16, 2, 32, 4.5, 1, esg.BASIS_HFO2)
norb = {72: 10, 8: 4}
sp = s.species; ref = g.export()
items = [(sp[i], sp[i], no[i]) for i in range(s.n_atoms)] + [(sp[a], sp[b], eo[k]) for k, (a, b) in enumerate(zip(ref["src"], ref["dst"]))]
at = 0; bad = 0
for idx, (za, zb, row) in enumerate(items):
    n = norb[za] * norb[zb]
    want = om.uncoupled_block(za, zb, row, norb[za], norb[zb])
    got = flat[at:at + n].reshape(norb[za], norb[zb])
    if np.abs(got - want).max() > 1e-5 and bad < 3:
        bad += 1
        np.set_printoptions(precision=3, suppress=True, linewidth=200)
        print("item", idx, za, zb); print("got\n", got); print("want\n", want)
    at += n
print("total", at, flat.size, "bad items", sum(1 for _ in []))
