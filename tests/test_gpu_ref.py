"""The B200 path against the REFERENCE implementation itself (oracle/_ref,
the /root/reference sources compiled unmodified against oracle/eigen_shim;
see tests/test_ref_pin.py for the restated oracle against the same).

Bars as tests/test_gpu_parity.py: graph and partitions bit-exact; heads of
the fp32 path within max-abs 2e-4 x max and rel-L2 2e-5 of the reference's
float forward (Network<float>::build_forward, network.h:115-164).
"""
import numpy as np
import pytest

import ref as R
from paper_2507_03840_b200 import esg

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not R.available(), reason="oracle/_ref not built")]
PBC1 = np.ones(3, np.uint8)


def err(a, b):
    return np.abs(a - b).max() / max(np.abs(b).max(), 1e-30), np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-30)


@pytest.mark.parametrize("name", ["C1", "C2"])
def test_device_graph_and_lownn_equal_reference(gpu_ctx, name):
    s, r, _, _ = esg.config_structure(name)
    want = R.build_graph(s.positions, s.species, s.cell, PBC1, r)
    g = esg.build_graph(gpu_ctx, s, r)
    got = g.export()
    for k in ("src", "dst", "shift"):
        assert np.array_equal(np.asarray(got[k]).reshape(-1), want[k].reshape(-1)), k
    for k in ("disp", "dist"):
        assert np.array_equal(got[k].view(np.uint64), want[k].view(np.uint64)), k
    deg = g.in_degrees()
    for depth in (1, 2, 3):
        assert np.array_equal(esg.lownn_partition_gpu(gpu_ctx, s, deg, depth, r),
                              R.lownn(s.positions, s.species, s.cell, PBC1, depth, r)), depth


@pytest.mark.parametrize("case", ["small", "C1"])
def test_fp32_forward_equals_reference(gpu_ctx, case):
    if case == "C1":
        s, r, layers, basis = esg.config_structure("C1")
    else:
        s, r, layers, basis = esg.make_jittered_lattice(40, 2.2, 0.45, [72, 8, 8], 4), 4.5, 2, esg.BASIS_HFO2
    rno, reo, _ = R.forward(s.positions, s.species, s.cell, PBC1, r, basis, layers=layers, precision=4)
    cfg = esg.ModelConfig(l_max=4, e_width=16, layers=layers, n_radial=32, r_cut=r, seed=1,
                          linear_precision=esg.LINEAR_FP32)
    net = esg.Network(gpu_ctx, cfg, basis)
    net.init_params()
    g = esg.build_graph(gpu_ctx, s, r)
    net.prepare(g, s.species)
    no, eo, _ = net.forward()
    for got, want in ((no, rno), (eo, reo)):
        mx, rl2 = err(got.astype(np.float64), want)
        assert mx < 2e-4 and rl2 < 2e-5, (case, mx, rl2)
    net.close()
    g.close()
