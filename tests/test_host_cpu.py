"""Host-side logic of libesg_b200.so against the oracle, and the C-ABI
surface -- no GPU needed (nothing here launches a kernel)."""
import ctypes as C
import os
import re

import numpy as np
import pytest

import oracle as O
from paper_2507_03840_b200 import esg

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_library_exports_every_declared_symbol():
    header = open(os.path.join(ROOT, "include", "esg.h")).read()
    names = sorted(set(re.findall(r"\b(esg_[a-z0-9_]+)\s*\(", header)))
    assert len(names) > 30
    lib = esg.lib()
    missing = [n for n in names if not hasattr(lib, n)]
    assert not missing, missing


@pytest.mark.parametrize("args", [(512, 2.71, 0.30, [14], 1), (3000, 2.20, 0.45, [72, 8, 8], 2),
                                  (40, 1.5, 0.4, [1, 8], 7)])
def test_jittered_lattice_bitwise(args):
    s = esg.make_jittered_lattice(*args)
    pos, cell, sp = O.jittered_lattice(*args)
    assert np.array_equal(s.positions, pos) and np.array_equal(s.cell, cell) and np.array_equal(s.species, sp)


def test_tile_bitwise():
    s = esg.make_jittered_lattice(60, 2.2, 0.45, [72, 8, 8], 2)
    t = esg.tile(s, [2, 3, 1])
    pos, cell, sp = O.tile(s.positions, s.cell, np.ones(3, np.uint8), s.species, [2, 3, 1])
    assert np.array_equal(t.positions, pos) and np.array_equal(t.cell, cell) and np.array_equal(t.species, sp)
    with pytest.raises(esg.UsageError):
        esg.tile(esg.AtomicStructure(s.positions, s.species, s.cell, np.array([1, 1, 0], bool)), [1, 1, 2])


@pytest.mark.parametrize("seed", [1, 2, 3, 4])
def test_wrap_bitwise(seed):
    rng = np.random.default_rng(seed)
    cell = np.array([[6.0, 0.4, 0.0], [0.9, 5.5, 0.3], [0.2, 0.6, 6.5]]) * (1 + seed)
    pos = rng.normal(scale=20.0, size=(50, 3))
    for pbc in ([1, 1, 1], [1, 0, 1], [0, 0, 0]):
        s = esg.AtomicStructure(pos, np.ones(50, np.int32), cell, np.array(pbc, bool))
        assert np.array_equal(esg.wrap_positions(s), O.wrap(pos, cell, np.array(pbc, np.uint8)))


@pytest.mark.parametrize("depth", [0, 1, 2, 3])
def test_lownn_matches_oracle(depth):
    for args, r in (((512, 2.71, 0.30, [14], 1), 8.0), ((3000, 2.20, 0.45, [72, 8, 8], 2), 12.0)):
        s = esg.make_jittered_lattice(*args)
        g = O.build_graph(s.positions, s.cell, np.ones(3, np.uint8), r)
        deg = O.in_degrees(s.n_atoms, g)
        want = O.lownn(s.positions, s.cell, np.ones(3, np.uint8), deg, depth, r)
        assert np.array_equal(esg.lownn_partition(s, deg, depth, r), want)


def test_lownn_errors_map_to_usage():
    s = esg.make_jittered_lattice(4, 2.0, 0.1, [1], 1)
    with pytest.raises(esg.UsageError):
        esg.lownn_partition(s, np.ones(4, np.int32), 3, 2.5)  # 8 parts > 4 atoms


def test_lownn_gpu_entry_rejects_null_context():
    # the device Low-NN has no host fallback: without a context it is a usage
    # error (checked before any device work, so this runs without a GPU)
    s = esg.make_jittered_lattice(8, 2.0, 0.1, [1], 1)
    part = np.zeros(8, np.int32)
    rc = esg.lib().esg_lownn_partition_gpu(None, C.c_int(8), esg._p(s.positions), esg._p(s.cell), esg._p(s._pbc8()),
                                           esg._p(np.ones(8, np.int32)), C.c_int(1), C.c_double(2.5), esg._p(part))
    assert rc == 2 and b"ctx" in esg.lib().esg_last_error()


@pytest.mark.parametrize("n_parts", [2, 4, 8])
def test_comm_plan_matches_oracle(n_parts):
    s = esg.make_jittered_lattice(400, 2.2, 0.45, [72, 8, 8], 3)
    pbc = np.ones(3, np.uint8)
    g = O.build_graph(s.positions, s.cell, pbc, 5.0)
    deg = O.in_degrees(400, g)
    part = O.lownn(s.positions, s.cell, pbc, deg, int(np.log2(n_parts)), 5.0)
    off = np.concatenate([[0], np.cumsum(deg)]).astype(np.int64)
    for rank in range(n_parts):
        want = O.comm_plan(400, g["src"], g["dst"], part, n_parts, rank)
        got = esg.CommPlan(None, s.species, part, n_parts, rank, csr=(off, g["src"])).export()
        for k in ("row_global", "edge_index", "src_row", "dst_row", "nbr_peer", "nbr_recv_row", "nbr_recv_count",
                  "nbr_send_count", "send_rows"):
            assert np.array_equal(got[k], want[k]), k


def hfo2_cfg(**kw):
    c = dict(l_max=4, e_width=16, layers=3, n_radial=32, r_cut=12.0, seed=1)
    c.update(kw)
    return esg.ModelConfig(**c)


def test_params_bitwise_and_named_like_reference():
    m = esg.Network(None, hfo2_cfg(), esg.BASIS_HFO2)
    m.init_params()
    om = O.Model(4, 16, 3, 32, 12.0, 1, esg.BASIS_HFO2)
    assert m.entries() == om.entries()
    assert np.array_equal(m.params(), om.params_f32())
    assert m.out_len == om.out_len == 160
    # ~1.05M parameters for M=3, HfO2 heads
    assert 1.0e6 < m.n_params < 1.1e6


def test_si_head_layout():
    m = esg.Network(None, esg.ModelConfig(l_max=4, e_width=16, layers=1, r_cut=8.0), esg.BASIS_SI)
    om = O.Model(4, 16, 1, 32, 8.0, 1, esg.BASIS_SI)
    assert m.out_len == om.out_len


def test_param_hash_changes_with_values():
    m = esg.Network(None, esg.ModelConfig(l_max=2, e_width=8, layers=1), {1: [0, 1], 8: [0, 1]})
    m.init_params()
    h0 = m.param_hash()
    p = m.params()
    p[5] += 1.0
    m.set_params(p)
    assert m.param_hash() != h0


def test_model_config_validation():
    with pytest.raises(esg.UsageError):
        esg.Network(None, esg.ModelConfig(l_max=7), {1: [0]})
    with pytest.raises(esg.UsageError):  # l_max cannot couple d x d shells
        esg.Network(None, esg.ModelConfig(l_max=2), {72: [0, 2]})
    with pytest.raises(esg.DataError):
        esg.Network(None, esg.ModelConfig(l_max=2), {1: [9]})


def test_acceptance_counts():
    """acceptance.cpp:466-496 criterion 6: 1000 Hf + 2000 O in the SZV basis
    is an 18,000-orbital Hamiltonian; the generator gives 1000 Hf of 3000;
    tiling 2x2x2 gives 24,000 atoms; a message row is 3 x 25 x 16 fp32 = 4,800 B."""
    n_orb = {z: sum(2 * l + 1 for l in ls) for z, ls in esg.BASIS_HFO2.items()}
    assert 1000 * n_orb[72] + 2000 * n_orb[8] == 18000
    cell = esg.make_jittered_lattice(3000, 2.4, 0.1, [72, 8, 8], 2)
    assert cell.n_atoms == 3000 and int((cell.species == 72).sum()) == 1000
    assert esg.tile(cell, (2, 2, 2)).n_atoms == 24000
    assert 3 * 25 * 16 * 4 == 4800


def test_facade_demo_host_only():
    """csrc/facade_demo.cpp through esgnn_b200.hpp without a GPU: parameter
    store, coupling tables and the error mapping (UsageError)."""
    import os
    import subprocess
    demo = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "paper_2507_03840_b200",
                        "facade_demo")
    if not os.path.exists(demo):
        pytest.skip("facade_demo not built")
    out = subprocess.run([demo, "--host-only"], capture_output=True, text=True, timeout=120)
    assert out.returncode == 0, out.stdout + out.stderr
    assert "usage error mapped" in out.stdout and "out_len 160" in out.stdout
    assert "extxyz round trip exact" in out.stdout
