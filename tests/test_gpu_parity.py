"""GPU parity: the CUDA path through the C ABI against the CPU oracle.

Bars (SURVEY.md §8 / BASELINE.json north_star):
  * graph (src, dst, shift) and fp64 displacement / distance: bit-exact
  * partition assignments and comm plans from the GPU graph: bit-exact
  * Hamiltonian heads, fp32 linears: max-abs error <= 2e-4 x max|ref| and
    relative-L2 <= 2e-5 against the float oracle (stated fp32 tolerance)
  * bf16 tcgen05 linears: relative-L2 <= 2e-2, max-abs <= 5e-2 x max|ref|
"""
import numpy as np
import pytest

import oracle as O
from paper_2507_03840_b200 import esg

pytestmark = pytest.mark.gpu

SKEW = np.array([[6.0, 0.4, 0.0], [0.9, 5.5, 0.3], [0.2, 0.6, 6.5]])


PLAN_KEYS = ("row_global", "edge_index", "src_row", "dst_row", "send_rows", "nbr_peer", "nbr_recv_row",
             "nbr_recv_count", "nbr_send_count")


def same_graph(g, ref):
    assert len(g["src"]) == len(ref["src"])
    for k in ("src", "dst", "shift"):
        assert np.array_equal(g[k], ref[k]), k
    # bitwise fp64 equality (not allclose)
    assert np.array_equal(g["disp"].view(np.uint64), ref["disp"].view(np.uint64))
    assert np.array_equal(g["dist"].view(np.uint64), ref["dist"].view(np.uint64))


@pytest.mark.parametrize("pbc", [(1, 1, 1), (0, 0, 0), (1, 0, 1)])
@pytest.mark.parametrize("seed", [1, 2, 3])
def test_graph_kat_random_skewed(gpu_ctx, pbc, seed):
    rng = np.random.default_rng(seed)
    pos = rng.random((8, 3)) @ SKEW
    s = esg.AtomicStructure(pos, np.ones(8, np.int32), SKEW.copy(), np.array(pbc, bool))
    g = esg.build_graph(gpu_ctx, s, 4.0).export()
    same_graph(g, O.build_graph(pos, SKEW, np.array(pbc, np.uint8), 4.0))


def test_graph_edge_cases(gpu_ctx):
    two = esg.AtomicStructure(np.array([[0.0, 0, 0], [3.0, 0, 0]]), np.ones(2, np.int32), np.eye(3),
                              np.zeros(3, bool))
    assert esg.build_graph(gpu_ctx, two, 3.0).n_edges == 2  # inclusive cutoff
    assert esg.build_graph(gpu_ctx, two, 2.9999999).n_edges == 0
    one = esg.AtomicStructure(np.array([[1.0, 1, 1]]), np.array([6], np.int32), np.eye(3) * 2.0, np.ones(3, bool))
    g = esg.build_graph(gpu_ctx, one, 2.5).export()
    assert len(g["src"]) == 6 and np.allclose(g["dist"], 2.0)
    lone = esg.AtomicStructure(np.array([[0.0, 0, 0], [50.0, 0, 0]]), np.ones(2, np.int32), np.eye(3),
                               np.zeros(3, bool))
    assert esg.build_graph(gpu_ctx, lone, 3.0).n_edges == 0  # empty graph
    with pytest.raises(esg.UsageError):
        esg.build_graph(gpu_ctx, two, -1.0)


@pytest.mark.parametrize("name", ["C1", "C2"])
def test_graph_configs_bit_exact(gpu_ctx, name):
    s, r, _, _ = esg.config_structure(name)
    g = esg.build_graph(gpu_ctx, s, r)
    ref = O.build_graph(s.positions, s.cell, np.ones(3, np.uint8), r)
    same_graph(g.export(), ref)
    # partitions from the GPU graph (depth 1..3) and every rank's plan
    deg = g.in_degrees()
    for depth in (1, 2, 3):
        part = esg.lownn_partition(s, deg, depth, r)
        assert np.array_equal(part, O.lownn(s.positions, s.cell, np.ones(3, np.uint8), deg, depth, r))
        for rank in range(1 << depth):
            got = esg.build_comm_plan(g, s.species, part, 1 << depth, rank).export()
            want = O.comm_plan(s.n_atoms, ref["src"], ref["dst"], part, 1 << depth, rank)
            for k in PLAN_KEYS:
                assert np.array_equal(got[k], want[k]), (name, depth, rank, k)


def test_graph_c4_bit_exact_and_plans(gpu_ctx):
    """The bench workload's graph (C4: 192k atoms, 69.6M edges at 10 A) is
    bit-exact against the oracle's build_graph (graph.cpp:55-131); Low-NN at
    depth 3 on the host and on the device equals the oracle
    (lownn.cpp:105-133); every rank's comm plan equals comm_plan.cpp:11-106."""
    s, r, _, _ = esg.config_structure("C4")
    g = esg.build_graph(gpu_ctx, s, r)
    ref = O.build_graph(s.positions, s.cell, np.ones(3, np.uint8), r)
    assert g.n_edges == 69626112
    same_graph(g.export(), ref)
    deg = g.in_degrees()
    assert np.array_equal(deg, O.in_degrees(s.n_atoms, ref))
    part = O.lownn(s.positions, s.cell, np.ones(3, np.uint8), deg, 3, r)
    assert np.array_equal(esg.lownn_partition(s, deg, 3, r), part)
    assert np.array_equal(esg.lownn_partition_gpu(gpu_ctx, s, deg, 3, r), part)
    for rank in range(8):
        got = esg.build_comm_plan(g, s.species, part, 8, rank).export()
        want = O.comm_plan(s.n_atoms, ref["src"], ref["dst"], part, 8, rank)
        for k in PLAN_KEYS:
            assert np.array_equal(got[k], want[k]), (rank, k)
    g.close()


def test_graph_sort_fallback(gpu_ctx, monkeypatch):
    """The per-destination key sort runs as a shared-memory bitonic sort when
    every segment fits (the other graph tests) and as cub's segmented radix
    sort otherwise; ESG_SEG_SORT_CAP=0 forces the latter."""
    monkeypatch.setenv("ESG_SEG_SORT_CAP", "0")
    s, r, _, _ = esg.config_structure("C1")
    same_graph(esg.build_graph(gpu_ctx, s, r).export(), O.build_graph(s.positions, s.cell, np.ones(3, np.uint8), r))


def test_graph_tiling_x8(gpu_ctx):
    """test_structures.cpp:166-189 on the skewed cell (no exact-cutoff ties)."""
    pos = np.random.default_rng(13).random((5, 3)) @ SKEW
    s = esg.AtomicStructure(pos, np.ones(5, np.int32), SKEW.copy(), np.ones(3, bool))
    t = esg.tile(s, [2, 2, 2])
    gs, gt = esg.build_graph(gpu_ctx, s, 4.0), esg.build_graph(gpu_ctx, t, 4.0)
    assert gt.n_edges == 8 * gs.n_edges
    assert np.array_equal(gt.in_degrees(), np.tile(gs.in_degrees(), 8))
    same_graph(gt.export(), O.build_graph(t.positions, t.cell, np.ones(3, np.uint8), 4.0))
    # a cell exactly 2 r_cut wide has distance ties at the cutoff: whatever the
    # reference arithmetic keeps, the GPU keeps too
    j = esg.tile(esg.make_jittered_lattice(5, 2.0, 0.3, [1, 8], 13), [2, 2, 2])
    same_graph(esg.build_graph(gpu_ctx, j, 4.0).export(), O.build_graph(j.positions, j.cell, np.ones(3, np.uint8), 4.0))


def run_both(ctx, s, r, layers, basis, l_max=4, e=16, prec=esg.LINEAR_FP32, dtype=np.float32):
    cfg = esg.ModelConfig(l_max=l_max, e_width=e, layers=layers, n_radial=32, r_cut=r, seed=1,
                          linear_precision=prec)
    net = esg.Network(ctx, cfg, basis)
    net.init_params()
    g = esg.build_graph(ctx, s, r)
    net.prepare(g, s.species)
    no, eo, tm = net.forward()
    ref = O.build_graph(s.positions, s.cell, np.ones(3, np.uint8), r)
    om = O.Model(l_max, e, layers, 32, r, 1, basis)
    rno, reo = om.forward(O.serial_view(s.n_atoms, s.species, ref), dtype)
    return net, (no, eo, tm), (rno, reo), om, ref


def err(a, b):
    scale = max(np.abs(b).max(), 1e-30)
    return np.abs(a - b).max() / scale, np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-30)


@pytest.mark.parametrize("l_max,e", [(4, 16), (2, 8)])
def test_forward_fp32_small(gpu_ctx, l_max, e):
    s = esg.make_jittered_lattice(40, 2.2, 0.45, [72, 8, 8], 4)
    basis = esg.BASIS_HFO2 if l_max == 4 else {72: [0, 1], 8: [0, 1]}
    net, (no, eo, tm), (rno, reo), _, _ = run_both(gpu_ctx, s, 4.5, 2, basis, l_max, e)
    for got, want in ((no, rno), (eo, reo)):
        mx, rl2 = err(got, want)
        assert mx < 2e-4 and rl2 < 2e-5, (mx, rl2)
    assert tm.gpu_launches > 0


def test_forward_fp32_c1(gpu_ctx):
    s, r, layers, basis = esg.config_structure("C1")
    net, (no, eo, tm), (rno, reo), _, _ = run_both(gpu_ctx, s, r, layers, basis)
    for got, want in ((no, rno), (eo, reo)):
        mx, rl2 = err(got, want)
        assert mx < 2e-4 and rl2 < 2e-5, (mx, rl2)
    # deterministic: a second forward is bitwise identical
    no2, eo2, _ = net.forward()
    assert np.array_equal(no, no2) and np.array_equal(eo, eo2)


def test_forward_c2_three_layers(gpu_ctx):
    """BASELINE config 2: the 3-layer forward (network.h:115-164 at M = 3) on
    the 3,000-atom HfO2 structure, 1.86M edges.  fp32 linears: heads and
    uncoupled blocks within the fp32 bar of the float oracle; bf16 linears
    within their stated bar; serial determinism."""
    s, r, layers, basis = esg.config_structure("C2")
    net, (no, eo, tm), (rno, reo), om, ref = run_both(gpu_ctx, s, r, layers, basis)
    assert tm.gpu_launches > 0 and net.n_edges == 1860036
    for got, want in ((no, rno), (eo, reo)):
        mx, rl2 = err(got, want)
        assert mx < 2e-4 and rl2 < 2e-5, (mx, rl2)
    # uncoupled blocks (block_matrix.cpp:66-88) of the device export against
    # the oracle's to_block of the oracle heads, on a sample of items
    flat = net.blocks_uncoupled()
    norb = {72: 10, 8: 4}
    sp = s.species
    sizes = np.array([norb[z] for z in sp])
    item_n = np.concatenate([sizes * sizes, sizes[ref["src"]] * sizes[ref["dst"]]])
    starts = np.concatenate([[0], np.cumsum(item_n)])
    assert starts[-1] == flat.size
    rng = np.random.default_rng(5)
    picks = np.concatenate([np.arange(64), s.n_atoms + rng.choice(len(ref["src"]), 400, replace=False)])
    for it in picks:
        if it < s.n_atoms:
            za, zb, row = sp[it], sp[it], rno[it]
        else:
            k = it - s.n_atoms
            za, zb, row = sp[ref["src"][k]], sp[ref["dst"][k]], reo[k]
        want = om.uncoupled_block(za, zb, row, norb[za], norb[zb]).ravel()
        got = flat[starts[it]:starts[it + 1]]
        scale = max(np.abs(reo).max(), np.abs(rno).max())
        assert np.abs(got - want).max() <= 2e-4 * scale, it
    no2, eo2, _ = net.forward()
    assert np.array_equal(no, no2) and np.array_equal(eo, eo2)
    net.set_precision(esg.LINEAR_BF16)
    nb, eb, _ = net.forward()
    for got, want in ((nb, rno), (eb, reo)):
        mx, rl2 = err(got, want)
        assert mx < 5e-2 and rl2 < 2e-2, (mx, rl2)


@pytest.mark.parametrize("prec", [esg.LINEAR_FP32, esg.LINEAR_BF16])
def test_forward_chunking_is_invisible(gpu_ctx, monkeypatch, prec):
    """The forward runs in destination-aligned edge chunks (model.cu
    model_prepare); every reduction is segment-local, so the chunk size must
    not change a bit.  C2 (1.86M edges) in one chunk against ~15 chunks, and
    a 300-atom case in 1,024-edge chunks against the oracle."""
    s, r, layers, basis = esg.config_structure("C2")
    cfg = esg.ModelConfig(l_max=4, e_width=16, layers=layers, n_radial=32, r_cut=r, seed=1, linear_precision=prec)
    g = esg.build_graph(gpu_ctx, s, r)
    outs = []
    for chunk in (None, "131072"):
        if chunk:
            monkeypatch.setenv("ESG_CHUNK_EDGES", chunk)
        net = esg.Network(gpu_ctx, cfg, basis)
        net.init_params()
        net.prepare(g, s.species)
        outs.append(net.forward()[:2])
        net.close()
    assert np.array_equal(outs[0][0], outs[1][0]) and np.array_equal(outs[0][1], outs[1][1])
    monkeypatch.setenv("ESG_CHUNK_EDGES", "1024")
    sm = esg.make_jittered_lattice(300, 2.2, 0.45, [72, 8, 8], 4)
    net, (no, eo, tm), (rno, reo), _, _ = run_both(gpu_ctx, sm, 4.5, 2, esg.BASIS_HFO2, prec=prec)
    assert net.n_edges > 4 * 1024
    bar = (2e-4, 2e-5) if prec == esg.LINEAR_FP32 else (5e-2, 2e-2)
    for got, want in ((no, rno), (eo, reo)):
        mx, rl2 = err(got, want)
        assert mx < bar[0] and rl2 < bar[1], (mx, rl2)


def test_forward_bf16_tensor_cores(gpu_ctx):
    s, r, layers, basis = esg.config_structure("C1")
    net, (no, eo, tm), (rno, reo), _, _ = run_both(gpu_ctx, s, r, layers, basis, prec=esg.LINEAR_BF16)
    for got, want in ((no, rno), (eo, reo)):
        mx, rl2 = err(got, want)
        assert mx < 5e-2 and rl2 < 2e-2, (mx, rl2)


def test_uncoupled_blocks_match_oracle(gpu_ctx):
    s = esg.make_jittered_lattice(40, 2.2, 0.45, [72, 8, 8], 4)
    net, (no, eo, tm), _, om, ref = run_both(gpu_ctx, s, 4.5, 2, esg.BASIS_HFO2)
    flat = net.blocks_uncoupled()
    norb = {72: 10, 8: 4}
    sp = s.species
    at = 0
    items = [(sp[i], sp[i], no[i]) for i in range(s.n_atoms)]
    items += [(sp[a], sp[b], eo[k]) for k, (a, b) in enumerate(zip(ref["src"], ref["dst"]))]
    for za, zb, row in items:
        n = norb[za] * norb[zb]
        want = om.uncoupled_block(za, zb, row, norb[za], norb[zb]).ravel()
        assert np.abs(flat[at:at + n] - want).max() <= 1e-5 * max(1.0, np.abs(want).max())
        at += n
    assert at == flat.size


def test_precision_switch_and_errors(gpu_ctx):
    s = esg.make_jittered_lattice(20, 2.2, 0.45, [72, 8, 8], 4)
    cfg = esg.ModelConfig(l_max=4, e_width=16, layers=1, r_cut=4.5)
    net = esg.Network(gpu_ctx, cfg, esg.BASIS_HFO2)
    with pytest.raises(esg.UsageError):
        net.forward()  # forward before prepare
    net.init_params()
    with pytest.raises(esg.DataError):  # species missing from the basis
        g = esg.build_graph(gpu_ctx, s, 4.5)
        net.prepare(g, np.full(20, 6, np.int32))


def test_streamed_outputs_match(gpu_ctx):
    """esg_forward into pinned host buffers streams the heads of each final
    chunk while the last edge block runs (C3: several chunks); the outputs
    are bit-identical to the copy-after-forward path of pageable buffers."""
    import torch
    s, r, layers, basis = esg.config_structure("C3")
    cfg = esg.ModelConfig(l_max=4, e_width=16, layers=layers, n_radial=32, r_cut=r, seed=1,
                          linear_precision=esg.LINEAR_BF16)
    net = esg.Network(gpu_ctx, cfg, basis)
    net.init_params()
    g = esg.build_graph(gpu_ctx, s, r)
    net.prepare(g, s.species)
    no, eo, _ = net.forward()
    pn = torch.empty((net.n_owned, net.out_len), dtype=torch.float32, pin_memory=True).numpy()
    pe = torch.empty((net.n_edges, net.out_len), dtype=torch.float32, pin_memory=True).numpy()
    pn[:] = np.nan
    pe[:] = np.nan
    net.forward_into(pn, pe)
    assert np.array_equal(pn.view(np.uint32), no.view(np.uint32))
    assert np.array_equal(pe.view(np.uint32), eo.view(np.uint32))
    net.close()
    g.close()


def test_async_outputs_do_not_race(gpu_ctx):
    """esg_forward_async: the next forward runs while the previous outputs
    drain, but its heads wait for those copies -- two back-to-back async
    forwards with different parameters deliver their own outputs, bit-exact."""
    import torch
    s, r, layers, basis = esg.config_structure("C3")
    cfg = esg.ModelConfig(l_max=4, e_width=16, layers=layers, n_radial=32, r_cut=r, seed=1,
                          linear_precision=esg.LINEAR_BF16)
    net = esg.Network(gpu_ctx, cfg, basis)
    net.init_params()
    g = esg.build_graph(gpu_ctx, s, r)
    net.prepare(g, s.species)
    p1 = net.params()
    p2 = (p1 * 1.01).astype(np.float32)
    want = []
    for p in (p1, p2):
        net.set_params(p)
        no, eo, _ = net.forward()
        want.append((no, eo))
    bufs = [(torch.empty((net.n_owned, net.out_len), dtype=torch.float32, pin_memory=True).numpy(),
             torch.empty((net.n_edges, net.out_len), dtype=torch.float32, pin_memory=True).numpy()) for _ in range(2)]
    for p, (bn, be) in zip((p1, p2), bufs):
        net.set_params(p)
        net.forward_into_async(bn, be)
    net.wait_outputs()
    for (bn, be), (no, eo) in zip(bufs, want):
        assert np.array_equal(bn.view(np.uint32), no.view(np.uint32))
        assert np.array_equal(be.view(np.uint32), eo.view(np.uint32))
    net.close()
    g.close()


def test_async_pipeline_builds_next_graph(gpu_ctx):
    """The e2e step pattern: an untimed esg_forward_async returns once the
    forward is queued, the next structure's graph builds on the context's
    build stream meanwhile, then prepare + forward on it.  Both outputs equal
    the synchronous forwards bit for bit."""
    import torch
    sa = esg.make_jittered_lattice(3000, 2.2, 0.45, [72, 8, 8], 2)
    sb = esg.make_jittered_lattice(3000, 2.2, 0.45, [72, 8, 8], 3)
    r = 8.0
    cfg = esg.ModelConfig(l_max=4, e_width=16, layers=2, n_radial=32, r_cut=r, seed=1,
                          linear_precision=esg.LINEAR_FP32)
    net = esg.Network(gpu_ctx, cfg, esg.BASIS_HFO2)
    net.init_params()
    want = []
    for st in (sa, sb):
        g = esg.build_graph(gpu_ctx, st, r)
        net.prepare(g, st.species)
        want.append(net.forward()[:2])
        g.close()
    ga = esg.build_graph(gpu_ctx, sa, r)
    net.prepare(ga, sa.species)
    bufs = []
    for k, st in enumerate((sa, sb)):
        if k:
            gb = esg.build_graph(gpu_ctx, st, r)  # while forward 0 runs
            net.prepare(gb, st.species)
        bn = torch.empty((net.n_owned, net.out_len), dtype=torch.float32, pin_memory=True).numpy()
        be = torch.empty((net.n_edges, net.out_len), dtype=torch.float32, pin_memory=True).numpy()
        assert net.forward_into_async(bn, be, timing=False) is None
        bufs.append((bn, be))
    net.wait_outputs()
    for (bn, be), (no, eo) in zip(bufs, want):
        assert np.array_equal(bn.view(np.uint32), no.view(np.uint32))
        assert np.array_equal(be.view(np.uint32), eo.view(np.uint32))
    net.close()
    ga.close()
    gb.close()


def test_forward_c3_golden_sample(gpu_ctx):
    """BASELINE config 3 (20,000-atom HfO2, 12.8M edges, 3 layers, seven
    edge chunks): the fp32 heads against the float oracle's on the committed
    sample (tests/golden/c3_heads_sample.npz, tools/make_c3_golden.py), fp32
    bar on the sample."""
    import os
    gd = np.load(os.path.join(os.path.dirname(__file__), "golden", "c3_heads_sample.npz"))
    s, r, layers, basis = esg.config_structure("C3")
    cfg = esg.ModelConfig(l_max=4, e_width=16, layers=layers, n_radial=32, r_cut=r, seed=1,
                          linear_precision=esg.LINEAR_FP32)
    net = esg.Network(gpu_ctx, cfg, basis)
    net.init_params()
    g = esg.build_graph(gpu_ctx, s, r)
    assert g.n_edges == int(gd["n_edges"])
    net.prepare(g, s.species)
    no, eo, _ = net.forward()
    got = np.concatenate([no[gd["node_index"]], eo[gd["edge_index"]]]).astype(np.float64)
    want = np.concatenate([gd["node_heads"], gd["edge_heads"]]).astype(np.float64)
    mx = np.abs(got - want).max() / max(float(gd["node_max"]), float(gd["edge_max"]))
    rl2 = np.linalg.norm(got - want) / np.linalg.norm(want)
    assert mx < 2e-4 and rl2 < 2e-5, (mx, rl2)
    net.close()
    g.close()
