"""Partition baselines (OUT OF SCOPE for the product): the
mincut edge-cut baseline lives only in the oracle (tests/oracle.py, a
restatement of mincut.cpp:16-201) as the comparison point for Low-NN.  The
reference's own KATs pin the restatement (test_partition.cpp:112-196) and
Low-NN (the product's host and device partitioners) must cut to no more
neighbours than it."""
import numpy as np
import pytest

import oracle as O
from paper_2507_03840_b200 import esg


def csr(g, n):
    off = np.zeros(n + 1, np.int64)
    np.cumsum(np.bincount(g["dst"], minlength=n), out=off[1:])
    return off, np.asarray(g["src"], np.int32)


def count_cut(off, src, part):
    dst = np.repeat(np.arange(len(off) - 1), np.diff(off))
    return int((part[src] != part[dst]).sum())


def test_mincut_kats():
    # separated clusters split with zero cut (test_partition.cpp:162-178)
    pos = np.array([[c * 50.0 + 0.9 * (i % 2), 0.9 * (i // 2), 0.0] for c in range(2) for i in range(4)])
    g = O.build_graph(pos, np.eye(3) * 200.0, np.zeros(3, np.uint8), 1.5)
    off, src = csr(g, 8)
    p = O.mincut(8, off, src, 2, 3)
    assert count_cut(off, src, p) == 0 and p[0] == p[1] == p[2] and p[4] == p[5] and p[0] != p[4]
    # beats random balanced bisections (test_partition.cpp:180-196)
    pos, cell, _ = O.jittered_lattice(60, 1.4, 0.3, [1], 9)
    g = O.build_graph(pos, cell, np.ones(3, np.uint8), 2.2)
    off, src = csr(g, 60)
    p = O.mincut(60, off, src, 2, 5)
    rng = np.random.default_rng(17)
    best = min(count_cut(off, src, (rng.permutation(60) >= 30).astype(np.int32)) for _ in range(50))
    assert count_cut(off, src, p) <= 2 * best
    assert np.array_equal(O.mincut(60, off, src, 2, 5), p)  # deterministic per seed


def test_lownn_fewer_neighbors_than_mincut():
    """test_partition.cpp:112-117 on the 8^3 lattice, depth 4 vs 16 parts."""
    pos = np.array([[(x + 0.5), (y + 0.5), (z + 0.5)] for x in range(8) for y in range(8) for z in range(8)])
    cell, pbc = np.eye(3) * 8.0, np.ones(3, np.uint8)
    g = O.build_graph(pos, cell, pbc, 1.01)
    off, src = csr(g, 512)
    low = O.lownn(pos, cell, pbc, np.diff(off).astype(np.int32), 4, 1.01)
    s = esg.AtomicStructure(pos, np.ones(512, np.int32), cell, np.ones(3, bool))
    assert np.array_equal(esg.lownn_partition(s, np.diff(off).astype(np.int32), 4, 1.01), low)
    cut = O.mincut(512, off, src, 16, 1)
    ml = O.compute_metrics(512, g["src"], g["dst"], low, 16)[1][2]
    mc = O.compute_metrics(512, g["src"], g["dst"], cut, 16)[1][2]
    assert ml <= mc + 1e-12
