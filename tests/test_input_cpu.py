"""Input side: extxyz ingest/output and the mincut baseline
partitioner, the product (C ABI) against pure-Python restatements in
tests/oracle.py, plus the reference's own KATs (test_structures.cpp:206-250,
test_partition.cpp:112-196)."""
import numpy as np
import pytest

import oracle as O
from paper_2507_03840_b200 import esg

SKEW = np.array([[6.0, 0.4, 0.0], [0.9, 5.5, 0.3], [0.2, 0.6, 6.5]])


def random_structure(n, seed, pbc):
    rng = np.random.default_rng(seed)
    pos = rng.random((n, 3)) @ SKEW
    return esg.AtomicStructure(pos, (1 + np.arange(n) % 3).astype(np.int32), SKEW.copy(), np.array(pbc, bool))


def csr(g, n):
    off = np.zeros(n + 1, np.int64)
    np.cumsum(np.bincount(g["dst"], minlength=n), out=off[1:])
    return off, np.asarray(g["src"], np.int32)


# ------------------------------------------------------------------ extxyz
@pytest.mark.parametrize("pbc", [(True, False, True), (False, False, False), (True, True, True)])
def test_extxyz_round_trip(tmp_path, pbc):
    """test_structures.cpp:206-218: exact positions, cell, pbc and species."""
    s = random_structure(7, 19, pbc)
    p = tmp_path / "s.xyz"
    esg.write_extxyz(str(p), s)
    assert p.read_text() == O.write_extxyz_text(s.positions, s.species, s.cell, s.pbc)
    r = esg.read_extxyz(str(p))
    assert np.array_equal(r.pbc, s.pbc) and np.array_equal(r.species, s.species)
    assert np.array_equal(r.positions, s.positions)
    if any(pbc):
        assert np.array_equal(r.cell, s.cell)
    else:
        assert np.array_equal(r.cell, np.eye(3))  # no Lattice written: the default cell


def test_extxyz_quoted_fields_and_extras(tmp_path):
    """test_structures.cpp:220-234."""
    text = ('2\nLattice="4 0 0 0 4 0 0 0 4" Properties=species:S:1:pos:R:3 pbc="T F T"\n'
            "Si 0.0 0.0 0.0 0.1 0.2\nO 1.5 1.5 1.5\n")
    p = tmp_path / "q.xyz"
    p.write_text(text)
    s = esg.read_extxyz(str(p))
    assert s.species.tolist() == [14, 8] and s.pbc.tolist() == [True, False, True]
    assert s.cell[1, 1] == 4.0 and s.positions[1, 2] == 1.5
    pos, sp, cell, pbc = O.read_extxyz_text(text)
    assert np.array_equal(pos, s.positions) and np.array_equal(cell, s.cell)


@pytest.mark.parametrize("text", [
    '2\nLattice="4 0 0 0 4"\nSi 0 0 0\nSi 1 1 1\n',  # short lattice
    '1\npbc="T T T"\nSi 0 0 0\n',  # pbc without a lattice
    "2\n\nSi 0 0 0\n",  # fewer atoms than declared
    '1\nkey="unterminated\nSi 0 0 0\n',
    "1\n\nSi 0 zero 0\n",  # not a number
    "1\n\nXx 0 0 0\n",  # unknown element
    "x\n\n",  # no atom count
    "",  # empty
    '1\npbc="T Q T" Lattice="1 0 0 0 1 0 0 0 1"\nSi 0 0 0\n',  # bad flag
])
def test_extxyz_errors(tmp_path, text):
    """test_structures.cpp:236-250 (ParseError is a DataError)."""
    p = tmp_path / "bad.xyz"
    p.write_text(text)
    with pytest.raises(esg.DataError):
        esg.read_extxyz(str(p))
    with pytest.raises((O.ParseError, ValueError)):
        O.read_extxyz_text(text)


def test_extxyz_of_the_bench_structure(tmp_path):
    """A full config through write -> read (C2, 3000 atoms) is bit-exact and
    its tiling reproduces tile()."""
    s, r, _, _ = esg.config_structure("C2")
    p = tmp_path / "c2.xyz"
    esg.write_extxyz(str(p), s)
    back = esg.read_extxyz(str(p))
    assert np.array_equal(back.positions, s.positions) and np.array_equal(back.cell, s.cell)
    t1, t2 = esg.tile(s, (2, 1, 1)), esg.tile(back, (2, 1, 1))
    assert np.array_equal(t1.positions, t2.positions)


# ------------------------------------------------------------------ mincut
@pytest.mark.parametrize("n_parts,seed", [(2, 1), (3, 5), (4, 3), (5, 1), (8, 2)])
def test_mincut_matches_restatement(n_parts, seed):
    pos, cell, species = O.jittered_lattice(80, 1.5, 0.35, [1, 8], 4)
    g = O.build_graph(pos, cell, np.ones(3, np.uint8), 2.6)
    off, src = csr(g, 80)
    got = esg.mincut_partition((off, src), n_parts, seed)
    want = O.mincut(80, off, src, n_parts, seed)
    assert np.array_equal(got, want)
    assert sorted(set(got.tolist())) == list(range(n_parts))


def count_cut(off, src, part):
    dst = np.repeat(np.arange(len(off) - 1), np.diff(off))
    return int((part[src] != part[dst]).sum())


def test_mincut_kats():
    # separated clusters split with zero cut (test_partition.cpp:162-178)
    pos = np.array([[c * 50.0 + 0.9 * (i % 2), 0.9 * (i // 2), 0.0] for c in range(2) for i in range(4)])
    g = O.build_graph(pos, np.eye(3) * 200.0, np.zeros(3, np.uint8), 1.5)
    off, src = csr(g, 8)
    p = esg.mincut_partition((off, src), 2, 3)
    assert count_cut(off, src, p) == 0 and p[0] == p[1] == p[2] and p[4] == p[5] and p[0] != p[4]
    # beats random balanced bisections (test_partition.cpp:180-196)
    pos, cell, _ = O.jittered_lattice(60, 1.4, 0.3, [1], 9)
    g = O.build_graph(pos, cell, np.ones(3, np.uint8), 2.2)
    off, src = csr(g, 60)
    p = esg.mincut_partition((off, src), 2, 5)
    rng = np.random.default_rng(17)
    best = min(count_cut(off, src, (rng.permutation(60) >= 30).astype(np.int32)) for _ in range(50))
    assert count_cut(off, src, p) <= 2 * best
    assert np.array_equal(esg.mincut_partition((off, src), 2, 5), p)  # deterministic per seed
    with pytest.raises(esg.UsageError):
        esg.mincut_partition((off, src), 0, 1)
    with pytest.raises(esg.UsageError):
        esg.mincut_partition((off, src), 61, 1)


def test_lownn_fewer_neighbors_than_mincut():
    """test_partition.cpp:112-117 on the 8^3 lattice, depth 4 vs 16 parts."""
    pos = np.array([[(x + 0.5), (y + 0.5), (z + 0.5)] for x in range(8) for y in range(8) for z in range(8)])
    cell, pbc = np.eye(3) * 8.0, np.ones(3, np.uint8)
    g = O.build_graph(pos, cell, pbc, 1.01)
    off, src = csr(g, 512)
    low = O.lownn(pos, cell, pbc, np.diff(off).astype(np.int32), 4, 1.01)
    cut = esg.mincut_partition((off, src), 16, 1)
    ml = O.compute_metrics(512, g["src"], g["dst"], low, 16)[1][2]
    mc = O.compute_metrics(512, g["src"], g["dst"], cut, 16)[1][2]
    assert ml <= mc + 1e-12
