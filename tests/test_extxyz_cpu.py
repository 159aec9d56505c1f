"""Extended-xyz input side (extxyz.h:11-20): the
product's reader / writer (csrc/extxyz_io.cpp, C ABI esg_extxyz_*) against
the reference's own read_extxyz_file / write_extxyz_file (oracle/_ref), and
its error behaviour (ParseError → ESG_ERR_DATA with the line number)."""
import os

import numpy as np
import pytest

import ref as R
from paper_2507_03840_b200 import esg

SKEW = np.array([[6.0, 0.4, 0.0], [0.9, 5.5, 0.3], [0.2, 0.6, 6.5]])
needs_ref = pytest.mark.skipif(not R.available(), reason="oracle/_ref not built (no /root/reference)")


def same(s, pos, sp, cell, pbc):
    assert np.array_equal(s.positions.view(np.uint64), np.asarray(pos).view(np.uint64))
    assert np.array_equal(s.species, sp)
    assert np.array_equal(s.cell.view(np.uint64), np.asarray(cell).view(np.uint64))
    assert np.array_equal(s.pbc, np.asarray(pbc).astype(bool))


def test_round_trip_exact(tmp_path):
    s = esg.tile(esg.make_jittered_lattice(300, 2.2, 0.45, [72, 8, 8], 3), [2, 1, 2])
    s.positions[0] = [-0.0, 1e-300, -123456.789]  # signed zero, subnormal-adjacent, large
    p = str(tmp_path / "s.xyz")
    esg.write_extxyz(p, s)
    t = esg.read_extxyz(p)
    same(t, s.positions, s.species, s.cell, s.pbc)


@needs_ref
def test_writer_text_equals_reference(tmp_path):
    s = esg.make_jittered_lattice(120, 2.2, 0.45, [72, 8, 8], 4)
    s.pbc[:] = [True, False, True]
    a, b = str(tmp_path / "ours.xyz"), str(tmp_path / "ref.xyz")
    esg.write_extxyz(a, s)
    R.write_extxyz(b, s.positions, s.species, s.cell, s._pbc8())
    assert open(a, "rb").read() == open(b, "rb").read()
    # a molecule (no periodic direction): empty comment line
    m = esg.AtomicStructure(s.positions[:5].copy(), s.species[:5].copy(), np.zeros((3, 3)), np.zeros(3, bool))
    esg.write_extxyz(a, m)
    R.write_extxyz(b, m.positions, m.species, m.cell, m._pbc8())
    assert open(a, "rb").read() == open(b, "rb").read()


HANDWRITTEN = [
    '3\nLattice="6.0 0.4 0 0.9 5.5 0.3 0.2 0.6 6.5" Properties=species:S:1:pos:R:3 pbc="F T F"\n'
    'Hf 0.1 0.2 0.3 extra columns 7\nO\t1.5e0 +2.25 -3\nO 4 5 6\n',
    '2\nLattice=" 1 0 0  0 2 0  0 0 3 " name=x  energy=-1.5\nSi 0 0 0\nSi 0.5 1 1.5\n',
    '2\n\nH 0 0 0\nH 0 0 0.74\n',
    '1\npbc="T T T" Lattice="2 0 0 0 2 0 0 0 2"\nC 1 1 1\n',
    '2 atoms here\nLattice="4 0 0 0 4 0 0 0 4" pbc="True false 1"\r\nO 1 2 3\r\nH 1 2 3.5\r\n',
]
BAD = {
    "empty": "",
    "count": "x\n\n",
    "negative": "-1\n\n",
    "no comment": "2\n",
    "lattice short": '1\nLattice="1 0 0 0 1 0 0 0"\nH 0 0 0\n',
    "pbc flag": '1\nLattice="1 0 0 0 1 0 0 0 1" pbc="T X T"\nH 0 0 0\n',
    "pbc short": '1\nLattice="1 0 0 0 1 0 0 0 1" pbc="T T"\nH 0 0 0\n',
    "pbc without lattice": '1\npbc="T F F"\nH 0 0 0\n',
    "quote": '1\nLattice="1 0 0 0 1 0 0 0 1\nH 0 0 0\n',
    "too few atoms": "3\n\nH 0 0 0\nH 1 1 1\n",
    "short atom line": "1\n\nH 0 0\n",
    "number": "1\n\nH 0 0 zero\n",
}


@needs_ref
@pytest.mark.parametrize("k", range(len(HANDWRITTEN)))
def test_reader_equals_reference(tmp_path, k):
    p = str(tmp_path / "h.xyz")
    with open(p, "w", newline="") as f:
        f.write(HANDWRITTEN[k])
    same(esg.read_extxyz(p), *R.read_extxyz(p))


@pytest.mark.parametrize("name", sorted(BAD))
def test_reader_errors(tmp_path, name):
    p = str(tmp_path / "bad.xyz")
    with open(p, "w") as f:
        f.write(BAD[name])
    with pytest.raises(esg.DataError) as e:
        esg.read_extxyz(p)
    assert "line" in str(e.value)
    if R.available():  # the reference rejects the same files
        with pytest.raises(RuntimeError):
            R.read_extxyz(p)


def test_missing_file(tmp_path):
    with pytest.raises(esg.DataError):
        esg.read_extxyz(str(tmp_path / "none.xyz"))


@needs_ref
def test_c4_file_reads_like_reference(tmp_path):
    """The bench workload as a file: 192k atoms, reader equal to the reference's."""
    s, _, _, _ = esg.config_structure("C4")
    p = str(tmp_path / "c4.xyz")
    esg.write_extxyz(p, s)
    same(esg.read_extxyz(p), *R.read_extxyz(p))
    assert os.path.getsize(p) > 192000 * 40
