"""Partition metrics, CPU side: the oracle's compute_metrics
pinned by the reference's own KATs (test_partition.cpp:61-120, 145-160,
198-224), and the product's host formatters (metrics JSON, DOT, assignment
files) against the restated reference writers."""
import numpy as np
import pytest

import oracle as O
from paper_2507_03840_b200 import esg


def ring(n, spacing):
    cell = np.eye(3) * 100.0
    cell[0, 0] = n * spacing
    pos = np.array([[(i + 0.5) * spacing, 50.0, 50.0] for i in range(n)])
    return pos, cell, np.array([1, 0, 0], np.uint8)


def cubic_lattice(n, a):
    pos = np.array([[(x + 0.5) * a, (y + 0.5) * a, (z + 0.5) * a] for x in range(n) for y in range(n)
                    for z in range(n)])
    return pos, np.eye(3) * n * a, np.ones(3, np.uint8)


def lownn_case(pos, cell, pbc, r, depth):
    g = O.build_graph(pos, cell, pbc, r)
    part = O.lownn(pos, cell, pbc, O.in_degrees(len(pos), g), depth, r)
    return g, part, 1 << depth


def volume(g, part, P):
    """write_dot's weights: distinct source nodes part f packs for part q."""
    v = np.zeros((P, P), np.int64)
    pairs = {(part[d], s) for s, d in zip(g["src"], g["dst"]) if part[s] != part[d]}
    for q, s in pairs:
        v[part[s], q] += 1
    return v


def test_oracle_metrics_kats():
    # depth zero keeps everything in one part (test_partition.cpp:61-72)
    g, part, P = lownn_case(*ring(6, 1.0), 1.2, 0)
    parts, d, i = O.compute_metrics(6, g["src"], g["dst"], part, P)
    assert parts[0, 2] == 0 and parts[0, 3] == 0 and d[0] == 1.0 and d[1] == 1.0
    # one periodic cut: a single neighbour each (:84-93)
    g, part, P = lownn_case(*cubic_lattice(8, 1.0), 1.01, 1)
    parts, d, i = O.compute_metrics(512, g["src"], g["dst"], part, P)
    assert parts[:, 2].tolist() == [1, 1] and d[0] == 1.0
    # depth 3 lattice: 64 nodes, <= 3 neighbours, edge imbalance ~1 (:95-110)
    g, part, P = lownn_case(*cubic_lattice(8, 1.0), 1.01, 3)
    parts, d, i = O.compute_metrics(512, g["src"], g["dst"], part, P)
    assert (parts[:, 0] == 64).all() and (parts[:, 2] <= 3).all() and d[0] == 1.0 and abs(d[1] - 1.0) <= 0.16
    # triangle, one part per node (:145-160)
    pos = np.array([[0.0, 0.0, 0.0], [1.0, 0.0, 0.0], [0.5, 0.9, 0.0]])
    g = O.build_graph(pos, np.eye(3) * 10.0, np.zeros(3, np.uint8), 2.0)
    assert len(g["src"]) == 6
    parts, d, i = O.compute_metrics(3, g["src"], g["dst"], np.arange(3, dtype=np.int32), 3)
    assert (parts == [1, 2, 2, 2]).all() and i[1] == 6 and i[2] == 6


def test_json_formatting_matches_nlohmann_rules():
    vals = [1.0, 1.0345, 2.5, 1 / 3, 1e-5, 1.5e-4, 0.001234, 1e15, 1e16, 123456.789, 7.0, 1.3333333333333333,
            12345678901234567.0, 0.1, 2.0 ** -30]
    for k in range(0, len(vals), 3):
        d = (vals[k], vals[(k + 1) % len(vals)], vals[(k + 2) % len(vals)])
        parts = np.array([[5, 7, 1, 3], [9, 11, 2, 4]], np.int64)
        i = np.array([2, 7, 13])
        got = esg.metrics_from_arrays(d, i, parts, np.zeros((2, 2))).json()
        assert got == O.metrics_json(parts, d, i), (got, O.metrics_json(parts, d, i))
    assert '"n_parts": 2' in got and '"parts"' in got and '"recv_volume"' in got  # test_partition.cpp:215-218


@pytest.mark.parametrize("depth", [1, 2, 3])
def test_dot_matches_reference_writer(tmp_path, depth):
    pos, cell, species = O.jittered_lattice(60, 2.2, 0.35, [1, 8], 3)
    g, part, P = lownn_case(pos, cell, np.ones(3, np.uint8), 3.5, depth)
    parts, d, i = O.compute_metrics(len(pos), g["src"], g["dst"], part, P)
    m = esg.metrics_from_arrays(d, i, parts, volume(g, part, P))
    O.write_dot(len(pos), g["src"], g["dst"], part, P, tmp_path / "ref.dot")
    assert m.dot() == (tmp_path / "ref.dot").read_text()
    assert m.dot().startswith("digraph parts {") and "p0 -> p1" in m.dot()  # test_partition.cpp:220-222


def test_assignment_files_round_trip(tmp_path):
    """test_partition.cpp:198-209."""
    p = tmp_path / "a.txt"
    esg.write_assignment(str(p), np.array([0, 2, 1, 1, 0]))
    assert p.read_text() == "0 0\n1 2\n2 1\n3 1\n4 0\n"
    back, n_parts = esg.read_assignment(str(p))
    assert n_parts == 3 and back.tolist() == [0, 2, 1, 1, 0]
    for bad in ("0 0\n2 1\n", "", "0 0\n1 -1\n", "0 0\nx\n"):
        p.write_text(bad)
        with pytest.raises(esg.DataError):
            esg.read_assignment(str(p))
    with pytest.raises(esg.DataError):
        esg.read_assignment(str(tmp_path / "missing.txt"))
