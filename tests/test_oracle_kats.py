"""Pins the CPU oracle (oracle/oracle.cpp) against the reference's own
known-answer tests: test_structures.cpp, test_partition.cpp,
test_harmonics.cpp, test_model.cpp, acceptance.cpp.  CPU only."""
import math

import numpy as np
import pytest

import oracle as O

SKEW = np.array([[6.0, 0.4, 0.0], [0.9, 5.5, 0.3], [0.2, 0.6, 6.5]])


def random_structure(n, seed, pbc):
    """test_structures.cpp:23-35: fractional uniform points in a skewed cell."""
    rng = np.random.default_rng(seed)
    f = rng.random((n, 3))
    pos = f @ SKEW  # cartesian = cellᵀ f
    return pos, SKEW.copy(), np.array(pbc, np.uint8), (1 + np.arange(n) % 3).astype(np.int32)


def brute_force(pos, cell, pbc, r_cut, lim=3):
    """test_structures.cpp:38-61 brute-force neighbour list."""
    out = []
    n = len(pos)
    for i in range(n):
        for j in range(n):
            for sx in range(-lim, lim + 1):
                for sy in range(-lim, lim + 1):
                    for sz in range(-lim, lim + 1):
                        if (not pbc[0] and sx) or (not pbc[1] and sy) or (not pbc[2] and sz):
                            continue
                        if i == j and sx == 0 and sy == 0 and sz == 0:
                            continue
                        sv = sx * cell[0] + sy * cell[1] + sz * cell[2]
                        d = pos[j] + sv - pos[i]
                        nd = math.sqrt(d @ d)
                        if nd <= r_cut:
                            out.append((j, i, (sx, sy, sz), d, nd))
    out.sort(key=lambda t: (t[0], t[1], t[2]))
    return out


@pytest.mark.parametrize("pbc", [(1, 1, 1), (0, 0, 0), (1, 0, 1)])
@pytest.mark.parametrize("seed", [1, 2, 3])
def test_neighbor_list_matches_brute_force(pbc, seed):
    pos, cell, pbc, _ = random_structure(8, seed, pbc)
    g = O.build_graph(pos, cell, pbc, 4.0)
    ref = brute_force(pos, cell, pbc, 4.0)
    assert len(g["src"]) == len(ref)
    for k, (dst, src, sh, d, nd) in enumerate(ref):
        assert g["src"][k] == src and g["dst"][k] == dst and tuple(g["shift"][k]) == sh
        assert np.abs(g["disp"][k] - d).max() < 1e-12
        assert abs(g["dist"][k] - nd) < 1e-12


def test_every_edge_has_its_mirror():
    pos, cell, pbc, _ = random_structure(10, 7, (1, 1, 1))
    g = O.build_graph(pos, cell, pbc, 4.5)
    keys = {(s, d, tuple(sh)) for s, d, sh in zip(g["src"], g["dst"], g["shift"])}
    for s, d, sh in zip(g["src"], g["dst"], g["shift"]):
        assert (d, s, tuple(-np.asarray(sh))) in keys


def test_edges_sorted_with_contiguous_ranges():
    pos, cell, pbc, _ = random_structure(9, 11, (1, 1, 1))
    g = O.build_graph(pos, cell, pbc, 4.0)
    keys = list(zip(g["dst"], g["src"], map(tuple, g["shift"])))
    assert all(keys[k - 1] < keys[k] for k in range(1, len(keys)))
    deg = O.in_degrees(9, g)
    assert deg.sum() == len(keys)


def test_cutoff_is_inclusive():
    pos = np.array([[0.0, 0, 0], [3.0, 0, 0]])
    cell = np.eye(3)
    pbc = np.zeros(3, np.uint8)
    assert len(O.build_graph(pos, cell, pbc, 3.0)["src"]) == 2
    assert len(O.build_graph(pos, cell, pbc, 2.9999999)["src"]) == 0


def test_single_atom_sees_its_periodic_images():
    g = O.build_graph(np.array([[1.0, 1, 1]]), np.eye(3) * 2.0, np.ones(3, np.uint8), 2.5)
    assert len(g["src"]) == 6
    assert np.all(g["src"] == 0) and np.all(g["dst"] == 0)
    assert np.allclose(g["dist"], 2.0)


def test_wrap_maps_into_unit_cell():
    pos, cell, _, _ = random_structure(6, 5, (1, 1, 0))
    pbc = np.array([1, 1, 0], np.uint8)
    shifted = pos + np.array([3.0, -2.0, 0.0]) @ cell
    w = O.wrap(shifted, cell, pbc)
    f = w @ np.linalg.inv(cell)
    f0 = shifted @ np.linalg.inv(cell)
    assert np.all(f[:, :2] >= 0) and np.all(f[:, :2] < 1)
    assert np.allclose(f[:, 2], f0[:, 2], rtol=1e-12, atol=1e-12)
    assert np.all(np.abs(np.remainder(f[:, :2] - f0[:, :2] + 0.5, 1.0) - 0.5) < 1e-9)


def test_tiling_replicates_atoms_and_edges():
    pos, cell, pbc, sp = random_structure(5, 13, (1, 1, 1))
    tp, tc, ts = O.tile(pos, cell, pbc, sp, [2, 2, 2])
    assert tp.shape[0] == 40 and np.allclose(tc, 2 * cell)
    gs = O.build_graph(pos, cell, pbc, 4.0)
    gt = O.build_graph(tp, tc, pbc, 4.0)
    assert len(gt["src"]) == 8 * len(gs["src"])
    ds, dt = O.in_degrees(5, gs), O.in_degrees(40, gt)
    assert np.all(dt == ds[np.arange(40) % 5])


def test_face_spacing():
    c = np.eye(3) * 5.0
    assert all(abs(O.face_spacing(c, d) - 5.0) < 1e-12 for d in range(3))
    c[0] = [4.0, 3.0, 0.0]
    assert abs(O.face_spacing(c, 0) - 4.0) < 1e-12


# ----------------------------------------------------------- partition
def ring(n, spacing):
    cell = np.eye(3) * 100.0
    cell[0, 0] = n * spacing
    pos = np.array([[(i + 0.5) * spacing, 50.0, 50.0] for i in range(n)])
    return pos, cell, np.array([1, 0, 0], np.uint8)


def cubic_lattice(n, a):
    pos = np.array([[(x + 0.5) * a, (y + 0.5) * a, (z + 0.5) * a] for x in range(n) for y in range(n)
                    for z in range(n)])
    return pos, np.eye(3) * n * a, np.ones(3, np.uint8)


def neighbors(g, part, n_parts):
    nb = [set() for _ in range(n_parts)]
    for s, d in zip(g["src"], g["dst"]):
        if part[s] != part[d]:
            nb[part[d]].add(part[s])
    return [len(x) for x in nb]


def test_ring_splits_into_quarters():
    pos, cell, pbc = ring(8, 1.0)
    g = O.build_graph(pos, cell, pbc, 1.2)
    deg = O.in_degrees(8, g)
    assert np.all(deg == 2)
    assert list(O.lownn(pos, cell, pbc, deg, 2, 1.2)) == [0, 0, 1, 1, 2, 2, 3, 3]
    assert np.all(O.lownn(pos, cell, pbc, deg, 0, 1.2) == 0)


def test_one_periodic_cut_gives_one_neighbor():
    pos, cell, pbc = cubic_lattice(8, 1.0)
    g = O.build_graph(pos, cell, pbc, 1.01)
    p = O.lownn(pos, cell, pbc, O.in_degrees(512, g), 1, 1.01)
    assert neighbors(g, p, 2) == [1, 1]
    assert np.bincount(p).tolist() == [256, 256]


def test_lattice_depth3_balanced_few_neighbors():
    pos, cell, pbc = cubic_lattice(8, 1.0)
    g = O.build_graph(pos, cell, pbc, 1.01)
    deg = O.in_degrees(512, g)
    p = O.lownn(pos, cell, pbc, deg, 3, 1.01)
    assert np.bincount(p).tolist() == [64] * 8
    assert max(neighbors(g, p, 8)) <= 3
    assert np.array_equal(p, O.lownn(pos, cell, pbc, deg, 3, 1.01))


def test_comm_plan_interlocks():
    """test_runtime.cpp:185-233: my send rows to q are q's halo block from me."""
    pos, cell, sp = O.jittered_lattice(64, 1.6, 0.3, [1, 8], 5)
    pbc = np.ones(3, np.uint8)
    g = O.build_graph(pos, cell, pbc, 2.5)
    part = O.lownn(pos, cell, pbc, O.in_degrees(64, g), 2, 2.5)
    plans = [O.comm_plan(64, g["src"], g["dst"], part, 4, r) for r in range(4)]
    for r, pl in enumerate(plans):
        at = 0
        for q, peer in enumerate(pl["nbr_peer"]):
            cnt = pl["nbr_send_count"][q]
            mine = pl["row_global"][pl["send_rows"][at:at + cnt]]
            at += cnt
            other = plans[peer]
            k = list(other["nbr_peer"]).index(r)
            rr, rc = other["nbr_recv_row"][k], other["nbr_recv_count"][k]
            assert np.array_equal(other["row_global"][rr:rr + rc], mine)
        # owned edges: exactly those with an owned destination, global order
        owned = np.where(part[g["dst"]] == r)[0]
        assert np.array_equal(pl["edge_index"], owned)


# ----------------------------------------------------------- harmonics
def random_rotation(rng):
    q, r = np.linalg.qr(rng.normal(size=(3, 3)))
    q = q * np.sign(np.diag(r))
    if np.linalg.det(q) < 0:
        q[:, 0] = -q[:, 0]
    return q


def rot_y(a):
    c, s = math.cos(a), math.sin(a)
    return np.array([[c, 0, s], [0, 1, 0], [-s, 0, c]])


def test_to_m_layout_kat():
    to_m, to_l, mo = O.m_layout(2)
    assert list(to_m) == [0, 3, 1, 5, 7, 4, 2, 6, 8]
    assert all(to_l[to_m[r]] == r for r in range(9))
    assert mo[1] == 3 and mo[2] == 7


def test_degree_one_block_is_rotation():
    R = random_rotation(np.random.default_rng(303))
    D = O.wigner(R, 2)
    assert D[0][0, 0] == 1.0 and np.abs(D[1] - R).max() < 1e-14


def test_wigner_homomorphism_and_orthogonality():
    rng = np.random.default_rng(404)
    for _ in range(10):
        r1, r2 = random_rotation(rng), random_rotation(rng)
        d1, d2, d12 = O.wigner(r1, 6), O.wigner(r2, 6), O.wigner(r1 @ r2, 6)
        for l in range(7):
            assert np.abs(d12[l] - d1[l] @ d2[l]).max() < 1e-11
            assert np.abs(d1[l] @ d1[l].T - np.eye(2 * l + 1)).max() < 1e-12


def test_rotation_about_y_is_block_diagonal():
    g = 0.7312
    D = O.wigner(rot_y(g), 4)
    for l in range(5):
        d = D[l]
        for m in range(-l, l + 1):
            for n in range(-l, l + 1):
                if abs(m) != abs(n):
                    assert abs(d[m + l, n + l]) < 1e-13
        for m in range(1, l + 1):
            c, s = math.cos(m * g), math.sin(m * g)
            assert abs(d[l + m, l + m] - c) < 1e-12 and abs(d[l - m, l - m] - c) < 1e-12
            assert abs(d[l - m, l + m] - s) < 1e-12 and abs(d[l + m, l - m] + s) < 1e-12


def test_alignment_collapses_harmonics_to_pole():
    rng = np.random.default_rng(606)
    for _ in range(40):
        u = rng.normal(size=3)
        u /= np.linalg.norm(u)
        R, D = O.align_wigner(u, 4)
        assert np.linalg.norm(R @ u - np.array([0, 1, 0])) < 1e-12
        y = O.real_sh(u, 4)
        for l in range(5):
            aligned = D[l] @ y[l * l:(l + 1) ** 2]
            want = np.zeros(2 * l + 1)
            want[l] = math.sqrt((2 * l + 1) / (4 * math.pi))
            assert np.abs(aligned - want).max() < 1e-11
    R, _ = O.align_wigner(np.array([0.0, -1.0, 0.0]), 1)
    assert np.linalg.norm(R @ np.array([0, -1.0, 0]) - np.array([0, 1.0, 0])) < 1e-14


def test_coupling_orthonormal_and_intertwining():
    rng = np.random.default_rng(707)
    Q = random_rotation(rng)
    D = O.wigner(Q, 6)
    for la in range(4):
        for lb in range(4):
            stack = np.vstack([O.coupling(la, lb, L) for L in range(abs(la - lb), la + lb + 1)])
            assert np.abs(stack @ stack.T - np.eye(stack.shape[0])).max() < 1e-12
            kr = np.kron(D[la], D[lb])
            for L in range(abs(la - lb), la + lb + 1):
                C = O.coupling(la, lb, L)
                assert np.abs(C @ kr - D[L] @ C).max() < 1e-10


def _racah_cg(j1, m1, j2, m2, J, M):
    """<j1 m1; j2 m2 | J M> by Racah's closed form (Condon-Shortley)."""
    from math import factorial as f, sqrt
    if m1 + m2 != M or abs(m1) > j1 or abs(m2) > j2 or abs(M) > J:
        return 0.0
    pre = sqrt((2 * J + 1) * f(J + j1 - j2) * f(J - j1 + j2) * f(j1 + j2 - J) / f(j1 + j2 + J + 1))
    pre *= sqrt(f(J + M) * f(J - M) * f(j1 - m1) * f(j1 + m1) * f(j2 - m2) * f(j2 + m2))
    s = 0.0
    for k in range(j1 + j2 - J + 1):
        d = (j1 + j2 - J - k, j1 - m1 - k, j2 + m2 - k, J - j2 + m1 + k, J - j1 - m2 + k)
        if min(d) < 0:
            continue
        s += (-1) ** k / (f(k) * f(d[0]) * f(d[1]) * f(d[2]) * f(d[3]) * f(d[4]))
    return pre * s


def _real_basis(l):
    d = 2 * l + 1
    b = np.zeros((d, d), complex)
    b[l, l] = 1.0
    s = np.sqrt(0.5)
    for m in range(1, l + 1):
        ph = -1.0 if m % 2 else 1.0
        b[l + m, l - m], b[l + m, l + m] = s, ph * s
        b[l - m, l - m], b[l - m, l + m] = 1j * s, -1j * ph * s
    return b


def test_coupling_matches_racah_closed_form():
    """An independent construction of clebsch_gordan.cpp's tables: Racah's
    closed form in the complex basis, the same real-basis change and phase
    convention, against the oracle's lowering-operator construction (which the
    product's tables equal bit for bit, tests/test_blocks_cpu.py)."""
    for la in range(5):
        for lb in range(5):
            ba, bb = _real_basis(la), _real_basis(lb)
            kron = np.kron(ba, bb)
            for L in range(abs(la - lb), la + lb + 1):
                cg = np.array([[_racah_cg(la, ma, lb, mb, L, M) for ma in range(-la, la + 1) for mb in range(-lb, lb + 1)]
                               for M in range(-L, L + 1)])
                u = _real_basis(L) @ cg @ kron.conj().T
                want = u.imag if (la + lb - L) % 2 else u.real
                assert np.abs(want - O.coupling(la, lb, L)).max() < 1e-12, (la, lb, L)


# --------------------------------------------------------------- model
SP_BASIS = {1: [0, 1], 8: [0, 1]}


def small_model(l_max=2, e=4, layers=2, gate=True):
    return O.Model(l_max, e, layers, 8, 2.5, 1, SP_BASIS, gate)


def small_graph(n=6, seed=21):
    pos, cell, sp = O.jittered_lattice(n, 2.2, 0.25, [1, 8], seed)
    pbc = np.ones(3, np.uint8)
    return pos, cell, pbc, sp


def head_keys(slot_l):
    keys, off = [], 0
    for la in slot_l:
        for lb in slot_l:
            for L in range(la + lb + 1):
                keys.append((L, off))
                off += 2 * L + 1
    return keys


@pytest.mark.parametrize("l_max", [2, 4])
@pytest.mark.parametrize("dtype,limit", [(np.float64, 1e-10), (np.float32, 1e-4)])
def test_forward_equivariance(l_max, dtype, limit):
    """acceptance.cpp:100-169: coupled L-segments rotate with D_L (relative)."""
    pos, cell, sp = O.jittered_lattice(20, 2.2, 0.45, [1, 8], 5)
    pbc = np.ones(3, np.uint8)
    m = O.Model(l_max, 8, 2, 8, 4.0, 5, SP_BASIS)
    g = O.build_graph(pos, cell, pbc, 4.0)
    no, eo = m.forward(O.serial_view(20, sp, g), dtype)
    scale = max(np.abs(no).max(), np.abs(eo).max())
    keys = head_keys([0, 1])
    rng = np.random.default_rng(11)
    worst = 0.0
    for _ in range(4):
        Q = random_rotation(rng)
        g2 = O.build_graph(pos @ Q.T, cell @ Q.T, pbc, 4.0)
        assert len(g2["src"]) == len(g["src"])
        no2, eo2 = m.forward(O.serial_view(20, sp, g2), dtype)
        D = O.wigner(Q, 2)
        for ref, rot in ((no, no2), (eo, eo2)):
            for L, off in keys:
                want = ref[:, off:off + 2 * L + 1].astype(np.float64) @ D[L].T
                worst = max(worst, np.abs(rot[:, off:off + 2 * L + 1] - want).max())
    assert worst / scale < limit


def test_zero_layer_heads_are_scalar_only():
    """test_model.cpp:408-435: with no message passing, L > 0 heads are 0."""
    pos, cell, pbc, sp = small_graph()
    m = small_model(layers=0)
    g = O.build_graph(pos, cell, pbc, 2.5)
    no, eo = m.forward(O.serial_view(len(pos), sp, g), np.float64)
    # head layout for slots (0: l=0, 1: l=1): keys (0,0,0) (0,1,0..1) (1,0,0..1) (1,1,0..2)
    l_of = []
    for sa, la in enumerate([0, 1]):
        for sb, lb in enumerate([0, 1]):
            for L in range(la + lb + 1):
                l_of += [L] * (2 * L + 1)
    l_of = np.array(l_of)
    assert np.all(no[:, l_of > 0] == 0) and np.all(eo[:, l_of > 0] == 0)
    assert np.any(no[:, l_of == 0] != 0)


def test_param_init_is_deterministic_and_named():
    m1, m2 = small_model(), small_model()
    assert np.array_equal(m1.params_f32(), m2.params_f32())
    names = [e[0] for e in m1.entries()]
    assert names[:3] == ["embed/H", "embed/O", "radial/lift"]
    assert "layer0/node/lin1/m0" in names and "layer1/edge/lin2/m2i" in names
    assert names[-1].startswith("head/edge/")


def test_single_vs_double_precision_agree():
    pos, cell, pbc, sp = small_graph()
    m = small_model()
    g = O.build_graph(pos, cell, pbc, 2.5)
    v = O.serial_view(len(pos), sp, g)
    a, b = m.forward(v, np.float32), m.forward(v, np.float64)
    scale = np.abs(b[1]).max()
    assert np.abs(a[1] - b[1]).max() < 1e-5 * max(scale, 1.0)
