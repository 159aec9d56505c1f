"""GPU per-edge rotation blocks against the oracle.

esg_edge_rotations runs the same device code the message kernels use
in-register (align_to_y + the generated Ivanic-Ruedenberg recursion, fp32)
and is compared with the oracle's fp64 align_to_y + wigner_blocks
(align.cpp:32-39, wigner.cpp:47-83).  Edges close to the +-y axis are the
hard case: sin(beta) must come from the lateral length, not sqrt(1 - uy^2)
(ADVICE r01).  KAT: the aligned frame collapses the real SH of the edge
direction to m = 0 with value sqrt((2l+1)/4pi) (test_harmonics.cpp:204-228).

Bar: every block entry within 2e-6 absolute of the fp64 oracle (fp32
arithmetic on an fp32-rounded displacement; entries are bounded by 1).
"""
import numpy as np
import pytest

import oracle as O
from paper_2507_03840_b200 import esg

pytestmark = pytest.mark.gpu

TOL = 2e-6


def near_axis_displacements():
    rng = np.random.default_rng(7)
    out = []
    for sign in (1.0, -1.0):
        for length in (2.2, 5.0, 9.97):
            for lateral in (0.0, 1e-7, 1e-5, 1e-4, 1e-3, 1e-2, 0.1, 0.3):
                phi = rng.uniform(0, 2 * np.pi)
                x, z = lateral * np.cos(phi), lateral * np.sin(phi)
                y = sign * np.sqrt(max(length * length - lateral * lateral, 0.0))
                out.append((x, y, z))
    # lattice directions (C4's y-aligned neighbours) and exact axes
    for v in ((0, 2.2, 0), (0, -2.2, 0), (2.2, 0, 0), (0, 0, -2.2), (2.2, 2.2, 0), (0, 4.4, 1e-9)):
        out.append(v)
    return np.array(out, np.float64)


def oracle_blocks(disp, l_max):
    rows = []
    for d in disp:
        _, D = O.align_wigner(d, l_max)
        rows.append(np.concatenate([b.ravel() for b in D]))
    return np.array(rows)


@pytest.mark.parametrize("l_max", [2, 4, 6])
def test_rotations_random_directions(gpu_ctx, l_max):
    rng = np.random.default_rng(l_max)
    disp = rng.normal(size=(2000, 3)) * rng.uniform(0.5, 12.0, size=(2000, 1))
    got = esg.edge_rotations(gpu_ctx, disp, l_max)
    want = oracle_blocks(disp, l_max)
    assert np.abs(got - want).max() < TOL * (2 if l_max == 6 else 1)


@pytest.mark.parametrize("l_max", [4])
def test_rotations_near_y_axis(gpu_ctx, l_max):
    disp = near_axis_displacements()
    got = esg.edge_rotations(gpu_ctx, disp, l_max)
    want = oracle_blocks(disp, l_max)
    err = np.abs(got - want).max(axis=1)
    assert err.max() < TOL, (err.max(), disp[err.argmax()])


def test_alignment_collapses_sh_on_device(gpu_ctx):
    """test_harmonics.cpp:204-228 with the device blocks: D_l(R) Y_l(u) =
    sqrt((2l+1)/4pi) e_(m=0)."""
    disp = np.concatenate([near_axis_displacements(), np.random.default_rng(3).normal(size=(64, 3))])
    l_max = 4
    D = esg.edge_rotations(gpu_ctx, disp, l_max).astype(np.float64)
    for k, d in enumerate(disp):
        sh = O.real_sh(d / np.linalg.norm(d), l_max)
        o = 0
        for l in range(l_max + 1):
            n = 2 * l + 1
            y = D[k, o:o + n * n].reshape(n, n) @ sh[l * l:l * l + n]
            want = np.zeros(n)
            want[l] = np.sqrt((2 * l + 1) / (4 * np.pi))
            assert np.abs(y - want).max() < 5e-6, (k, l, y)
            o += n * n


def test_rotations_errors(gpu_ctx):
    with pytest.raises(esg.UsageError):
        esg.edge_rotations(gpu_ctx, np.zeros((1, 3)), 7)
    assert esg.edge_rotations(gpu_ctx, np.zeros((0, 3)), 4).shape == (0, 165)
