"""Low-NN partition on the device (lownn_gpu.cu) against the
oracle's lownn_partition restatement (lownn.cpp:23-133): the assignments must
be identical, including coordinate ties (broken by atom id), -0.0 / 0.0 ties,
non-periodic axes, zero in-degrees (unit weights) and the bench structure."""
import numpy as np
import pytest

import oracle as O
from paper_2507_03840_b200 import esg

pytestmark = pytest.mark.gpu


def structure(pos, cell, pbc):
    return esg.AtomicStructure(np.asarray(pos, np.float64), np.full(len(pos), 14, np.int32),
                               np.asarray(cell, np.float64), np.asarray(pbc, bool))


def check(ctx, s, deg, depth, r):
    pbc8 = np.asarray(s.pbc, np.uint8)
    want = O.lownn(s.positions, s.cell, pbc8, deg, depth, r)
    got = esg.lownn_partition_gpu(ctx, s, deg, depth, r)
    assert np.array_equal(got, want)
    assert np.array_equal(got, esg.lownn_partition(s, deg, depth, r))
    return got


@pytest.mark.parametrize("name", ["C1", "C2"])
@pytest.mark.parametrize("depth", [0, 1, 2, 3])
def test_lownn_gpu_configs(gpu_ctx, name, depth):
    s, r, _, _ = esg.config_structure(name)
    deg = esg.build_graph(gpu_ctx, s, r).in_degrees()
    part = check(gpu_ctx, s, deg, depth, r)
    assert np.array_equal(np.bincount(part, minlength=1 << depth) > 0, np.ones(1 << depth, bool))


@pytest.mark.parametrize("depth", [1, 2, 3, 4, 5])
def test_lownn_gpu_lattice_ties(gpu_ctx, depth):
    n, a = 8, 1.0
    pos = [[(x + 0.5) * a, (y + 0.5) * a, (z + 0.5) * a] for x in range(n) for y in range(n) for z in range(n)]
    rng = np.random.default_rng(depth)
    perm = rng.permutation(len(pos))  # ties broken by atom id, not input order of equal keys
    s = structure(np.asarray(pos)[perm], np.eye(3) * n * a, [1, 1, 1])
    check(gpu_ctx, s, np.full(len(pos), 6, np.int32), depth, 1.01)
    check(gpu_ctx, s, rng.integers(0, 9, len(pos)).astype(np.int32), depth, 1.01)


def test_lownn_gpu_zero_degrees_and_signed_zero(gpu_ctx):
    rng = np.random.default_rng(7)
    pos = rng.uniform(-3.0, 3.0, (500, 3))
    pos[::7, 0] = 0.0
    pos[3::7, 0] = -0.0
    pos[::5, 1] = pos[0, 1]
    s = structure(pos, np.eye(3) * 6.0, [0, 1, 0])
    for depth in (1, 2, 3, 4):
        check(gpu_ctx, s, np.zeros(500, np.int32), depth, 2.5)
        check(gpu_ctx, s, rng.integers(0, 40, 500).astype(np.int32), depth, 2.5)


def test_lownn_gpu_ring_and_open_box(gpu_ctx):
    n = 64
    pos = [[(i + 0.5) * 1.0, 50.0, 50.0] for i in range(n)]
    cell = np.eye(3) * 100.0
    cell[0, 0] = n
    s = structure(pos, cell, [1, 0, 0])
    for depth in (1, 2, 3, 6):
        check(gpu_ctx, s, np.full(n, 2, np.int32), depth, 1.2)
    sk = esg.make_jittered_lattice(3000, 2.20, 0.45, [72, 8, 8], 2)
    s2 = structure(sk.positions, sk.cell + np.array([[0.0, 0.0, 0.0], [1.5, 0.0, 0.0], [0.0, -2.0, 0.0]]), [0, 0, 1])
    for depth in (1, 2, 3):
        check(gpu_ctx, s2, np.arange(3000, dtype=np.int32) % 97, depth, 6.0)


def test_lownn_gpu_bench_structure(gpu_ctx):
    s, r, _, _ = esg.config_structure("C4")
    deg = esg.build_graph(gpu_ctx, s, r).in_degrees()
    for depth in (1, 2, 3):
        check(gpu_ctx, s, deg, depth, r)


def test_lownn_gpu_errors_map_to_usage(gpu_ctx):
    s = esg.make_jittered_lattice(4, 2.0, 0.1, [1], 1)
    with pytest.raises(esg.UsageError):
        esg.lownn_partition_gpu(gpu_ctx, s, np.ones(4, np.int32), 3, 2.5)  # 8 parts > 4 atoms
    with pytest.raises(esg.UsageError):
        esg.lownn_partition_gpu(gpu_ctx, s, np.ones(4, np.int32), 1, 0.0)
