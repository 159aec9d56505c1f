"""Block export host side: the shard format, the
rank-0 merge and the text writer, checked against the oracle's restatement
of write_blocks (block_matrix.cpp:90-101, std::ostream precision 17) over
gather_blocks' merged map (model_run.cpp:103-120).  No device needed."""
import numpy as np
import pytest

import oracle as O
from paper_2507_03840_b200 import esg

SHAPES = [(10, 10), (10, 4), (4, 10), (4, 4), (1, 1), (14, 9)]
TRICKY = np.array([1 / 3, -0.0, 0.0, 5e-324, 2.2250738585072014e-308, 1e300, -2.0, 0.1, 123456789.0,
                   -1.0000000000000002, 6.02214076e23, np.pi])


def write_shard(path, keys, shapes, values, basis=1, vb=8, flags=0, rank=0, world=1):
    """The documented shard layout (csrc/blocks_io.h)."""
    nb, nv = len(keys), len(values)
    h = np.zeros(1, esg.SHARD_HEADER)
    h["magic"], h["version"], h["basis"], h["value_bytes"], h["flags"] = b"ESGBLKS1", 1, basis, vb, flags
    h["rank"], h["world"], h["n_blocks"], h["n_values"] = rank, world, nb, nv
    h["keys_offset"] = 64
    h["values_offset"] = (64 + 24 * nb + 63) // 64 * 64
    rec = np.zeros(nb, esg.BLOCK_KEY)
    for f, col in zip(("i", "j", "ix", "iy", "iz"), np.asarray(keys).T):
        rec[f] = col
    rec["rows"], rec["cols"] = np.asarray(shapes).T
    with open(path, "wb") as fh:
        fh.write(h.tobytes())
        fh.write(rec.tobytes())
        fh.write(b"\0" * (int(h["values_offset"][0]) - 64 - 24 * nb))
        fh.write(np.asarray(values, np.float64 if vb == 8 else np.float32).tobytes())


def random_set(rng, n, n_atoms=30):
    keys = np.stack([rng.integers(0, n_atoms, n), rng.integers(0, n_atoms, n), rng.integers(-2, 3, n),
                     rng.integers(-2, 3, n), rng.integers(-2, 3, n)], axis=1).astype(np.int32)
    shapes = np.array([SHAPES[k] for k in rng.integers(0, len(SHAPES), n)], np.int32)
    nv = int((shapes[:, 0] * shapes[:, 1]).sum())
    vals = rng.standard_normal(nv) * 10.0 ** rng.integers(-8, 9, nv)
    vals[rng.integers(0, nv, len(TRICKY))] = TRICKY
    return keys, shapes, vals


def test_coupling_tables_bit_equal_oracle():
    """The product's CG tables (host.cpp) equal the oracle's
    clebsch_gordan.cpp restatement bit for bit, so the uncoupled export can be
    bit-exact."""
    for la in range(5):
        for lb in range(5):
            for L in range(abs(la - lb), la + lb + 1):
                a = esg.coupling_matrix(la, lb, L)
                assert np.array_equal(a.ravel().view(np.uint64), O.coupling(la, lb, L).ravel().view(np.uint64))


def test_merge_matches_reference_writer(tmp_path):
    """Three 'rank' shards with overlapping keys (the last rank wins) and
    tricky doubles: the merged text is byte-identical to the reference writer."""
    rng = np.random.default_rng(3)
    sets = [random_set(rng, n) for n in (40, 1, 25)]
    k0, s0, _ = sets[0]
    k2, s2, v2 = sets[2]  # rank 2 repeats five of rank 0's keys with new values
    n5 = int((s0[:5, 0] * s0[:5, 1]).sum())
    sets[2] = (np.concatenate([k2[:3], k0[:5], k2[3:]]), np.concatenate([s2[:3], s0[:5], s2[3:]]),
               np.concatenate([v2[:int((s2[:3, 0] * s2[:3, 1]).sum())], rng.standard_normal(n5),
                               v2[int((s2[:3, 0] * s2[:3, 1]).sum()):]]))
    paths = []
    for r, (k, s, v) in enumerate(sets):
        paths.append(str(tmp_path / f"r{r}.blk"))
        write_shard(paths[-1], k, s, v, rank=r, world=3)
    esg.merge_block_shards_to_text(paths, str(tmp_path / "got.txt"))
    O.write_blocks(np.concatenate([x[0] for x in sets]), np.concatenate([x[1] for x in sets]),
                   np.concatenate([x[2] for x in sets]), tmp_path / "want.txt")
    got, want = (tmp_path / "got.txt").read_bytes(), (tmp_path / "want.txt").read_bytes()
    assert got == want
    assert got.count(b"\n") < sum(len(x[0]) for x in sets)  # duplicates collapsed


def test_text_round_trips_values(tmp_path):
    """test_blocks.cpp:149-160: write then read gives the same blocks (17
    significant digits round-trip every double)."""
    rng = np.random.default_rng(5)
    k, s, v = random_set(rng, 30)
    k[:, 0] = np.arange(30)  # distinct keys
    write_shard(tmp_path / "a.blk", k, s, v)
    esg.merge_block_shards_to_text([str(tmp_path / "a.blk")], str(tmp_path / "a.txt"))
    got = {}
    for line in (tmp_path / "a.txt").read_text().splitlines():
        f = line.split()
        key, r, c = tuple(int(x) for x in f[:5]), int(f[5]), int(f[6])
        got[key] = np.array([float(x) for x in f[7:]]).reshape(r, c)
    off = np.concatenate([[0], np.cumsum(s[:, 0] * s[:, 1])])
    for b in range(30):
        blk = got[tuple(int(x) for x in k[b])]
        assert np.array_equal(blk.ravel().view(np.uint64), v[off[b]:off[b + 1]].view(np.uint64))


def test_fp32_shard_and_reader(tmp_path):
    rng = np.random.default_rng(9)
    k, s, v = random_set(rng, 12)
    with np.errstate(over="ignore"):  # 1e300 -> inf is part of the set
        v32 = v.astype(np.float32)
    p = tmp_path / "f.blk"
    write_shard(p, k, s, v32, vb=4, rank=1, world=2)
    hd, keys, shapes, off, vals = esg.read_block_shard(str(p))
    assert hd["value_bytes"] == 4 and hd["rank"] == 1 and hd["world"] == 2 and hd["basis"] == 1
    assert np.array_equal(keys, k) and np.array_equal(shapes, s) and np.array_equal(vals, v32)
    assert off[-1] == len(v)
    esg.merge_block_shards_to_text([str(p)], str(tmp_path / "got.txt"))
    O.write_blocks(k, s, v32.astype(np.float64), tmp_path / "want.txt")
    assert (tmp_path / "got.txt").read_bytes() == (tmp_path / "want.txt").read_bytes()


def test_merge_rejects_bad_shards(tmp_path):
    rng = np.random.default_rng(1)
    k, s, v = random_set(rng, 4)
    good = tmp_path / "good.blk"
    write_shard(good, k, s, v)
    out = str(tmp_path / "o.txt")
    bad = tmp_path / "bad.blk"
    bad.write_bytes(b"XXXXXXXX" + good.read_bytes()[8:])
    trunc = tmp_path / "trunc.blk"
    trunc.write_bytes(good.read_bytes()[:-8])
    coupled = tmp_path / "coupled.blk"
    write_shard(coupled, k, s, v, basis=0)
    for paths in ([str(bad)], [str(trunc)], [str(good), str(coupled)], [str(tmp_path / "missing.blk")]):
        with pytest.raises(esg.DataError):
            esg.merge_block_shards_to_text(paths, out)
    esg.merge_block_shards_to_text([], out)  # no shards: empty file
    assert (tmp_path / "o.txt").read_bytes() == b""


def test_read_blocks_round_trip_and_errors(tmp_path):
    """test_blocks.cpp:147-163: write_blocks then read_blocks gives the same
    blocks (in BlockKey order); malformed lines, short value lists and
    duplicate keys are data errors."""
    rng = np.random.default_rng(11)
    k, s, v = random_set(rng, 40)
    k[:, 0] = np.arange(40)  # distinct keys
    write_shard(tmp_path / "a.blk", k, s, v)
    esg.merge_block_shards_to_text([str(tmp_path / "a.blk")], str(tmp_path / "a.txt"))
    keys, shapes, off, vals = esg.read_blocks_text(str(tmp_path / "a.txt"))
    order = np.lexsort(k.T[::-1])  # BlockKey order
    src_off = np.concatenate([[0], np.cumsum(s[:, 0] * s[:, 1])])
    assert np.array_equal(keys, k[order]) and np.array_equal(shapes, s[order])
    want = np.concatenate([v[src_off[b]:src_off[b + 1]] for b in order])
    assert np.array_equal(vals.view(np.uint64), want.view(np.uint64))
    (tmp_path / "c.txt").write_text("# comment\n\n0 0 0 0 0 1 1 2.5\n")
    assert esg.read_blocks_text(str(tmp_path / "c.txt"))[3].tolist() == [2.5]
    for bad in ("0 0 0 0 0 1\n", "0 0 0 0 0 2 2 1 2 3\n", "0 0 0 0 0 0 1\n", "0 0 0 0 0 1 1 nan\n",
                "0 0 0 0 0 1 1 1\n0 0 0 0 0 1 1 2\n"):
        (tmp_path / "b.txt").write_text(bad)
        with pytest.raises(esg.DataError):
            esg.read_blocks_text(str(tmp_path / "b.txt"))
