"""Block export on the GPU against the oracle.

Bars (all bit-exact, given the GPU's own fp32 head rows as input):
  * keys: owned atoms (g, g, 0) then edges (src, dst, shift) in graph order
  * coupled values == fill_block (network.h:296-315)
  * uncoupled values == to_block per shell pair (block_matrix.cpp:66-88)
  * symmetrised on-site blocks == 0.5 (B + B^T), other blocks unchanged
  * shard file == in-memory export (fp64 and fp32), over a multi-chunk
    pipeline; text == the reference writer (block_matrix.cpp:90-101)
"""
import numpy as np
import pytest

import oracle as O
from paper_2507_03840_b200 import esg

pytestmark = pytest.mark.gpu
NORB = {72: 10, 8: 4}


@pytest.fixture(scope="module")
def run(gpu_ctx):
    s = esg.make_jittered_lattice(40, 2.2, 0.45, [72, 8, 8], 4)
    cfg = esg.ModelConfig(l_max=4, e_width=16, layers=2, n_radial=32, r_cut=4.5, seed=1)
    net = esg.Network(gpu_ctx, cfg, esg.BASIS_HFO2)
    net.init_params()
    g = esg.build_graph(gpu_ctx, s, 4.5)
    net.prepare(g, s.species)
    no, eo, _ = net.forward()
    om = O.Model(4, 16, 2, 32, 4.5, 1, esg.BASIS_HFO2)
    return net, s, g.export(), no, eo, om


def items(s, gx, no, eo):
    sp = s.species
    out = [(sp[i], sp[i], no[i]) for i in range(s.n_atoms)]
    out += [(sp[a], sp[b], eo[k]) for k, (a, b) in enumerate(zip(gx["src"], gx["dst"]))]
    return out


def bits(a):
    return np.ascontiguousarray(a, np.float64).view(np.uint64)


def test_keys_and_shapes(run):
    net, s, gx, no, eo, om = run
    keys, shapes, off, vals = net.blocks(esg.BLOCKS_UNCOUPLED)
    n = s.n_atoms
    assert len(keys) == n + len(gx["src"])
    assert np.array_equal(keys[:n, 0], np.arange(n)) and np.array_equal(keys[:n, 1], np.arange(n))
    assert not keys[:n, 2:].any()
    assert np.array_equal(keys[n:, 0], gx["src"]) and np.array_equal(keys[n:, 1], gx["dst"])
    assert np.array_equal(keys[n:, 2:], np.asarray(gx["shift"]).reshape(-1, 3))
    sa = np.concatenate([s.species, s.species[gx["src"]]])
    sb = np.concatenate([s.species, s.species[gx["dst"]]])
    assert np.array_equal(shapes[:, 0], [NORB[z] for z in sa]) and np.array_equal(shapes[:, 1], [NORB[z] for z in sb])
    assert off[-1] == len(vals) == net.blocks_count()[1]


@pytest.mark.parametrize("basis", [esg.BLOCKS_COUPLED, esg.BLOCKS_UNCOUPLED])
def test_values_bit_exact(run, basis):
    net, s, gx, no, eo, om = run
    keys, shapes, off, vals = net.blocks(basis)
    ref = om.coupled_block if basis == esg.BLOCKS_COUPLED else om.uncoupled_block
    for b, (za, zb, row) in enumerate(items(s, gx, no, eo)):
        want = ref(za, zb, row, NORB[za], NORB[zb]).ravel()
        assert np.array_equal(bits(vals[off[b]:off[b + 1]]), bits(want)), b
    if basis == esg.BLOCKS_UNCOUPLED:
        assert np.array_equal(vals, net.blocks_uncoupled())  # legacy entry point


def test_symmetrised_onsite(run):
    net, s, gx, no, eo, om = run
    keys, shapes, off, u = net.blocks(esg.BLOCKS_UNCOUPLED)
    _, _, _, sym = net.blocks(esg.BLOCKS_UNCOUPLED, symmetrize_onsite=True)
    for b in range(s.n_atoms):
        r, c = shapes[b]
        blk = u[off[b]:off[b + 1]].reshape(r, c)
        assert np.array_equal(bits(sym[off[b]:off[b + 1]]), bits((0.5 * (blk + blk.T)).ravel()))
    assert np.array_equal(bits(sym[off[s.n_atoms]:]), bits(u[off[s.n_atoms]:]))
    with pytest.raises(esg.UsageError):
        net.blocks(esg.BLOCKS_COUPLED, symmetrize_onsite=True)


@pytest.mark.parametrize("chunk", [None, "8192"])
def test_shard_matches_export(run, tmp_path, monkeypatch, chunk):
    net, s, gx, no, eo, om = run
    if chunk:
        monkeypatch.setenv("ESG_BLOCK_CHUNK_BYTES", chunk)  # many chunks through the pinned pipeline
    keys, shapes, off, vals = net.blocks(esg.BLOCKS_UNCOUPLED)
    for vb in (8, 4):
        p = tmp_path / f"r0_{vb}.blk"
        net.write_block_shard(str(p), esg.BLOCKS_UNCOUPLED, value_bytes=vb)
        hd, k2, s2, o2, v2 = esg.read_block_shard(str(p))
        assert (hd["basis"], hd["value_bytes"], hd["rank"], hd["world"]) == (1, vb, 0, 1)
        assert np.array_equal(k2, keys) and np.array_equal(s2, shapes) and np.array_equal(o2, off)
        want = vals if vb == 8 else vals.astype(np.float32)
        assert np.array_equal(np.asarray(v2).view(np.uint8), want.view(np.uint8))


def test_text_matches_reference_writer(run, tmp_path):
    net, s, gx, no, eo, om = run
    for basis, name in ((esg.BLOCKS_COUPLED, "coupled"), (esg.BLOCKS_UNCOUPLED, "uncoupled")):
        keys, shapes, off, vals = net.blocks(basis)
        net.write_blocks_text(str(tmp_path / f"{name}.txt"), basis)
        net.write_block_shard(str(tmp_path / f"{name}.blk"), basis)
        esg.merge_block_shards_to_text([str(tmp_path / f"{name}.blk")], str(tmp_path / f"{name}_merged.txt"))
        O.write_blocks(keys, shapes, vals, tmp_path / f"{name}_ref.txt")
        ref = (tmp_path / f"{name}_ref.txt").read_bytes()
        assert (tmp_path / f"{name}.txt").read_bytes() == ref
        assert (tmp_path / f"{name}_merged.txt").read_bytes() == ref


def test_device_export(run):
    import torch
    net, s, gx, no, eo, om = run
    keys, shapes, off, vals = net.blocks(esg.BLOCKS_UNCOUPLED)
    nb, nv = net.blocks_count()
    dk = torch.zeros(nb * 24, dtype=torch.uint8, device="cuda:0")
    dv = torch.zeros(nv, dtype=torch.float64, device="cuda:0")
    ms = net.blocks_to_device(dk.data_ptr(), dv.data_ptr(), esg.BLOCKS_UNCOUPLED)
    torch.cuda.synchronize()
    assert ms > 0
    k = dk.cpu().numpy().view(esg.BLOCK_KEY)
    assert np.array_equal(np.stack([k["i"], k["j"], k["ix"], k["iy"], k["iz"]], 1), keys)
    assert np.array_equal(bits(dv.cpu().numpy()), bits(vals))


def test_reference_output_stage(run, tmp_path):
    """model_run.cpp:141-153 for one rank (oracle restatement: coupled map,
    its text, blocks_to_uncoupled, its text) == the two text files written
    from the GPU export, byte for byte."""
    net, s, gx, no, eo, om = run
    keys, _, _, _ = net.blocks(esg.BLOCKS_COUPLED)
    om.export_text(keys, np.concatenate([no, eo]), s.species, tmp_path / "ref_c.txt", tmp_path / "ref_u.txt")
    net.write_blocks_text(str(tmp_path / "c.txt"), esg.BLOCKS_COUPLED)
    net.write_blocks_text(str(tmp_path / "u.txt"), esg.BLOCKS_UNCOUPLED)
    assert (tmp_path / "c.txt").read_bytes() == (tmp_path / "ref_c.txt").read_bytes()
    assert (tmp_path / "u.txt").read_bytes() == (tmp_path / "ref_u.txt").read_bytes()


def test_build_targets_inverts_blocks(run, tmp_path):
    """test_model.cpp:472-498: encoding the uncoupled blocks of a forward as
    targets gives back the head outputs (fp32 heads -> fp64 blocks -> fp32);
    every slot of an item's species pair is active; items without a block
    stay masked."""
    net, s, gx, no, eo, om = run
    keys, shapes, off, vals = net.blocks(esg.BLOCKS_UNCOUPLED)
    nt, nm, et, em, cnt = net.build_targets(keys, shapes, vals)
    for t, m, ref in ((nt, nm, no), (et, em, eo)):
        sel = m.astype(bool)
        assert np.abs(t[sel] - ref[sel]).max() <= 1e-5 * np.abs(ref).max()
    assert cnt == int(nm.sum() + em.sum()) == int((shapes[:, 0] * shapes[:, 1]).sum())
    # a numpy restatement of encode_target for a few items
    for b in (0, s.n_atoms, len(keys) - 1):
        za, zb = (s.species[keys[b, 0]], s.species[keys[b, 1]])
        blk = vals[off[b]:off[b + 1]].reshape(shapes[b])
        row = nt[b] if b < s.n_atoms else et[b - s.n_atoms]
        want = om.uncoupled_block(za, zb, row, *shapes[b])  # encode then decode must round-trip
        assert np.abs(want - blk).max() <= 1e-5 * max(1.0, np.abs(blk).max())
    # through the text format, as model_run reads training targets
    net.write_blocks_text(str(tmp_path / "targets.txt"), esg.BLOCKS_UNCOUPLED)
    tk, ts, to, tv = esg.read_blocks_text(str(tmp_path / "targets.txt"))
    nt3, nm3, et3, em3, cnt3 = net.build_targets(tk, ts, tv)
    assert cnt3 == cnt and np.array_equal(nm3, nm) and np.array_equal(em3, em)
    assert np.array_equal(nt3, nt) and np.array_equal(et3, et)
    # only half of the blocks given: the others keep mask 0
    half = np.arange(len(keys)) % 2 == 0
    hv = np.concatenate([vals[off[b]:off[b + 1]] for b in np.nonzero(half)[0]])
    nt2, nm2, et2, em2, cnt2 = net.build_targets(keys[half], shapes[half], hv)
    masks = np.concatenate([nm2.any(axis=1), em2.any(axis=1)])
    assert np.array_equal(masks, half) and cnt2 == int((shapes[half, 0] * shapes[half, 1]).sum())
