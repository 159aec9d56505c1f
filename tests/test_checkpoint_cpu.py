"""Checkpoints and the optimizer on the host-only model.

The parameter section is checkpoint.h:15-92's version-1 container, read here
by `reference_load`: a restatement of the reference's load_checkpoint that
reads the named arrays and nothing else.  The optimizer section that follows
(which the reference lacks) must give a bit-exact resume.
"""
import struct

import numpy as np
import pytest

import oracle as O
from paper_2507_03840_b200 import esg

SP_BASIS = {1: [0, 1], 8: [0, 1]}


def host_model(seed=11, l_max=2):
    net = esg.Network(None, esg.ModelConfig(l_max=l_max, e_width=8, layers=2, n_radial=8, r_cut=4.0, seed=seed),
                      SP_BASIS)
    net.init_params()
    return net


def reference_load(path):
    """checkpoint.h:50-92: magic, version, config, scalar width, entries."""
    with open(path, "rb") as f:
        buf = f.read()
    assert buf[:8] == b"ESGNNCK1"
    off = 8

    def u64():
        nonlocal off
        (v,) = struct.unpack_from("<Q", buf, off)
        off += 8
        return v

    assert u64() == 1
    n = u64()
    cfg = buf[off:off + n].decode()
    off += n
    assert u64() == 4
    out = []
    for _ in range(u64()):
        n = u64()
        name = buf[off:off + n].decode()
        off += n
        r, c = u64(), u64()
        data = np.frombuffer(buf, np.float32, r * c, off)
        off += 4 * r * c
        out.append((name, r, c, data))
    return cfg, out, off, len(buf)


def test_params_only_file_is_the_reference_container(tmp_path):
    net = host_model()
    p = tmp_path / "a.ckpt"
    net.save_checkpoint(str(p), config_text="l_max=2\nwidth=8\n")
    cfg, arrays, end, size = reference_load(p)
    assert cfg == "l_max=2\nwidth=8\n"
    assert end == size  # nothing after the arrays without an optimizer
    params = net.params()
    ents = net.entries()
    assert [(a[0], a[1], a[2]) for a in arrays] == [(e[0], e[1], e[2]) for e in ents]
    for (name, r, c, data), (_, _, _, o) in zip(arrays, ents):
        assert np.array_equal(data, params[o:o + r * c])


def test_roundtrip_restores_parameters(tmp_path):
    a, b = host_model(seed=11), host_model(seed=99)
    assert not np.array_equal(a.params(), b.params())
    p = tmp_path / "a.ckpt"
    a.save_checkpoint(str(p), config_text="cfg")
    assert b.load_checkpoint(str(p)) == "cfg"
    assert np.array_equal(a.params().view(np.uint32), b.params().view(np.uint32))


def test_load_rejects_mismatches(tmp_path):
    a = host_model()
    p = tmp_path / "a.ckpt"
    a.save_checkpoint(str(p))
    with pytest.raises(esg.DataError):  # other architecture: entry shapes differ
        host_model(l_max=4).load_checkpoint(str(p))
    bad = tmp_path / "bad.ckpt"
    bad.write_bytes(b"NOTACKPT" + p.read_bytes()[8:])
    with pytest.raises(esg.DataError):
        a.load_checkpoint(str(bad))
    trunc = tmp_path / "trunc.ckpt"
    trunc.write_bytes(p.read_bytes()[:-100])
    with pytest.raises(esg.DataError):
        a.load_checkpoint(str(trunc))
    with pytest.raises(esg.DataError):  # asked for optimizer state the file does not hold
        a.load_checkpoint(str(p), esg.Adam(a))
    with pytest.raises(esg.DataError):
        a.load_checkpoint(str(tmp_path / "missing.ckpt"))


def grad_stream(n, steps, seed=3):
    rng = np.random.default_rng(seed)
    # losses first fall then plateau so reduce-on-plateau fires (patience 3)
    losses = [1.0 / (k + 1) if k < steps // 2 else 0.25 for k in range(steps)]
    return [(rng.standard_normal(n).astype(np.float32) * 0.1, losses[k]) for k in range(steps)]


def test_adam_apply_matches_optimizer_restatement():
    net = host_model()
    opt = esg.Adam(net, patience=3)
    ref = O.Adam(net.n_params, patience=3)
    p = net.params()
    for g, loss in grad_stream(net.n_params, 12):
        opt.apply(net, g, loss)
        p = ref.step(p, g, loss)
        assert np.array_equal(net.params().view(np.uint32), p.view(np.uint32))
    assert opt.lr == ref.lr < 5e-3  # the plateau halved the rate


def test_exact_resume_through_checkpoint(tmp_path):
    stream = grad_stream(host_model().n_params, 12)
    cont = host_model()
    copt = esg.Adam(cont, patience=3)
    for g, loss in stream:
        copt.apply(cont, g, loss)

    first = host_model()
    fopt = esg.Adam(first, patience=3)
    for g, loss in stream[:5]:
        fopt.apply(first, g, loss)
    p = tmp_path / "mid.ckpt"
    first.save_checkpoint(str(p), fopt, "resume")
    cfg, arrays, end, size = reference_load(p)  # the reference still reads it
    assert end < size and cfg == "resume"

    resumed = host_model(seed=123)
    ropt = esg.Adam(resumed)  # defaults; the file's optimizer config wins
    resumed.load_checkpoint(str(p), ropt)
    for g, loss in stream[5:]:
        ropt.apply(resumed, g, loss)
    assert np.array_equal(resumed.params().view(np.uint32), cont.params().view(np.uint32))
    assert ropt.lr == copt.lr

    # without the moments the same resume diverges: the section is what makes it exact
    fresh = host_model(seed=123)
    fresh.load_checkpoint(str(p))
    nopt = esg.Adam(fresh, patience=3)
    for g, loss in stream[5:]:
        nopt.apply(fresh, g, loss)
    assert not np.array_equal(fresh.params(), cont.params())
