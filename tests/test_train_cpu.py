"""Training path on the CPU oracle: the reference's own
known-answer tests for the loss and the gradients (test_model.cpp:233-275,
437-470), which pin the oracle's backward that the GPU tests compare with."""
import numpy as np
import pytest

import oracle as O

SP_BASIS = {1: [0, 1], 8: [0, 1]}  # test_model.cpp:22-27 sp_basis


def small_model():
    # test_model.cpp:29-37 small_config: l_max 2, E 4, 2 layers, 8 Gaussians, r_cut 3.4, seed 11
    return O.Model(2, 4, 2, 8, 3.4, 11, SP_BASIS)


def toy_problem(model, n, spacing, jitter, seed, r_cut):
    pos, cell, species = O.jittered_lattice(n, spacing, jitter, [1, 8], seed)
    g = O.build_graph(pos, cell, np.ones(3, np.uint8), r_cut)
    view = O.serial_view(n, species, g)
    nt, nm, et, em, nt64, et64 = model.toy_targets(n, species, g)
    return species, g, view, (nt, nm, et, em), (nt64, nm, et64, em)


def test_masked_loss_matches_elementwise():
    """test_model.cpp:437-470: partial sums and the seeded gradient."""
    rng = np.random.default_rng(71)
    pred = rng.standard_normal((3, 4))
    tgt = rng.standard_normal((3, 4))
    mask = np.zeros((3, 4), np.uint8)
    mask.reshape(-1)[::2] = 1
    (sa, sq, cnt), g = O.masked_loss(pred, tgt, mask, 6)
    d = (pred - tgt).reshape(-1)[::2]
    assert cnt == 6
    assert sa == pytest.approx(np.abs(d).sum(), rel=1e-14)
    assert sq == pytest.approx((d * d).sum(), rel=1e-14)
    gf = g.reshape(-1)
    assert np.all(gf[1::2] == 0.0)
    np.testing.assert_allclose(gf[::2], (np.sign(d) + 2 * d) / 6.0, rtol=1e-14)


def test_toy_targets_mirror_blocks_and_mask():
    """Every graph edge and node gets a target; mirror pair blocks are
    transposes (synthetic.cpp:79-95): for same-species pairs the coupled
    encodings of (i,j,s) and (j,i,-s) agree up to the (-1)^(la+lb+L) parity."""
    m = small_model()
    s, g, view, t32, t64 = toy_problem(m, 6, 2.2, 0.25, 21, 3.4)
    nt, nm, et, em = t32
    assert nm.any(axis=1).all() and em.any(axis=1).all()
    assert np.isfinite(nt).all() and np.isfinite(et).all()


def test_oracle_gradients_match_finite_differences():
    """test_model.cpp:233-275: 150 random parameters, central differences in
    double against the oracle's reverse pass, |fd - an| / max(1e-3, |fd|, |an|) < 1e-5."""
    m = small_model()
    s, g, view, t32, t64 = toy_problem(m, 6, 2.2, 0.25, 21, 3.4)
    nt64, nm, et64, em = t64
    targets = (nt64, nm, et64, em)
    n_total = int(nm.sum() + em.sum())
    assert len(g["src"]) > 0 and n_total > 0
    p0 = m.params_f64()
    _, grads = O.loss_grad(m, view, targets, n_total, np.float64)

    def loss(p):
        m.set_params_f64(p)
        no, eo = m.forward(view, np.float64)
        (a, b, _), _ = O.masked_loss(no, nt64, nm, n_total)
        (c, d, _), _ = O.masked_loss(eo, et64, em, n_total)
        return (a + b + c + d) / n_total

    # ParamStore entries picked as the reference does (rng() % n_entries, rng() % count)
    entries = m.entries()
    rng = np.random.default_rng(5)
    checked, worst = 0, 0.0
    for _ in range(150):
        name, r, c, off = entries[int(rng.integers(len(entries)))]
        k = off + int(rng.integers(r * c))
        save = p0[k]
        h = 1e-6 * max(1.0, abs(save))
        p = p0.copy()
        p[k] = save + h
        lp = loss(p)
        p[k] = save - h
        lm = loss(p)
        fd = (lp - lm) / (2.0 * h)
        an = grads[k]
        scale = max(1e-3, abs(fd), abs(an))
        worst = max(worst, abs(fd - an) / scale)
        checked += 1
    m.set_params_f64(p0)
    assert checked == 150
    assert worst < 1e-5, worst


def test_oracle_gradients_fd_lmax4():
    """The same finite-difference check at l_max 4, E 8 (the GPU kernels'
    instantiation), 40 parameters, one layer."""
    m = O.Model(4, 8, 1, 8, 3.4, 13, SP_BASIS)
    species, g, view, t32, t64 = toy_problem(m, 6, 2.2, 0.25, 21, 3.4)
    nt64, nm, et64, em = t64
    n_total = int(nm.sum() + em.sum())
    p0 = m.params_f64()
    _, grads = O.loss_grad(m, view, (nt64, nm, et64, em), n_total, np.float64)

    def loss(p):
        m.set_params_f64(p)
        no, eo = m.forward(view, np.float64)
        (a, b, _), _ = O.masked_loss(no, nt64, nm, n_total)
        (c, d, _), _ = O.masked_loss(eo, et64, em, n_total)
        return (a + b + c + d) / n_total

    rng = np.random.default_rng(7)
    entries = m.entries()
    worst = 0.0
    for _ in range(40):
        name, r, c, off = entries[int(rng.integers(len(entries)))]
        k = off + int(rng.integers(r * c))
        h = 1e-6 * max(1.0, abs(p0[k]))
        p = p0.copy()
        p[k] += h
        lp = loss(p)
        p[k] -= 2 * h
        lm = loss(p)
        fd = (lp - lm) / (2 * h)
        worst = max(worst, abs(fd - grads[k]) / max(1e-3, abs(fd), abs(grads[k])))
    m.set_params_f64(p0)
    assert worst < 1e-5, worst
