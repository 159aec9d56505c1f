"""GPU training path against the CPU oracle.

Bars:
  * loss: relative error <= 1e-5 against the fp64 oracle (fp32 forward)
  * gradients: relative-L2 over the full parameter gradient <= 1e-5 and
    max-abs <= 1e-4 x max|ref| against the fp64 oracle's reverse pass (itself
    pinned by finite differences, tests/test_train_cpu.py)
  * deterministic: two evaluations give bit-identical gradients
  * the Adam step equals optimizer.h applied to the returned gradients
"""
import numpy as np
import pytest

import oracle as O
from paper_2507_03840_b200 import esg

pytestmark = pytest.mark.gpu

SP_BASIS = {1: [0, 1], 8: [0, 1]}


def problem(gpu_ctx, L, E, layers=2, n=24, r_cut=4.0, seed=5):
    pos, cell, species = O.jittered_lattice(n, 2.2, 0.3, [1, 8], seed)
    s = esg.AtomicStructure(pos, species, cell, np.ones(3, bool))
    g = esg.build_graph(gpu_ctx, s, r_cut)
    gx = g.export()
    cfg = esg.ModelConfig(l_max=L, e_width=E, layers=layers, n_radial=8, r_cut=r_cut, seed=11,
                          linear_precision=esg.LINEAR_FP32)
    net = esg.Network(gpu_ctx, cfg, SP_BASIS)
    net.init_params()
    net.prepare(g, species)
    om = O.Model(L, E, layers, 8, r_cut, 11, SP_BASIS)
    view = O.serial_view(n, species, gx)
    nt, nm, et, em, nt64, et64 = om.toy_targets(n, species, gx)
    n_total = int(nm.sum() + em.sum())
    net.set_targets(nt, nm, et, em)
    return net, om, view, (nt, nm, et, em), (nt64, nm, et64, em), n_total, g


def rel(a, b):
    return float(np.linalg.norm(a.astype(np.float64) - b) / max(np.linalg.norm(b), 1e-300))


@pytest.mark.parametrize("L,E", [(4, 16), (2, 8)])
def test_loss_and_gradients_match_oracle(gpu_ctx, L, E):
    net, om, view, t32, t64, n_total, g = problem(gpu_ctx, L, E)
    loss, partials, grads = net.loss_grad(n_total)
    (sa, sq, cnt), ref = O.loss_grad(om, view, t64, n_total, np.float64)
    ref_loss = (sa + sq) / n_total
    assert partials[2] == cnt == n_total
    assert abs(loss - ref_loss) <= 1e-5 * abs(ref_loss), (loss, ref_loss)
    r = rel(grads, ref)
    mx = float(np.abs(grads.astype(np.float64) - ref).max() / np.abs(ref).max())
    print(f"L={L} E={E} edges={len(view['src_row'])} loss {loss:.8g} vs {ref_loss:.8g}  grad relL2 {r:.3g} max {mx:.3g}")
    assert r <= 1e-5, r
    assert mx <= 1e-4, mx
    # per parameter entry: every entry's gradient is right, not just the bulk
    for name, rows, cols, off in om.entries():
        a = grads[off:off + rows * cols].astype(np.float64)
        b = ref[off:off + rows * cols]
        if np.abs(b).max() > 1e-6 * np.abs(ref).max():
            assert rel(a, b) <= 1e-4, (name, rel(a, b))


def test_gradients_many_splits_and_chunks(gpu_ctx, monkeypatch):
    """A graph of ~6k edges: the tensor-core weight gradients run over a dozen
    512-edge splits (dw_tc.cu, fp64 split sum) and the training forward over
    several 1,024-edge chunks -- same bars as the small problem."""
    monkeypatch.setenv("ESG_CHUNK_EDGES", "1024")
    net, om, view, t32, t64, n_total, g = problem(gpu_ctx, 4, 16, n=240, r_cut=4.5, seed=7)
    assert len(view["src_row"]) > 12 * 512
    loss, partials, grads = net.loss_grad(n_total)
    (sa, sq, cnt), ref = O.loss_grad(om, view, t64, n_total, np.float64)
    assert abs(loss - (sa + sq) / n_total) <= 1e-5 * abs(loss)
    r = rel(grads, ref)
    mx = float(np.abs(grads.astype(np.float64) - ref).max() / np.abs(ref).max())
    assert r <= 1e-5 and mx <= 1e-4, (r, mx)


def test_gradients_deterministic(gpu_ctx):
    net, *_, n_total, g = problem(gpu_ctx, 4, 16)
    l1, _, g1 = net.loss_grad(n_total)
    l2, _, g2 = net.loss_grad(n_total)
    assert l1 == l2
    assert np.array_equal(g1.view(np.uint32), g2.view(np.uint32))


def test_train_step_is_adam_on_the_gradients(gpu_ctx):
    net, om, view, t32, t64, n_total, g = problem(gpu_ctx, 4, 16)
    p0 = net.params()
    loss0, _, grads = net.loss_grad(n_total)
    opt = esg.Adam(net)
    loss_step, fwd_ms, bwd_ms = net.train_step(opt, n_total)
    assert loss_step == loss0
    want = O.Adam(net.n_params).step(p0, grads, loss0)
    assert np.array_equal(net.params().view(np.uint32), want.view(np.uint32))
    # a few steps reduce the loss (toy targets, Adam lr 5e-3)
    losses = [loss_step] + [net.train_step(opt, n_total)[0] for _ in range(5)]
    assert losses[-1] < losses[0], losses
    assert fwd_ms > 0 and bwd_ms > 0


def test_exact_resume_from_checkpoint(gpu_ctx, tmp_path):
    """§8(f) 2: 4 training steps straight vs 2 steps, checkpoint (params +
    Adam moments), load into a fresh network and optimizer, 2 more steps:
    bit-identical parameters and losses (the GPU step is deterministic)."""
    net, om, view, t32, t64, n_total, g = problem(gpu_ctx, 4, 16)
    opt = esg.Adam(net)
    straight = [net.train_step(opt, n_total)[0] for _ in range(4)]
    p_straight = net.params()

    net2, *_ = problem(gpu_ctx, 4, 16)
    opt2 = esg.Adam(net2)
    first = [net2.train_step(opt2, n_total)[0] for _ in range(2)]
    path = str(tmp_path / "mid.ckpt")
    net2.save_checkpoint(path, opt2, "l_max=4")

    net3, *_ = problem(gpu_ctx, 4, 16)
    net3.set_params(np.zeros(net3.n_params, np.float32))
    opt3 = esg.Adam(net3)
    assert net3.load_checkpoint(path, opt3) == "l_max=4"
    second = [net3.train_step(opt3, n_total)[0] for _ in range(2)]
    assert first + second == straight
    assert np.array_equal(net3.params().view(np.uint32), p_straight.view(np.uint32))
