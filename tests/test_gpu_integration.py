"""INTEGRATION.md's forward_rank patch, compiled against the reference's own
headers and types (tools/integration/forward_rank_b200.cpp, built by
oracle/ref.mk) and run on the GPU: the reference's call site drives
libesg_b200 through the façade.

Checks: the device graph equals the reference's structures::build_graph bit
for bit (the program's exit code), usage errors surface as the reference's
esgnn::UsageError, the heads are within the fp32 bar of the reference's own
Network<float> forward, and blocks_coupled.txt / blocks_uncoupled.txt carry
the reference run's keys in its order with values within the same bar.
"""
import os
import subprocess

import numpy as np
import pytest

import ref as R
from paper_2507_03840_b200 import esg

BIN = os.path.join(R.ROOT, "oracle", "_ref", "forward_rank_b200")
pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not (R.available() and os.path.exists(BIN)),
                                                  reason="oracle/_ref not built")]
PBC1 = np.ones(3, np.uint8)


@pytest.mark.parametrize("case", ["small", "C1"])
def test_patched_forward_rank(tmp_path, case):
    out = subprocess.run([BIN, str(tmp_path), case], capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stdout + out.stderr
    assert "bit-identical to the reference's build_graph" in out.stdout
    assert "esgnn::UsageError (core/error.h)" in out.stdout
    if case == "C1":
        s, r, layers, basis = esg.config_structure("C1")
    else:
        s, r, layers, basis = esg.make_jittered_lattice(40, 2.2, 0.45, [72, 8, 8], 4), 4.5, 2, esg.BASIS_HFO2
    rc, ru = str(tmp_path / "ref_coupled.txt"), str(tmp_path / "ref_uncoupled.txt")
    rno, reo, g = R.forward(s.positions, s.species, s.cell, PBC1, r, basis, layers=layers, precision=4,
                            coupled_path=rc, uncoupled_path=ru)
    heads = np.fromfile(str(tmp_path / "heads.bin"), np.float32).astype(np.float64)
    want = np.concatenate([rno.ravel(), reo.ravel()])
    assert heads.size == want.size
    assert np.abs(heads - want).max() <= 2e-4 * np.abs(want).max()
    assert np.linalg.norm(heads - want) <= 2e-5 * np.linalg.norm(want)
    for mine, theirs in (("blocks_coupled.txt", rc), ("blocks_uncoupled.txt", ru)):
        k1, sh1, o1, v1 = esg.read_blocks_text(str(tmp_path / mine))
        k2, sh2, o2, v2 = esg.read_blocks_text(theirs)
        assert np.array_equal(k1, k2) and np.array_equal(sh1, sh2), mine
        assert np.abs(v1 - v2).max() <= 2e-4 * np.abs(v2).max(), mine


DEMO = os.path.join(R.ROOT, "paper_2507_03840_b200", "facade_demo")


@pytest.mark.skipif(not os.path.exists(DEMO), reason="facade_demo not built")
def test_facade_demo_runs_on_gpu():
    """The façade's own demo (csrc/facade_demo.cpp): model_run.cpp's
    forward_rank call sequence written against esgnn_b200.hpp, on the GPU."""
    out = subprocess.run([DEMO], capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stdout + out.stderr
