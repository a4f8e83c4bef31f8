"""Colour-wise exchange on the device (pf_hierarchy_set_colorwise_exchange) against the
oracle's restatement (orc_set_colorwise), bit for bit: K subdomains on one GPU (per-level
kernels and the cooperative bottom kernel) and K ranks through the peer transport."""
import os
import subprocess
import sys

import numpy as np
import pytest

from helpers import cfg, download, structured, upload
from oracle.restated import Oracle
from paper_1609_04809_b200 import _lib, gmg
from paper_1609_04809_b200.fe import LOGNORMAL, ROTATED_Q1, FESetup
from paper_1609_04809_b200.levels import StructuredSetup

pytestmark = pytest.mark.gpu
HERE = os.path.dirname(os.path.abspath(__file__))


def exact(a, b):
    return all(np.array_equal(x, y) for x, y in zip(a, b))


@pytest.mark.parametrize("K,L", [(2, 4), (4, 4), (8, 4), (3, 3)])
@pytest.mark.parametrize("kind", [gmg.PF_SMOOTHER_GAUSS_SEIDEL, gmg.PF_SMOOTHER_MULTICOLOR_SOR], ids=["gs", "sor"])
@pytest.mark.parametrize("bottom", ["0", "1024"], ids=["multilaunch", "bottom"])
def test_colorwise_q1_bit_exact(cuda, K, L, kind, bottom):
    ss = [StructuredSetup(3, 2, L, K, r, _lib.PF_PROBLEM_LOGNORMAL, seed=7) for r in range(K)]
    lv = [s.levels for s in ss]
    c = cfg(kind, damping=1.2 if kind == gmg.PF_SMOOTHER_MULTICOLOR_SOR else 1.0, max_cycles=100)
    h = gmg.Hierarchy(lv, options={"bottom_rows": int(bottom)}).set_colorwise_exchange()
    x = upload(h, L - 1, [s.x0 for s in ss])
    st = gmg.solve_outer(h, x, upload(h, L - 1, [s.b for s in ss]), c)
    xo, res, ost, rc = Oracle(lv, colorwise=True).solve_outer([s.x0 for s in ss], [s.b for s in ss], c)
    assert rc == 0 and st.iterations == ost.iterations
    np.testing.assert_allclose(st.residuals, res, rtol=1e-12)
    assert exact(download(h, x, K), xo)


def test_colorwise_rotated_q1_k8_converges_bit_exact(cuda):
    """configs[3]'s element and coefficient (32^3 cells) on 8 subdomains, SOR w = 1.2: the
    processor-local sweep diverges (NoConvergenceError), the colour-wise one converges in the
    single-domain cycle count, equal to the oracle bit for bit."""
    fs = [FESetup(ROTATED_Q1, 2, 5, LOGNORMAL, seed=2024, n_ranks=8, rank=r) for r in range(8)]
    lv = [f.levels for f in fs]
    c = cfg(gmg.PF_SMOOTHER_MULTICOLOR_SOR, damping=1.2, max_cycles=300)
    h = gmg.Hierarchy(lv)
    x = upload(h, 4, [f.x0 for f in fs])
    b = upload(h, 4, [f.b for f in fs])
    with pytest.raises(gmg.NoConvergenceError):
        gmg.solve_outer(h, x, b, c)
    h.set_colorwise_exchange()
    x = upload(h, 4, [f.x0 for f in fs])
    st = gmg.solve_outer(h, x, b, c)
    xo, res, ost, rc = Oracle(lv, colorwise=True).solve_outer([f.x0 for f in fs], [f.b for f in fs], c)
    one = FESetup(ROTATED_Q1, 2, 5, LOGNORMAL, seed=2024)
    _, _, st1, _ = Oracle([one.levels]).solve_outer([one.x0], [one.b], c)
    assert rc == 0 and st.iterations == ost.iterations == st1.iterations
    assert exact(download(h, x, 8), xo)


@pytest.mark.parametrize("fused", [False, True], ids=["standard", "fused"])
def test_colorwise_through_the_peer_transport(cuda, tmp_path, fused):
    """4 ranks as hierarchies of one process over the peer transport, colour-wise SOR on the
    lognormal Q1 problem: equal to the oracle's 4-rank colour-wise solve bit for bit."""
    env = {**os.environ, "CUDA_MODULE_LOADING": "EAGER", "CUDA_DEVICE_MAX_CONNECTIONS": "32", "PF_WATCHDOG_S": "60"}
    cmd = [sys.executable, os.path.join(HERE, "peer_threads.py"), "--out", str(tmp_path), "--world", "4",
           "--levels", "4", "--kind", "2", "--rep", "bottom", "--colorwise", "--problem", "4"] + (["--fused"] if fused else [])
    r = subprocess.run(cmd, env=env, capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, (r.stdout + r.stderr)[-3000:]
    ss = [StructuredSetup(3, 2, 4, 4, q, _lib.PF_PROBLEM_LOGNORMAL, seed=1, direct_halos=fused) for q in range(4)]
    lv = [s.levels for s in ss]
    c = cfg(gmg.PF_SMOOTHER_MULTICOLOR_SOR, damping=1.2)
    xs, res, ost, rc = Oracle(lv, colorwise=True).solve_outer([s.x0 for s in ss], [s.b for s in ss], c)
    for q in range(4):
        z = np.load(os.path.join(str(tmp_path), f"result_{q}.npz"))
        assert int(z["iterations"]) == ost.iterations
        assert np.array_equal(z["x"], xs[q]) and np.array_equal(z["x_again"], xs[q])
