"""The bench configuration pinned bit for bit: C2 (128^3 Q1, 7 levels, V(2,2) damped Jacobi,
1e-10) solved on the device from the product setup must reproduce the UNMODIFIED
reference's whole solution — sha256 of every authoritative value in Key4 order
(tests/golden/c2_jacobi_k{1,8}_digest.npz, made by make_golden.py --c2-digest) — with 1
subdomain, with 8 subdomains on one GPU, and with 8 ranks exchanging through the peer
transport; residual histories within the norm-roundoff gate (device norms are tree sums)."""
import os
import subprocess
import sys

import numpy as np
import pytest

from helpers import cfg, download, keyed_digest, structured, upload
from paper_1609_04809_b200 import gmg

pytestmark = pytest.mark.gpu
HERE = os.path.dirname(os.path.abspath(__file__))


def golden(K):
    return np.load(os.path.join(HERE, "golden", f"c2_jacobi_k{K}_digest.npz"))


@pytest.mark.parametrize("K", [1, 8])
def test_c2_solution_digest_single_device(cuda, K):
    g = golden(K)
    setups, levels = structured(3, 2, 7, K)
    h = gmg.Hierarchy(levels)
    x = upload(h, 6, [s.x0 for s in setups])
    st = gmg.solve_outer(h, x, upload(h, 6, [s.b for s in setups]), cfg())
    assert st.iterations == int(g["iterations"]) == 9
    assert keyed_digest([lv[-1] for lv in levels], download(h, x, K)) == str(g["digest"])
    # the device norm is a tree sum of 2M squares, the reference's a sequential one: the
    # two agree to a few ulps of the sum (n eps bounds it at 2e-10)
    np.testing.assert_allclose(st.residuals, g["residuals"], rtol=1e-10)


def test_c2_solution_digest_peer_ranks(cuda, tmp_path):
    """8 ranks, one hierarchy each, exchanging through the peer transport inside the
    captured outer-cycle graphs (replicated bottom): the reference's 8-rank solution."""
    g = golden(8)
    env = {**os.environ, "CUDA_MODULE_LOADING": "EAGER", "CUDA_DEVICE_MAX_CONNECTIONS": "32", "PF_WATCHDOG_S": "120"}
    cmd = [sys.executable, os.path.join(HERE, "peer_threads.py"), "--out", str(tmp_path), "--world", "8",
           "--levels", "7", "--kind", "0", "--rep", "coarse"]
    r = subprocess.run(cmd, env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, (r.stdout + r.stderr)[-3000:]
    setups, levels = structured(3, 2, 7, 8)
    xs = [np.load(os.path.join(str(tmp_path), f"result_{q}.npz"))["x"] for q in range(8)]
    z0 = np.load(os.path.join(str(tmp_path), "result_0.npz"))
    assert int(z0["iterations"]) == int(g["iterations"])
    assert keyed_digest([lv[-1] for lv in levels], xs) == str(g["digest"])
