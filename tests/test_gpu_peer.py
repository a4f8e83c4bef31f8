"""The peer-memory transport (pf_peer.cu): the multi-process data plane running the way a
multi-GPU run runs it — one subdomain per hierarchy, every exchange one kernel storing into
the peer's mapped memory, and the whole outer cycle recorded into a CUDA graph (the
captured branch of solve_outer that NCCL-free multi-GPU runs take).

Two placements of the ranks, both bit-exact against the oracle's K-rank solve
(fecomm.cpp:25-72 exchange order, test_multigrid.cpp:218-250's rank-count invariance):
  * K hierarchies of one process on K host threads (arena pointers shared directly);
  * K separate processes on cuda:0, arenas mapped with CUDA IPC (tests/peer_rank.py),
    the cross-process path a one-process-per-GPU run over NVLink takes.
"""
import os
import subprocess
import sys

import numpy as np
import pytest

from helpers import cfg, key_noise, structured
from oracle.restated import Oracle
from paper_1609_04809_b200 import _lib, gmg

pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))


def _run(cmds, timeout=240, env=None):
    """Run the rank processes (or the one threaded process) and fail with their output."""
    env = {**os.environ, "PF_WATCHDOG_S": "60", **(env or {})}
    procs = [subprocess.Popen(c, env=env, stdout=subprocess.PIPE, stderr=subprocess.STDOUT) for c in cmds]
    outs = []
    for p in procs:
        try:
            out, _ = p.communicate(timeout=timeout)
        except subprocess.TimeoutExpired:
            for q in procs:
                q.kill()
            raise
        outs.append(out.decode(errors="replace"))
    for r, p in enumerate(procs):
        assert p.returncode == 0, f"process {r} failed:\n{outs[r][-3000:]}"


def _check(d, K, L, fused, kind):
    setups, levels = structured(3, 2, L, K, direct_halos=fused)
    c = cfg(kind, damping=1.2 if kind == gmg.PF_SMOOTHER_MULTICOLOR_SOR else 0.8)
    xs, resid, ost, acc = _oracle(levels, setups, c, L)
    rn0 = None
    for r in range(K):
        z = np.load(os.path.join(d, f"result_{r}.npz"))
        assert int(z["graphs"]) >= 1, "the multi-process solve must run from a captured graph"
        assert int(z["iterations"]) == ost.iterations
        np.testing.assert_allclose(z["residuals"], resid, rtol=1e-12)
        assert np.array_equal(z["x"], xs[r]), f"rank {r}"
        assert np.array_equal(z["x_again"], xs[r]), f"rank {r} (graph replay)"
        assert np.array_equal(z["acc"], acc[r]), f"accumulate rank {r}"
        rn0 = float(z["rn"]) if rn0 is None else rn0
        assert float(z["rn"]) == rn0


# ranks that share one process share its CUDA context: eager module loading and a hardware
# work queue per stream (pf_hierarchy_init_peer checks both)
THREAD_ENV = {"CUDA_MODULE_LOADING": "EAGER", "CUDA_DEVICE_MAX_CONNECTIONS": "32"}


def _oracle(levels, setups, c, L):
    o = Oracle(levels)
    xs, resid, ost, rc = o.solve_outer([s.x0 for s in setups], [s.b for s in setups], c)
    acc = o.update_master_slave(L - 2, key_noise([lv[L - 2] for lv in levels], 3), 1)
    return xs, resid, ost, acc


CASES = [(2, 4, "coarse", False), (4, 4, "bottom", False), (8, 3, "coarse", False),
         (4, 4, "bottom", True), (2, 4, "bottom", True), (3, 3, "coarse", True), (8, 4, "bottom", True)]


def _args(K, L, rep, fused, kind):
    return ["--world", str(K), "--levels", str(L), "--kind", str(kind), "--rep", rep] + (["--fused"] if fused else [])


@pytest.mark.parametrize("K,L,rep,fused", CASES, ids=lambda v: str(v))
@pytest.mark.parametrize("kind", [gmg.PF_SMOOTHER_JACOBI, gmg.PF_SMOOTHER_MULTICOLOR_SOR], ids=["jacobi", "sor"])
def test_peer_threads_captured(cuda, tmp_path, K, L, rep, fused, kind):
    """K hierarchies on K threads of one process (tests/peer_threads.py) exchange through
    the peer transport; solve_outer takes the captured outer-cycle graph (exchange kernels,
    fused exchanges, the replicated bottom) and must equal the oracle bit for bit, twice in
    a row (graph replay).  (In-process ranks run without the side-stream overlap; the
    process tests below cover it.)"""
    _run([[sys.executable, os.path.join(HERE, "peer_threads.py"), "--out", str(tmp_path)] + _args(K, L, rep, fused, kind)],
         env=THREAD_ENV)
    _check(str(tmp_path), K, L, fused, kind)


@pytest.mark.parametrize("K,L,rep,fused,kind", [(2, 4, "coarse", False, 0), (2, 4, "bottom", True, 0),
                                                (4, 4, "bottom", True, 0), (4, 3, "coarse", False, 2),
                                                (3, 3, "coarse", True, 0), (4, 4, "bottom", True, 2),
                                                (2, 4, "coarse", True, 2), (3, 4, "coarse", True, 1)],
                         ids=lambda v: str(v))
def test_peer_processes_ipc(cuda, tmp_path, K, L, rep, fused, kind):
    """K processes on cuda:0, each one rank (tests/peer_rank.py), arenas mapped with CUDA
    IPC — the path of one process per GPU over NVLink: the captured multi-process solve
    (fused exchanges with the side-stream overlap of the Jacobi sweep / the last colour of
    the coloured sweep, replicated bottom) equals the oracle's K-rank solve bit for bit."""
    d = str(tmp_path)
    _run([[sys.executable, os.path.join(HERE, "peer_rank.py"), "--dir", d, "--rank", str(r)] + _args(K, L, rep, fused, kind)
          for r in range(K)])
    _check(d, K, L, fused, kind)


def test_peer_watchdog_raises_transport_error(cuda, tmp_path):
    """A rank that never reaches the exchange: the waiting kernels give up after
    PF_WATCHDOG_S and the solve raises TransportError (transport.cpp:54-60) instead of
    hanging the device."""
    _run([[sys.executable, os.path.join(HERE, "peer_threads.py"), "--out", str(tmp_path), "--idle-rank", "1"]
          + _args(2, 3, "coarse", False, 0)], env=dict(THREAD_ENV, PF_WATCHDOG_S="2"))
    z = np.load(os.path.join(str(tmp_path), "result_0.npz"))
    assert str(z["error"]).startswith("TransportError: peer watchdog")


def test_in_process_peers_need_eager_loading(cuda):
    """Without eager module loading / enough hardware queues, in-process peer ranks are
    refused at init (they could deadlock), not silently run."""
    K, L = 2, 3
    setups, levels = structured(3, 2, L, K)
    replicas = [s[0] for s in levels]
    hs = [gmg.Hierarchy([levels[r]], rank_base=r, world_size=K, coarse_replicas=replicas) for r in range(K)]
    blobs = [h.peer_export() for h in hs]
    if os.environ.get("CUDA_MODULE_LOADING") != "EAGER":
        with pytest.raises(_lib.PfError, match="EAGER"):
            hs[0].init_peer(blobs)


def test_peer_blob_mismatch_is_rejected(cuda):
    """Blobs of a different hierarchy shape (or out of rank order) are refused."""
    K, L = 2, 3
    setups, levels = structured(3, 2, L, K)
    replicas = [s[0] for s in levels]
    h0 = gmg.Hierarchy([levels[0]], rank_base=0, world_size=K, coarse_replicas=replicas)
    h1 = gmg.Hierarchy([levels[1]], rank_base=1, world_size=K, coarse_replicas=replicas)
    b0, b1 = h0.peer_export(), h1.peer_export()
    with pytest.raises(_lib.InvalidArgument):
        h0.init_peer([b1, b0])
