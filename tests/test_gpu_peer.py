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
import threading

import numpy as np
import pytest

from helpers import cfg, key_noise, structured
from oracle.restated import Oracle
from paper_1609_04809_b200 import _lib, gmg

pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))


def _threads(K, body):
    out, errs = [None] * K, []
    bar = threading.Barrier(K)

    def wrap(r):
        try:
            out[r] = body(r, bar)
        except Exception as e:  # noqa: BLE001
            errs.append(e)
            bar.abort()
    th = [threading.Thread(target=wrap, args=(r,)) for r in range(K)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    if errs:
        raise errs[0]
    return out


def _oracle(levels, setups, c, L):
    o = Oracle(levels)
    xs, resid, ost, rc = o.solve_outer([s.x0 for s in setups], [s.b for s in setups], c)
    acc = o.update_master_slave(L - 2, key_noise([lv[L - 2] for lv in levels], 3), 1)
    return xs, resid, ost, acc


CASES = [(2, 4, "coarse", False), (4, 4, "bottom", False), (8, 3, "coarse", False),
         (4, 4, "bottom", True), (8, 4, "bottom", True), (3, 3, "coarse", True)]


@pytest.mark.parametrize("K,L,rep,fused", CASES, ids=lambda v: str(v))
@pytest.mark.parametrize("kind", [gmg.PF_SMOOTHER_JACOBI, gmg.PF_SMOOTHER_MULTICOLOR_SOR], ids=["jacobi", "sor"])
def test_peer_threads_captured(cuda, K, L, rep, fused, kind):
    """K hierarchies on K threads exchange through the peer transport; solve_outer takes the
    captured outer-cycle graph (exchange kernels, the overlap's fork/join and the
    replicated bottom inside it) and must equal the oracle bit for bit, twice in a row."""
    setups, levels = structured(3, 2, L, K, direct_halos=fused)
    c = cfg(kind, damping=1.2 if kind == gmg.PF_SMOOTHER_MULTICOLOR_SOR else 0.8)
    replicas = [s[0] for s in levels] if rep == "coarse" else [s[:L - 1] for s in levels]
    blobs = [None] * K

    def body(r, bar):
        h = gmg.Hierarchy([levels[r]], rank_base=r, world_size=K, coarse_replicas=replicas, fused_exchanges=fused)
        blobs[r] = h.peer_export()
        bar.wait()
        h.init_peer(blobs)
        x = h.vector(L - 1)
        b = h.vector(L - 1, setups[r].b)
        v = h.vector(L - 2, key_noise([levels[r][L - 2]], 3)[0])
        # ranks sharing a device: every allocation (a device-synchronising call) is done
        # before any rank parks a kernel waiting for a peer
        bar.wait()
        sols = []
        for _ in range(2):
            x.upload(setups[r].x0)
            st = gmg.solve_outer(h, x, b, c)
            sols.append(x.download())
        rn = gmg.residual_norm(h, L - 1, x, b)
        gmg.update_master_slave(h, L - 2, v, gmg.PF_UPDATE_ACCUMULATE_THEN_SCATTER)
        bar.wait()  # no rank tears its arena down while a peer may still store into it
        return st, sols, rn, v.download(), h.graph_count()

    res = _threads(K, body)
    xs, resid, ost, acc = _oracle(levels, setups, c, L)
    for r in range(K):
        st, sols, rn, v, graphs = res[r]
        assert graphs >= 1, "the multi-process solve must run from a captured graph"
        assert st.iterations == ost.iterations
        np.testing.assert_allclose(st.residuals, resid, rtol=1e-12)
        assert np.array_equal(sols[0], xs[r]), f"rank {r}"
        assert np.array_equal(sols[1], xs[r]), f"rank {r} (graph replay)"
        assert np.array_equal(v, acc[r]), f"accumulate rank {r}"
        assert rn == res[0][2]


@pytest.mark.parametrize("K,L,rep,fused,kind", [(2, 4, "coarse", False, 0), (2, 4, "bottom", True, 0),
                                                (4, 4, "bottom", True, 2), (4, 3, "coarse", False, 2)],
                         ids=lambda v: str(v))
def test_peer_processes_ipc(cuda, tmp_path, K, L, rep, fused, kind):
    """K processes on cuda:0, each one rank (tests/peer_rank.py), arenas mapped with CUDA
    IPC: the captured multi-process solve equals the oracle's K-rank solve bit for bit."""
    d = str(tmp_path)
    cmd = [sys.executable, os.path.join(HERE, "peer_rank.py"), "--dir", d, "--world", str(K), "--levels", str(L),
           "--kind", str(kind), "--rep", rep] + (["--fused"] if fused else [])
    env = dict(os.environ, PF_WATCHDOG_S="60")
    procs = [subprocess.Popen(cmd + ["--rank", str(r)], env=env, stdout=subprocess.PIPE, stderr=subprocess.STDOUT)
             for r in range(K)]
    outs = []
    for p in procs:
        try:
            out, _ = p.communicate(timeout=240)
        except subprocess.TimeoutExpired:
            for q in procs:
                q.kill()
            raise
        outs.append(out.decode(errors="replace"))
    for r, p in enumerate(procs):
        assert p.returncode == 0, f"rank {r} failed:\n{outs[r][-3000:]}"
    setups, levels = structured(3, 2, L, K, direct_halos=fused)
    c = cfg(kind, damping=1.2 if kind == gmg.PF_SMOOTHER_MULTICOLOR_SOR else 0.8)
    xs, resid, ost, acc = _oracle(levels, setups, c, L)
    rn0 = None
    for r in range(K):
        z = np.load(os.path.join(d, f"result_{r}.npz"))
        assert int(z["graphs"]) >= 1
        assert int(z["iterations"]) == ost.iterations
        np.testing.assert_allclose(z["residuals"], resid, rtol=1e-12)
        assert np.array_equal(z["x"], xs[r]), f"rank {r}"
        assert np.array_equal(z["x_again"], xs[r]), f"rank {r} (graph replay)"
        assert np.array_equal(z["acc"], acc[r]), f"accumulate rank {r}"
        rn0 = float(z["rn"]) if rn0 is None else rn0
        assert float(z["rn"]) == rn0


def test_peer_watchdog_raises_transport_error(cuda, monkeypatch):
    """A rank that never reaches the exchange: the waiting kernels give up after
    PF_WATCHDOG_S and the solve raises TransportError (transport.cpp:54-60) instead of
    hanging the device."""
    monkeypatch.setenv("PF_WATCHDOG_S", "2")
    K, L = 2, 3
    setups, levels = structured(3, 2, L, K)
    replicas = [s[0] for s in levels]
    blobs = [None] * K

    def body(r, bar):
        h = gmg.Hierarchy([levels[r]], rank_base=r, world_size=K, coarse_replicas=replicas)
        blobs[r] = h.peer_export()
        bar.wait()
        h.init_peer(blobs)
        x = h.vector(L - 1, setups[r].x0)
        b = h.vector(L - 1, setups[r].b)
        bar.wait()
        if r == 1:
            bar.wait()  # rank 1 never solves
            return None
        try:
            with pytest.raises(_lib.TransportError, match="watchdog"):
                gmg.solve_outer(h, x, b, cfg())
        finally:
            bar.wait()
        return True

    assert _threads(K, body)[0]


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
