"""CPU, world_size 2 (gloo): the N>1 host path across real processes (Q1, and the Q2 /
rotated-Q1 box partitions of pf_fe.h).

Each process plays one rank exactly as a GPU rank of `bench.py --gpus 2` does: it builds
only its own subdomain with the product's communication-free setup, then
  1. checks channel symmetry across processes (the i-th send carrier of r->p is the i-th
     recv carrier of p<-r, femapper.hpp:38-41) by exchanging carrier keys;
  2. runs one damped-Jacobi smooth() step with the ParFECommunicator exchanges (MS
     scatter then Halo1, solvers.cpp:62-67) moved over gloo send/recv, in the reference's
     expression order, and compares its rows with the single-process oracle's 2-rank
     sweep bit for bit;
  3. reduces the residual norm with an allgather + ascending-rank sum
     (transport.cpp:139-149) and compares with the oracle.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _jacobi_rows(lv, x, b, omega):
    """one_local_sweep Jacobi branch (solvers.cpp:35-51), rows in host order."""
    out = x.copy()
    for r in range(lv.n_own):
        acc, diag = b[r], 0.0
        for k in range(lv.row_offsets[r], lv.row_offsets[r + 1]):
            c = lv.cols[k]
            if c == r:
                diag = lv.vals[k]
            else:
                acc -= lv.vals[k] * x[c]
        out[r] = (1.0 - omega) * x[r] + omega * acc / diag
    return out


def _exchange(lv, v, kind, rank):
    """ParFECommunicator::scatter (fecomm.cpp:25-39) over gloo p2p."""
    reqs, bufs = [], []
    for c in lv.channels:
        if c.kind == kind and len(c.send):
            t = torch.from_numpy(v[c.send].copy())
            bufs.append(t)
            reqs.append(dist.isend(t, c.peer))
    for c in lv.channels:
        if c.kind == kind and len(c.recv):
            t = torch.empty(len(c.recv), dtype=torch.float64)
            dist.recv(t, c.peer)
            v[c.recv] = t.numpy()
    for q in reqs:
        q.wait()


def _setup(family, world, rank):
    """q1: the reference's Q1 hierarchy (pf_setup.h); q2 / rt: the element families of
    pf_fe.h, box-partitioned the same way."""
    if family == "q1":
        from paper_1609_04809_b200.levels import StructuredSetup
        return StructuredSetup(3, 2, 4, world, rank)
    from paper_1609_04809_b200.fe import LOGNORMAL, Q2, ROTATED_Q1, CONSTANT, FESetup
    if family == "q2":
        return FESetup(Q2, 2, 2, CONSTANT, n_ranks=world, rank=rank)
    return FESetup(ROTATED_Q1, 2, 3, LOGNORMAL, seed=4, n_ranks=world, rank=rank)


def _worker(rank, world, port, out_dir, family):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    s = _setup(family, world, rank)
    top = s.levels[-1]
    # 1. channel symmetry by carrier key
    mine = {(c.kind, c.peer): ([tuple(top.keys[i]) for i in c.send],
                               [tuple(top.keys[i]) for i in c.recv]) for c in top.channels}
    allc = [None] * world
    dist.all_gather_object(allc, mine)
    for (kind, peer), (send, recv) in mine.items():
        theirs = allc[peer].get((kind, rank), ([], []))
        assert send == theirs[1] and recv == theirs[0], (kind, peer)
    # 2. one smooth() step: local sweep, MS scatter, Halo1 scatter
    x = _jacobi_rows(top, s.x0, s.b, 0.8)
    _exchange(top, x, 0, rank)
    _exchange(top, x, 1, rank)
    # 3. residual norm with the ascending-rank sum
    local = 0.0
    for r in range(top.n_own):
        acc = s.b[r]
        for k in range(top.row_offsets[r], top.row_offsets[r + 1]):
            acc -= top.vals[k] * x[top.cols[k]]
        local += acc * acc
    parts = [None] * world
    dist.all_gather_object(parts, local)
    total = 0.0
    for p in parts:
        total += p
    np.save(os.path.join(out_dir, f"x{rank}.npy"), x)
    np.save(os.path.join(out_dir, f"n{rank}.npy"), np.array([np.sqrt(total)]))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("family", ["q1", "q2", "rt"])
def test_two_process_sweep_matches_oracle(tmp_path, family):
    world = 2
    mp.start_processes(_worker, args=(world, _free_port(), str(tmp_path), family), nprocs=world,
                       join=True, start_method="spawn")
    from oracle.restated import Oracle
    from paper_1609_04809_b200 import gmg
    setups = [_setup(family, world, r) for r in range(world)]
    top = len(setups[0].levels) - 1
    o = Oracle([s.levels for s in setups])
    want = o.smooth(top, [s.x0 for s in setups], [s.b for s in setups], gmg.PF_SMOOTHER_JACOBI,
                    sweeps=1, damping=0.8)
    norm = o.residual_norm(top, want, [s.b for s in setups])
    for r in range(world):
        got = np.load(tmp_path / f"x{r}.npy")
        assert np.array_equal(got, want[r]), f"rank {r}"
        assert np.load(tmp_path / f"n{r}.npy")[0] == norm


class _FakeHierarchy:
    """Stands in for gmg.Hierarchy in attach_transport (no device here): records what the
    product's transport selection did."""

    def __init__(self, fail):
        self.fail, self.calls = fail, []

    def peer_export(self):
        self.calls.append("export")
        return b"blob-%d" % int(os.environ["RANK"])

    def init_peer(self, blobs):
        self.calls.append(("init_peer", tuple(blobs)))
        if self.fail:
            raise RuntimeError("cannot map peers")

    def drop_transport(self):
        self.calls.append("drop")

    def init_nccl(self, uid):
        self.calls.append(("nccl", len(uid)))


def _plumbing_worker(rank, world, port, out_dir):
    """The host side of bench.py --gpus 2 across real processes: replica levels gathered
    from their owners (gmg.gather_replica_levels) equal the locally rebuilt ones; the peer
    blobs allgather over torch.distributed and over a directory; a peer-mapping failure on
    one rank makes every rank fall back to NCCL together (bench.attach_transport)."""
    import sys
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, root)
    import bench
    from paper_1609_04809_b200 import _lib, gmg
    from paper_1609_04809_b200 import dist as pdist
    from paper_1609_04809_b200.levels import StructuredSetup

    def gather(obj):
        out = [None] * world
        dist.all_gather_object(out, obj)
        return out
    s = StructuredSetup(3, 2, 6, world, rank, _lib.PF_PROBLEM_LOGNORMAL, seed=3, direct_halos=True,
                        materialize=False)
    got = gmg.gather_replica_levels(s, gather)
    want = gmg.replica_levels(3, 2, 6, world, _lib.PF_PROBLEM_LOGNORMAL, direct_halos=True)
    # (replica_levels builds fewer levels per setup; the lognormal seed default is 1)
    want = [[StructuredSetup(3, 2, 6, world, q, _lib.PF_PROBLEM_LOGNORMAL, seed=3, direct_halos=True).levels[l]
             for l in range(len(want[q]))] for q in range(world)]
    assert len(got) == world and all(len(g) == len(w) for g, w in zip(got, want))
    for g_r, w_r in zip(got, want):
        for a, b in zip(g_r, w_r):
            assert a.n == b.n and np.array_equal(a.row_offsets, b.row_offsets)
            assert np.array_equal(a.cols, b.cols) and np.array_equal(a.vals, b.vals)
    blob = b"rank%d" % rank
    assert pdist.allgather_blobs_torch(blob) == [b"rank0", b"rank1"]
    assert pdist.allgather_blobs_dir(os.path.join(out_dir, "rdv"), rank, world, blob) == [b"rank0", b"rank1"]
    gmg.Hierarchy.nccl_unique_id = staticmethod(lambda: bytes(128))  # no NCCL bootstrap on CPU
    ok = _FakeHierarchy(fail=False)
    assert bench.attach_transport(ok, world, rank, "peer", dist) == "peer"
    assert ok.calls == ["export", ("init_peer", (b"blob-0", b"blob-1"))]
    bad = _FakeHierarchy(fail=rank == 1)
    used = bench.attach_transport(bad, world, rank, "peer", dist)
    assert used.startswith("nccl (peer transport failed on rank 1"), used
    assert bad.calls[-2:] == ["drop", ("nccl", 128)]
    np.save(os.path.join(out_dir, f"ok{rank}.npy"), np.array([1]))
    dist.barrier()
    dist.destroy_process_group()


def test_two_process_host_plumbing(tmp_path):
    """gloo, world size 2: the multi-process host path of the product (replica gathering,
    blob allgathers, the all-or-nothing transport fallback)."""
    world = 2
    mp.start_processes(_plumbing_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world,
                       join=True, start_method="spawn")
    for r in range(world):
        assert np.load(tmp_path / f"ok{r}.npy")[0] == 1
