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
