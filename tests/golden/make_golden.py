"""Generate tests/golden/*.npz from the UNMODIFIED reference (oracle/_ref, built from
/root/reference/proj by oracle/Makefile).  Run in the CPU container, where the reference
sources exist:

    python tests/golden/make_golden.py

The fixtures are what the reference itself computes for the BASELINE inputs (f = 3 pi^2
sin sin sin, g = 0, V(2,2), tol 1e-10) and for its own PoissonProblem; the CPU tests pin
the C restatement (oracle/gmg_oracle.c) and the product's setup to them, the GPU tests
pin libpf_gpu.so to them.  Keyed values are indexed by the reference's Key4 (entity kind,
lattice key) so they do not depend on any rank-local numbering.
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from oracle import ref  # noqa: E402


def keyed_solution(R, xs):
    keys, vals = [], []
    for r in range(R.K):
        lv = R.ranks[r][-1]
        own = np.flatnonzero(lv.owns_row)
        keys.append(lv.keys[own])
        vals.append(xs[r][own])
    keys = np.concatenate(keys)
    vals = np.concatenate(vals)
    order = np.lexsort(keys.T[::-1])
    return keys[order], vals[order]


def structure(R):
    """Per rank and level: class counts, n_own, nnz, channel (kind, peer, n_send, n_recv)."""
    rows = []
    for r in range(R.K):
        for l, lv in enumerate(R.ranks[r]):
            counts = np.bincount(lv.class_of, minlength=8)
            rows.append([r, l, lv.n_dofs, lv.n_own, int(lv.row_offsets[-1])] + counts.tolist())
    chans = []
    for r in range(R.K):
        for l, lv in enumerate(R.ranks[r]):
            for c in lv.channels:
                chans.append([r, l, c.kind, c.peer, len(c.send), len(c.recv)])
    return np.array(rows, np.int64), np.array(chans, np.int64).reshape(-1, 6)


def solve_case(name, dim, nc, levels, K, smoother, problem=0, keep_solution=True):
    R = ref.build(dim, nc, levels, K, problem)
    sizes = [R.ranks[r][-1].n_dofs for r in range(K)]
    xs, res, st = ref.run(dim, nc, levels, K, problem=problem, smoother=smoother, pre=2, post=2,
                          outer_tol=1e-10, sizes=sizes)
    assert st["status"] == 0, st
    keys, vals = keyed_solution(R, xs)
    srows, schans = structure(R)
    out = dict(dim=dim, n_coarse=nc, levels=levels, K=K, smoother=smoother, problem=problem,
               residuals=res, initial_residual=st["initial_residual"], iterations=st["iterations"],
               n_global=R.ranks[0][-1].n_global, structure=srows, channels=schans,
               solution_sum=float(vals.sum()), solution_l2=float(np.sqrt((vals ** 2).sum())))
    if keep_solution:
        out.update(keys=keys, values=vals)
    else:  # a deterministic sample of 512 carriers keeps big fixtures small
        idx = np.linspace(0, len(vals) - 1, 512).astype(np.int64)
        out.update(keys=keys[idx], values=vals[idx])
    np.savez_compressed(os.path.join(HERE, name + ".npz"), **out)
    print(f"{name}: {st['iterations']} cycles, r0 {st['initial_residual']:.6e}, "
          f"final {res[-1]:.6e}, solve {st['solve_seconds']:.2f}s")


def digest_case(name, dim, nc, levels, K, smoother):
    """A whole solution pinned by a digest: sha256 of the keyed values in key order (the
    GPU recomputes it from its own solution), plus the residual history and a sample."""
    import hashlib
    R = ref.build(dim, nc, levels, K, 0)
    sizes = [R.ranks[r][-1].n_dofs for r in range(K)]
    xs, res, st = ref.run(dim, nc, levels, K, smoother=smoother, pre=2, post=2, outer_tol=1e-10, sizes=sizes)
    assert st["status"] == 0, st
    keys, vals = keyed_solution(R, xs)
    idx = np.linspace(0, len(vals) - 1, 512).astype(np.int64)
    np.savez_compressed(os.path.join(HERE, name + ".npz"), dim=dim, n_coarse=nc, levels=levels, K=K,
                        smoother=smoother, residuals=res, initial_residual=st["initial_residual"],
                        iterations=st["iterations"], n_carriers=len(vals),
                        digest=hashlib.sha256(np.ascontiguousarray(vals, np.float64).tobytes()).hexdigest(),
                        keys=keys[idx], values=vals[idx])
    print(f"{name}: {st['iterations']} cycles, {len(vals)} carriers, solve {st['solve_seconds']:.2f}s")


def sweep_case(name, dim, nc, levels, K, smoother, n_ops):
    """Iterates of `n_ops` single smooth() calls from x0 (per-sweep parity)."""
    R = ref.build(dim, nc, levels, K, 0)
    sizes = [R.ranks[r][-1].n_dofs for r in range(K)]
    xs, _, st = ref.run(dim, nc, levels, K, op=ref.OP_SMOOTH, n_ops=n_ops, smoother=smoother,
                        sizes=sizes)
    keys, vals = keyed_solution(R, xs)
    np.savez_compressed(os.path.join(HERE, name + ".npz"), dim=dim, n_coarse=nc, levels=levels, K=K,
                        smoother=smoother, n_ops=n_ops, keys=keys, values=vals)
    print(f"{name}: {len(vals)} carriers")


def small_cases():
    # C1 (32^3, 5 levels): BASELINE configs[0], Jacobi and the reference GS, 1 and 8 ranks
    solve_case("c1_jacobi_k1", 3, 2, 5, 1, 0)
    solve_case("c1_jacobi_k8", 3, 2, 5, 8, 0)
    solve_case("c1_gs_k1", 3, 2, 5, 1, 1)
    # small multi-rank cases with full keyed solutions
    solve_case("q1_3d_l3_k4_jacobi", 3, 2, 3, 4, 0)
    solve_case("q1_2d_l4_k3_gs_refpoisson", 2, 2, 4, 3, 1, problem=1)
    solve_case("q1_2d_nc4_l3_k6_jacobi_refpoisson", 2, 4, 3, 6, 0, problem=1)
    # per-sweep iterates
    sweep_case("sweeps_3d_l4_k2_jacobi", 3, 2, 4, 2, 0, 3)
    sweep_case("sweeps_3d_l4_k1_gs", 3, 2, 4, 1, 1, 2)


if __name__ == "__main__":
    if "--only-c2-digest" not in sys.argv:
        small_cases()
    # C2 (128^3, 7 levels) residual history on 8 reference ranks (SURVEY: 9 cycles)
    if "--c2" in sys.argv:
        solve_case("c2_jacobi_k8", 3, 2, 7, 8, 0, keep_solution=False)
        solve_case("c2_gs_k8", 3, 2, 7, 8, 1, keep_solution=False)
    # C2 whole-solution digests (1 and 8 reference ranks): the bench configuration pinned bit
    # for bit (--c2-digest / --only-c2-digest)
    if "--c2-digest" in sys.argv or "--only-c2-digest" in sys.argv:
        digest_case("c2_jacobi_k1_digest", 3, 2, 7, 1, 0)
        digest_case("c2_jacobi_k8_digest", 3, 2, 7, 8, 0)
