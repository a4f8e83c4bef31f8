"""GPU: the reference's own hot-path property tests, restated against the
device implementation.  Each test cites the reference test it mirrors
(/root/reference/proj/tests/...).  Data: the product setup, K subdomains on one device
(the single-GPU stand-in for K ranks, exchanges as device copies)."""
import numpy as np
import pytest

from helpers import cfg, download, key_noise, keyed, structured, upload
from paper_1609_04809_b200 import _lib, gmg
from paper_1609_04809_b200.levels import StructuredSetup, export_matrixmarket

pytestmark = pytest.mark.gpu

HALO2, DIRICHLET = 6, 7


@pytest.mark.parametrize("K", [1, 2, 4, 8])
@pytest.mark.parametrize("kind", [gmg.PF_SMOOTHER_JACOBI, gmg.PF_SMOOTHER_GAUSS_SEIDEL], ids=["jacobi", "gs"])
def test_smooth_never_writes_halo2_or_dirichlet(cuda, K, kind):
    """test_solvers.cpp:140-180: a smooth() (sweeps + master/slave + halo1 updates) leaves
    the Halo2 and Dirichlet entries untouched."""
    setups, levels = structured(3, 2, 4, K)
    h = gmg.Hierarchy(levels)
    top = h.finest
    x0 = key_noise([lv[top] for lv in levels], 11)
    x = upload(h, top, x0)
    b = upload(h, top, key_noise([lv[top] for lv in levels], 12))
    gmg.smooth(h, top, x, b, gmg.SmootherConfig(kind=kind, sweeps=2, damping=0.8))
    for r, xr in enumerate(download(h, x, K)):
        cls = levels[r][top].class_of
        keep = (cls == HALO2) | (cls == DIRICHLET)
        assert np.array_equal(xr[keep], x0[r][keep])
        own = np.arange(levels[r][top].n) < levels[r][top].n_own
        assert not np.array_equal(xr[own], x0[r][own])


@pytest.mark.parametrize("K", [1, 2, 4, 8])
def test_prolongation_restriction_adjoint(cuda, K):
    """test_multigrid.cpp:113-142 (acceptance criterion 6): <R r, xc> = <r, P xc> over the
    authoritative rows to 1e-12 relative."""
    setups, levels = structured(3, 2, 4, K)
    h = gmg.Hierarchy(levels)
    f, c = h.finest, h.finest - 1
    r_h = key_noise([lv[f] for lv in levels], 21)
    xc_h = key_noise([lv[c] for lv in levels], 22)
    # consistent coarse vector: every copy of a carrier holds the same value (key_noise)
    xc = upload(h, c, xc_h)
    r = upload(h, f, r_h)
    rc, px = h.vector(c), h.vector(f)
    gmg.restrict_residual(h, f, r, rc)
    gmg.prolongate(h, f, xc, px)
    lhs = sum(float(np.dot(rcr[lv[c].owns_row.astype(bool)], xc_h[s][lv[c].owns_row.astype(bool)]))
              for s, (rcr, lv) in enumerate(zip(download(h, rc, K), levels)))
    rhs = sum(float(np.dot(r_h[s][lv[f].owns_row.astype(bool)], pxr[lv[f].owns_row.astype(bool)]))
              for s, (pxr, lv) in enumerate(zip(download(h, px, K), levels)))
    assert abs(lhs - rhs) <= 1e-12 * max(abs(lhs), 1.0)


def test_partition_of_unity_and_constants(cuda):
    """test_multigrid.cpp:58-86: prolongating the constant 1 gives 1 on every fine dof."""
    setups, levels = structured(3, 2, 4, 2)
    h = gmg.Hierarchy(levels)
    f = h.finest
    one = h.vector(f - 1).fill(1.0)
    out = h.vector(f)
    gmg.prolongate(h, f, one, out)
    assert all(np.array_equal(o, np.ones_like(o)) for o in download(h, out, 2))


def test_exact_solution_is_a_fixed_point(cuda):
    """test_multigrid.cpp:144-162: a V-cycle started at the converged solution changes it by
    at most 1e-12 relative."""
    setups, levels = structured(3, 2, 5, 1)
    h = gmg.Hierarchy(levels)
    x = upload(h, 4, [s.x0 for s in setups])
    b = upload(h, 4, [s.b for s in setups])
    gmg.solve_outer(h, x, b, cfg(tol=1e-13, max_cycles=60))  # the roundoff floor is ~1.4e-14
    before = download(h, x, 1)[0]
    gmg.v_cycle(h, x, b, cfg())
    after = download(h, x, 1)[0]
    assert np.abs(after - before).max() <= 1e-12 * np.abs(before).max()


@pytest.mark.parametrize("K", [1, 2])
def test_cycle_count_and_contraction(cuda, K):
    """test_multigrid.cpp:176-216 (acceptance criterion 3): at most 12 cycles, a monotonically
    decreasing residual, contraction <= 0.2 per cycle, identical on every rank."""
    setups, levels = structured(3, 2, 5, K)
    h = gmg.Hierarchy(levels)
    st = gmg.solve_outer(h, upload(h, 4, [s.x0 for s in setups]), upload(h, 4, [s.b for s in setups]), cfg())
    res = np.array([st.initial_residual] + list(st.residuals))
    assert st.converged and st.iterations <= 12
    assert np.all(np.diff(res) < 0)
    assert (res[1:] / res[:-1]).max() <= 0.2


def test_rank_counts_agree(cuda):
    """test_multigrid.cpp:218-250: K = 1, 2, 4 give the same solution per key to 1e-8 (here:
    bit-identical, the damped Jacobi iterate does not depend on the partition)."""
    sols = []
    for K in (1, 2, 4):
        setups, levels = structured(3, 2, 4, K)
        h = gmg.Hierarchy(levels)
        x = upload(h, 3, [s.x0 for s in setups])
        gmg.solve_outer(h, x, upload(h, 3, [s.b for s in setups]), cfg())
        sols.append(keyed([lv[3] for lv in levels], download(h, x, K)))
    ref = sols[0]
    for s in sols[1:]:
        assert s.keys() == ref.keys()
        assert max(abs(s[k] - ref[k]) for k in ref) <= 1e-8 * max(abs(v) for v in ref.values())


@pytest.mark.parametrize("K", [2, 4, 8])
def test_exchanges_make_every_copy_consistent_and_are_idempotent(cuda, K):
    """test_fecomm.cpp:135-146, :219-256: after update_master_slave(Scatter) + halo1 + halo2
    every local copy of a carrier holds its owner's value; repeating changes no bit."""
    setups, levels = structured(3, 2, 4, K)
    h = gmg.Hierarchy(levels)
    f = h.finest
    rng = np.random.default_rng(5)
    v0 = [rng.standard_normal(lv[f].n) for lv in levels]
    v = upload(h, f, v0)
    for _ in range(2):
        gmg.update_master_slave(h, f, v, gmg.PF_UPDATE_SCATTER)
        gmg.update_halo1(h, f, v)
        gmg.update_halo2(h, f, v)
        got = download(h, v, K)
        if _ == 0:
            first = [g.copy() for g in got]
    assert all(np.array_equal(a, b) for a, b in zip(first, got))
    owner_val = {}
    for lv, g in zip(levels, got):
        for i in np.flatnonzero(lv[f].owns_row):
            owner_val[tuple(lv[f].keys[i])] = g[i]
    for lv, g in zip(levels, got):
        cls = lv[f].class_of
        for i in range(lv[f].n):
            if cls[i] == DIRICHLET:
                continue  # Dirichlet copies are not exchanged (their values never change)
            assert g[i] == owner_val[tuple(lv[f].keys[i])]


def test_reruns_are_bit_identical(cuda):
    """Acceptance criterion 10: the same solve run twice gives identical bits."""
    setups, levels = structured(3, 2, 5, 4)
    outs = []
    for _ in range(2):
        h = gmg.Hierarchy(levels)
        x = upload(h, 4, [s.x0 for s in setups])
        st = gmg.solve_outer(h, x, upload(h, 4, [s.b for s in setups]), cfg(kind=gmg.PF_SMOOTHER_MULTICOLOR_SOR, damping=1.2))
        outs.append((download(h, x, 4), list(st.residuals)))
    assert outs[0][1] == outs[1][1]
    assert all(np.array_equal(a, b) for a, b in zip(outs[0][0], outs[1][0]))


def test_export_against_multigrid(cuda, tmp_path):
    """Acceptance criterion 8: the exported system (729 DOFs) solved densely matches the
    multigrid solution to 1e-8."""
    K = 2
    S = [StructuredSetup(3, 2, 3, K, r, _lib.PF_PROBLEM_REFERENCE_POISSON, keep=True) for r in range(K)]
    n, nnz = export_matrixmarket(S, str(tmp_path / "a.mtx"), str(tmp_path / "a_rhs.mtx"))
    assert n == 729
    A = np.zeros((n, n))
    for line in (tmp_path / "a.mtx").read_text().splitlines()[2:]:
        r, c, v = line.split()
        A[int(r) - 1, int(c) - 1] = float(v)
    b = np.array([float(t) for t in (tmp_path / "a_rhs.mtx").read_text().splitlines()[2:]])
    dense = np.linalg.solve(A, b)
    h = gmg.Hierarchy([s.levels for s in S])
    x = upload(h, 2, [s.x0 for s in S])
    gmg.solve_outer(h, x, upload(h, 2, [s.b for s in S]), cfg(tol=1e-13, max_cycles=60))
    # global numbering of the export: own rows rank by rank, then the owned Dirichlet rows
    sol = download(h, x, K)
    own = np.concatenate([sol[r][:S[r].levels[-1].n_own] for r in range(K)])
    assert np.abs(own - dense[:len(own)]).max() <= 1e-8 * np.abs(dense).max()
    for s in S:
        s.close()


@pytest.mark.parametrize("K", [1, 2])
def test_single_level_hierarchy_is_the_coarse_solve(cuda, K):
    """multigrid.cpp:150-158: on a one-level hierarchy a V-cycle is coarse_solve; the
    device and the oracle agree bit for bit (Q1 with 4^3 coarse cells: 27 unknowns per
    subdomain pair), and so do the element families (one subdomain)."""
    from oracle.restated import Oracle
    from paper_1609_04809_b200.fe import CONSTANT, LOGNORMAL, Q2, ROTATED_Q1, FESetup
    cases = [[StructuredSetup(3, 4, 1, K, r) for r in range(K)]]
    if K == 1:
        cases += [[FESetup(Q2, 3, 1)], [FESetup(ROTATED_Q1, 3, 1, LOGNORMAL, seed=2)]]
    for setups in cases:
        levels = [s.levels for s in setups]
        h = gmg.Hierarchy(levels)
        x = upload(h, 0, [s.x0 for s in setups])
        c = cfg(tol=1e-12, max_cycles=5)
        st = gmg.solve_outer(h, x, upload(h, 0, [s.b for s in setups]), c)
        xo, res, ost, rc = Oracle(levels).solve_outer([s.x0 for s in setups], [s.b for s in setups], c)
        assert rc == 0 and st.converged and st.iterations == ost.iterations
        assert all(np.array_equal(a, b) for a, b in zip(download(h, x, K), xo))


def test_ragged_subdomains(cuda):
    """K = 3, 5, 6, 7 (boxes of unequal size, partition.cpp:51-63): device == oracle."""
    from oracle.restated import Oracle
    for K in (3, 5, 6, 7):
        setups, levels = structured(3, 2, 4, K)
        h = gmg.Hierarchy(levels)
        x = upload(h, 3, [s.x0 for s in setups])
        st = gmg.solve_outer(h, x, upload(h, 3, [s.b for s in setups]), cfg())
        xo, res, ost, rc = Oracle(levels).solve_outer([s.x0 for s in setups], [s.b for s in setups], cfg())
        assert st.iterations == ost.iterations, K
        assert all(np.array_equal(a, b) for a, b in zip(download(h, x, K), xo)), K
