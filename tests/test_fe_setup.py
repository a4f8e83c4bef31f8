"""CPU: the Q2 and rotated-Q1 hierarchies (include/pf_fe.h; BASELINE configs[2] and
configs[3]) against the numpy restatement oracle/fe_restated.py, plus the properties that
pin the discretisations themselves (the reference has neither family: parity unpinned by
the reference, pinned by restatement and by these properties)."""
import numpy as np
import pytest
import scipy.sparse as sp
import scipy.sparse.linalg as spl

from oracle import fe_restated as R
from paper_1609_04809_b200 import _lib
from paper_1609_04809_b200.fe import CONSTANT, LOGNORMAL, Q2, ROTATED_Q1, FESetup

CASES = [(Q2, CONSTANT, 1), (Q2, CONSTANT, 2), (Q2, CONSTANT, 3), (ROTATED_Q1, CONSTANT, 1),
         (ROTATED_Q1, CONSTANT, 3), (ROTATED_Q1, LOGNORMAL, 2), (ROTATED_Q1, LOGNORMAL, 3)]
IDS = ["%s_%s_L%d" % ("q2" if f == Q2 else "rt", "ln" if c else "k1", L) for f, c, L in CASES]


@pytest.mark.parametrize("family,coef,L", CASES, ids=IDS)
def test_setup_equals_restatement(family, coef, L):
    """Every level array equal to the restatement's: numbering, keys, classes, colours,
    the assembled operator (values bit for bit), the rhs and the exact-solution values;
    the prolongation pattern exactly, its weights to 1e-15 (rotated Q1: closed form vs
    2 x 2 Gauss means; Q2: exact)."""
    s = FESetup(family, 2, L, coef, seed=77)
    ref, b, x0, exact, kap = R.build(family, 2, L, coef == LOGNORMAL, seed=77)
    for l, (a, r) in enumerate(zip(s.levels, ref)):
        assert (a.n, a.n_own) == (r.n, r.n_own), l
        for name in ("row_offsets", "cols", "vals", "owns_row", "is_dir", "color", "keys", "class_of", "order"):
            assert np.array_equal(getattr(a, name), getattr(r, name)), (l, name)
        if l:
            assert np.array_equal(a.p_offsets, r.p_offsets) and np.array_equal(a.p_cols, r.p_cols), l
            np.testing.assert_allclose(a.p_w, r.p_w, rtol=0, atol=1e-15)
    assert np.array_equal(s.b, b) and np.array_equal(s.x0, x0) and np.array_equal(s.exact, exact)
    assert np.array_equal(s.kappa, kap)


def test_unit_stiffness_matches_exact_rationals():
    """The quadrature element matrices equal the exact integrals (fractions) to 4 ulps:
    rows sum to zero (constants in the kernel), symmetric, positive semi-definite."""
    from fractions import Fraction as Fr
    # rotated Q1 on [0,1]^3: d/dt of (1/6 + s X_o/2 + (2X_o^2 - X_p^2 - X_q^2)/4), X = 2t - 1
    # integrate the products exactly: int X dt = 0, int X^2 dt = 1/3
    def rt_exact(a, b):
        oa, sa, ob, sb = a // 2, (1 if a & 1 else -1), b // 2, (1 if b & 1 else -1)
        tot = Fr(0)
        for ax in range(3):
            # gradient component = c0 + c1 X_ax
            ca = (Fr(sa), Fr(2)) if ax == oa else (Fr(0), Fr(-1))
            cb = (Fr(sb), Fr(2)) if ax == ob else (Fr(0), Fr(-1))
            tot += ca[0] * cb[0] + ca[1] * cb[1] * Fr(1, 3)
        return tot
    K = R.rt_unit_stiffness()
    E = np.array([[float(rt_exact(a, b)) for b in range(6)] for a in range(6)])
    np.testing.assert_allclose(K, E, rtol=4e-16, atol=4e-16)
    for K in (R.rt_unit_stiffness(), R.q2_unit_stiffness()):
        assert np.abs(K - K.T).max() == 0.0
        assert np.abs(K.sum(1)).max() < 1e-14
        assert np.linalg.eigvalsh(K).min() > -1e-13


@pytest.mark.parametrize("family,order", [(Q2, 3.5), (ROTATED_Q1, 1.7)], ids=["q2", "rt"])
def test_discretisation_converges(family, order):
    """Direct solves of the finest system against sin(pi x) sin(pi y) sin(pi z): Q2 nodal
    error O(h^4) (superconvergent at the nodes), rotated-Q1 face means O(h^2)."""
    errs = []
    for L in (2, 3, 4):
        s = FESetup(family, 2, L)
        lv = s.levels[-1]
        A = sp.csr_matrix((lv.vals, lv.cols, lv.row_offsets), shape=(lv.n, lv.n)).tocsc()
        errs.append(np.abs(spl.spsolve(A, s.b) - s.exact).max())
    rates = np.log2(np.array(errs[:-1]) / np.array(errs[1:]))
    assert rates.min() > order, (errs, rates)


@pytest.mark.parametrize("family", [Q2, ROTATED_Q1], ids=["q2", "rt"])
def test_prolongation_properties(family):
    """Q2: partition of unity on every fine dof, and exact interpolation of quadratics.
    Rotated Q1: the coarse face means of a linear function prolongate to its fine face
    means on every own face; no entries onto Dirichlet faces."""
    s = FESetup(family, 2, 4)
    F, Cl = s.levels[-1], s.levels[-2]
    P = sp.csr_matrix((F.p_w, F.p_cols, F.p_offsets), shape=(F.n, Cl.n))
    if family == Q2:
        assert np.array_equal(P @ np.ones(Cl.n), np.ones(F.n))
        def quad(lv):
            x = lv.keys[:, 1:] / (2.0 * (2 << (lv is F and 3 or 2)))
            return x[:, 0] ** 2 - 3 * x[:, 1] * x[:, 2] + x[:, 2]
        np.testing.assert_allclose(P @ quad(Cl), quad(F), atol=1e-14)
    else:
        assert np.all(np.diff(F.p_offsets)[F.n_own:] == 0)
        def lin(lv, N):
            o, a = lv.keys[:, 0], lv.keys[:, 1:].astype(float)
            c = (a + 0.5) / N
            c[np.arange(lv.n), o] = a[np.arange(lv.n), o] / N  # face centroid
            return 1.0 + 2.0 * c[:, 0] - 3.0 * c[:, 1] + 0.5 * c[:, 2]
        got = P @ lin(Cl, 8)
        np.testing.assert_allclose(got[:F.n_own], lin(F, 16)[:F.n_own], atol=1e-14)


def test_bad_arguments_raise():
    with pytest.raises(_lib.InvalidArgument):
        FESetup(Q2, 2, 2, LOGNORMAL)
    with pytest.raises(_lib.InvalidArgument):
        FESetup(7, 2, 2)
    with pytest.raises(_lib.InvalidArgument):
        FESetup(ROTATED_Q1, 1, 2)


@pytest.mark.parametrize("family,coef", [(Q2, CONSTANT), (ROTATED_Q1, LOGNORMAL)], ids=["q2", "rt_lognormal"])
def test_partitioned_setup(family, coef):
    """Box partitions (1, 2, 3, 4, 8 ranks): the master/slave channels pair up (the i-th
    entries of r -> p and p <- r name the same entity), every entity has exactly one
    authoritative copy, and the partitioned solve (oracle, K subdomains) takes the same
    cycles as one subdomain, its solution equal by key to roundoff (the restricted partial
    sums are accumulated in another order)."""
    from helpers import cfg, keyed
    from oracle.restated import Oracle
    from paper_1609_04809_b200 import gmg
    ref = None
    pp = 3 if family == Q2 else 2
    for K in (1, 2, 3, 4, 8):
        S = [FESetup(family, 2, 3, coef, seed=5, n_ranks=K, rank=r) for r in range(K)]
        for l in range(3):
            lv = [s.levels[l] for s in S]
            auth = {}
            for r, a in enumerate(lv):
                for i in np.flatnonzero(a.owns_row):
                    k = tuple(a.keys[i])
                    assert k not in auth
                    auth[k] = r
            assert len(auth) == len({tuple(k) for a in lv for k in a.keys})
            for r, a in enumerate(lv):
                for c in a.channels:
                    back = [d for d in lv[c.peer].channels if d.peer == r][0]
                    assert np.array_equal(a.keys[c.send], lv[c.peer].keys[back.recv])
        o = Oracle([s.levels for s in S])
        x, res, st, rc = o.solve_outer([s.x0 for s in S], [s.b for s in S],
                                       cfg(gmg.PF_SMOOTHER_JACOBI, pre=pp, post=pp, max_cycles=300))
        assert rc == 0
        got = keyed([s.levels[-1] for s in S], x)
        if ref is None:
            ref, cycles = got, st.iterations
        assert st.iterations == cycles and got.keys() == ref.keys()
        scale = max(abs(v) for v in ref.values())
        assert max(abs(got[k] - ref[k]) for k in ref) <= 1e-13 * scale
