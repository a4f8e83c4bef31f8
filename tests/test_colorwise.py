"""Colour-wise exchange of the coloured smoothers (pf_hierarchy_set_colorwise_exchange,
restated as orc_set_colorwise): the oracle side (CPU).

The reference's smooth() (solvers.cpp:56-68) sweeps each subdomain's own rows and only
then refreshes the slave / halo copies, so a K-subdomain Gauss-Seidel / SOR sweep is
Jacobi-like across subdomain boundaries.  On the rotated-Q1 lognormal operator of BASELINE
configs[3] over-relaxed SOR then diverges at K = 8.  Exchanging after every colour makes the
partitioned sweep relax like the single-domain coloured sweep: the same cycle count as
K = 1 for any K.  (tests/test_gpu_colorwise.py checks the device against this oracle bit
for bit.)"""
import numpy as np
import pytest

from helpers import cfg
from oracle.restated import Oracle
from paper_1609_04809_b200 import _lib, gmg
from paper_1609_04809_b200.fe import LOGNORMAL, ROTATED_Q1, FESetup
from paper_1609_04809_b200.levels import StructuredSetup


def _solve(levels, setups, c, colorwise):
    return Oracle(levels, colorwise=colorwise).solve_outer([s.x0 for s in setups], [s.b for s in setups], c)


def test_rotated_q1_lognormal_sor_k8_converges_colorwise():
    """configs[3]'s element and coefficient at 32^3 cells, SOR w = 1.2: processor-local
    smoothing diverges at K = 8; colour-wise converges in the K = 1 cycle count."""
    c = cfg(gmg.PF_SMOOTHER_MULTICOLOR_SOR, damping=1.2, max_cycles=300)
    one = [FESetup(ROTATED_Q1, 2, 5, LOGNORMAL, seed=2024)]
    _, _, st1, rc1 = _solve([s.levels for s in one], one, c, False)
    assert rc1 == 0
    eight = [FESetup(ROTATED_Q1, 2, 5, LOGNORMAL, seed=2024, n_ranks=8, rank=r) for r in range(8)]
    lv = [s.levels for s in eight]
    _, res_l, st_l, rc_l = _solve(lv, eight, c, False)
    assert rc_l == 3 or st_l.final_residual > st_l.initial_residual  # processor-local: diverges
    _, res_c, st_c, rc_c = _solve(lv, eight, c, True)
    assert rc_c == 0 and st_c.iterations == st1.iterations
    assert st_c.final_residual <= 1e-10 * st_c.initial_residual


@pytest.mark.parametrize("K", [2, 4, 8])
def test_q1_lognormal_colorwise_matches_single_domain_cycles(K):
    """Q1 with the lognormal coefficient, SOR w = 1.2: colour-wise K-subdomain smoothing takes
    the single-domain cycle count (processor-local needs more), and the residual histories
    agree to roundoff (the subdomains sum each row in their own local order)."""
    c = cfg(gmg.PF_SMOOTHER_MULTICOLOR_SOR, damping=1.2, max_cycles=100)
    one = [StructuredSetup(3, 2, 5, 1, 0, _lib.PF_PROBLEM_LOGNORMAL, seed=7)]
    _, res1, st1, _ = _solve([s.levels for s in one], one, c, False)
    ss = [StructuredSetup(3, 2, 5, K, r, _lib.PF_PROBLEM_LOGNORMAL, seed=7) for r in range(K)]
    lv = [s.levels for s in ss]
    _, res_l, st_l, _ = _solve(lv, ss, c, False)
    _, res_c, st_c, rc = _solve(lv, ss, c, True)
    assert rc == 0 and st_c.iterations == st1.iterations < st_l.iterations
    np.testing.assert_allclose(res_c, res1, rtol=1e-6, atol=1e-14 * st1.initial_residual)


def test_colorwise_is_inert_for_jacobi_and_one_subdomain():
    """Damped Jacobi ignores the mode; one subdomain has no copies to refresh."""
    ss = [StructuredSetup(3, 2, 4, 2, r) for r in range(2)]
    lv = [s.levels for s in ss]
    c = cfg(gmg.PF_SMOOTHER_JACOBI)
    xa, ra, sa, _ = _solve(lv, ss, c, False)
    xb, rb, sb, _ = _solve(lv, ss, c, True)
    assert sa.iterations == sb.iterations and all(np.array_equal(a, b) for a, b in zip(xa, xb))
    one = [StructuredSetup(3, 2, 4, 1, 0)]
    c = cfg(gmg.PF_SMOOTHER_MULTICOLOR_SOR, damping=1.2)
    xa, _, _, _ = _solve([s.levels for s in one], one, c, False)
    xb, _, _, _ = _solve([s.levels for s in one], one, c, True)
    assert np.array_equal(xa[0], xb[0])
