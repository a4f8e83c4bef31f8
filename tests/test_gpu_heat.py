"""GPU parity of the Crank-Nicolson heat loop (SURVEY.md §8f rank 3, app.cpp:146-230).

Chain: the restated loop (oracle/restated.py::heat_loop) equals the reference's run_heat
bit for bit (tests/test_oracle.py); the product's heat setup equals the reference's level
data, rhs operator and loads bit for bit (tests/test_setup.py).  Here the device pieces —
load assembly (k_load + accumulate), the rhs operator, the fused CN right-hand side with
the Dirichlet rows, and the whole device-driven time loop — are checked against the
setup's host load, the oracle, and the reference's run_heat itself, all with ==.
"""
import numpy as np
import pytest

from helpers import cfg, keyed
from oracle.restated import csr_spmv, heat_exact
from paper_1609_04809_b200 import _lib, gmg
from paper_1609_04809_b200.heat import HeatRun, apply_dirichlet_rhs, assemble_load, cn_rhs, time_steps

pytestmark = pytest.mark.gpu

CASES = [(3, 2, 3, 1), (3, 2, 3, 2), (3, 2, 4, 4), (2, 3, 3, 3), (3, 2, 3, 8), (3, 3, 3, 5)]
IDS = ["d%d_nc%d_L%d_K%d" % c for c in CASES]


@pytest.mark.parametrize("dim,nc,L,K", CASES, ids=IDS)
def test_device_load_equals_host_and_reference(cuda, ref_lib, dim, nc, L, K):
    """assemble_load on the device == the setup's host load (every row) == the reference's
    assemble_load (every row it reads: all but Dirichlet), at t = dt and 2 dt."""
    dt = 0.02
    run = HeatRun(dim, nc, L, dt, n_ranks=K)
    R = ref_lib.build(dim, nc, L, K, 3, dt=dt, n_loads=2)
    v = run.h.vector()
    for k in range(2):
        t = (k + 1) * dt
        s, _, _ = run.setups[0].scales(t)
        assemble_load(run.load, s, v)
        for r in range(K):
            got = v.download(r)
            assert np.array_equal(got, run.setups[r].load_at(t)), (k, r)
            kb = {tuple(int(x) for x in key): i for i, key in enumerate(run.setups[r].levels[-1].keys)}
            top = R.ranks[r][-1]
            perm = np.array([kb[tuple(int(x) for x in key)] for key in top.keys])
            live = top.class_of != 7
            assert np.array_equal(got[perm][live], R.loads[r][k][live]), (k, r)
    run.close()


@pytest.mark.parametrize("dim,nc,L,K", CASES[:4], ids=IDS[:4])
def test_rhs_operator_and_cn_rhs_match_oracle(cuda, dim, nc, L, K):
    """Operator.apply == serial CSR spmv (linalg.cpp:45-57); cn_rhs == spmv + dt/2 (ln +
    lnx) with the Dirichlet rows of b and u from g(t) (app.cpp:191-200)."""
    dt = 0.05
    run = HeatRun(dim, nc, L, dt, n_ranks=K)
    rng = np.random.default_rng(7)
    top = [s.levels[-1] for s in run.setups]
    x = [rng.standard_normal(lv.n) for lv in top]
    ln = [rng.standard_normal(lv.n) for lv in top]
    lnx = [rng.standard_normal(lv.n) for lv in top]
    X, LN, LNX = run.h.vector(values=x), run.h.vector(values=ln), run.h.vector(values=lnx)
    Y, B = run.h.vector(), run.h.vector()
    run.op.apply(X, Y)
    want_y = [csr_spmv(lv.row_offsets, lv.cols, s.rhs_op, xi) for lv, s, xi in zip(top, run.setups, x)]
    assert all(np.array_equal(Y.download(r), want_y[r]) for r in range(K))
    t = 3 * dt
    _, has, g = run.setups[0].scales(t)
    U = run.h.vector(values=x)
    cn_rhs(run.op, run.load, X, LN, LNX, 0.5 * dt, has, g, B, U)
    denom = nc * 2 ** (L - 1)
    for r in range(K):
        want = want_y[r] + 0.5 * dt * (ln[r] + lnx[r])
        d = np.flatnonzero(top[r].is_dir)
        gd = heat_exact(top[r].keys[d], denom, dim, t)
        want[d] = gd
        assert np.array_equal(B.download(r), want), r
        u_want = x[r].copy()
        u_want[d] = gd
        assert np.array_equal(U.download(r), u_want), r
    # apply_dirichlet_rhs alone, no u
    B2 = run.h.vector(values=x)
    apply_dirichlet_rhs(run.load, has, g, B2)
    for r in range(K):
        want = x[r].copy()
        d = np.flatnonzero(top[r].is_dir)
        want[d] = heat_exact(top[r].keys[d], denom, dim, t)
        assert np.array_equal(B2.download(r), want)
    run.close()


@pytest.mark.parametrize("dim,nc,L,K", CASES, ids=IDS)
def test_heat_run_equals_reference_run_heat(cuda, ref_lib, dim, nc, L, K):
    """The whole device time loop (pf_heat_run) == the reference's run_heat: the solution
    per carrier key after the last step bit for bit, that step's residual history to the
    last ulp (norm summation order)."""
    dt, end = 0.02, 0.06
    steps = time_steps(end, dt)
    assert steps == 3
    run = HeatRun(dim, nc, L, dt, n_ranks=K)
    st = run.run(steps, cfg())
    rep = ref_lib.heat(dim, nc, L, K, dt=dt, end_time=end, smoother=0, pre=2, post=2, outer_tol=1e-10)
    # norms: device tree reduction vs the reference's sequential sum (last-ulp level)
    np.testing.assert_allclose(st.residuals, rep["residuals"], rtol=1e-13, atol=0)
    assert run.keyed() == rep["solution"]
    run.close()


def test_heat_steps_compose_and_reset(cuda):
    """run(3) == run(1) x 3 (the loop carries u and load_now); reset() restarts."""
    run = HeatRun(3, 2, 4, 0.01, n_ranks=2)
    run.run(3, cfg())
    a = run.solution()
    run.reset()
    for _ in range(3):
        run.run(1, cfg())
    b = run.solution()
    assert all(np.array_equal(x, y) for x, y in zip(a, b))
    run.close()


def test_heat_gauss_seidel_close_to_reference(cuda, ref_lib):
    """Gauss-Seidel: the device sweeps in colour order, the reference lexicographically
    (DESIGN.md "GS ordering"), so iterates differ; both converge to 1e-10, the solutions
    agree to that level."""
    dim, nc, L, K, dt = 3, 2, 4, 2, 0.02
    run = HeatRun(dim, nc, L, dt, n_ranks=K)
    st = run.run(3, cfg(kind=gmg.PF_SMOOTHER_GAUSS_SEIDEL))
    rep = ref_lib.heat(dim, nc, L, K, dt=dt, end_time=0.06, smoother=1, pre=2, post=2, outer_tol=1e-10)
    got = run.keyed()
    assert got.keys() == rep["solution"].keys()
    scale = max(abs(v) for v in rep["solution"].values())
    assert max(abs(got[k] - rep["solution"][k]) for k in got) <= 1e-8 * scale
    assert abs(st.iterations - len(rep["residuals"])) <= 1
    run.close()


def test_heat_no_convergence_names_the_step(cuda):
    """NoConvergenceError is rethrown with the step index (app.cpp:205-207)."""
    run = HeatRun(3, 2, 4, 0.01)
    run.run(1, cfg())
    with pytest.raises(_lib.NoConvergenceError, match="time step 2") as ei:
        run.run(2, cfg(tol=1e-300, max_cycles=2))
    assert ei.value.step == 2
    run.close()


@pytest.mark.slow
def test_heat_c2_error_against_exact_solution(cuda):
    """C2 (128^3, 7 levels, 2,146,689 dofs): a few CN steps on the device; every step
    converges and the nodal error against exp(-t/10) sin(pi x) cos(pi y) cos(pi z) stays at
    the O(h^2 + dt^2) discretisation level; the device load equals the host load."""
    dt = 0.01
    run = HeatRun(3, 2, 7, dt)
    s, _, _ = run.setups[0].scales(dt)
    v = run.h.vector()
    assemble_load(run.load, s, v)
    assert np.array_equal(v.download(0), run.setups[0].load_at(dt))
    st = run.run(3, cfg())
    assert st.converged and st.iterations <= 12
    top = run.setups[0].levels[-1]
    u = run.u.download(0)
    ex = heat_exact(top.keys, 128, 3, 3 * dt)
    assert np.abs(u - ex).max() < 2e-4
    run.close()
