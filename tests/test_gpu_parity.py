"""GPU parity: every hot-path operation of libpf_gpu.so against the C restatement (bit for
bit, same input bytes) and against the compiled reference itself.

The restatement (oracle/gmg_oracle.c) is pinned bit-exactly to the reference by
tests/test_oracle.py, so "GPU == oracle" on the reference's own level data means
"GPU == reference".  Jacobi iterates, coloured GS/SOR iterates, the cycle residual,
restriction (+ accumulate), prolongation, the exchanges and the coarse solve are
compared with ==; norms (device tree reduction vs sequential sum) within 1e-13.
"""
import numpy as np
import pytest

from helpers import cfg, download, key_noise, keyed, structured, upload
from oracle.restated import Oracle
from paper_1609_04809_b200 import _lib, gmg
from paper_1609_04809_b200.levels import StructuredSetup

pytestmark = pytest.mark.gpu

KINDS = [gmg.PF_SMOOTHER_JACOBI, gmg.PF_SMOOTHER_GAUSS_SEIDEL, gmg.PF_SMOOTHER_MULTICOLOR_SOR]
CASES = [(3, 2, 4, 1), (3, 2, 4, 2), (3, 2, 4, 4), (3, 2, 3, 8), (2, 4, 3, 6), (3, 2, 3, 3)]


def exact(a_list, b_list):
    return all(np.array_equal(a, b) for a, b in zip(a_list, b_list))


@pytest.fixture(scope="module", params=CASES, ids=lambda c: "d%d_nc%d_L%d_K%d" % c)
def system(request, cuda):
    dim, nc, L, K = request.param
    setups, levels = structured(dim, nc, L, K)
    h = gmg.Hierarchy(levels)
    o = Oracle(levels)
    return dict(h=h, o=o, levels=levels, setups=setups, K=K, L=L)


@pytest.mark.parametrize("kind", KINDS, ids=["jacobi", "gs", "sor"])
def test_smooth_bit_exact(system, kind):
    h, o, levels, K, L = system["h"], system["o"], system["levels"], system["K"], system["L"]
    top = L - 1
    tl = [lv[top] for lv in levels]
    x0 = key_noise(tl, 11)
    b = key_noise(tl, 12)
    omega = 1.2 if kind == gmg.PF_SMOOTHER_MULTICOLOR_SOR else 0.8
    for sweeps in (1, 2, 3):
        x = upload(h, top, x0)
        bb = upload(h, top, b)
        gmg.smooth(h, top, x, bb, gmg.SmootherConfig(kind=kind, sweeps=sweeps, damping=omega))
        got = download(h, x, K)
        want = o.smooth(top, x0, b, kind, sweeps=sweeps, damping=omega)
        assert exact(got, want), f"sweeps={sweeps}"


def test_spmv_residual_transfers_bit_exact(system):
    h, o, levels, K, L = system["h"], system["o"], system["levels"], system["K"], system["L"]
    for l in range(L):
        lv = [s[l] for s in levels]
        x = key_noise(lv, 21 + l)
        b = key_noise(lv, 31 + l)
        xd, bd, yd = upload(h, l, x), upload(h, l, b), h.vector(l)
        gmg.spmv(h, l, xd, yd)
        assert exact(download(h, yd, K), o.spmv(l, x))
        rn = gmg.residual_norm(h, l, xd, bd)
        assert rn == pytest.approx(o.residual_norm(l, x, b), rel=1e-13)
        for kind in (0, 1, 2):
            v = upload(h, l, x)
            {0: lambda: gmg.update_master_slave(h, l, v, gmg.PF_UPDATE_SCATTER),
             1: lambda: gmg.update_halo1(h, l, v), 2: lambda: gmg.update_halo2(h, l, v)}[kind]()
            want = (o.update_master_slave(l, x, 0) if kind == 0 else o.update_halo(l, kind, x))
            assert exact(download(h, v, K), want), f"scatter kind {kind}"
        v = upload(h, l, x)
        gmg.update_master_slave(h, l, v, gmg.PF_UPDATE_ACCUMULATE_THEN_SCATTER)
        assert exact(download(h, v, K), o.update_master_slave(l, x, 1))
        if l > 0:
            lc = [s[l - 1] for s in levels]
            xc = key_noise(lc, 41 + l)
            out = h.vector(l)
            gmg.prolongate(h, l, upload(h, l - 1, xc), out)
            assert exact(download(h, out, K), o.prolongate(l, xc))
            rc = h.vector(l - 1)
            gmg.restrict_residual(h, l, upload(h, l, x), rc)
            assert exact(download(h, rc, K), o.restrict_residual(l, x))


@pytest.mark.parametrize("kind", KINDS, ids=["jacobi", "gs", "sor"])
def test_vcycle_and_solve_bit_exact(system, kind):
    h, o, levels, setups, K, L = (system[k] for k in ("h", "o", "levels", "setups", "K", "L"))
    c = cfg(kind, damping=1.2 if kind == gmg.PF_SMOOTHER_MULTICOLOR_SOR else 0.8)
    b = [s.b for s in setups]
    x0 = [s.x0 for s in setups]
    x = upload(h, L - 1, x0)
    bd = upload(h, L - 1, b)
    gmg.v_cycle(h, x, bd, c)
    xo, _ = o.v_cycle(x0, b, c)
    assert exact(download(h, x, K), xo)
    x = upload(h, L - 1, x0)
    st = gmg.solve_outer(h, x, bd, c)
    xs, res, ost, rc = o.solve_outer(x0, b, c)
    assert rc == 0 and st.converged
    assert st.iterations == ost.iterations
    np.testing.assert_allclose(st.residuals, res, rtol=1e-12)
    assert exact(download(h, x, K), xs)
    assert st.final_residual <= 1e-10 * st.initial_residual


def test_coarse_solve_matches_oracle(system):
    h, o, levels, K = system["h"], system["o"], system["levels"], system["K"]
    lv = [s[0] for s in levels]
    b = key_noise(lv, 5)
    x0 = [np.zeros(l.n) for l in lv]
    xd, bd = upload(h, 0, x0), upload(h, 0, b)
    st = gmg.coarse_solve(h, 0, xd, bd, 1e-12, 20000)
    xo, ost = o.coarse_solve(0, x0, b, 1e-12, 20000)
    assert st.iterations == ost.iterations and st.converged == bool(ost.converged)
    assert st.initial_residual == ost.initial_residual and st.final_residual == ost.final_residual
    assert exact(download(h, xd, K), xo)


def test_reference_level_data_bit_exact(cuda, ref_lib):
    """The drop-in path: the reference's own CSR / P / channels (host order, class-sorted,
    Z-order first touch) through the GPU library; solve_outer must reproduce the
    reference's residual history and solution bit for bit (Jacobi, C1 = 32^3)."""
    for K in (1, 2, 8):
        R = ref_lib.build(3, 2, 5 if K == 1 else 4, K)
        levels = [[lv.to_level_arrays() for lv in R.ranks[r]] for r in range(K)]
        h = gmg.Hierarchy(levels)
        c = cfg(gmg.PF_SMOOTHER_JACOBI)
        x = upload(h, h.finest, R.x0)
        b = upload(h, h.finest, R.b)
        st = gmg.solve_outer(h, x, b, c)
        xr, resr, sr = ref_lib.run(3, 2, h.n_levels, K, smoother=0, pre=2, post=2, outer_tol=1e-10)
        assert st.iterations == sr["iterations"]
        np.testing.assert_allclose(st.residuals, resr, rtol=1e-13, atol=0)
        assert exact(download(h, x, K), xr), f"K={K}: solution differs from the reference"


def test_structured_solution_matches_reference_by_key(cuda, ref_lib):
    """Product setup + GPU solve vs the reference's own setup + solve, per carrier key.

    The product's setup numbers the dofs as the reference does and sums every assembled
    entry over the same cells in the same (gcn) order, so its level data are the
    reference's byte for byte (tests/test_setup.py) — and the damped-Jacobi solve is then
    identical: same cycle count, same solution bit for bit, residual norms to the last
    ulp (summation order of the norm)."""
    for K, L in ((1, 5), (8, 4), (4, 4)):
        setups, levels = structured(3, 2, L, K)
        h = gmg.Hierarchy(levels)
        x = upload(h, L - 1, [s.x0 for s in setups])
        b = upload(h, L - 1, [s.b for s in setups])
        st = gmg.solve_outer(h, x, b, cfg())
        R = ref_lib.build(3, 2, L, K)
        xr, resr, sr = ref_lib.run(3, 2, L, K, smoother=0, pre=2, post=2, outer_tol=1e-10)
        assert st.iterations == sr["iterations"]
        np.testing.assert_allclose(st.residuals, resr, rtol=1e-13, atol=0)
        got = keyed([s[-1] for s in levels], download(h, x, K))
        want = keyed([R.ranks[r][-1].to_level_arrays() for r in range(K)], xr)
        assert got == want, K


def test_host_entry_point_matches_device_solve(cuda):
    setups, levels = structured(3, 2, 5, 1)
    h = gmg.Hierarchy(levels)
    c = cfg()
    x = upload(h, 4, [setups[0].x0])
    st = gmg.solve_outer(h, x, upload(h, 4, [setups[0].b]), c)
    xh = [setups[0].x0.copy()]
    st2 = gmg.solve_outer_host(h, xh, [setups[0].b], c)
    assert st2.iterations == st.iterations
    assert np.array_equal(xh[0], x.download())


def test_errors_are_raised(cuda):
    setups, levels = structured(3, 2, 3, 1)
    h = gmg.Hierarchy(levels)
    x = upload(h, 2, [setups[0].x0])
    b = upload(h, 2, [setups[0].b])
    with pytest.raises(gmg.NoConvergenceError):
        gmg.solve_outer(h, x, b, cfg(tol=1e-14, max_cycles=1))
    with pytest.raises(_lib.InvalidArgument):
        gmg.spmv(h, 2, h.vector(1), h.vector(2))
    bad = levels[0][2].normalized()
    bad.vals = bad.vals.copy()
    for k in range(bad.row_offsets[0], bad.row_offsets[1]):
        if bad.cols[k] == 0:
            bad.vals[k] = 0.0
    lv = list(levels[0])
    lv[2] = bad
    with pytest.raises(gmg.SingularDiagonalError):
        gmg.Hierarchy([lv])


def _run_ranks(K, body):
    """Run body(rank) on K host threads (ctypes releases the GIL inside the library)."""
    import threading
    out, errs = [None] * K, []

    def wrap(r):
        try:
            out[r] = body(r)
        except Exception as e:  # noqa: BLE001
            errs.append(e)
    th = [threading.Thread(target=wrap, args=(r,)) for r in range(K)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    if errs:
        raise errs[0]
    return out


@pytest.mark.parametrize("K,L", [(2, 4), (4, 4), (8, 3), (3, 3), (8, 4)])
@pytest.mark.parametrize("kind", [gmg.PF_SMOOTHER_JACOBI, gmg.PF_SMOOTHER_MULTICOLOR_SOR], ids=["jacobi", "sor"])
@pytest.mark.parametrize("rep", ["coarse", "bottom"])
def test_multiprocess_path_loopback(cuda, K, L, kind, rep):
    """The one-subdomain-per-process code path (pack/unpack kernels, segment transport,
    master accumulate from a receive buffer, allgather-based allreduce, the replicated
    coarse solve or the replicated bottom V-cycle) with the loopback transport standing in
    for NCCL: K hierarchies on K threads must reproduce the oracle's K-rank solve bit for
    bit."""
    setups, levels = structured(3, 2, L, K)
    c = cfg(kind, damping=1.2 if kind == gmg.PF_SMOOTHER_MULTICOLOR_SOR else 0.8)
    replicas = [s[0] for s in levels] if rep == "coarse" else [s[:L - 1] for s in levels]
    hub = gmg.LoopbackHub(K)

    def body(r):
        h = gmg.Hierarchy([levels[r]], rank_base=r, world_size=K, coarse_replicas=replicas)
        h.init_loopback(hub)
        x = h.vector(L - 1, setups[r].x0)
        b = h.vector(L - 1, setups[r].b)
        st = gmg.solve_outer(h, x, b, c)
        rn = gmg.residual_norm(h, L - 1, x, b)
        v = h.vector(L - 2, key_noise([levels[r][L - 2]], 3)[0])
        gmg.update_master_slave(h, L - 2, v, gmg.PF_UPDATE_ACCUMULATE_THEN_SCATTER)
        return st, x.download(), rn, v.download()

    res = _run_ranks(K, body)
    hub.close()
    o = Oracle(levels)
    xs, resid, ost, rc = o.solve_outer([s.x0 for s in setups], [s.b for s in setups], c)
    acc = o.update_master_slave(L - 2, key_noise([lv[L - 2] for lv in levels], 3), 1)
    for r in range(K):
        st, x, rn, v = res[r]
        assert st.iterations == ost.iterations
        np.testing.assert_allclose(st.residuals, resid, rtol=1e-12)
        assert np.array_equal(x, xs[r]), f"rank {r}"
        assert np.array_equal(v, acc[r]), f"accumulate rank {r}"
        assert rn == pytest.approx(res[0][2], rel=0, abs=0)


@pytest.mark.parametrize("bottom_rows", ["0", "1024", "65536", "1000000"],
                         ids=["multilaunch", "bottom", "bottom-64k", "bottom-all"])
@pytest.mark.parametrize("kind", KINDS, ids=["jacobi", "gs", "sor"])
def test_bottom_kernel_equals_multilaunch(cuda, bottom_rows, kind):
    """The cooperative bottom-of-cycle kernel is a launch-structure change only: with it
    disabled, covering the default levels, or covering every level below the finest, the
    solve must equal the oracle bit for bit (1 and 4 subdomains).  Jacobi is forced onto
    it too (by default it runs per-level kernels).  Per-hierarchy options."""
    c = cfg(kind, damping=1.2 if kind == gmg.PF_SMOOTHER_MULTICOLOR_SOR else 0.8)
    for K in (1, 4):
        setups, levels = structured(3, 2, 5, K)
        h = gmg.Hierarchy(levels, options={"bottom_rows": int(bottom_rows), "bottom_jacobi": 1})
        x = upload(h, 4, [s.x0 for s in setups])
        st = gmg.solve_outer(h, x, upload(h, 4, [s.b for s in setups]), c)
        xo, res, ost, rc = Oracle(levels).solve_outer([s.x0 for s in setups], [s.b for s in setups], c)
        assert st.iterations == ost.iterations
        assert exact(download(h, x, K), xo)


@pytest.mark.parametrize("mode", ["host", "graph"])
@pytest.mark.parametrize("kind", KINDS, ids=["jacobi", "gs", "sor"])
def test_solve_drivers_agree(cuda, mode, kind):
    """solve_outer driven from the host (one graph per outer cycle + host convergence
    test) and as one device-driven graph (WHILE/IF conditional nodes, the Jacobi norm
    fused into the next cycle's first sweep) give the oracle's iterate and cycle count."""
    c = cfg(kind, damping=1.2 if kind == gmg.PF_SMOOTHER_MULTICOLOR_SOR else 0.8)
    for K in (1, 2):
        setups, levels = structured(3, 2, 4, K)
        h = gmg.Hierarchy(levels, options={"solve_mode_host": int(mode == "host")})
        x = upload(h, 3, [s.x0 for s in setups])
        st = gmg.solve_outer(h, x, upload(h, 3, [s.b for s in setups]), c)
        xo, res, ost, rc = Oracle(levels).solve_outer([s.x0 for s in setups], [s.b for s in setups], c)
        assert st.iterations == ost.iterations and len(st.residuals) == st.iterations
        np.testing.assert_allclose(st.residuals, res, rtol=1e-12)
        assert st.initial_residual == pytest.approx(ost.initial_residual, rel=1e-13)
        assert exact(download(h, x, K), xo)
        # zero rhs converges in zero cycles (test_multigrid.cpp:164-174)
        z = h.vector(3)
        st0 = gmg.solve_outer(h, z, h.vector(3), c)
        assert st0.iterations == 0 and st0.converged


def test_repeated_solves_at_c2(cuda):
    """C2 (128^3) solved three times through the same cached solve graph: 9 Jacobi cycles,
    the reference's residual history (golden, 8 reference ranks) within the roundoff gate,
    identical iterates every time."""
    import os
    g = np.load(os.path.join(os.path.dirname(__file__), "golden", "c2_jacobi_k8.npz"))
    setups, levels = structured(3, 2, 7, 1)
    h = gmg.Hierarchy(levels)
    x = h.vector(6)
    b = upload(h, 6, [setups[0].b])
    first = None
    for _ in range(3):
        x.upload(setups[0].x0)
        st = gmg.solve_outer(h, x, b, cfg())
        assert st.iterations == int(g["iterations"]) == 9
        np.testing.assert_allclose(st.residuals, g["residuals"], rtol=1e-6,
                                   atol=1e-14 * float(g["initial_residual"]))
        sol = x.download()
        if first is None:
            first = sol
        assert np.array_equal(sol, first)
    got = keyed([levels[0][-1]], [first])
    want = dict(zip(map(tuple, g["keys"]), g["values"]))
    scale = np.abs(g["values"]).max()
    assert max(abs(got[k] - want[k]) for k in want) <= 1e-11 * scale


@pytest.mark.parametrize("K", [1, 2, 4, 8])
@pytest.mark.parametrize("smoother", [0, 1], ids=["jacobi", "gs"])
def test_drop_in_bridge_inside_the_reference(cuda, ref_lib, K, smoother):
    """The drop-in: the UNMODIFIED reference builds its hierarchy on K rank threads
    (run_on_ranks) and calls parfem::gpu::solve_outer (integration/parfem_gpu_bridge.cpp)
    where it would call parfem::solve_outer.  Jacobi must equal the reference's own solve
    bit for bit; Gauss-Seidel (device: multicolour) must converge to the same solution
    within the SURVEY §8d gate with +-1 cycle."""
    if not ref_lib.bridge_available():
        pytest.skip("oracle/_ref/libparfem_bridge.so not built")
    L = 5 if K == 1 else 4
    R = ref_lib.build(3, 2, L, K)
    sizes = [R.ranks[r][-1].n_dofs for r in range(K)]
    xr, resr, sr = ref_lib.run(3, 2, L, K, smoother=smoother, pre=2, post=2, outer_tol=1e-10, sizes=sizes)
    xg, resg, sg = ref_lib.run(3, 2, L, K, smoother=smoother, pre=2, post=2, outer_tol=1e-10, sizes=sizes,
                               gpu=True)
    assert sg["status"] == 0, sg["error"]
    if smoother == 0:
        assert sg["iterations"] == sr["iterations"]
        np.testing.assert_allclose(resg, resr, rtol=1e-13)
        assert all(np.array_equal(a, b) for a, b in zip(xg, xr))
    else:
        assert abs(sg["iterations"] - sr["iterations"]) <= 1
        assert resg[-1] <= 1e-10 * sg["initial_residual"]
        num = sum(float(np.sum((a - b) ** 2)) for a, b in zip(xg, xr))
        den = sum(float(np.sum(b ** 2)) for b in xr)
        assert np.sqrt(num) <= 1e-8 * np.sqrt(den)


@pytest.mark.parametrize("kind", KINDS, ids=["jacobi", "gs", "sor"])
def test_lognormal_coefficient_solve_bit_exact(cuda, kind):
    """BASELINE's lognormal(0,1) per-cell coefficient (PF_PROBLEM_LOGNORMAL; the setup is
    pinned to oracle/coef.py by tests/test_setup.py): every operator value distinct, so the
    device keeps fp64 values — GPU solve == oracle bit for bit, 1 and 2 subdomains."""
    c = cfg(kind, damping=1.2 if kind == gmg.PF_SMOOTHER_MULTICOLOR_SOR else 0.8, max_cycles=200)
    for K in (1, 2):
        setups = [StructuredSetup(3, 2, 5, K, r, _lib.PF_PROBLEM_LOGNORMAL, seed=99) for r in range(K)]
        levels = [s.levels for s in setups]
        h = gmg.Hierarchy(levels)
        x = upload(h, 4, [s.x0 for s in setups])
        st = gmg.solve_outer(h, x, upload(h, 4, [s.b for s in setups]), c)
        xo, res, ost, rc = Oracle(levels).solve_outer([s.x0 for s in setups], [s.b for s in setups], c)
        assert rc == 0 and st.converged
        assert st.iterations == ost.iterations
        np.testing.assert_allclose(st.residuals, res, rtol=1e-12)
        assert exact(download(h, x, K), xo)


def test_nccl_transport_selftest(cuda):
    """The dlopen'd NCCL wrapper the multi-process exchanges use (pf_nccl.cpp): a one-rank
    communicator, grouped send/recv to itself and an allgather deliver their payloads.
    (Multi-rank NCCL needs one GPU per rank; its exchange logic is covered bit-exactly by
    the loopback transport, test_multiprocess_path_loopback.)"""
    import ctypes as C
    import torch  # noqa: F401  (loads the NCCL the bench uses)
    import torch.distributed  # noqa: F401
    ok = C.c_int(0)
    _lib.check(_lib.lib().pf_nccl_selftest(0, C.byref(ok)))
    assert ok.value == 1


@pytest.mark.parametrize("K,L", [(4, 4), (8, 4), (3, 3)])
@pytest.mark.parametrize("kind", [gmg.PF_SMOOTHER_JACOBI, gmg.PF_SMOOTHER_MULTICOLOR_SOR], ids=["jacobi", "sor"])
@pytest.mark.parametrize("rep", ["coarse", "bottom"])
def test_fused_exchanges_bit_exact(cuda, K, L, kind, rep):
    """Direct halo lists (pf_setup_options.direct_halos) + fused exchanges (one message group
    per sweep for master/slave + halo1, + halo2 after a smoothing phase): the solve equals
    the oracle's — and the standard-lists solve — bit for bit, with K subdomains on one
    device and through the loopback transport (the multi-process code path)."""
    c = cfg(kind, damping=1.2 if kind == gmg.PF_SMOOTHER_MULTICOLOR_SOR else 0.8)
    setups, levels = structured(3, 2, L, K, direct_halos=True)
    xs, resid, ost, rc = Oracle(levels).solve_outer([s.x0 for s in setups], [s.b for s in setups], c)
    std_setups, std_levels = structured(3, 2, L, K)
    xstd, _, _, _ = Oracle(std_levels).solve_outer([s.x0 for s in std_setups], [s.b for s in std_setups], c)
    assert exact(xs, xstd)
    h = gmg.Hierarchy(levels, fused_exchanges=True)
    x = upload(h, L - 1, [s.x0 for s in setups])
    st = gmg.solve_outer(h, x, upload(h, L - 1, [s.b for s in setups]), c)
    assert st.iterations == ost.iterations
    assert exact(download(h, x, K), xs)
    replicas = [s[0] for s in levels] if rep == "coarse" else [s[:L - 2] for s in levels]
    hub = gmg.LoopbackHub(K)

    def body(r):
        hr = gmg.Hierarchy([levels[r]], rank_base=r, world_size=K, coarse_replicas=replicas, fused_exchanges=True)
        hr.init_loopback(hub)
        xr = hr.vector(L - 1, setups[r].x0)
        str_ = gmg.solve_outer(hr, xr, hr.vector(L - 1, setups[r].b), c)
        return str_.iterations, xr.download()

    res = _run_ranks(K, body)
    hub.close()
    for r in range(K):
        assert res[r][0] == ost.iterations
        assert np.array_equal(res[r][1], xs[r]), r


def test_fused_exchanges_need_direct_lists(cuda):
    setups, levels = structured(3, 2, 4, 4)  # standard lists forward Slave-held values
    with pytest.raises(_lib.InvalidArgument, match="direct_halos"):
        gmg.Hierarchy(levels, fused_exchanges=True)


def test_hierarchy_from_native_setups(cuda):
    """Hierarchy.from_setups (no numpy copies; the setups' matrices released after the
    upload — the large-grid path) solves exactly like the materialized path."""
    K, L = 2, 4
    setups, levels = structured(3, 2, L, K)
    h = gmg.Hierarchy(levels)
    x = upload(h, L - 1, [s.x0 for s in setups])
    st = gmg.solve_outer(h, x, upload(h, L - 1, [s.b for s in setups]), cfg())
    native = [StructuredSetup(3, 2, L, K, r, materialize=False) for r in range(K)]
    hn = gmg.Hierarchy.from_setups(native)
    xn = upload(hn, L - 1, [s.x0 for s in native])
    stn = gmg.solve_outer(hn, xn, upload(hn, L - 1, [s.b for s in native]), cfg())
    assert stn.iterations == st.iterations and list(stn.residuals) == list(st.residuals)
    assert exact(download(hn, xn, K), download(h, x, K))
    with pytest.raises(_lib.PfError):
        native[0].level_desc(0)  # released


@pytest.mark.parametrize("mode", ["graph", "host"])
def test_graph_cache_keys_every_config_bit(cuda, mode):
    """The cached solve graph is keyed by the exact bits of every config double: a second
    solve on the same vectors with a tighter outer_tol (or a damping that prints the same
    to 6 digits) must not replay the first graph."""
    setups, levels = structured(3, 2, 4, 1)
    h = gmg.Hierarchy(levels, options={"solve_mode_host": int(mode == "host")})
    x = h.vector(3)
    b = upload(h, 3, [setups[0].b])
    o = Oracle(levels)
    for tol, damping in ((1e-6, 0.8), (1e-10, 0.8), (1e-10, 2.0 / 3.0), (1e-10, 0.666667)):
        c = cfg(damping=damping, tol=tol)
        x.upload(setups[0].x0)
        st = gmg.solve_outer(h, x, b, c)
        xo, res, ost, rc = o.solve_outer([setups[0].x0], [setups[0].b], c)
        assert st.iterations == ost.iterations, (tol, damping)
        assert exact([x.download()], xo), (tol, damping)


def test_destroyed_vector_graphs_are_dropped(cuda):
    """Graphs are keyed by vector id, not address: destroying the solve's vectors and
    creating new ones (the allocator may hand back the same addresses) captures a fresh
    graph on the new device buffers, and the stale graphs are released."""
    setups, levels = structured(3, 2, 4, 1)
    h = gmg.Hierarchy(levels)
    o = Oracle(levels)
    xo, res, ost, rc = o.solve_outer([setups[0].x0], [setups[0].b], cfg())
    for i in range(4):
        x = h.vector(3, setups[0].x0)
        b = h.vector(3, setups[0].b)
        st = gmg.solve_outer(h, x, b, cfg())
        assert st.iterations == ost.iterations
        assert exact([x.download()], xo), i
        x.close()
        b.close()
        assert h.graph_count() <= 1


def test_options_are_per_hierarchy(cuda):
    """Tuning options live on the hierarchy: two hierarchies of one process with opposite
    settings of every launch-structure option both reproduce the oracle bit for bit; a
    launch option changed between solves drops the cached graphs and the next solve is
    again bit-exact; a build option after finalize and an unknown name are refused."""
    setups, levels = structured(3, 2, 5, 1)
    o = Oracle(levels)
    alt = {"bottom_rows": 0, "vtab_smem": 0, "value_index_min": 1 << 30, "fused_rr_rows": 0, "wide_max_rows": 0,
           "bottom_stage": 0, "pdl": 0}
    for kind in KINDS:
        c = cfg(kind, damping=1.2 if kind == gmg.PF_SMOOTHER_MULTICOLOR_SOR else 0.8)
        xo, res, ost, rc = o.solve_outer([s.x0 for s in setups], [s.b for s in setups], c)
        for opts in ({}, alt):
            h = gmg.Hierarchy(levels, options=opts)
            for k, v in opts.items():
                assert h.get_option(k) == v
            x = upload(h, 4, [setups[0].x0])
            b = upload(h, 4, [setups[0].b])
            st = gmg.solve_outer(h, x, b, c)
            assert st.iterations == ost.iterations and exact(download(h, x, 1), xo)
            h.set_option("wide_max_rows", 0 if h.get_option("wide_max_rows") != 0 else -1)
            h.set_option("solve_mode_host", 1)
            x.upload(setups[0].x0)
            st = gmg.solve_outer(h, x, b, c)
            assert st.iterations == ost.iterations and exact(download(h, x, 1), xo)
            with pytest.raises(_lib.PfError):
                h.set_option("value_index", 0)  # build option after finalize
            with pytest.raises(_lib.InvalidArgument):
                h.set_option("no_such_option", 1)
