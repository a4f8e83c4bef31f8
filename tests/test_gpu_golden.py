"""GPU: the reference's known answers and the committed golden fixtures (tests/golden/,
made from the unmodified reference by make_golden.py) replayed on the device — no
reference or oracle needed at run time.  Mirrors tests/test_oracle.py's CPU checks."""
import glob
import os

import numpy as np
import pytest

from helpers import cfg, download, keyed, upload
from paper_1609_04809_b200 import _lib, gmg
from paper_1609_04809_b200.levels import LevelArrays, StructuredSetup

pytestmark = pytest.mark.gpu
GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def dense_level(rows):
    n = len(rows)
    rp = np.arange(0, n * n + 1, n, dtype=np.int64)
    cols = np.tile(np.arange(n, dtype=np.int32), n)
    vals = np.array(rows, dtype=np.float64).ravel()
    return LevelArrays(n, n, rp, cols, vals, np.ones(n, np.uint8), np.zeros(n, np.uint8))


@pytest.mark.parametrize("kind", [gmg.PF_SMOOTHER_GAUSS_SEIDEL, gmg.PF_SMOOTHER_MULTICOLOR_SOR],
                         ids=["gs", "sor_1.0"])
def test_textbook_gauss_seidel_iterate(cuda, kind):
    """test_solvers.cpp:77-92: one GS sweep on [[4,1],[1,3]], b = [1,2] gives exactly
    [0.25, 1.75/3] (the two rows couple, so they get two colours, swept in order)."""
    h = gmg.Hierarchy([[dense_level([[4, 1], [1, 3]])]])
    x = upload(h, 0, [np.zeros(2)])
    gmg.smooth(h, 0, x, upload(h, 0, [np.array([1.0, 2.0])]), gmg.SmootherConfig(kind=kind, sweeps=1, damping=1.0))
    got = download(h, x, 1)[0]
    assert got[0] == 0.25 and got[1] == 1.75 / 3.0


def test_undamped_jacobi_on_identity(cuda):
    """test_solvers.cpp:60-75: one undamped Jacobi sweep on the identity returns b."""
    h = gmg.Hierarchy([[dense_level(np.eye(3).tolist())]])
    b = np.array([3.0, -1.0, 0.5])
    x = upload(h, 0, [np.zeros(3)])
    gmg.smooth(h, 0, x, upload(h, 0, [b]), gmg.SmootherConfig(kind=gmg.PF_SMOOTHER_JACOBI, sweeps=1, damping=1.0))
    assert np.array_equal(download(h, x, 1)[0], b)


def test_zero_diagonal_is_reported(cuda):
    """test_solvers.cpp:94-116: SingularDiagonalError (checked once, at upload)."""
    with pytest.raises(_lib.SingularDiagonalError):
        gmg.Hierarchy([[dense_level([[0.0]])]])


def golden_solves():
    return sorted(p for p in glob.glob(os.path.join(GOLDEN, "*.npz"))
                  if not os.path.basename(p).startswith("sweeps") and not p.endswith("_digest.npz"))


@pytest.mark.parametrize("path", golden_solves(), ids=os.path.basename)
def test_golden_solve_on_device(cuda, path):
    """The reference's own solves (C1 and C2 included, 1-8 ranks as subdomains on one GPU)
    replayed through the device on the product setup: Jacobi — the reference's cycle
    count, residual history within the roundoff gate, keyed solution within 1e-12 of its
    magnitude; Gauss-Seidel (the device colours it) — converged, +-1 cycle, relative L2
    difference <= 1e-8."""
    g = np.load(path)
    dim, nc, L, K, prob = (int(g[k]) for k in ("dim", "n_coarse", "levels", "K", "problem"))
    setups = [StructuredSetup(dim, nc, L, K, r, prob) for r in range(K)]
    levels = [s.levels for s in setups]
    h = gmg.Hierarchy(levels)
    jac = int(g["smoother"]) == 0
    c = cfg(gmg.PF_SMOOTHER_JACOBI if jac else gmg.PF_SMOOTHER_GAUSS_SEIDEL)
    x = upload(h, L - 1, [s.x0 for s in setups])
    st = gmg.solve_outer(h, x, upload(h, L - 1, [s.b for s in setups]), c)
    got = keyed([lv[-1] for lv in levels], download(h, x, K))
    want = dict(zip(map(tuple, g["keys"]), g["values"]))
    assert st.converged and set(want) <= set(got)
    w = np.array(list(want.values()))
    a = np.array([got[k] for k in want])
    if jac:
        assert st.iterations == int(g["iterations"])
        np.testing.assert_allclose(st.residuals, g["residuals"], rtol=1e-6,
                                   atol=1e-14 * float(g["initial_residual"]))
        assert np.abs(a - w).max() <= 1e-12 * np.abs(w).max()
    else:
        assert abs(st.iterations - int(g["iterations"])) <= 1
        assert np.linalg.norm(a - w) <= 1e-8 * np.linalg.norm(w)


def test_golden_jacobi_sweeps_on_device(cuda):
    """Per-sweep iterates of the reference (3 smooth() calls, 2 ranks) on the device."""
    g = np.load(os.path.join(GOLDEN, "sweeps_3d_l4_k2_jacobi.npz"))
    dim, nc, L, K = (int(g[k]) for k in ("dim", "n_coarse", "levels", "K"))
    setups = [StructuredSetup(dim, nc, L, K, r) for r in range(K)]
    levels = [s.levels for s in setups]
    h = gmg.Hierarchy(levels)
    x, b = upload(h, L - 1, [s.x0 for s in setups]), upload(h, L - 1, [s.b for s in setups])
    for _ in range(int(g["n_ops"])):
        gmg.smooth(h, L - 1, x, b, gmg.SmootherConfig(kind=gmg.PF_SMOOTHER_JACOBI, sweeps=1, damping=0.8))
    got = keyed([lv[-1] for lv in levels], download(h, x, K))
    want = dict(zip(map(tuple, g["keys"]), g["values"]))
    scale = max(abs(v) for v in want.values())
    assert max(abs(got[k] - want[k]) for k in want) <= 1e-14 * scale
