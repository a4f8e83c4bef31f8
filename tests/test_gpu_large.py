"""Above 2^31 stored entries (slow; PF_RUN_SLOW=1): one finest-level sweep of a 448^3 Q1
grid (n_coarse 7, 7 levels: 90.9M rows, 2.44e9 entries — the int64 slice offsets, and the
colour-interleaved block schedule since x is 727 MB) against the C restatement on the same
level data, bit for bit: damped Jacobi, multicolour SOR, and the residual norm.

The oracle reads the native setup's level arrays in place (Oracle.from_level_descs), then
the hierarchy takes them over (Hierarchy.from_setups), so the host holds one copy plus the
oracle's (~100 GB peak on the 196 GB GPU box)."""
import ctypes
import os

import numpy as np
import pytest

from oracle.restated import Oracle
from paper_1609_04809_b200 import gmg
from paper_1609_04809_b200.levels import StructuredSetup

pytestmark = [pytest.mark.gpu, pytest.mark.slow,
              pytest.mark.skipif(os.environ.get("PF_RUN_SLOW") != "1", reason="PF_RUN_SLOW=1 (448^3, ~100 GB host)")]


def test_sweeps_above_2_31_entries_bit_exact(cuda):
    L = 7
    s = StructuredSetup(3, 7, L, 1, 0, materialize=False)
    d = s.level_desc(L - 1)
    n = int(d.n_dofs)
    z = int(ctypes.cast(d.row_offsets, ctypes.POINTER(ctypes.c_int64))[n])
    assert z > 2 ** 31
    rng = np.random.default_rng(7)
    x0 = rng.standard_normal(n)
    o = Oracle.from_level_descs([[d]])
    want_j = o.smooth(0, [x0], [s.b], gmg.PF_SMOOTHER_JACOBI, sweeps=1, damping=0.8)[0]
    want_s = o.smooth(0, [x0], [s.b], gmg.PF_SMOOTHER_MULTICOLOR_SOR, sweeps=1, damping=1.2)[0]
    want_rn = o.residual_norm(0, [x0], [s.b])
    del o
    h = gmg.Hierarchy.from_setups([s])
    top = h.finest
    bd = h.vector(top, s.b)
    x = h.vector(top, x0)
    gmg.smooth(h, top, x, bd, gmg.SmootherConfig(kind=gmg.PF_SMOOTHER_JACOBI, sweeps=1, damping=0.8))
    assert np.array_equal(x.download(), want_j), "Jacobi sweep"
    x.upload(x0)
    gmg.smooth(h, top, x, bd, gmg.SmootherConfig(kind=gmg.PF_SMOOTHER_MULTICOLOR_SOR, sweeps=1, damping=1.2))
    assert np.array_equal(x.download(), want_s), "SOR sweep"
    x.upload(x0)
    rn = gmg.residual_norm(h, top, x, bd)
    assert rn == pytest.approx(want_rn, rel=1e-11)
