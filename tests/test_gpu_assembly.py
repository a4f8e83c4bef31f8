"""GPU: device assembly of the finest-level Q1 system (pf_assembly_*,
assemble_system + apply_dirichlet_rows, assembly.cpp:103-170).

The host setup's level data equal the reference's byte for byte (tests/test_setup.py) and,
for the lognormal coefficient, the restatement oracle/coef.py; the device kernel must
reproduce every stored value exactly (same products, same gcn-ordered cell sums)."""
import numpy as np
import pytest

from paper_1609_04809_b200 import _lib, gmg
from paper_1609_04809_b200.heat import Assembly, Operator
from paper_1609_04809_b200.levels import StructuredSetup

pytestmark = pytest.mark.gpu

CASES = [(3, 2, 3, 1, 0), (3, 2, 4, 2, 1), (3, 2, 3, 8, 0), (2, 3, 3, 5, 1), (3, 3, 3, 3, 2),
         (3, 2, 4, 1, 4), (3, 2, 3, 4, 4), (2, 4, 3, 6, 4)]


@pytest.mark.parametrize("dim,nc,L,K,prob", CASES, ids=["d%d_nc%d_L%d_K%d_p%d" % c for c in CASES])
def test_device_assembly_equals_host(cuda, dim, nc, L, K, prob):
    S = [StructuredSetup(dim, nc, L, K, r, prob, keep=True, seed=7) for r in range(K)]
    h = gmg.Hierarchy([s.levels for s in S])
    top = h.finest
    asm = Assembly(h, top, [s.assembly_desc() for s in S])
    op = asm.assemble(Operator(h, top))
    for r in range(K):
        lv = S[r].levels[-1]
        got = op.values(r, len(lv.vals))
        assert np.array_equal(got, lv.vals), r
    # the device-assembled operator drives the same spmv as the uploaded one
    x = h.vector(top, [np.sin(np.arange(s.levels[-1].n) * 0.37) for s in S])
    y1, y2 = h.vector(top), h.vector(top)
    op.apply(x, y1)
    gmg.spmv(h, top, x, y2)
    assert all(np.array_equal(y1.download(r), y2.download(r)) for r in range(K))
    h.close()
    for s in S:
        s.close()


def test_device_assembly_rejects_mismatch(cuda):
    a = StructuredSetup(3, 2, 3, keep=True)
    b = StructuredSetup(3, 2, 4, keep=True)
    h = gmg.Hierarchy([b.levels])
    with pytest.raises(_lib.InvalidArgument):
        Assembly(h, h.finest, [a.assembly_desc()])
    h.close()
