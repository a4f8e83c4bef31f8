"""CPU: MatrixMarket export (export_system, app.cpp:379-396,
export_matrixmarket, matrix_market.cpp:47-112, global numbering femapper.cpp:353-472).

The product writes the finest level of all ranks from its own setup; the files must be the
reference's byte for byte.
"""
import filecmp

import numpy as np
import pytest

from paper_1609_04809_b200 import _lib
from paper_1609_04809_b200.levels import StructuredSetup, export_matrixmarket


def _setups(dim, nc, L, K):
    return [StructuredSetup(dim, nc, L, K, r, _lib.PF_PROBLEM_REFERENCE_POISSON, keep=True) for r in range(K)]


@pytest.mark.parametrize("dim,nc,L,K", [(3, 2, 3, 1), (3, 2, 3, 4), (2, 3, 3, 5), (3, 2, 4, 8), (2, 4, 3, 6),
                                        (3, 3, 2, 7)])
def test_export_is_byte_identical_to_reference(ref_lib, tmp_path, dim, nc, L, K):
    ref_lib.export(dim, nc, L, K, str(tmp_path / "ref"))
    S = _setups(dim, nc, L, K)
    export_matrixmarket(S, str(tmp_path / "pf.mtx"), str(tmp_path / "pf_rhs.mtx"))
    assert filecmp.cmp(tmp_path / "ref.mtx", tmp_path / "pf.mtx", shallow=False)
    assert filecmp.cmp(tmp_path / "ref_rhs.mtx", tmp_path / "pf_rhs.mtx", shallow=False)


def test_export_round_trip(tmp_path):
    """Reading the files back gives every owned row of every rank and the rhs: the global
    matrix is the union of the owned rows, each entry present exactly once."""
    dim, nc, L, K = 3, 2, 3, 2
    S = _setups(dim, nc, L, K)
    n, nnz = export_matrixmarket(S, str(tmp_path / "a.mtx"), str(tmp_path / "a_rhs.mtx"))
    lines = (tmp_path / "a.mtx").read_text().splitlines()
    assert lines[0] == "%%MatrixMarket matrix coordinate real general"
    assert lines[1] == f"{n} {n} {nnz}"
    ent = np.array([ln.split() for ln in lines[2:]], dtype=float)
    assert len(ent) == nnz
    pairs = {(int(r), int(c)) for r, c, _ in ent}
    assert len(pairs) == nnz  # no duplicates across ranks
    assert {int(r) for r, _, _ in ent} == set(range(1, n + 1))
    rhs = (tmp_path / "a_rhs.mtx").read_text().splitlines()
    assert rhs[:2] == ["%%MatrixMarket matrix array real general", f"{n} 1"] and len(rhs) == n + 2
    # the global matrix is the 3D Q1 stiffness of the 8^3 grid: every row sums to 0 off
    # the boundary (constants are in the kernel of the Laplacian)
    rowsum = np.zeros(n + 1)
    for r, c, v in ent:
        rowsum[int(r)] += v
    interior = sum(s.levels[-1].n_own for s in S)
    assert np.abs(rowsum[1:interior + 1]).max() < 1e-12


def test_export_rejects_mixed_setups(tmp_path):
    a = StructuredSetup(3, 2, 2, 2, 0, keep=True)
    b = StructuredSetup(3, 2, 3, 2, 1, keep=True)
    with pytest.raises(_lib.InvalidArgument):
        export_matrixmarket([a, b], str(tmp_path / "x.mtx"), str(tmp_path / "x_rhs.mtx"))
    with pytest.raises(_lib.InvalidArgument):
        export_matrixmarket([b, a], str(tmp_path / "x.mtx"), str(tmp_path / "x_rhs.mtx"))
