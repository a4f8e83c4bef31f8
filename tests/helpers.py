"""Shared fixtures-as-functions for the parity tests."""
from __future__ import annotations

import numpy as np

from paper_1609_04809_b200 import gmg
from paper_1609_04809_b200.levels import StructuredSetup


def structured(dim, n_coarse, levels, K, problem=0, direct_halos=False):
    setups = [StructuredSetup(dim, n_coarse, levels, K, r, problem, direct_halos=direct_halos) for r in range(K)]
    return setups, [s.levels for s in setups]


def keyed(level_arrays, values):
    """{Key4: value} over authoritative rows (owns_row), as gather_vector does
    (tests/support.cpp:182-201)."""
    out = {}
    for lv, v in zip(level_arrays, values):
        for i in np.flatnonzero(lv.owns_row):
            out[tuple(lv.keys[i])] = v[i]
    return out


def key_noise(level_arrays, salt):
    """Deterministic keyed values in [-1, 1) (the reference fixture key_noise, restated in
    numpy: tests/support.cpp:17-25), identical on every rank for the same carrier."""
    M = (1 << 64) - 1
    out = []
    for lv in level_arrays:
        vals = np.empty(lv.n)
        for i in range(lv.n):
            h = (salt * 0x9e3779b97f4a7c15) & M
            for part in lv.keys[i]:
                h ^= ((int(part) & M) + 0x9e3779b97f4a7c15 + ((h << 6) & M) + (h >> 2)) & M
                h = (h * 0xbf58476d1ce4e5b9) & M
                h ^= h >> 31
            vals[i] = (h >> 11) / float(1 << 52) - 1.0
        out.append(vals)
    return out


def upload(h, level, arrays):
    v = h.vector(level)
    for s, a in enumerate(arrays):
        v.upload(a, s)
    return v


def download(h, v, K):
    return [v.download(s) for s in range(K)]


def cfg(kind=gmg.PF_SMOOTHER_JACOBI, damping=0.8, pre=2, post=2, tol=1e-10, max_cycles=100):
    return gmg.MultigridConfig(smoother=gmg.SmootherConfig(kind=kind, damping=damping),
                               pre_smooth=pre, post_smooth=post, outer_tol=tol,
                               outer_max_cycles=max_cycles)


def keyed_digest(level_arrays, values):
    """sha256 of the authoritative (owns_row) values in Key4 order — the form of the
    reference fixtures' whole-solution digests (tests/golden/make_golden.py digest_case)."""
    import hashlib
    keys = np.concatenate([lv.keys[np.flatnonzero(lv.owns_row)] for lv in level_arrays])
    vals = np.concatenate([v[np.flatnonzero(lv.owns_row)] for lv, v in zip(level_arrays, values)])
    order = np.lexsort(keys.T[::-1])
    return hashlib.sha256(np.ascontiguousarray(vals[order], np.float64).tobytes()).hexdigest()
