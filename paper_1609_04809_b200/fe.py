"""The Q2 and rotated-Q1 (Rannacher-Turek) hierarchies of BASELINE configs[2] and
configs[3] (include/pf_fe.h).  ``FESetup.levels`` are ordinary
``LevelArrays``: the same V-cycle (gmg.Hierarchy) and the same oracle run on them."""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import _lib
from .levels import Channel, LevelArrays, _arr

Q2, ROTATED_Q1 = _lib.PF_FE_Q2, _lib.PF_FE_ROTATED_Q1
CONSTANT, LOGNORMAL = _lib.PF_COEF_CONSTANT, _lib.PF_COEF_LOGNORMAL


class FESetup:
    """One-subdomain hierarchy of `family` on n_coarse^3 cells refined n_levels - 1 times;
    rhs f = 3 pi^2 sin sin sin, g = 0, x0 = 0.  `exact` holds the dof values of the
    constant-coefficient solution sin(pi x) sin(pi y) sin(pi z)."""

    def __init__(self, family: int, n_coarse: int, n_levels: int, coefficient: int = CONSTANT,
                 seed: int = 2024, keep: bool = False, n_ranks: int = 1, rank: int = 0):
        L = _lib.lib()
        self._h = C.c_void_p()
        _lib.check(L.pf_fe_setup_create_part(family, n_coarse, n_levels, coefficient, seed, n_ranks, rank,
                                             C.byref(self._h)), setup="fe")
        self.n_ranks, self.rank = n_ranks, rank
        self.family, self.n_coarse, self.n_levels = family, n_coarse, n_levels
        self.coefficient, self.seed = coefficient, seed
        try:
            self.levels = [self._level(l) for l in range(n_levels)]
            bp, xp, ep, n = C.c_void_p(), C.c_void_p(), C.c_void_p(), C.c_int64()
            _lib.check(L.pf_fe_setup_rhs(self._h, C.byref(bp), C.byref(xp), C.byref(ep), C.byref(n)),
                       setup="fe")
            self.b = _arr(bp, n.value, C.c_double, np.float64)
            self.x0 = _arr(xp, n.value, C.c_double, np.float64)
            self.exact = _arr(ep, n.value, C.c_double, np.float64)
            kp, kn = C.c_void_p(), C.c_int64()
            _lib.check(L.pf_fe_setup_kappa(self._h, C.byref(kp), C.byref(kn)), setup="fe")
            self.kappa = _arr(kp, kn.value, C.c_double, np.float64)
            s = C.c_double()
            _lib.check(L.pf_fe_setup_seconds(self._h, C.byref(s)), setup="fe")
            self.seconds = s.value
        except BaseException:
            self.close()
            raise
        if not keep:
            self.close()
        self.n_global = self.levels[-1].n

    def close(self):
        if self._h:
            _lib.lib().pf_fe_setup_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def assembly_desc(self, level: int) -> _lib.FeAssemblyDesc:
        """The device assembly description of a level (needs keep=True; pointers valid while
        this setup lives)."""
        if not self._h:
            raise _lib.PfError("native setup released: build it with keep=True")
        d = _lib.FeAssemblyDesc()
        _lib.check(_lib.lib().pf_fe_setup_assembly_desc(self._h, level, C.byref(d)), setup="fe")
        return d

    def _level(self, l: int) -> LevelArrays:
        L = _lib.lib()
        d = _lib.LevelDesc()
        _lib.check(L.pf_fe_setup_level(self._h, l, C.byref(d)), setup="fe")
        n, n_own = d.n_dofs, d.n_own_dofs
        rp = _arr(d.row_offsets, n + 1, C.c_int64, np.int64)
        nnz = int(rp[-1])
        kp, cp = C.c_void_p(), C.c_void_p()
        _lib.check(L.pf_fe_setup_level_keys(self._h, l, C.byref(kp), C.byref(cp)), setup="fe")
        chans = []
        for i in range(d.n_channels):
            c = d.channels[i]
            chans.append(Channel(c.kind, c.peer, _arr(c.send_dofs, c.n_send, C.c_int32, np.int32),
                                 _arr(c.recv_dofs, c.n_recv, C.c_int32, np.int32)))
        out = LevelArrays(n, n_own, rp, _arr(d.col_indices, nnz, C.c_int32, np.int32),
                          _arr(d.values, nnz, C.c_double, np.float64),
                          _arr(d.owns_row, n, C.c_uint8, np.uint8),
                          _arr(d.is_dirichlet, n, C.c_uint8, np.uint8),
                          _arr(d.color, n_own, C.c_int32, np.int32), chans,
                          keys=_arr(kp, 4 * n, C.c_int64, np.int64).reshape(n, 4),
                          class_of=_arr(cp, n, C.c_uint8, np.uint8),
                          order=_arr(d.row_order, n, C.c_int64, np.int64))
        if l > 0:
            out.p_offsets = _arr(d.p_offsets, n + 1, C.c_int64, np.int64)
            pn = int(out.p_offsets[-1])
            out.p_cols = _arr(d.p_cols, pn, C.c_int32, np.int32)
            out.p_w = _arr(d.p_weights, pn, C.c_double, np.float64)
        return out
