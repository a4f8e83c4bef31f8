"""ORACLE / TEST INFRASTRUCTURE — ctypes view of the C restatement (gmg_oracle.c).

Takes the same ``LevelArrays`` the product takes and runs the reference algorithm
on host arrays.  Only tests, smoke() and bench.py's cpu_baseline leg use it.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

from paper_1609_04809_b200 import _lib

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libpf_oracle.so")
ORC_SMOOTHER_LEX_GS = 3

_lib_o = None


def lib():
    global _lib_o
    if _lib_o is None:
        if not os.path.exists(LIB_PATH):
            raise FileNotFoundError(f"{LIB_PATH} missing (make -C oracle oracle)")
        L = C.CDLL(LIB_PATH)
        P = C.c_void_p
        L.orc_last_error.restype = C.c_char_p
        L.orc_create.argtypes = [C.c_int, C.c_int, C.POINTER(C.c_void_p)]
        L.orc_set_level.argtypes = [P, C.c_int, C.c_int, C.POINTER(_lib.LevelDesc)]
        L.orc_finalize.argtypes = [P]
        L.orc_set_coarse_direct.argtypes = [P, C.c_int]
        L.orc_set_colorwise.argtypes = [P, C.c_int]
        L.orc_destroy.argtypes = [P]
        L.orc_destroy.restype = None
        vec = P  # double* const*
        L.orc_spmv.argtypes = [P, C.c_int, vec, vec]
        L.orc_cycle_residual.argtypes = [P, C.c_int, vec, vec, vec]
        L.orc_residual_norm.argtypes = [P, C.c_int, vec, vec, C.POINTER(C.c_double)]
        L.orc_smooth.argtypes = [P, C.c_int, vec, vec, C.POINTER(_lib.SmootherConfig)]
        L.orc_coarse_solve.argtypes = [P, C.c_int, vec, vec, C.c_double, C.c_int,
                                       C.POINTER(_lib.SolveStats)]
        L.orc_prolongate.argtypes = [P, C.c_int, vec, vec]
        L.orc_restrict_residual.argtypes = [P, C.c_int, vec, vec]
        L.orc_update_master_slave.argtypes = [P, C.c_int, vec, C.c_int]
        L.orc_update_halo.argtypes = [P, C.c_int, C.c_int, vec]
        L.orc_v_cycle.argtypes = [P, vec, vec, C.POINTER(_lib.MultigridConfig),
                                  C.POINTER(_lib.SolveStats)]
        L.orc_solve_outer.argtypes = [P, vec, vec, C.POINTER(_lib.MultigridConfig),
                                      C.POINTER(_lib.SolveStats), C.POINTER(C.c_double), C.c_int]
        _lib_o = L
    return _lib_o


def _vec(arrs):
    return (C.c_void_p * len(arrs))(*[a.ctypes.data for a in arrs])


class Oracle:
    """K subdomains (ranks 0..K-1) of one hierarchy, host order, reference semantics."""

    def __init__(self, levels, coarse_direct=False, colorwise=False):
        L = lib()
        self.K, self.n_levels = len(levels), len(levels[0])
        self.sizes = [[lv.n for lv in sub] for sub in levels]
        self._h = C.c_void_p()
        self._check(L.orc_create(self.n_levels, self.K, C.byref(self._h)))
        for s, sub in enumerate(levels):
            for l, lv in enumerate(sub):
                d, keep = lv.desc()
                self._check(L.orc_set_level(self._h, l, s, C.byref(d)))
                del keep
        self._check(L.orc_finalize(self._h))
        if coarse_direct:
            self._check(L.orc_set_coarse_direct(self._h, 1))
        if colorwise:
            self._check(L.orc_set_colorwise(self._h, 1))

    @classmethod
    def from_level_descs(cls, descs, colorwise=False):
        """Oracle over raw pf_level_desc structs (descs[s][l]; e.g. pointers into a native
        setup, StructuredSetup.level_desc): no numpy copy of large levels."""
        self = cls.__new__(cls)
        L = lib()
        self.K, self.n_levels = len(descs), len(descs[0])
        self.sizes = [[int(d.n_dofs) for d in sub] for sub in descs]
        self._h = C.c_void_p()
        self._check(L.orc_create(self.n_levels, self.K, C.byref(self._h)))
        for s, sub in enumerate(descs):
            for l, d in enumerate(sub):
                self._check(L.orc_set_level(self._h, l, s, C.byref(d)))
        self._check(L.orc_finalize(self._h))
        if colorwise:
            self._check(L.orc_set_colorwise(self._h, 1))
        return self

    @staticmethod
    def _check(rc):
        if rc:
            raise RuntimeError(f"oracle error {rc}: {lib().orc_last_error().decode()}")

    def zeros(self, level):
        return [np.zeros(self.sizes[s][level]) for s in range(self.K)]

    @staticmethod
    def _own(arrs):
        return [np.ascontiguousarray(a, np.float64).copy() for a in arrs]

    def smooth(self, level, x, b, kind, sweeps=1, damping=0.8, local_sweeps=1):
        x = self._own(x)
        b = self._own(b)
        c = _lib.SmootherConfig(kind, sweeps, local_sweeps, damping)
        self._check(lib().orc_smooth(self._h, level, _vec(x), _vec(b), C.byref(c)))
        return x

    def residual_norm(self, level, x, b):
        out = C.c_double()
        x, b = self._own(x), self._own(b)
        self._check(lib().orc_residual_norm(self._h, level, _vec(x), _vec(b), C.byref(out)))
        return out.value

    def spmv(self, level, x):
        x = self._own(x)
        y = self.zeros(level)
        self._check(lib().orc_spmv(self._h, level, _vec(x), _vec(y)))
        return y

    def cycle_residual(self, level, x, b):
        x, b = self._own(x), self._own(b)
        r = self.zeros(level)
        self._check(lib().orc_cycle_residual(self._h, level, _vec(x), _vec(b), _vec(r)))
        return r

    def prolongate(self, fine, xc):
        xc = self._own(xc)
        out = self.zeros(fine)
        self._check(lib().orc_prolongate(self._h, fine, _vec(xc), _vec(out)))
        return out

    def restrict_residual(self, fine, r):
        r = self._own(r)
        rc = self.zeros(fine - 1)
        self._check(lib().orc_restrict_residual(self._h, fine, _vec(r), _vec(rc)))
        return rc

    def update_master_slave(self, level, v, mode):
        v = self._own(v)
        self._check(lib().orc_update_master_slave(self._h, level, _vec(v), mode))
        return v

    def update_halo(self, level, kind, v):
        v = self._own(v)
        self._check(lib().orc_update_halo(self._h, level, kind, _vec(v)))
        return v

    def coarse_solve(self, level, x, b, tol=1e-12, max_iter=20000):
        x, b = self._own(x), self._own(b)
        st = _lib.SolveStats()
        self._check(lib().orc_coarse_solve(self._h, level, _vec(x), _vec(b), tol, max_iter,
                                           C.byref(st)))
        return x, st

    def v_cycle(self, x, b, cfg):
        x, b = self._own(x), self._own(b)
        st = _lib.SolveStats()
        c = cfg.c()
        self._check(lib().orc_v_cycle(self._h, _vec(x), _vec(b), C.byref(c), C.byref(st)))
        return x, st

    def solve_outer(self, x, b, cfg):
        """Returns (x, residuals, stats, status); status 3 = NoConvergenceError."""
        x, b = self._own(x), self._own(b)
        st = _lib.SolveStats()
        c = cfg.c()
        res = np.zeros(max(cfg.outer_max_cycles, 1))
        rc = lib().orc_solve_outer(self._h, _vec(x), _vec(b), C.byref(c), C.byref(st),
                                   res.ctypes.data_as(C.POINTER(C.c_double)), res.size)
        if rc not in (0, 3):
            self._check(rc)
        return x, res[:st.iterations].copy(), st, rc

    def __del__(self):
        try:
            if self._h:
                lib().orc_destroy(self._h)
                self._h = None
        except Exception:
            pass


# ------------------------------------------------------------ heat (Crank-Nicolson) --

def csr_spmv(row_offsets, cols, vals, x):
    """spmv (linalg.cpp:45-57): every row summed serially in stored order from 0.0
    (numpy elementwise products and sums are single IEEE operations, no contraction)."""
    n = len(row_offsets) - 1
    lens = np.diff(row_offsets)
    y = np.zeros(n)
    for j in range(int(lens.max()) if n else 0):
        m = lens > j
        e = row_offsets[:-1][m] + j
        y[m] = y[m] + vals[e] * x[cols[e]]
    return y


def heat_exact(keys, denom, dim, t):
    """HeatProblem::exact (model.cpp:11-22) at the dof coordinates key / denom
    (fespace.cpp:66-70), with the host libm like the reference."""
    import math
    out = np.empty(len(keys))
    e = math.exp(-0.1 * t)
    for i, k in enumerate(keys):
        x = [float(k[1]) / denom, float(k[2]) / denom, float(k[3]) / denom]
        u = math.sin(math.pi * x[0]) * math.cos(math.pi * x[1])
        if dim == 3:
            u *= math.cos(math.pi * x[2])
        out[i] = e * u
    return out


def heat_loop(oracle, tops, rhs_ops, u0, load0, loads, dt, steps, cfg, dim, denom):
    """heat_rank_body's time loop (app.cpp:180-213) composed from the restated pieces:
    the reference's own rhs operator values and loads (per rank: loads[r][k] at t_{k+1}),
    csr_spmv, the Dirichlet rows from heat_exact, and Oracle.solve_outer.
    Returns (u per rank, last residual history)."""
    K = len(tops)
    u = [np.array(a, np.float64) for a in u0]
    ln = [np.array(a, np.float64) for a in load0]
    res = None
    for k in range(steps):
        t = float(k + 1) * dt
        b = []
        for r in range(K):
            lv = tops[r]
            br = csr_spmv(lv.row_offsets, lv.cols, rhs_ops[r], u[r])
            br = br + 0.5 * dt * (ln[r] + loads[r][k])
            dir_rows = np.flatnonzero(lv.class_of == 7)
            g = heat_exact(lv.keys[dir_rows], denom, dim, t)
            br[dir_rows] = g
            u[r][dir_rows] = g
            b.append(br)
        u, res, st, rc = oracle.solve_outer(u, b, cfg)
        if rc == 3:
            raise RuntimeError(f"time step {k + 1}: no convergence")
        ln = [loads[r][k] for r in range(K)]
    return u, res
