"""The reference's Crank-Nicolson heat run on the B200.

    reference (C++)                                  here
    ------------------------------------------------ -----------------------------------------
    rhs_op = M - dt/2 K              app.cpp:185-189 Operator(h, level, values)
    assemble_load(mapper, comm, f, t) assembly.cpp:144-160
                                                     assemble_load(load, source_scale, out)
    apply_dirichlet_rhs(b, g, t, mapper) assembly.cpp:172-179
                                                     apply_dirichlet_rhs(load, has, scale, b, u)
    spmv + b += dt/2 (ln + lnx) + Dirichlet          cn_rhs(op, load, u, ln, lnx, dt/2, ..., b, u)
                                     app.cpp:191-200
    the time loop of heat_rank_body  app.cpp:180-213 heat_run(h, op, load, u, load_now, ...)
    run_heat (one rank per thread)   app.cpp:299-305 HeatRun(...).run(...)

The load f(t, x) = s(t) * profile(x) is assembled on the device from per-axis factor
tables (pf_load_desc); s(t) and the boundary scale are evaluated on the host with the
same libm as the reference, so the device products equal the reference's bit for bit.
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import _lib
from .gmg import DeviceVector, Hierarchy, MultigridConfig, NoConvergenceError, SolveStats
from .levels import StructuredSetup


def time_steps(end_time: float, dt: float) -> int:
    """AppConfig::time_steps (config.cpp:47-50): round(end_time / dt), at least 1."""
    x = end_time / dt
    n = int(x)
    if x - n >= 0.5:  # llround: halves away from zero
        n += 1
    return max(n, 1)


class Operator:
    """A second matrix on a level's sparsity pattern (pf_operator_create)."""

    def __init__(self, h: Hierarchy, level: int, values=()):
        self.h, self.level = h, level
        self._p = C.c_void_p()
        _lib.check(_lib.lib().pf_operator_create(h._h, level, C.byref(self._p)))
        h._vectors.add(self)
        for s, v in enumerate(values):
            a = np.ascontiguousarray(v, np.float64)
            _lib.check(_lib.lib().pf_operator_set_values(self._p, s, a.ctypes.data, a.size))

    def apply(self, x: DeviceVector, y: DeviceVector) -> None:
        """spmv (linalg.cpp:45-57) with this operator."""
        _lib.check(_lib.lib().pf_operator_apply(self._p, x._p, y._p))

    def values(self, sub: int, nnz: int) -> np.ndarray:
        """The values of one subdomain in its level desc's CSR entry order."""
        out = np.empty(nnz)
        _lib.check(_lib.lib().pf_operator_get_values(self._p, sub, out.ctypes.data, nnz))
        return out

    def close(self):
        if self._p:
            _lib.lib().pf_operator_destroy(self._p)
            self._p = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class Load:
    """The finest-level load description on the device (pf_load_create / pf_load_set)."""

    def __init__(self, h: Hierarchy, level: int, descs):
        self.h, self.level = h, level
        self._p = C.c_void_p()
        _lib.check(_lib.lib().pf_load_create(h._h, level, C.byref(self._p)))
        h._vectors.add(self)
        for s, d in enumerate(descs):
            _lib.check(_lib.lib().pf_load_set(self._p, s, C.byref(d)))

    def close(self):
        if self._p:
            _lib.lib().pf_load_destroy(self._p)
            self._p = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def assemble_load(load: Load, source_scale: float, out: DeviceVector) -> None:
    _lib.check(_lib.lib().pf_load_assemble(load._p, source_scale, out._p))


def apply_dirichlet_rhs(load: Load, has_dirichlet: bool, scale: float, b: DeviceVector,
                        u: DeviceVector | None = None) -> None:
    _lib.check(_lib.lib().pf_load_apply_dirichlet(load._p, int(has_dirichlet), scale, b._p,
                                                  u._p if u is not None else None))


def cn_rhs(op: Operator, load: Load, u_in: DeviceVector, load_now: DeviceVector,
           load_next: DeviceVector, half_dt: float, has_dirichlet: bool, scale: float,
           b: DeviceVector, u: DeviceVector | None = None) -> None:
    _lib.check(_lib.lib().pf_cn_rhs(op._p, load._p, u_in._p, load_now._p, load_next._p, half_dt,
                                    int(has_dirichlet), scale, b._p, u._p if u is not None else None))


def heat_run(h: Hierarchy, op: Operator, load: Load, u: DeviceVector, load_now: DeviceVector,
             steps: int, dt: float, scales, cfg: MultigridConfig, first_step: int = 0) -> SolveStats:
    """The time loop of heat_rank_body (app.cpp:180-213) in one library call: steps
    first_step+1 .. first_step+steps.

    scales[k] = (source_scale, has_dirichlet, dirichlet_scale) of step first_step+k+1.
    Returns the last step's solve statistics; raises NoConvergenceError("time step k: ...")."""
    s = np.array([sc[0] for sc in scales[:steps]], np.float64)
    has = bool(scales[0][1]) if steps else False
    g = np.array([sc[2] for sc in scales[:steps]], np.float64)
    st = _lib.SolveStats()
    c = cfg.c()
    res = np.zeros(max(cfg.outer_max_cycles, 1))
    failed = C.c_int(0)
    dp = C.POINTER(C.c_double)
    rc = _lib.lib().pf_heat_run(h._h, op._p, load._p, u._p, load_now._p, first_step, steps, 0.5 * dt,
                                s.ctypes.data_as(dp), int(has), g.ctypes.data_as(dp), C.byref(c),
                                C.byref(st), res.ctypes.data_as(dp), res.size, C.byref(failed))
    stats = SolveStats.from_c(st, res[:st.iterations])
    if rc == _lib.PF_ERR_NO_CONVERGENCE:
        err = NoConvergenceError(_lib.lib().pf_last_error().decode())
        err.stats, err.step = stats, failed.value
        raise err
    _lib.check(rc)
    return stats


class HeatRun:
    """heat_rank_body (app.cpp:146-230) for the given ranks on one device: product setup
    (StructuredSetup with the heat problem), device hierarchy, rhs operator, load, u(0)
    and load(0) resident in HBM."""

    def __init__(self, dim: int, n_coarse: int, n_levels: int, dt: float, n_ranks: int = 1,
                 ranks: list | None = None, device: int = 0, world_size: int | None = None,
                 coarse_replicas=None):
        ranks = list(range(n_ranks)) if ranks is None else ranks
        self.dt = dt
        self.setups = [StructuredSetup(dim, n_coarse, n_levels, n_ranks, r, _lib.PF_PROBLEM_HEAT, dt=dt)
                       for r in ranks]
        self.h = Hierarchy([s.levels for s in self.setups], device=device, rank_base=ranks[0],
                           world_size=n_ranks if world_size is None else world_size,
                           coarse_replicas=coarse_replicas)
        top = self.h.finest
        self.op = Operator(self.h, top, [s.rhs_op for s in self.setups])
        self.load = Load(self.h, top, [s.load_desc() for s in self.setups])
        self.u = self.h.vector(top, [s.x0 for s in self.setups])
        self.load_now = self.h.vector(top, [s.b for s in self.setups])
        self.t = 0.0
        self.step = 0

    def reset(self):
        """Back to u(0), load(0)."""
        for i, s in enumerate(self.setups):
            self.u.upload(s.x0, i)
            self.load_now.upload(s.b, i)
        self.t, self.step = 0.0, 0

    def scales(self, steps: int):
        return [self.setups[0].scales(float(self.step + k + 1) * self.dt) for k in range(steps)]

    def run(self, steps: int, cfg: MultigridConfig) -> SolveStats:
        sc = self.scales(steps)
        st = heat_run(self.h, self.op, self.load, self.u, self.load_now, steps, self.dt, sc, cfg,
                      first_step=self.step)
        self.step += steps
        self.t = float(self.step) * self.dt
        return st

    def solution(self):
        return [self.u.download(i) for i in range(len(self.setups))]

    def keyed(self) -> dict:
        """{Key4: value} over the authoritative dofs (gather_solution, app.cpp:56-88)."""
        out = {}
        for s, u in zip(self.setups, self.solution()):
            lv = s.levels[-1]
            for i in np.flatnonzero(lv.owns_row):
                out[tuple(int(k) for k in lv.keys[i])] = float(u[i])
        return out

    def close(self):
        self.h.close()
        for s in self.setups:
            s.close()


class Assembly:
    """Device assembly of a level's stiffness system (pf_assembly_*; assemble_system +
    apply_dirichlet_rows, assembly.cpp:103-170): Q1 with an optional per-cell coefficient
    (pf_assembly_desc), or Q2 / rotated Q1 (pf_fe_assembly_desc, FESetup.assembly_desc)."""

    def __init__(self, h: Hierarchy, level: int, descs):
        self.h, self.level = h, level
        self._p = C.c_void_p()
        _lib.check(_lib.lib().pf_assembly_create(h._h, level, C.byref(self._p)))
        h._vectors.add(self)
        for s, d in enumerate(descs):
            if isinstance(d, _lib.FeAssemblyDesc):  # Q2 / rotated Q1 (pf_fe.h)
                _lib.check(_lib.lib().pf_fe_assembly_set(self._p, s, C.byref(d)))
            else:
                _lib.check(_lib.lib().pf_assembly_set(self._p, s, C.byref(d)))

    def assemble(self, op: Operator) -> Operator:
        _lib.check(_lib.lib().pf_assemble_operator(self._p, op._p))
        return op

    def close(self):
        if self._p:
            _lib.lib().pf_assembly_destroy(self._p)
            self._p = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
