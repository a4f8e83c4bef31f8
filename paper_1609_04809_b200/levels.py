"""Host-side level data: the Python form of ``pf_level_desc`` (include/pf_gpu.h).

A ``LevelArrays`` is one rank's view of one ``MultigridLevel``
(/root/reference/proj/include/parfem/multigrid.hpp:15-31) in the reference's host
order: the level operator as CSR, the ParFEMapper fields the hot path reads
(n_own_dofs, owns_row, the Dirichlet class, the channels, femapper.hpp:45-70) and the
prolongation map (multigrid.cpp:35-72).
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np

from . import _lib


@dataclass
class Channel:
    kind: int
    peer: int
    send: np.ndarray  # int32, host order
    recv: np.ndarray  # int32, host order


@dataclass
class LevelArrays:
    n: int
    n_own: int
    row_offsets: np.ndarray
    cols: np.ndarray
    vals: np.ndarray
    owns_row: np.ndarray
    is_dir: np.ndarray
    color: np.ndarray | None = None
    channels: list = field(default_factory=list)
    p_offsets: np.ndarray | None = None
    p_cols: np.ndarray | None = None
    p_w: np.ndarray | None = None
    keys: np.ndarray | None = None      # (n, 4) int64: entity kind, lattice key
    class_of: np.ndarray | None = None  # uint8 DofClass
    order: np.ndarray | None = None     # int64 device placement hint (pf_level_desc.row_order)

    def normalized(self) -> "LevelArrays":
        def a(x, t):
            return None if x is None else np.ascontiguousarray(x, dtype=t)
        chans = [Channel(int(c.kind), int(c.peer), a(c.send, np.int32), a(c.recv, np.int32))
                 for c in self.channels]
        return LevelArrays(int(self.n), int(self.n_own), a(self.row_offsets, np.int64),
                           a(self.cols, np.int32), a(self.vals, np.float64),
                           a(self.owns_row, np.uint8), a(self.is_dir, np.uint8),
                           a(self.color, np.int32), chans, a(self.p_offsets, np.int64),
                           a(self.p_cols, np.int32), a(self.p_w, np.float64),
                           a(self.keys, np.int64), a(self.class_of, np.uint8), a(self.order, np.int64))

    def desc(self):
        """(LevelDesc, keepalive) pointing into this object's arrays."""
        L = self.normalized()
        chans = (_lib.ChannelDesc * max(len(L.channels), 1))()
        for i, c in enumerate(L.channels):
            chans[i] = _lib.ChannelDesc(c.kind, c.peer, len(c.send), len(c.recv),
                                        c.send.ctypes.data, c.recv.ctypes.data)
        p = lambda x: None if x is None else x.ctypes.data  # noqa: E731
        d = _lib.LevelDesc(L.n, L.n_own, p(L.row_offsets), p(L.cols), p(L.vals), p(L.owns_row),
                           p(L.is_dir), p(L.color), len(L.channels), chans, p(L.p_offsets),
                           p(L.p_cols), p(L.p_w), p(L.order))
        return d, (L, chans)


def _arr(ptr, n, ctype, dtype):
    if n == 0:
        return np.zeros(0, dtype)
    return np.ctypeslib.as_array(C.cast(ptr, C.POINTER(ctype)), shape=(n,)).astype(dtype, copy=True)


class StructuredSetup:
    """The product's communication-free setup (include/pf_setup.h) for one rank.

    problem = PF_PROBLEM_HEAT builds the Crank-Nicolson hierarchy of the reference's heat
    run (every level's system M + dt/2 K) and keeps the native setup alive for the time
    loop: `rhs_op`, `load_at(t)`, `load_desc()`, `scales(t)`."""

    def __init__(self, dim: int, n_coarse: int, n_levels: int, n_ranks: int = 1, rank: int = 0,
                 problem: int = _lib.PF_PROBLEM_BASELINE, dt: float | None = None, keep: bool = False,
                 seed: int = 1, direct_halos: bool = False, materialize: bool = True):
        L = _lib.lib()
        self._h = C.c_void_p()
        if direct_halos:
            o = _lib.SetupOptions(dim, n_coarse, n_levels, n_ranks, rank, problem,
                                  0.01 if dt is None else dt, seed, 1)
            _lib.check(L.pf_setup_create_opts(C.byref(o), C.byref(self._h)), setup=True)
        elif problem == _lib.PF_PROBLEM_HEAT:
            _lib.check(L.pf_setup_create_heat(dim, n_coarse, n_levels, n_ranks, rank,
                                              0.01 if dt is None else dt, C.byref(self._h)), setup=True)
        elif problem == _lib.PF_PROBLEM_LOGNORMAL:
            _lib.check(L.pf_setup_create_lognormal(dim, n_coarse, n_levels, n_ranks, rank, seed,
                                                   C.byref(self._h)), setup=True)
        else:
            _lib.check(L.pf_setup_create(dim, n_coarse, n_levels, n_ranks, rank, problem,
                                         C.byref(self._h)), setup=True)
        self.dim, self.n_coarse, self.n_levels = dim, n_coarse, n_levels
        self.n_ranks, self.rank, self.problem = n_ranks, rank, problem
        self.dt = dt if problem == _lib.PF_PROBLEM_HEAT else None
        if problem == _lib.PF_PROBLEM_HEAT and dt is None:
            self.dt = 0.01
        # materialize=False: no numpy copies of the level data (large grids); the native
        # setup stays alive and gmg.Hierarchy.from_setups reads it directly
        self.levels = [self._level(l) for l in range(n_levels)] if materialize else None
        self.sizes = []
        for l in range(n_levels):
            nd = C.c_int64()
            _lib.check(L.pf_setup_counts(self._h, l, None, C.byref(nd), None, None), setup=True)
            self.sizes.append(nd.value)
        bp, xp, n = C.c_void_p(), C.c_void_p(), C.c_int64()
        _lib.check(L.pf_setup_rhs(self._h, C.byref(bp), C.byref(xp), C.byref(n)), setup=True)
        self.b = _arr(bp, n.value, C.c_double, np.float64)
        self.x0 = _arr(xp, n.value, C.c_double, np.float64)
        ng = C.c_int64()
        _lib.check(L.pf_setup_counts(self._h, n_levels - 1, C.byref(ng), None, None, None), setup=True)
        self.n_global = ng.value
        s = C.c_double()
        _lib.check(L.pf_setup_seconds(self._h, C.byref(s)), setup=True)
        self.seconds = s.value
        self.rhs_op = None
        self.kappa = None
        if problem == _lib.PF_PROBLEM_LOGNORMAL:
            kp, kn = C.c_void_p(), C.c_int64()
            _lib.check(L.pf_setup_kappa(self._h, C.byref(kp), C.byref(kn)), setup=True)
            self.kappa = _arr(kp, kn.value, C.c_double, np.float64)
        if problem == _lib.PF_PROBLEM_HEAT:
            vp, nnz = C.c_void_p(), C.c_int64()
            _lib.check(L.pf_setup_rhs_operator(self._h, C.byref(vp), C.byref(nnz)), setup=True)
            self.rhs_op = _arr(vp, nnz.value, C.c_double, np.float64)
        elif not keep and materialize:
            self.close()

    def close(self):
        if self._h:
            _lib.lib().pf_setup_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _live(self):
        if not self._h:
            raise _lib.PfError("native setup released (heat setups, or keep=True, keep it)")
        return self._h

    def level_desc(self, l: int) -> _lib.LevelDesc:
        """Level l as the native setup holds it (pointers valid while this setup lives and
        until release_matrices)."""
        d = _lib.LevelDesc()
        _lib.check(_lib.lib().pf_setup_level(self._live(), l, C.byref(d)), setup=True)
        return d

    def release_matrices(self):
        _lib.check(_lib.lib().pf_setup_release_matrices(self._live()), setup=True)

    def load_at(self, t: float) -> np.ndarray:
        """Finest-level load at time t (assemble_load, assembly.cpp:144-160), host order,
        Dirichlet rows 0."""
        out = np.zeros(self.sizes[-1])
        _lib.check(_lib.lib().pf_setup_load_at(self._live(), t, out.ctypes.data, out.size), setup=True)
        return out

    def load_desc(self) -> _lib.LoadDesc:
        """The device load description (pointers valid while this setup lives)."""
        d = _lib.LoadDesc()
        _lib.check(_lib.lib().pf_setup_load_desc(self._live(), C.byref(d)), setup=True)
        return d

    def assembly_desc(self) -> _lib.AssemblyDesc:
        """The device assembly description of the finest level (pointers valid while this
        setup lives; needs keep=True for non-heat problems)."""
        d = _lib.AssemblyDesc()
        _lib.check(_lib.lib().pf_setup_assembly_desc(self._live(), C.byref(d)), setup=True)
        return d

    def scales(self, t: float):
        """(source_scale, has_dirichlet, dirichlet_scale) at time t, host libm."""
        s, g, hd = C.c_double(), C.c_double(), C.c_int32()
        _lib.check(_lib.lib().pf_setup_scales(self._live(), t, C.byref(s), C.byref(hd), C.byref(g)),
                   setup=True)
        return s.value, bool(hd.value), g.value

    def _level(self, l: int) -> LevelArrays:
        L = _lib.lib()
        d = _lib.LevelDesc()
        _lib.check(L.pf_setup_level(self._h, l, C.byref(d)), setup=True)
        n, n_own = d.n_dofs, d.n_own_dofs
        rp = _arr(d.row_offsets, n + 1, C.c_int64, np.int64)
        nnz = int(rp[-1])
        chans = []
        for i in range(d.n_channels):
            c = d.channels[i]
            chans.append(Channel(c.kind, c.peer, _arr(c.send_dofs, c.n_send, C.c_int32, np.int32),
                                 _arr(c.recv_dofs, c.n_recv, C.c_int32, np.int32)))
        kp, cp = C.c_void_p(), C.c_void_p()
        _lib.check(L.pf_setup_level_keys(self._h, l, C.byref(kp), C.byref(cp)), setup=True)
        out = LevelArrays(n, n_own, rp, _arr(d.col_indices, nnz, C.c_int32, np.int32),
                          _arr(d.values, nnz, C.c_double, np.float64),
                          _arr(d.owns_row, n, C.c_uint8, np.uint8),
                          _arr(d.is_dirichlet, n, C.c_uint8, np.uint8),
                          _arr(d.color, n_own, C.c_int32, np.int32), chans,
                          keys=_arr(kp, 4 * n, C.c_int64, np.int64).reshape(n, 4),
                          class_of=_arr(cp, n, C.c_uint8, np.uint8),
                          order=_arr(d.row_order, n, C.c_int64, np.int64) if d.row_order else None)
        if l > 0:
            out.p_offsets = _arr(d.p_offsets, n + 1, C.c_int64, np.int64)
            pn = int(out.p_offsets[-1])
            out.p_cols = _arr(d.p_cols, pn, C.c_int32, np.int32)
            out.p_w = _arr(d.p_weights, pn, C.c_double, np.float64)
        return out


def export_matrixmarket(setups, matrix_path: str, rhs_path: str):
    """export_system (app.cpp:379-396): the finest level of all ranks as MatrixMarket files,
    byte-identical to the reference's.  setups[r] = rank r, built with keep=True.
    Returns (n_global, nnz)."""
    arr = (C.c_void_p * len(setups))(*[s._live() for s in setups])
    ng, nz = C.c_int64(), C.c_int64()
    _lib.check(_lib.lib().pf_setup_export_matrixmarket(arr, len(setups), matrix_path.encode(),
                                                       rhs_path.encode(), C.byref(ng), C.byref(nz)), setup=True)
    return ng.value, nz.value
