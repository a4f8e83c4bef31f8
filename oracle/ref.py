"""ORACLE / TEST INFRASTRUCTURE — ctypes view of the compiled reference.

Loads ``oracle/_ref/libparfem_ref.so`` (the unmodified reference library built
from /root/reference/proj/src by oracle/Makefile, plus ref_driver.cpp) and
returns its level data and results as numpy arrays in the reference's host
order.  Only tests, ``__graft_entry__.smoke()`` and bench.py's CPU-baseline /
``--impl reference`` leg use this module.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "_ref", "libparfem_ref.so")
BRIDGE_PATH = os.path.join(HERE, "_ref", "libparfem_bridge.so")

_lib = None
_bridge = None


def available() -> bool:
    return os.path.exists(LIB_PATH)


def bridge_available() -> bool:
    return os.path.exists(BRIDGE_PATH)


def lib(bridge: bool = False):
    """The reference library; bridge=True: the same reference with solve_outer routed
    through integration/parfem_gpu_bridge.cpp into libpf_gpu.so (ref_set_gpu(1))."""
    global _lib, _bridge
    if bridge:
        if _bridge is None:
            if not bridge_available():
                raise FileNotFoundError(f"{BRIDGE_PATH} not built (make -C oracle bridge)")
            _bridge = _bind(C.CDLL(BRIDGE_PATH))
            _bridge.ref_set_gpu(1)
        return _bridge
    if _lib is None:
        if not available():
            raise FileNotFoundError(f"reference oracle not built: {LIB_PATH} (run make -C oracle)")
        _lib = _bind(C.CDLL(LIB_PATH))
    return _lib


def _bind(L):
    if True:
        P = C.c_void_p
        i64p = C.POINTER(C.c_int64)
        L.ref_last_error.restype = C.c_char_p
        L.ref_build.restype = P
        L.ref_build.argtypes = [C.c_int] * 5
        L.ref_free.argtypes = [P]
        L.ref_level_sizes.argtypes = [P, C.c_int, C.c_int, i64p]
        L.ref_level_copy.argtypes = [P, C.c_int, C.c_int] + [P] * 10
        L.ref_level_channels.argtypes = [P, C.c_int, C.c_int, P, P]
        L.ref_rhs.argtypes = [P, C.c_int, P, P]
        L.ref_key_noise.restype = C.c_double
        L.ref_key_noise.argtypes = [i64p, C.c_uint64]
        L.ref_run.argtypes = [C.c_int] * 8 + [C.c_double, C.c_int, C.c_int, C.c_double, C.c_int,
                                              P, P, P, C.c_int, C.POINTER(C.c_int), P]
        L.ref_bench.argtypes = [C.c_int] * 6 + [C.c_double, C.c_int, C.c_int, C.c_double,
                                                C.c_int, C.c_int, P, P, i64p, C.POINTER(C.c_int)]
        L.ref_set_gpu.argtypes = [C.c_int]
        L.ref_heat.restype = P
        L.ref_heat.argtypes = [C.c_int] * 4 + [C.c_double, C.c_double, C.c_int, C.c_double,
                                               C.c_int, C.c_int, C.c_double]
        L.ref_heat_info.argtypes = [P, i64p, C.POINTER(C.c_int), P, P, P]
        L.ref_heat_copy.argtypes = [P, P, P, P]
        L.ref_heat_free.argtypes = [P]
        L.ref_set_heat.argtypes = [C.c_double, C.c_int]
        L.ref_export.argtypes = [C.c_int] * 4 + [C.c_char_p]
        L.ref_heat_bench.argtypes = [C.c_int] * 4 + [C.c_double, C.c_int, C.c_double, C.c_int, C.c_int,
                                                     C.c_double, C.c_int, C.c_int, P, P, i64p,
                                                     C.POINTER(C.c_int)]
        L.ref_heat_data.argtypes = [P, C.c_int, P, P]
    return L


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(C.c_void_p)


@dataclass
class RefChannel:
    kind: int
    peer: int
    send: np.ndarray
    recv: np.ndarray


@dataclass
class RefLevel:
    n_dofs: int
    n_own: int
    n_global: int
    row_offsets: np.ndarray
    cols: np.ndarray
    vals: np.ndarray
    owns_row: np.ndarray
    class_of: np.ndarray
    keys: np.ndarray  # (n_dofs, 4): kind, key[0..2]
    global_of: np.ndarray
    channels: list = field(default_factory=list)
    p_offsets: np.ndarray | None = None
    p_cols: np.ndarray | None = None
    p_w: np.ndarray | None = None

    @property
    def is_dirichlet(self) -> np.ndarray:
        return (self.class_of == 7).astype(np.uint8)

    @property
    def n(self) -> int:
        return self.n_dofs

    def to_level_arrays(self, color=None):
        """The same level as the product's LevelArrays (host order unchanged)."""
        from paper_1609_04809_b200.levels import Channel, LevelArrays
        return LevelArrays(self.n_dofs, self.n_own, self.row_offsets, self.cols, self.vals,
                           self.owns_row, self.is_dirichlet, color,
                           [Channel(c.kind, c.peer, c.send, c.recv) for c in self.channels],
                           self.p_offsets, self.p_cols, self.p_w, self.keys, self.class_of)


@dataclass
class RefHierarchy:
    dim: int
    n_coarse: int
    n_levels: int
    K: int
    problem: int
    ranks: list  # ranks[r] = list of RefLevel, 0 = coarsest
    b: list      # finest rhs per rank (heat: load at t = 0)
    x0: list     # finest start vector per rank (heat: exact solution at t = 0)
    rhs_op: list | None = None  # heat: finest M - dt/2 K values per rank
    loads: list | None = None   # heat: per rank, [n_loads, n_dofs] loads at t_k = k dt


def build(dim: int, n_coarse: int, levels: int, K: int, problem: int = 0, *, dt: float = 0.01,
          n_loads: int = 2) -> RefHierarchy:
    """problem 3 (heat): the HeatCrankNicolson hierarchy with time step dt, plus the rhs
    operator and the loads at t_k = k dt, k = 1..n_loads."""
    L = lib()
    L.ref_set_heat(dt, n_loads)
    h = L.ref_build(dim, n_coarse, levels, K, problem)
    if not h:
        raise RuntimeError(L.ref_last_error().decode())
    try:
        ranks, bs, xs = [], [], []
        for r in range(K):
            lv = []
            for l in range(levels):
                s = np.zeros(7, np.int64)
                L.ref_level_sizes(h, r, l, s.ctypes.data_as(C.POINTER(C.c_int64)))
                n, n_own, nnz, pnnz, nch, ng, ne = (int(v) for v in s)
                d = RefLevel(n, n_own, ng,
                             np.zeros(n + 1, np.int64), np.zeros(nnz, np.int32), np.zeros(nnz),
                             np.zeros(n, np.uint8), np.zeros(n, np.uint8), np.zeros((n, 4), np.int64),
                             np.zeros(n, np.int64))
                if l > 0:
                    d.p_offsets = np.zeros(n + 1, np.int64)
                    d.p_cols = np.zeros(pnnz, np.int32)
                    d.p_w = np.zeros(pnnz)
                L.ref_level_copy(h, r, l, _ptr(d.row_offsets), _ptr(d.cols), _ptr(d.vals),
                                 _ptr(d.owns_row), _ptr(d.class_of), _ptr(d.keys), _ptr(d.global_of),
                                 _ptr(d.p_offsets) if l > 0 else None,
                                 _ptr(d.p_cols) if l > 0 else None,
                                 _ptr(d.p_w) if l > 0 else None)
                meta = np.zeros(max(4 * nch, 1), np.int32)
                ent = np.zeros(max(ne, 1), np.int32)
                L.ref_level_channels(h, r, l, _ptr(meta), _ptr(ent))
                e = 0
                for i in range(nch):
                    kind, peer, ns, nr = (int(v) for v in meta[4 * i:4 * i + 4])
                    d.channels.append(RefChannel(kind, peer, ent[e:e + ns].copy(),
                                                 ent[e + ns:e + ns + nr].copy()))
                    e += ns + nr
                lv.append(d)
            ranks.append(lv)
            n = lv[-1].n_dofs
            b = np.zeros(n)
            x0 = np.zeros(n)
            L.ref_rhs(h, r, _ptr(b), _ptr(x0))
            bs.append(b)
            xs.append(x0)
        out = RefHierarchy(dim, n_coarse, levels, K, problem, ranks, bs, xs)
        if problem == 3:
            out.rhs_op, out.loads = [], []
            for r in range(K):
                top = ranks[r][-1]
                op = np.zeros(len(top.vals))
                ld = np.zeros((n_loads, top.n_dofs))
                L.ref_heat_data(h, r, _ptr(op), _ptr(ld))
                out.rhs_op.append(op)
                out.loads.append(ld)
        return out
    finally:
        L.ref_free(h)


OP_SOLVE, OP_SMOOTH, OP_VCYCLE, OP_RESNORM, OP_RESIDUAL = range(5)


def run(dim, n_coarse, levels, K, *, problem=0, op=OP_SOLVE, n_ops=1, smoother=0, damping=0.8,
        pre=2, post=2, outer_tol=1e-10, max_cycles=100, x_in=None, sizes=None, gpu=False):
    """Run the reference hot path; returns (x_per_rank, residuals, stats dict).
    gpu=True: the unmodified reference with its solve_outer replaced by the GPU bridge."""
    L = lib(bridge=gpu)
    if sizes is None:
        hb = build(dim, n_coarse, levels, K, problem)
        sizes = [hb.ranks[r][-1].n_dofs for r in range(K)]
    xo = [np.zeros(n) for n in sizes]
    xo_ptrs = (C.c_void_p * K)(*[x.ctypes.data for x in xo])
    xi_ptrs = None
    if x_in is not None:
        x_in = [np.ascontiguousarray(x, np.float64) for x in x_in]
        xi_ptrs = (C.c_void_p * K)(*[x.ctypes.data for x in x_in])
    res = np.zeros(1000)
    nres = C.c_int(0)
    st = np.zeros(7)
    rc = L.ref_run(dim, n_coarse, levels, K, problem, op, n_ops, smoother, damping, pre, post,
                   outer_tol, max_cycles, xi_ptrs, xo_ptrs, _ptr(res), 1000, C.byref(nres), _ptr(st))
    stats = dict(iterations=int(st[0]), initial_residual=st[1], final_residual=st[2],
                 solve_seconds=st[3], setup_seconds=st[4], converged=bool(st[5]),
                 comm_seconds=st[6], status=rc,
                 error=L.ref_last_error().decode() if rc else "")
    return xo, res[:nres.value].copy(), stats


def bench(dim, n_coarse, levels, K, *, problem=0, smoother=0, damping=0.8, pre=2, post=2,
          outer_tol=1e-10, warmup=1, steps=1):
    L = lib()
    per = np.zeros(steps)
    setup = np.zeros(1)
    ng = C.c_int64(0)
    its = C.c_int(0)
    rc = L.ref_bench(dim, n_coarse, levels, K, problem, smoother, damping, pre, post, outer_tol,
                     warmup, steps, _ptr(per), _ptr(setup), C.byref(ng), C.byref(its))
    if rc:
        raise RuntimeError(L.ref_last_error().decode())
    return dict(step_seconds=per, setup_seconds=float(setup[0]), n_global=int(ng.value),
                iterations=int(its.value))


def key_noise(keys: np.ndarray, salt: int) -> np.ndarray:
    """The reference fixture key_noise (tests/support.cpp:17-25) for each Key4 row."""
    L = lib()
    keys = np.ascontiguousarray(keys, np.int64)
    out = np.empty(len(keys))
    for i in range(len(keys)):
        out[i] = L.ref_key_noise(keys[i].ctypes.data_as(C.POINTER(C.c_int64)), salt)
    return out


def heat(dim, n_coarse, levels, K, *, dt=0.01, end_time=0.05, smoother=0, damping=0.8, pre=2,
         post=2, outer_tol=1e-10):
    """The reference's own run_heat (app.cpp:146-230, :299-305): Crank-Nicolson over
    round(end_time/dt) steps.  Returns dict(solution={Key4: value} over all ranks,
    residuals=last solve's history, l2, linf, phases={...})."""
    L = lib()
    hv = L.ref_heat(dim, n_coarse, levels, K, dt, end_time, smoother, damping, pre, post, outer_tol)
    if not hv:
        raise RuntimeError(L.ref_last_error().decode())
    try:
        n = C.c_int64(0)
        nr = C.c_int(0)
        l2, linf, ph = np.zeros(1), np.zeros(1), np.zeros(5)
        L.ref_heat_info(hv, C.byref(n), C.byref(nr), _ptr(l2), _ptr(linf), _ptr(ph))
        keys = np.zeros((n.value, 4), np.int64)
        vals = np.zeros(n.value)
        res = np.zeros(max(nr.value, 1))
        L.ref_heat_copy(hv, _ptr(keys), _ptr(vals), _ptr(res))
    finally:
        L.ref_heat_free(hv)
    sol = {tuple(int(v) for v in k): float(x) for k, x in zip(keys, vals)}
    names = ("initialization", "assembling", "solving", "communication", "total")
    return dict(solution=sol, residuals=res[:nr.value], l2=float(l2[0]), linf=float(linf[0]),
                phases=dict(zip(names, ph.tolist())))


def heat_bench(dim, n_coarse, levels, K, *, dt=0.01, smoother=0, damping=0.8, pre=2, post=2,
               outer_tol=1e-10, warmup=0, steps=1):
    """Seconds per Crank-Nicolson step of the reference (heat_rank_body's loop body through
    its public functions), max over K rank threads."""
    L = lib()
    per = np.zeros(steps)
    setup = np.zeros(1)
    ng = C.c_int64(0)
    its = C.c_int(0)
    rc = L.ref_heat_bench(dim, n_coarse, levels, K, dt, smoother, damping, pre, post, outer_tol,
                          warmup, steps, _ptr(per), _ptr(setup), C.byref(ng), C.byref(its))
    if rc:
        raise RuntimeError(L.ref_last_error().decode())
    return dict(step_seconds=per, setup_seconds=float(setup[0]), n_global=int(ng.value),
                iterations=int(its.value))


def export(dim, n_coarse, levels, K, prefix: str) -> None:
    """The reference's export_system (app.cpp:379-396): writes prefix.mtx, prefix_rhs.mtx."""
    L = lib()
    if L.ref_export(dim, n_coarse, levels, K, prefix.encode()):
        raise RuntimeError(L.ref_last_error().decode())
