"""Host-side mirror of the reference's multigrid / linear-algebra / communicator API.

Names, argument meaning and error behaviour follow /root/reference/proj:

    reference (C++)                                  here (Python, device-resident data)
    ------------------------------------------------ -----------------------------------------
    build_hierarchy            multigrid.cpp:76-119  Hierarchy(levels_per_subdomain, ...)
    DistributedVector          fecomm.hpp:16-26      DeviceVector (hierarchy.vector(level))
    spmv                       linalg.cpp:45-57      spmv(h, level, x, y)
    residual_norm              linalg.cpp:59-74      residual_norm(h, level, x, b)
    smooth                     solvers.cpp:56-68     smooth(h, level, x, b, SmootherConfig)
    coarse_solve               solvers.cpp:70-92     coarse_solve(h, level, x, b, tol, max_iter)
    prolongate                 multigrid.cpp:121-129 prolongate(h, fine, coarse, out)
    restrict_residual          multigrid.cpp:131-146 restrict_residual(h, fine, r, rc)
    v_cycle                    multigrid.cpp:194-208 v_cycle(h, x, b, MultigridConfig)
    solve_outer                multigrid.cpp:210-246 solve_outer(h, x, b, MultigridConfig)
    ParFECommunicator::update_* fecomm.cpp:41-72     update_master_slave / update_halo1 / _halo2
    allreduce_sum              transport.cpp:163-165 allreduce_sum(h, values)

All computation happens in libpf_gpu.so on the B200; this module only moves
descriptors and host arrays across the C ABI.  Errors raise the Python mirror of the
reference's exception (``_lib.SingularDiagonalError``, ``_lib.NoConvergenceError``,
``_lib.TransportError``, ``_lib.InvalidArgument``).
"""
from __future__ import annotations

import ctypes as C
import weakref
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from ._lib import (PF_SMOOTHER_GAUSS_SEIDEL, PF_SMOOTHER_JACOBI,  # noqa: F401
                   PF_SMOOTHER_MULTICOLOR_SOR, PF_UPDATE_ACCUMULATE_THEN_SCATTER,
                   PF_UPDATE_SCATTER, NoConvergenceError, SingularDiagonalError, TransportError)
from .levels import LevelArrays, StructuredSetup  # noqa: F401

SMOOTHERS = {"jacobi": PF_SMOOTHER_JACOBI, "gauss_seidel": PF_SMOOTHER_GAUSS_SEIDEL,
             "multicolor_sor": PF_SMOOTHER_MULTICOLOR_SOR}


@dataclass
class SmootherConfig:
    """parfem::SmootherConfig (solvers.hpp:9-14)."""
    kind: int = PF_SMOOTHER_GAUSS_SEIDEL
    sweeps: int = 3
    local_sweeps: int = 1
    damping: float = 0.8

    def c(self) -> _lib.SmootherConfig:
        return _lib.SmootherConfig(self.kind, self.sweeps, self.local_sweeps, self.damping)


@dataclass
class MultigridConfig:
    """parfem::MultigridConfig (multigrid.hpp:53-62)."""
    cycles: int = 1
    smoother: SmootherConfig = field(default_factory=SmootherConfig)
    pre_smooth: int = 3
    post_smooth: int = 3
    coarse_tol: float = 1e-12
    coarse_max_iter: int = 20000
    outer_tol: float = 1e-9
    outer_max_cycles: int = 100

    def c(self) -> _lib.MultigridConfig:
        return _lib.MultigridConfig(self.cycles, self.smoother.c(), self.pre_smooth, self.post_smooth,
                                    self.coarse_tol, self.coarse_max_iter, self.outer_tol,
                                    self.outer_max_cycles)


@dataclass
class SolveStats:
    """parfem::SolveStats (linalg.hpp:37-45)."""
    iterations: int = 0
    initial_residual: float = 0.0
    final_residual: float = 0.0
    converged: bool = True
    residuals: list = field(default_factory=list)
    solve_seconds: float = 0.0
    comm_seconds: float = 0.0

    @classmethod
    def from_c(cls, s: _lib.SolveStats, residuals=()):
        return cls(s.iterations, s.initial_residual, s.final_residual, bool(s.converged),
                   list(residuals), s.solve_seconds, s.comm_seconds)


class DeviceVector:
    """A level's DistributedVector held on the device (one array per local subdomain)."""

    def __init__(self, h: "Hierarchy", level: int):
        self.h, self.level = h, level
        self._p = C.c_void_p()
        _lib.check(_lib.lib().pf_vector_create(h._h, level, C.byref(self._p)))
        h._vectors.add(self)

    def upload(self, values, sub: int = 0) -> "DeviceVector":
        a = np.ascontiguousarray(values, np.float64)
        _lib.check(_lib.lib().pf_vector_upload(self._p, sub, a.ctypes.data, a.size))
        return self

    def download(self, sub: int = 0, out: np.ndarray | None = None) -> np.ndarray:
        """Host-order copy of subdomain `sub`; into `out` (contiguous float64, e.g. a pinned
        buffer) when given, else into a new array."""
        n = self.h.n_dofs(self.level, sub)
        if out is None:
            out = np.empty(n)
        elif out.dtype != np.float64 or out.size != n or not out.flags.c_contiguous:
            raise ValueError(f"out must be a contiguous float64 array of {n} entries")
        _lib.check(_lib.lib().pf_vector_download(self._p, sub, out.ctypes.data, out.size))
        return out

    def fill(self, value: float) -> "DeviceVector":
        _lib.check(_lib.lib().pf_vector_fill(self._p, value))
        return self

    def copy_from(self, src: "DeviceVector") -> "DeviceVector":
        _lib.check(_lib.lib().pf_vector_copy(src._p, self._p))
        return self

    def close(self):
        if self._p:
            _lib.lib().pf_vector_destroy(self._p)
            self._p = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class LoopbackHub:
    """Shared transport of several single-subdomain hierarchies on one GPU (the
    single-GPU test bench of the multi-process path, include/pf_gpu.h)."""

    def __init__(self, world_size: int):
        self._p = C.c_void_p()
        _lib.check(_lib.lib().pf_loopback_create(world_size, C.byref(self._p)))

    def close(self):
        if self._p:
            _lib.lib().pf_loopback_destroy(self._p)
            self._p = C.c_void_p()


class Hierarchy:
    """Device mirror of MultigridHierarchy (multigrid.hpp:43-51).

    ``levels[s][l]`` is LevelArrays of local subdomain s (= rank rank_base + s) at level l
    (0 = coarsest).  Several subdomains on one device stand in for several ranks; with one
    process per GPU pass one subdomain, its rank and world_size, then call init_nccl.
    """

    def __init__(self, levels, device: int = 0, rank_base: int = 0, world_size: int | None = None,
                 finalize: bool = True, coarse_replicas=None, fused_exchanges: bool = False,
                 options: dict | None = None):
        n_sub = len(levels)
        n_levels = len(levels[0])
        world = n_sub if world_size is None else world_size
        L = _lib.lib()
        self._h = C.c_void_p()
        self._vectors = weakref.WeakSet()
        _lib.check(L.pf_hierarchy_create(device, n_levels, n_sub, rank_base, world, C.byref(self._h)))
        self.n_levels, self.n_sub, self.rank_base, self.world = n_levels, n_sub, rank_base, world
        for k, v in (options or {}).items():
            self.set_option(k, v)
        self._sizes = [[lv.n for lv in sub] for sub in levels]
        for s, sub in enumerate(levels):
            for l, lv in enumerate(sub):
                d, keep = lv.desc()
                _lib.check(L.pf_hierarchy_set_level(self._h, l, s, C.byref(d)))
                del keep
        if coarse_replicas is not None:
            # multi-process runs: coarse_replicas[r] = rank r's level 0, or the list of its
            # levels 0..top (the replicated bottom of the V-cycle)
            for r, lvs in enumerate(coarse_replicas):
                for l, lv in enumerate(lvs if isinstance(lvs, (list, tuple)) else [lvs]):
                    d, keep = lv.desc()
                    _lib.check(L.pf_hierarchy_set_replica_level(self._h, l, r, C.byref(d)))
                    del keep
        if fused_exchanges:
            _lib.check(L.pf_hierarchy_set_fused_exchanges(self._h, 1))
        if finalize:
            self.finalize()

    @classmethod
    def from_setups(cls, setups, device: int = 0, rank_base: int = 0, world_size: int | None = None,
                    coarse_replicas=None, fused_exchanges: bool = False, options: dict | None = None) -> "Hierarchy":
        """A hierarchy straight from native StructuredSetups (materialize=False): the level
        arrays move from each setup into the hierarchy and on to the device, without numpy
        copies or a second host copy (large grids: 512^3 fits in host memory)."""
        self = cls.__new__(cls)
        L = _lib.lib()
        n_sub, n_levels = len(setups), setups[0].n_levels
        world = n_sub if world_size is None else world_size
        self._h = C.c_void_p()
        self._vectors = weakref.WeakSet()
        _lib.check(L.pf_hierarchy_create(device, n_levels, n_sub, rank_base, world, C.byref(self._h)))
        self.n_levels, self.n_sub, self.rank_base, self.world = n_levels, n_sub, rank_base, world
        for k, v in (options or {}).items():
            self.set_option(k, v)
        self._sizes = [list(s.sizes) for s in setups]
        for si, s in enumerate(setups):
            for l in range(n_levels):  # the arrays move from the setup: one host copy
                _lib.check(L.pf_hierarchy_set_level_from_setup(self._h, l, si, s._live()))
        if coarse_replicas is not None:
            for r, lvs in enumerate(coarse_replicas):
                for l, lv in enumerate(lvs if isinstance(lvs, (list, tuple)) else [lvs]):
                    d, keep = lv.desc()
                    _lib.check(L.pf_hierarchy_set_replica_level(self._h, l, r, C.byref(d)))
                    del keep
        if fused_exchanges:
            _lib.check(L.pf_hierarchy_set_fused_exchanges(self._h, 1))
        self.finalize()
        return self

    def set_option(self, name: str, value: int) -> "Hierarchy":
        """pf_hierarchy_set_option: a tuning option of this hierarchy (option_names())."""
        _lib.check(_lib.lib().pf_hierarchy_set_option(self._h, name.encode(), int(value)))
        return self

    def get_option(self, name: str) -> int:
        out = C.c_int64()
        _lib.check(_lib.lib().pf_hierarchy_get_option(self._h, name.encode(), C.byref(out)))
        return out.value

    def finalize(self):
        _lib.check(_lib.lib().pf_hierarchy_finalize(self._h))

    def init_nccl(self, unique_id: bytes):
        buf = C.create_string_buffer(unique_id, len(unique_id))
        _lib.check(_lib.lib().pf_hierarchy_init_nccl(self._h, buf, len(unique_id)))

    def init_loopback(self, hub: "LoopbackHub"):
        _lib.check(_lib.lib().pf_hierarchy_init_loopback(self._h, hub._p))

    def peer_export(self) -> bytes:
        """This rank's peer-transport blob (pf_hierarchy_peer_export): allocates the
        peer-visible exchange arena; allgather the blobs and pass them to init_peer."""
        n = C.c_int64(0)
        _lib.check(_lib.lib().pf_hierarchy_peer_export(self._h, None, 0, C.byref(n)))
        buf = C.create_string_buffer(n.value)
        _lib.check(_lib.lib().pf_hierarchy_peer_export(self._h, buf, n.value, C.byref(n)))
        return buf.raw[:n.value]

    def init_peer(self, blobs) -> None:
        """Activate the peer-memory transport from every rank's blob (rank order): each
        exchange becomes one kernel storing into the peers' mapped memory (CUDA IPC across
        processes / NVLink), capturable into the solve graph."""
        stride = max(len(b) for b in blobs)
        buf = C.create_string_buffer(b"".join(b.ljust(stride, b"\0") for b in blobs), stride * len(blobs))
        _lib.check(_lib.lib().pf_hierarchy_init_peer(self._h, buf, stride))

    def drop_transport(self) -> None:
        """Detach the transport (every rank together) so another can be attached."""
        _lib.check(_lib.lib().pf_hierarchy_drop_transport(self._h))

    @staticmethod
    def nccl_unique_id() -> bytes:
        buf = C.create_string_buffer(128)
        _lib.check(_lib.lib().pf_nccl_unique_id(buf, 128))
        return buf.raw

    @property
    def finest(self) -> int:
        return self.n_levels - 1

    def n_dofs(self, level: int, sub: int = 0) -> int:
        return self._sizes[sub][level]

    def vector(self, level: int | None = None, values=None) -> DeviceVector:
        v = DeviceVector(self, self.finest if level is None else level)
        if values is not None:
            if isinstance(values, (list, tuple)):
                for s, a in enumerate(values):
                    v.upload(a, s)
            else:
                v.upload(values, 0)
        return v

    def set_colorwise_exchange(self, on: bool = True) -> "Hierarchy":
        """Coloured smoothers exchange after every colour (pf_hierarchy_set_colorwise_exchange):
        a K-subdomain sweep then relaxes like the single-domain coloured sweep."""
        _lib.check(_lib.lib().pf_hierarchy_set_colorwise_exchange(self._h, 1 if on else 0))
        return self

    def set_coarse_direct(self, on: bool = True) -> "Hierarchy":
        """Direct coarse solve on level 0 (pf_hierarchy_set_coarse_direct): one subdomain."""
        _lib.check(_lib.lib().pf_hierarchy_set_coarse_direct(self._h, 1 if on else 0))
        return self

    def device_bytes(self) -> int:
        out = C.c_int64()
        _lib.check(_lib.lib().pf_hierarchy_device_bytes(self._h, C.byref(out)))
        return out.value

    def level_info(self, level: int, sub: int = 0) -> dict:
        a, b, c, d = C.c_int64(), C.c_int64(), C.c_int64(), C.c_int64()
        _lib.check(_lib.lib().pf_level_info(self._h, level, sub, C.byref(a), C.byref(b), C.byref(c),
                                            C.byref(d)))
        return dict(n_dofs=a.value, n_own=b.value, nnz=c.value, n_colors=d.value)

    def stream_handle(self) -> int:
        """cudaStream_t of this hierarchy (an int for torch.cuda.ExternalStream)."""
        out = C.c_void_p()
        _lib.check(_lib.lib().pf_hierarchy_stream(self._h, C.byref(out)))
        return out.value or 0

    def launch_count(self) -> int:
        out = C.c_int64()
        _lib.check(_lib.lib().pf_launch_count(self._h, C.byref(out)))
        return out.value

    def graph_count(self) -> int:
        """CUDA graphs cached by the hierarchy (solve / outer-cycle / V-cycle captures)."""
        out = C.c_int64()
        _lib.check(_lib.lib().pf_hierarchy_graph_count(self._h, C.byref(out)))
        return out.value

    def reset_launch_count(self):
        _lib.check(_lib.lib().pf_reset_launch_count(self._h))

    def time_sweep(self, level: int, kind: int, iters: int = 20):
        ms, b = C.c_double(), C.c_double()
        _lib.check(_lib.lib().pf_time_sweep(self._h, level, kind, iters, C.byref(ms), C.byref(b)))
        return ms.value, b.value

    def time_vcycle(self, x: DeviceVector, b: DeviceVector, cfg: MultigridConfig, iters: int = 10):
        ms = C.c_double()
        c = cfg.c()
        _lib.check(_lib.lib().pf_time_vcycle(self._h, x._p, b._p, C.byref(c), iters, C.byref(ms)))
        return ms.value

    def close(self):
        if getattr(self, "_h", None):
            # vectors first: a vector must never outlive the hierarchy it was made from
            for v in list(getattr(self, "_vectors", ())):
                v.close()
            _lib.lib().pf_hierarchy_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


# ---------------------------------------------------------------- reference API --

def set_host_threads(n: int) -> int:
    """pf_set_host_threads: the library's OpenMP host threads (n <= 0: every processor)."""
    out = C.c_int(0)
    _lib.check(_lib.lib().pf_set_host_threads(int(n), C.byref(out)))
    return out.value


def option_names() -> dict:
    """Every tuning option: {name: "build" | "launch"} (pf_option_names; no GPU needed)."""
    buf = C.create_string_buffer(4096)
    _lib.check(_lib.lib().pf_option_names(buf, len(buf)))
    return dict(item.split(":") for item in buf.value.decode().split())


def spmv(h: Hierarchy, level: int, x: DeviceVector, y: DeviceVector) -> None:
    _lib.check(_lib.lib().pf_spmv(h._h, level, x._p, y._p))


def residual_norm(h: Hierarchy, level: int, x: DeviceVector, b: DeviceVector) -> float:
    out = C.c_double()
    _lib.check(_lib.lib().pf_residual_norm(h._h, level, x._p, b._p, C.byref(out)))
    return out.value


def smooth(h: Hierarchy, level: int, x: DeviceVector, b: DeviceVector, cfg: SmootherConfig) -> None:
    c = cfg.c()
    _lib.check(_lib.lib().pf_smooth(h._h, level, x._p, b._p, C.byref(c)))


def coarse_solve(h: Hierarchy, level: int, x: DeviceVector, b: DeviceVector, tol: float,
                 max_iter: int) -> SolveStats:
    st = _lib.SolveStats()
    _lib.check(_lib.lib().pf_coarse_solve(h._h, level, x._p, b._p, tol, max_iter, C.byref(st)))
    return SolveStats.from_c(st)


def prolongate(h: Hierarchy, fine: int, coarse: DeviceVector, out: DeviceVector) -> None:
    _lib.check(_lib.lib().pf_prolongate(h._h, fine, coarse._p, out._p))


def restrict_residual(h: Hierarchy, fine: int, r: DeviceVector, rc: DeviceVector) -> None:
    _lib.check(_lib.lib().pf_restrict_residual(h._h, fine, r._p, rc._p))


def update_master_slave(h: Hierarchy, level: int, v: DeviceVector, mode: int) -> None:
    _lib.check(_lib.lib().pf_update_master_slave(h._h, level, v._p, mode))


def update_halo1(h: Hierarchy, level: int, v: DeviceVector) -> None:
    _lib.check(_lib.lib().pf_update_halo1(h._h, level, v._p))


def update_halo2(h: Hierarchy, level: int, v: DeviceVector) -> None:
    _lib.check(_lib.lib().pf_update_halo2(h._h, level, v._p))


def allreduce_sum(h: Hierarchy, values) -> float:
    a = np.ascontiguousarray(values, np.float64)
    out = C.c_double()
    _lib.check(_lib.lib().pf_allreduce_sum(h._h, a.ctypes.data_as(C.POINTER(C.c_double)),
                                           C.byref(out)))
    return out.value


def v_cycle(h: Hierarchy, x: DeviceVector, b: DeviceVector, cfg: MultigridConfig) -> SolveStats:
    st = _lib.SolveStats()
    c = cfg.c()
    _lib.check(_lib.lib().pf_v_cycle(h._h, x._p, b._p, C.byref(c), C.byref(st)))
    return SolveStats.from_c(st)


def solve_outer(h: Hierarchy, x: DeviceVector, b: DeviceVector, cfg: MultigridConfig) -> SolveStats:
    st = _lib.SolveStats()
    c = cfg.c()
    res = np.zeros(max(cfg.outer_max_cycles, 1))
    rc = _lib.lib().pf_solve_outer(h._h, x._p, b._p, C.byref(c), C.byref(st),
                                   res.ctypes.data_as(C.POINTER(C.c_double)), res.size)
    stats = SolveStats.from_c(st, res[:st.iterations])
    if rc == _lib.PF_ERR_NO_CONVERGENCE:
        err = NoConvergenceError(_lib.lib().pf_last_error().decode())
        err.stats = stats
        raise err
    _lib.check(rc)
    return stats


def solve_outer_host(h: Hierarchy, x_host: list, b_host: list, cfg: MultigridConfig) -> SolveStats:
    """End-to-end solve from host arrays (per local subdomain); x_host is overwritten."""
    xs = [np.ascontiguousarray(a, np.float64) for a in x_host]
    bs = [np.ascontiguousarray(a, np.float64) for a in b_host]
    xp = (C.c_void_p * len(xs))(*[a.ctypes.data for a in xs])
    bp = (C.c_void_p * len(bs))(*[a.ctypes.data for a in bs])
    st = _lib.SolveStats()
    c = cfg.c()
    res = np.zeros(max(cfg.outer_max_cycles, 1))
    rc = _lib.lib().pf_solve_outer_host(h._h, xp, bp, C.byref(c), C.byref(st),
                                        res.ctypes.data_as(C.POINTER(C.c_double)), res.size)
    for dst, src in zip(x_host, xs):
        if dst is not src:
            dst[...] = src
    stats = SolveStats.from_c(st, res[:st.iterations])
    if rc == _lib.PF_ERR_NO_CONVERGENCE:
        err = NoConvergenceError(_lib.lib().pf_last_error().decode())
        err.stats = stats
        raise err
    _lib.check(rc)
    return stats


def replica_levels(dim: int, n_coarse: int, n_levels: int, world: int, problem: int = 0,
                   max_rows: int = 65536, direct_halos: bool = False):
    """Every rank's bottom levels 0..top for a multi-process hierarchy (coarse_replicas):
    top is the highest level below the finest whose rows over all ranks stay <= max_rows
    (those levels then run redundantly on every GPU after one allgather)."""
    # only the levels that can qualify: the global vertex count bounds every rank sum
    nl = 1
    while nl < n_levels - 1 and (n_coarse * 2 ** nl + 1) ** dim <= max_rows:
        nl += 1
    per_rank = [StructuredSetup(dim, n_coarse, max(1, min(n_levels - 1, nl)), world, q, problem,
                                direct_halos=direct_halos).levels
                for q in range(world)]
    top = 0
    for l in range(len(per_rank[0])):
        if sum(p[l].n for p in per_rank) <= max_rows:
            top = l
    return [p[:top + 1] for p in per_rank]


def gather_replica_levels(setup, allgather, max_rows: int = 65536):
    """coarse_replicas for a multi-process hierarchy without building any other rank's
    setup: every rank contributes its own levels 0..top (taken from its setup before the
    upload moves them) through `allgather(obj) -> list` (e.g. torch.distributed
    all_gather_object).  top as in replica_levels."""
    nl = 1
    while nl < setup.n_levels - 1 and (setup.n_coarse * 2 ** nl + 1) ** setup.dim <= max_rows:
        nl += 1
    mine = [setup._level(l) for l in range(min(setup.n_levels - 1, nl))]
    per_rank = allgather(mine)
    top = 0
    for l in range(len(per_rank[0])):
        if sum(p[l].n for p in per_rank) <= max_rows:
            top = l
    return [p[:top + 1] for p in per_rank]


def structured_hierarchy(dim: int, n_coarse: int, n_levels: int, n_ranks: int = 1,
                         problem: int = _lib.PF_PROBLEM_BASELINE, device: int = 0,
                         ranks: list | None = None, world_size: int | None = None):
    """Setup + device hierarchy for the given ranks (default: all ranks on this device).

    Returns (hierarchy, setups) where setups[s] holds the host data (keys, b, x0)."""
    ranks = list(range(n_ranks)) if ranks is None else ranks
    setups = [StructuredSetup(dim, n_coarse, n_levels, n_ranks, r, problem) for r in ranks]
    h = Hierarchy([s.levels for s in setups], device=device, rank_base=ranks[0],
                  world_size=n_ranks if world_size is None else world_size)
    return h, setups
