"""Small runs of every kernel family for compute-sanitizer (memcheck / racecheck /
synccheck / initcheck): row kernels (Jacobi, residual, norms, transfers), the cooperative
bottom kernel with its grid barriers and last-block ticket reductions, the coarse solves,
the exchange kernels (device-local copies, pack / unpack / ordered accumulate through the
loopback transport), the CN heat kernels, the FE assembly, and — with PF_SOR_TMA=1 — the
TMA-staged colour sweep.  Each phase checks its result against the oracle, so the runs
under the sanitizer are also parity runs.

    compute-sanitizer --tool memcheck python tools/sanitize_run.py [phase ...]
"""
import os
import sys
import threading

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

from helpers import cfg, download, structured, upload  # noqa: E402
from oracle.restated import Oracle  # noqa: E402
from paper_1609_04809_b200 import _lib, gmg  # noqa: E402


def solve_phase(K, kind, L=4, problem=0):
    setups, levels = structured(3, 2, L, K) if problem == 0 else (None, None)
    if problem:
        from paper_1609_04809_b200.levels import StructuredSetup
        setups = [StructuredSetup(3, 2, L, K, r, problem, seed=5) for r in range(K)]
        levels = [s.levels for s in setups]
    c = cfg(kind, damping=1.2 if kind == 2 else 0.8, max_cycles=200)
    h = gmg.Hierarchy(levels)
    x = upload(h, L - 1, [s.x0 for s in setups])
    st = gmg.solve_outer(h, x, upload(h, L - 1, [s.b for s in setups]), c)
    xo, res, ost, rc = Oracle(levels).solve_outer([s.x0 for s in setups], [s.b for s in setups], c)
    assert st.iterations == ost.iterations and all(np.array_equal(a, b) for a, b in zip(download(h, x, K), xo))
    h.close()


def loopback_phase(K=2, L=4, kind=0):
    setups, levels = structured(3, 2, L, K, direct_halos=True)
    c = cfg(kind, damping=1.2 if kind == 2 else 0.8)
    reps = [s[:L - 1] for s in levels]
    hub = gmg.LoopbackHub(K)
    out = [None] * K

    def body(r):
        h = gmg.Hierarchy([levels[r]], rank_base=r, world_size=K, coarse_replicas=reps, fused_exchanges=True)
        h.init_loopback(hub)
        x = h.vector(L - 1, setups[r].x0)
        gmg.solve_outer(h, x, h.vector(L - 1, setups[r].b), c)
        v = h.vector(L - 2)
        gmg.update_master_slave(h, L - 2, v, gmg.PF_UPDATE_ACCUMULATE_THEN_SCATTER)
        out[r] = x.download()
        h.close()
    th = [threading.Thread(target=body, args=(r,)) for r in range(K)]
    [t.start() for t in th]
    [t.join() for t in th]
    xo, _, _, _ = Oracle(levels).solve_outer([s.x0 for s in setups], [s.b for s in setups], c)
    assert all(np.array_equal(a, b) for a, b in zip(out, xo))
    hub.close()


def heat_phase():
    from paper_1609_04809_b200.heat import HeatRun
    run = HeatRun(3, 2, 4, 0.01)
    c = cfg()
    run.run(2, c)
    run.close()


def fe_phase():
    from paper_1609_04809_b200.fe import LOGNORMAL, Q2, ROTATED_Q1, FESetup
    for fam, coef, L in ((Q2, 0, 3), (ROTATED_Q1, LOGNORMAL, 4)):
        fs = FESetup(fam, 2, L, coef, seed=3)
        h = gmg.Hierarchy([fs.levels])
        c = cfg(2, damping=1.2, max_cycles=200)
        x = h.vector(L - 1, fs.x0)
        st = gmg.solve_outer(h, x, h.vector(L - 1, fs.b), c)
        xo, _, ost, _ = Oracle([fs.levels]).solve_outer([fs.x0], [fs.b], c)
        assert st.iterations == ost.iterations and np.array_equal(x.download(), xo[0])
        h.close()


PHASES = {
    "jacobi_k1": lambda: solve_phase(1, 0),
    "sor_k2": lambda: solve_phase(2, 2),
    "gs_k4_lognormal": lambda: solve_phase(4, 1, problem=_lib.PF_PROBLEM_LOGNORMAL),
    "loopback_k2": lambda: loopback_phase(2, 4, 0),
    "loopback_k3_sor": lambda: loopback_phase(3, 3, 2),
    "heat": heat_phase,
    "fe": fe_phase,
}

if __name__ == "__main__":
    names = sys.argv[1:] or list(PHASES)
    for n in names:
        PHASES[n]()
        print("phase", n, "ok", flush=True)
