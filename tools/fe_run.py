"""Q2 (BASELINE configs[2]: 64^3 cells, 129^3 dofs, 6 levels, V(3,3)) and rotated Q1
(configs[3]: 128^3 cells, 6.3M face dofs, lognormal(0,1) coefficient, 7 levels, V(2,2))
on one B200: setup time, device bytes, finest sweep GB/s, V-cycle ms, solve ms and
cycles per smoother.  Usage: python tools/fe_run.py [q2|rt|rt1] [levels] [--direct]"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from paper_1609_04809_b200 import gmg  # noqa: E402
from paper_1609_04809_b200.fe import CONSTANT, LOGNORMAL, Q2, ROTATED_Q1, FESetup  # noqa: E402


def main():
    which = sys.argv[1] if len(sys.argv) > 1 else "q2"
    family, coef, pp = {"q2": (Q2, CONSTANT, 3), "rt": (ROTATED_Q1, LOGNORMAL, 2),
                        "rt1": (ROTATED_Q1, CONSTANT, 2)}[which]
    args = [a for a in sys.argv[2:] if not a.startswith("--")]
    direct = "--direct" in sys.argv
    L = int(args[0]) if args else (6 if family == Q2 else 7)
    t = time.time()
    s = FESetup(family, 2, L, coef, seed=2024, keep=True)
    t_setup = time.time() - t
    fin = s.levels[-1]
    h = gmg.Hierarchy([s.levels])
    if direct:
        h.set_coarse_direct()
    out = dict(family=which, levels=L, coarse="direct" if direct else "gauss-seidel", n_global=s.n_global, nnz=int(fin.row_offsets[-1]),
               setup_s=round(t_setup, 2), device_gb=round(h.device_bytes() / 1e9, 2))
    # device assembly of the finest system (pf_fe_assembly_set + pf_assemble_operator)
    from paper_1609_04809_b200.heat import Assembly, Operator
    asm, op = Assembly(h, L - 1, [s.assembly_desc(L - 1)]), Operator(h, L - 1)
    ta = []
    for _ in range(4):
        t0 = time.time()
        asm.assemble(op)
        ta.append(time.time() - t0)
    out["device_assembly_ms"] = round(min(ta[1:]) * 1e3, 3)
    out["device_assembly_equal"] = bool(np.array_equal(op.values(0, len(fin.vals)), fin.vals))
    out["host_setup_all_levels_s"] = round(s.seconds, 2)
    asm.close()
    op.close()
    s.close()
    n_own = fin.n_own
    nnz_own = int(fin.row_offsets[n_own])
    sor_omega = float(os.environ.get("FE_SOR_OMEGA", "1.2"))
    for kind, omega, name in [(gmg.PF_SMOOTHER_JACOBI, 0.8, "jacobi"),
                              (gmg.PF_SMOOTHER_MULTICOLOR_SOR, sor_omega, "sor_%g" % sor_omega)]:
        c = gmg.MultigridConfig(smoother=gmg.SmootherConfig(kind=kind, damping=omega), pre_smooth=pp,
                                post_smooth=pp, outer_tol=1e-10, outer_max_cycles=500)
        x, b = h.vector(L - 1), h.vector(L - 1)
        b.upload(s.b)
        times = []
        for rep in range(3):
            x.upload(s.x0)
            t0 = time.time()
            st = gmg.solve_outer(h, x, b, c)
            times.append(time.time() - t0)
        err = float(np.abs(x.download(0) - s.exact).max())
        sweep_ms, sweep_bytes = h.time_sweep(L - 1, kind, 20)
        out[name] = dict(cycles=st.iterations, converged=bool(st.converged), solve_ms=round(min(times) * 1e3, 2),
                         dofs_per_s=s.n_global / min(times), err_vs_exact=err,
                         vcycle_ms=round(h.time_vcycle(x, b, c, 10), 3), finest_sweep_us=round(sweep_ms * 1e3, 1),
                         finest_sweep_gbs=round(sweep_bytes / (sweep_ms * 1e-3) / 1e9, 1))
    out["finest_stored_nnz_own"] = nnz_own
    print(json.dumps(out))


if __name__ == "__main__":
    main()
