"""C2 with the lognormal coefficient (BASELINE configs 3-4's coefficient on the Q1 C2 grid)."""
import sys, time
sys.path.insert(0, '.')
from paper_1609_04809_b200 import gmg, _lib
from paper_1609_04809_b200.levels import StructuredSetup
L = int(sys.argv[1]) if len(sys.argv) > 1 else 7
t = time.time(); s = StructuredSetup(3, 2, L, 1, 0, _lib.PF_PROBLEM_LOGNORMAL, seed=2024); print("setup", round(time.time() - t, 2), flush=True)
h = gmg.Hierarchy([s.levels])
print({l: h.level_info(l) for l in range(L)})
for kind, om in ((0, 0.8), (2, 1.2)):
    c = gmg.MultigridConfig(smoother=gmg.SmootherConfig(kind=kind, damping=om), pre_smooth=2, post_smooth=2, outer_tol=1e-10, outer_max_cycles=200)
    x = h.vector(L - 1, s.x0); b = h.vector(L - 1, s.b)
    st = gmg.solve_outer(h, x, b, c)
    ts = []
    for i in range(3):
        x.upload(s.x0)
        st = gmg.solve_outer(h, x, b, c)
        ts.append(st.solve_seconds)
    print(f"kind {kind}: cycles {st.iterations} converged {st.converged} solve {min(ts)*1e3:.2f} ms DOF/s {s.n_global/min(ts):.3e} vcycle {h.time_vcycle(x, b, c, 10):.3f} ms", flush=True)
ms, by = h.time_sweep(L - 1, 0, 20)
print(f"sweep: {ms*1e3:.1f} us {by/ms/1e6:.1f} GB/s")
ms, by = h.time_sweep(L - 1, 2, 20)
print(f"SOR sweep: {ms*1e3:.1f} us {by/ms/1e6:.1f} GB/s")
