"""Quick C2 timing probe (development aid)."""
import sys, time
import numpy as np
sys.path.insert(0, '.')
from paper_1609_04809_b200 import gmg
from paper_1609_04809_b200.levels import StructuredSetup
L = int(sys.argv[1]) if len(sys.argv) > 1 else 7
t = time.time(); s = StructuredSetup(3, 2, L, 1, 0); print("setup", time.time() - t, flush=True)
t = time.time(); h = gmg.Hierarchy([s.levels]); print("upload", time.time() - t, flush=True)
for kind, om in ((0, 0.8), (2, 1.2), (1, 1.0)):
    c = gmg.MultigridConfig(smoother=gmg.SmootherConfig(kind=kind, damping=om), pre_smooth=2, post_smooth=2, outer_tol=1e-10)
    x = h.vector(L - 1, s.x0); b = h.vector(L - 1, s.b)
    st = gmg.solve_outer(h, x, b, c)
    ts = []
    for i in range(5):
        x.upload(s.x0)
        st = gmg.solve_outer(h, x, b, c)
        ts.append(st.solve_seconds)
    vc = h.time_vcycle(x, b, c, 20)
    print(f"kind {kind}: cycles {st.iterations} res {st.residuals[-1]/st.initial_residual:.3e} solve {min(ts)*1e3:.3f} ms  DOF/s {s.n_global/min(ts):.3e} vcycle {vc:.3f} ms", flush=True)
for kind in (0, 2):
    ms, by = h.time_sweep(L - 1, kind, 50)
    print(f"sweep kind {kind}: {ms*1e3:.1f} us  {by/ms/1e6:.1f} GB/s", flush=True)
print("launches", h.launch_count())
