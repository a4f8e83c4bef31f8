"""A/B timing probe at C2 (development aid): solve times, V-cycle, finest sweeps, and the
solutions saved to argv[1] for a bit-exactness check between two builds / settings."""
import sys, time
import numpy as np
sys.path.insert(0, '.')
from paper_1609_04809_b200 import gmg
from paper_1609_04809_b200.levels import StructuredSetup
L = int(sys.argv[2]) if len(sys.argv) > 2 else 7
s = StructuredSetup(3, 2, L, 1, 0)
h = gmg.Hierarchy([s.levels])
sols = []
for kind, om in ((0, 0.8), (2, 1.2)):
    c = gmg.MultigridConfig(smoother=gmg.SmootherConfig(kind=kind, damping=om), pre_smooth=2, post_smooth=2, outer_tol=1e-10)
    x = h.vector(L - 1, s.x0); b = h.vector(L - 1, s.b)
    ts = []
    for i in range(8):
        x.upload(s.x0)
        st = gmg.solve_outer(h, x, b, c)
        ts.append(st.solve_seconds)
    sols.append(x.download())
    vc = h.time_vcycle(x, b, c, 30)
    print(f"kind {kind}: cycles {st.iterations} solve min {min(ts[1:])*1e3:.3f} med {np.median(ts[1:])*1e3:.3f} ms vcycle {vc:.3f} ms", flush=True)
for kind in (0, 2):
    ms, by = h.time_sweep(L - 1, kind, 50)
    print(f"sweep kind {kind}: {ms*1e3:.1f} us", flush=True)
np.save(sys.argv[1], np.stack(sols))
