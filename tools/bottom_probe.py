"""V-cycle time with the bottom kernel disabled / enabled / different grids (dev aid)."""
import os, subprocess, sys
code = r'''
import sys; sys.path.insert(0, ".")
from paper_1609_04809_b200 import gmg
from paper_1609_04809_b200.levels import StructuredSetup
s = StructuredSetup(3, 2, 7, 1, 0)
h = gmg.Hierarchy([s.levels])
for kind, om in ((0, 0.8), (2, 1.2)):
    c = gmg.MultigridConfig(smoother=gmg.SmootherConfig(kind=kind, damping=om), pre_smooth=2, post_smooth=2, outer_tol=1e-10)
    x = h.vector(6, s.x0); b = h.vector(6, s.b)
    vc = min(h.time_vcycle(x, b, c, 20) for _ in range(3))
    print(f"  kind {kind}: vcycle {vc*1e3:.1f} us")
'''
for env in [{"PF_BOTTOM_ROWS": "0"}, {}, {"PF_BOTTOM_GRID": "74"}, {"PF_BOTTOM_GRID": "37"}, {"PF_BOTTOM_GRID": "16"},
            {"PF_BOTTOM_ROWS": "5000"}, {"PF_BOTTOM_ROWS": "300000"}]:
    print(env, flush=True)
    e = dict(os.environ); e.update(env)
    subprocess.run([sys.executable, "-c", code], env=e)
