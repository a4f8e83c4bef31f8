"""One C2 V-cycle (after a warm-up solve), for an ncu launch list:
ncu --metrics gpu__time_duration.sum --csv python tools/vcycle_profile.py [kind]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1609_04809_b200 import gmg  # noqa: E402
from paper_1609_04809_b200.levels import StructuredSetup  # noqa: E402

kind = int(sys.argv[1]) if len(sys.argv) > 1 else 0
s = StructuredSetup(3, 2, 7, 1, 0)
h = gmg.Hierarchy([s.levels])
c = gmg.MultigridConfig(smoother=gmg.SmootherConfig(kind=kind, damping=0.8 if kind == 0 else 1.2),
                        pre_smooth=2, post_smooth=2, outer_tol=1e-10)
x, b = h.vector(6, s.x0), h.vector(6, s.b)
gmg.v_cycle(h, x, b, c)
print("done")
