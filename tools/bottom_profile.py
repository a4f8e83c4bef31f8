import sys; sys.path.insert(0, ".")
from paper_1609_04809_b200 import gmg
from paper_1609_04809_b200.levels import StructuredSetup
s = StructuredSetup(3, 2, 7, 1, 0)
h = gmg.Hierarchy([s.levels])
for kind, om in ((0, 0.8), (2, 1.2)):
    c = gmg.MultigridConfig(smoother=gmg.SmootherConfig(kind=kind, damping=om), pre_smooth=2, post_smooth=2, outer_tol=1e-10)
    x = h.vector(6, s.x0); b = h.vector(6, s.b)
    print("kind", kind, "vcycle", h.time_vcycle(x, b, c, 20), flush=True)
