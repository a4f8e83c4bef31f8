"""One warm-up C2 solve, then one measured solve (development aid for ncu launch lists).

    PF_SOLVE_MODE=host ncu --metrics gpu__time_duration.sum -s $(python tools/one_solve.py --count) ...
prints, with --count, the number of library kernel launches before the second solve.
"""
import sys

sys.path.insert(0, ".")
from paper_1609_04809_b200 import gmg  # noqa: E402
from paper_1609_04809_b200.levels import StructuredSetup  # noqa: E402

kind = int(sys.argv[2]) if len(sys.argv) > 2 else 0
s = StructuredSetup(3, 2, 7, 1, 0)
h = gmg.Hierarchy([s.levels])
c = gmg.MultigridConfig(smoother=gmg.SmootherConfig(kind=kind, damping=0.8 if kind == 0 else 1.2),
                        pre_smooth=2, post_smooth=2, outer_tol=1e-10)
x = h.vector(6, s.x0)
b = h.vector(6, s.b)
gmg.solve_outer(h, x, b, c)
n0 = h.launch_count()
x.upload(s.x0)
n1 = h.launch_count()
st = gmg.solve_outer(h, x, b, c)
if "--count" in sys.argv:
    print(n1)
else:
    print("cycles", st.iterations, "launches", h.launch_count() - n1, "skip", n1, file=sys.stderr)
