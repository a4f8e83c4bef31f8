"""One V-cycle of the Q2 / rotated-Q1 hierarchy, for an ncu launch list:
ncu --metrics gpu__time_duration.sum --csv python tools/fe_profile.py q2"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1609_04809_b200 import gmg  # noqa: E402
from paper_1609_04809_b200.fe import CONSTANT, LOGNORMAL, Q2, ROTATED_Q1, FESetup  # noqa: E402

which = sys.argv[1] if len(sys.argv) > 1 else "q2"
kind = int(sys.argv[2]) if len(sys.argv) > 2 else gmg.PF_SMOOTHER_JACOBI
family, coef, pp, L = {"q2": (Q2, CONSTANT, 3, 6), "rt": (ROTATED_Q1, LOGNORMAL, 2, 7)}[which]
s = FESetup(family, 2, L, coef, seed=2024)
h = gmg.Hierarchy([s.levels])
c = gmg.MultigridConfig(smoother=gmg.SmootherConfig(kind=kind, damping=1.2 if kind == 2 else 0.8),
                        pre_smooth=pp, post_smooth=pp, outer_tol=1e-10, outer_max_cycles=500)
x, b = h.vector(L - 1), h.vector(L - 1)
b.upload(s.b)
x.upload(s.x0)
gmg.v_cycle(h, x, b, c)
print("done")
