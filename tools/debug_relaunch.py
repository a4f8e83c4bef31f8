import sys, os
sys.path.insert(0, ".")
import numpy as np
from paper_1609_04809_b200 import gmg
from paper_1609_04809_b200.levels import StructuredSetup
L = int(sys.argv[1])
s = StructuredSetup(3, 2, L, 1, 0)
h = gmg.Hierarchy([s.levels])
c = gmg.MultigridConfig(smoother=gmg.SmootherConfig(kind=0, damping=0.8), pre_smooth=2, post_smooth=2, outer_tol=1e-10)
x = h.vector(L - 1, s.x0); b = h.vector(L - 1, s.b)
for i in range(4):
    x.upload(s.x0)
    st = gmg.solve_outer(h, x, b, c)
    print(i, st.iterations, st.initial_residual, st.residuals[:3], np.abs(x.download()).max(), flush=True)
