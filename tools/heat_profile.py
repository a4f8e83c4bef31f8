"""Two CN time steps at C2 (the first warms up), for an ncu launch list:
ncu --metrics gpu__time_duration.sum --csv python tools/heat_profile.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1609_04809_b200 import gmg  # noqa: E402
from paper_1609_04809_b200.heat import HeatRun  # noqa: E402

run = HeatRun(3, 2, 7, 0.01)
c = gmg.MultigridConfig(smoother=gmg.SmootherConfig(kind=0, damping=0.8), pre_smooth=2, post_smooth=2,
                        outer_tol=1e-10)
st = run.run(1, c)
st = run.run(1, c)
print("cycles", st.iterations, "solve_s", st.solve_seconds, "residuals", st.residuals[:3])
