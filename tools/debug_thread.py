import sys, threading; sys.path.insert(0, '.')
from paper_1609_04809_b200 import gmg
from paper_1609_04809_b200.levels import StructuredSetup
mode = sys.argv[1]
s = StructuredSetup(3, 2, 3, 1, 0)
def body():
    h = gmg.Hierarchy([s.levels])
    c = gmg.MultigridConfig(smoother=gmg.SmootherConfig(kind=0, damping=0.8), pre_smooth=2, post_smooth=2, outer_tol=1e-10)
    x = h.vector(2, s.x0); b = h.vector(2, s.b)
    st = gmg.solve_outer(h, x, b, c)
    print("ok", st.iterations, flush=True)
if mode == "main":
    body()
else:
    t = threading.Thread(target=body); t.start(); t.join()
