"""Launches the finest-level hot kernels of C2 for ncu captures (development aid).

    python tools/profile_sweep.py [levels] [kind]   # kind: 0 Jacobi, 2 SOR
Each kernel of interest runs after a few warm-up launches so `-k regex:<name> -s 3 -c 1`
captures a steady-state finest-level launch.
"""
import sys

sys.path.insert(0, ".")
from paper_1609_04809_b200 import gmg  # noqa: E402
from paper_1609_04809_b200.levels import StructuredSetup  # noqa: E402

L = int(sys.argv[1]) if len(sys.argv) > 1 else 7
kind = int(sys.argv[2]) if len(sys.argv) > 2 else 0
s = StructuredSetup(3, 2, L, 1, 0)
h = gmg.Hierarchy([s.levels])
ms, by = h.time_sweep(L - 1, kind, 10)
print(f"sweep kind {kind}: {ms * 1e3:.1f} us, {by / ms / 1e6:.1f} GB/s algorithmic")
c = gmg.MultigridConfig(smoother=gmg.SmootherConfig(kind=kind, damping=0.8 if kind == 0 else 1.2),
                        pre_smooth=2, post_smooth=2, outer_tol=1e-10)
x = h.vector(L - 1, s.x0)
b = h.vector(L - 1, s.b)
st = gmg.solve_outer(h, x, b, c)
print("cycles", st.iterations)
