"""Per-level cost of a C2-shaped V-cycle, measured live (graph replay, PDL, CUDA events):
T(L) = mean V-cycle time of the L-level hierarchy (n_coarse 2, so 2^(L) cells per axis);
the cost of level L-1 (the finest of that hierarchy) is T(L) - T(L-1).

python tools/level_costs.py [max_levels] [kinds...]   (kinds: 0 Jacobi w=0.8, 2 SOR w=1.2)"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1609_04809_b200 import gmg  # noqa: E402
from paper_1609_04809_b200.levels import StructuredSetup  # noqa: E402

max_l = int(sys.argv[1]) if len(sys.argv) > 1 else 7
kinds = [int(k) for k in sys.argv[2:]] or [0, 2]
for kind in kinds:
    prev = 0.0
    for L in range(2, max_l + 1):
        s = StructuredSetup(3, 2, L, 1, 0)
        h = gmg.Hierarchy([s.levels])
        c = gmg.MultigridConfig(smoother=gmg.SmootherConfig(kind=kind, damping=0.8 if kind == 0 else 1.2),
                                pre_smooth=2, post_smooth=2, outer_tol=1e-10)
        x, b = h.vector(L - 1, s.x0), h.vector(L - 1, s.b)
        t = min(h.time_vcycle(x, b, c, iters=50) for _ in range(3))
        n = h.n_dofs(L - 1)
        print(f"kind {kind} levels {L} finest rows {n:9d}: V-cycle {1e3 * t:8.1f} us, finest level adds "
              f"{1e3 * (t - prev):8.1f} us", flush=True)
        prev = t
        h.close()
