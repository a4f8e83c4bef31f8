"""Per-level cost of a V-cycle, measured live (graph replay, PDL, CUDA events):
T(L) = mean V-cycle time of the L-level hierarchy; the cost of level L-1 (the finest of that
hierarchy) is T(L) - T(L-1).

python tools/level_costs.py [max_levels] [kinds...]          Q1 (C2 shape; kinds: 0 Jacobi w=0.8, 2 SOR w=1.2)
python tools/level_costs.py --fe q2|rt [max_levels] [kinds]   Q2 V(3,3) / rotated Q1 V(2,2), direct coarse solve"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1609_04809_b200 import gmg  # noqa: E402
from paper_1609_04809_b200.levels import StructuredSetup  # noqa: E402

argv = sys.argv[1:]
fe = None
if argv and argv[0] == "--fe":
    fe, argv = argv[1], argv[2:]
max_l = int(argv[0]) if argv else (6 if fe == "q2" else 7)
kinds = [int(k) for k in argv[1:]] or [0, 2]
pp = 3 if fe == "q2" else 2


def build(L):
    if fe is None:
        s = StructuredSetup(3, 2, L, 1, 0)
        return s, gmg.Hierarchy([s.levels])
    from paper_1609_04809_b200.fe import CONSTANT, Q2, ROTATED_Q1, FESetup
    s = FESetup(Q2 if fe == "q2" else ROTATED_Q1, 2, L, CONSTANT, seed=2024)
    h = gmg.Hierarchy([s.levels])
    h.set_coarse_direct()
    return s, h


for kind in kinds:
    prev = 0.0
    for L in range(2, max_l + 1):
        s, h = build(L)
        c = gmg.MultigridConfig(smoother=gmg.SmootherConfig(kind=kind, damping=0.8 if kind == 0 else 1.2),
                                pre_smooth=pp, post_smooth=pp, outer_tol=1e-10)
        x, b = h.vector(L - 1, s.x0), h.vector(L - 1, s.b)
        t = min(h.time_vcycle(x, b, c, iters=50) for _ in range(3))
        n = h.n_dofs(L - 1)
        print(f"{fe or 'q1'} kind {kind} levels {L} finest rows {n:9d}: V-cycle {1e3 * t:8.1f} us, finest level adds "
              f"{1e3 * (t - prev):8.1f} us", flush=True)
        prev = t
        h.close()
