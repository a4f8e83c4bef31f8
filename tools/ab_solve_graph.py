"""A/B of the two shapes of the device-driven solve graph (Options::solve_graph_if) on one
GPU (development aid): C2 solve times, cycle counts, residual histories and solution
digests must agree.

    python tools/ab_solve_graph.py [levels]
"""
import hashlib
import sys

import numpy as np

sys.path.insert(0, ".")
from paper_1609_04809_b200 import gmg  # noqa: E402
from paper_1609_04809_b200.levels import StructuredSetup  # noqa: E402

L = int(sys.argv[1]) if len(sys.argv) > 1 else 7
s = StructuredSetup(3, 2, L, 1, 0)
h = gmg.Hierarchy([s.levels])
seen = {}
for rep in range(2):
    for shape in (1, 0):
        h.set_option("solve_graph_if", shape)
        for kind, om in ((0, 0.8), (2, 1.2)):
            c = gmg.MultigridConfig(smoother=gmg.SmootherConfig(kind=kind, damping=om), pre_smooth=2, post_smooth=2,
                                    outer_tol=1e-10)
            x = h.vector(L - 1, s.x0)
            b = h.vector(L - 1, s.b)
            st = gmg.solve_outer(h, x, b, c)
            d = hashlib.sha256(np.ascontiguousarray(x.download()).tobytes()).hexdigest()[:16]
            ts = []
            for _ in range(10):
                x.upload(s.x0)
                st = gmg.solve_outer(h, x, b, c)
                ts.append(st.solve_seconds)
            print(f"solve_graph_if {shape} kind {kind}: cycles {st.iterations} solve min {min(ts) * 1e3:.3f} "
                  f"median {sorted(ts)[5] * 1e3:.3f} ms launches {h.launch_count()} digest {d}", flush=True)
            seen.setdefault(kind, set()).add((st.iterations, d, tuple(st.residuals)))
for kind, v in seen.items():
    print(f"kind {kind}: {'identical' if len(v) == 1 else 'DIFFERENT'}")
