"""A/B of the block-window row kernels (pf_window.cuh) against the plain ones on one GPU
(development aid): sweep / V-cycle / solve times and bit-identity of the solutions.

    PF_TIMING=1 python tools/ab_win.py [levels] [lognormal]
"""
import hashlib
import sys

import numpy as np

sys.path.insert(0, ".")
from paper_1609_04809_b200 import _lib, gmg  # noqa: E402
from paper_1609_04809_b200.levels import StructuredSetup  # noqa: E402

L = int(sys.argv[1]) if len(sys.argv) > 1 else 7
if len(sys.argv) > 2 and sys.argv[2] == "lognormal":
    s = StructuredSetup(3, 2, L, 1, 0, _lib.PF_PROBLEM_LOGNORMAL, seed=2024)
else:
    s = StructuredSetup(3, 2, L, 1, 0)
h = gmg.Hierarchy([s.levels], options={"win": 1})
digests = {}
for wk in (0, 1, 2):
    h.set_option("win_kernels", wk)
    for kind, om in ((0, 0.8), (2, 1.2)):
        c = gmg.MultigridConfig(smoother=gmg.SmootherConfig(kind=kind, damping=om), pre_smooth=2, post_smooth=2,
                                outer_tol=1e-10, outer_max_cycles=200)
        x = h.vector(L - 1, s.x0)
        b = h.vector(L - 1, s.b)
        st = gmg.solve_outer(h, x, b, c)
        d = hashlib.sha256(np.ascontiguousarray(x.download()).tobytes()).hexdigest()[:16]
        ts = []
        for _ in range(3):
            x.upload(s.x0)
            st = gmg.solve_outer(h, x, b, c)
            ts.append(st.solve_seconds)
        vc = h.time_vcycle(x, b, c, 20)
        ms, by = h.time_sweep(L - 1, kind, 50)
        print(f"win_kernels {wk} kind {kind}: cycles {st.iterations} solve {min(ts) * 1e3:.3f} ms vcycle {vc:.3f} ms "
              f"sweep {ms * 1e3:.1f} us digest {d}", flush=True)
        digests.setdefault(kind, set()).add((st.iterations, d))
for kind, v in digests.items():
    print(f"kind {kind}: {'bit-identical' if len(v) == 1 else 'DIFFERENT ' + str(v)}")
