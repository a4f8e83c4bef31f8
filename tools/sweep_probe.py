import sys, os, subprocess
code = r'''
import sys; sys.path.insert(0, ".")
from paper_1609_04809_b200 import gmg
from paper_1609_04809_b200.levels import StructuredSetup
s = StructuredSetup(3, 2, 7, 1, 0)
h = gmg.Hierarchy([s.levels])
r = []
for k in (0, 2):
    r.append(min(h.time_sweep(6, k, 30)[0] for _ in range(3)) * 1e3)
c = gmg.MultigridConfig(smoother=gmg.SmootherConfig(kind=0, damping=0.8), pre_smooth=2, post_smooth=2, outer_tol=1e-10)
x = h.vector(6, s.x0); b = h.vector(6, s.b)
vc = min(h.time_vcycle(x, b, c, 20) for _ in range(3))
print(f"  jacobi sweep {r[0]:.1f} us  sor sweep {r[1]:.1f} us  vcycle {vc*1e3:.1f} us", flush=True)
'''
for env in [{"PF_ROW_ORDER": "plain", "PF_SELL_COMPRESS": "0"}, {"PF_ROW_ORDER": "plain", "PF_SELL_COMPRESS": "1"},
            {"PF_ROW_ORDER": "pattern", "PF_SELL_COMPRESS": "0"}, {"PF_ROW_ORDER": "pattern", "PF_SELL_COMPRESS": "1"}]:
    print(env, flush=True)
    e = dict(os.environ); e.update(env)
    subprocess.run([sys.executable, "-c", code], env=e)
