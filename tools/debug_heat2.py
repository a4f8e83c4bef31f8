"""Debug: 3 CN steps, device heat_run step by step vs the restated loop on the same data."""
import sys
import numpy as np
sys.path.insert(0, "/root/repo"); sys.path.insert(0, "/root/repo/tests")
from helpers import cfg
from oracle.restated import Oracle, heat_loop
from paper_1609_04809_b200.heat import HeatRun

dim, nc, L, K, dt = 3, 2, 3, 1, 0.02
run = HeatRun(dim, nc, L, dt, n_ranks=K)
S = run.setups
tops = [s.levels[-1] for s in S]
O = Oracle([s.levels for s in S])
denom = nc * 2 ** (L - 1)
for steps in (1, 2, 3):
    loads = [np.stack([s.load_at((k + 1) * dt) for k in range(steps)]) for s in S]
    u, res = heat_loop(O, tops, [s.rhs_op for s in S], [s.x0 for s in S], [s.b for s in S], loads, dt,
                       steps, cfg(), dim, denom)
    run.reset()
    st = run.run(steps, cfg())
    print(steps, "iters dev", st.iterations, "orc", len(res), "u eq",
          [np.array_equal(run.u.download(r), u[r]) for r in range(K)],
          "maxdiff", max(np.abs(run.u.download(r) - u[r]).max() for r in range(K)))
    print("  dev", st.residuals[-2:], "orc", list(res[-2:]))
