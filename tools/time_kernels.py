"""Live per-call times of the finest-level operations at C2 (development aid): each public
call (one kernel, or a kernel + its exchange) enqueued `iters` times back to back on the
hierarchy's stream between two CUDA events.  The stream is kept busy, so per-call launch
overhead hides behind the previous call.

    python tools/time_kernels.py [levels]"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1609_04809_b200 import gmg  # noqa: E402
from paper_1609_04809_b200.levels import StructuredSetup  # noqa: E402

L = int(sys.argv[1]) if len(sys.argv) > 1 else 7
s = StructuredSetup(3, 2, L, 1, 0)
h = gmg.Hierarchy([s.levels])
f, c = L - 1, L - 2
rng = np.random.default_rng(1)
xf = h.vector(f, rng.standard_normal(h.n_dofs(f)))
bf = h.vector(f, s.b)
yf = h.vector(f)
xc = h.vector(c, rng.standard_normal(h.n_dofs(c)))
rc = h.vector(c)
stream = torch.cuda.ExternalStream(h.stream_handle())
ops = {
    "prolongate (k_prolong_add)": lambda: gmg.prolongate(h, f, xc, yf),
    "restrict_residual (k_restrict)": lambda: gmg.restrict_residual(h, f, bf, rc),
    "spmv (k_spmv)": lambda: gmg.spmv(h, f, xf, yf),
    "jacobi sweep (k_jacobi)": lambda: gmg.smooth(h, f, xf, bf, gmg.SmootherConfig(kind=0, sweeps=1, damping=0.8)),
}
for name, op in ops.items():
    for _ in range(5):
        op()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    iters = 100
    e0.record(stream)
    for _ in range(iters):
        op()
    e1.record(stream)
    torch.cuda.synchronize()
    print(f"{name:34s} {1e3 * e0.elapsed_time(e1) / iters:8.1f} us per call", flush=True)
