"""Large single-GPU runs (BASELINE configs[4] sizes) through the lean path: native setup ->
device without numpy copies, host matrices released after the upload.

    python tools/large_run.py <levels> [problem] [kinds] [n_coarse]   # 9 levels, nc 2 = 512^3
Prints setup / upload seconds, peak host RSS, device bytes, and per smoother the cycles and
the time of the second solve (the first one includes the graph capture)."""
import resource
import sys
import time

sys.path.insert(0, ".")
from paper_1609_04809_b200 import _lib, gmg  # noqa: E402
from paper_1609_04809_b200.levels import StructuredSetup  # noqa: E402

L = int(sys.argv[1]) if len(sys.argv) > 1 else 8
prob = int(sys.argv[2]) if len(sys.argv) > 2 else _lib.PF_PROBLEM_LOGNORMAL
kinds = [int(k) for k in sys.argv[3].split(",")] if len(sys.argv) > 3 else [2, 0]
nc = int(sys.argv[4]) if len(sys.argv) > 4 else 2


def rss_gb():
    return resource.getrusage(resource.RUSAGE_SELF).ru_maxrss / 1e6


t = time.time()
s = StructuredSetup(3, nc, L, 1, 0, prob, seed=2024, materialize=False)
print(f"levels {L}: {s.n_global} dofs; setup {time.time() - t:.1f} s, peak RSS {rss_gb():.1f} GB", flush=True)
t = time.time()
h = gmg.Hierarchy.from_setups([s])
print(f"upload {time.time() - t:.1f} s, peak RSS {rss_gb():.1f} GB, device {h.device_bytes() / 1e9:.1f} GB", flush=True)
print({l: h.level_info(l) for l in (L - 2, L - 1)}, flush=True)
top = L - 1
import os  # noqa: E402

sor_omegas = [float(w) for w in os.environ.get("LARGE_SOR_OMEGA", "1.2").split(",")]
runs = [(k, w) for k in kinds for w in (sor_omegas if k == 2 else [0.8])]
for kind, om in runs:
    c = gmg.MultigridConfig(smoother=gmg.SmootherConfig(kind=kind, damping=om), pre_smooth=2, post_smooth=2,
                            outer_tol=1e-10, outer_max_cycles=400)
    x, b = h.vector(top, s.x0), h.vector(top, s.b)
    st = gmg.solve_outer(h, x, b, c)  # first solve: graph capture and lazy module loading
    first_ms = st.solve_seconds * 1e3
    x.upload(s.x0)
    st = gmg.solve_outer(h, x, b, c)
    print(f"kind {kind} omega {om}: first solve {first_ms:.1f} ms; cycles {st.iterations} converged {st.converged} solve {st.solve_seconds * 1e3:.1f} ms "
          f"({s.n_global / st.solve_seconds:.3e} DOF/s), V-cycle {h.time_vcycle(x, b, c, 3):.2f} ms", flush=True)
    x.close()
    b.close()
ms, by = h.time_sweep(top, 0, 5)
print(f"finest Jacobi sweep {ms * 1e3:.0f} us, {by / ms / 1e6:.0f} GB/s", flush=True)
