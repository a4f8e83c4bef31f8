"""A/B probe of the colour-interleaved block schedule on a grid whose x exceeds L2
(development aid): python tools/ab_interleave.py <n_coarse> <levels> [problem].
Prints the finest Jacobi sweep and residual times, the Jacobi solve, and a digest of the
solution (compare the digest between PF_INTERLEAVE_MIN_BYTES settings)."""
import hashlib
import sys
import time

sys.path.insert(0, ".")
from paper_1609_04809_b200 import gmg  # noqa: E402
from paper_1609_04809_b200.levels import StructuredSetup  # noqa: E402

nc, L = int(sys.argv[1]), int(sys.argv[2])
prob = int(sys.argv[3]) if len(sys.argv) > 3 else 0
t = time.time()
s = StructuredSetup(3, nc, L, 1, 0, prob, seed=2024, materialize=False)
h = gmg.Hierarchy.from_setups([s])
print(f"{s.n_global} dofs, setup+upload {time.time() - t:.1f} s", flush=True)
top = L - 1
ms, by = h.time_sweep(top, 0, 10)
print(f"finest Jacobi sweep {ms * 1e3:.0f} us, {by / ms / 1e6:.0f} GB/s on stored bytes", flush=True)
c = gmg.MultigridConfig(smoother=gmg.SmootherConfig(kind=0, damping=0.8), pre_smooth=2, post_smooth=2,
                        outer_tol=1e-10, outer_max_cycles=200)
x, b = h.vector(top, s.x0), h.vector(top, s.b)
gmg.solve_outer(h, x, b, c)
x.upload(s.x0)
st = gmg.solve_outer(h, x, b, c)
print(f"Jacobi: {st.iterations} cycles, solve {st.solve_seconds * 1e3:.1f} ms, V-cycle {h.time_vcycle(x, b, c, 3):.2f} ms",
      flush=True)
print("digest", hashlib.sha256(x.download().tobytes()).hexdigest()[:16], flush=True)
