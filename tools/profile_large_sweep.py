"""Finest-level sweeps of a large grid for ncu captures (development aid):
python tools/profile_large_sweep.py <n_coarse> <levels> <kind> [problem]"""
import sys

sys.path.insert(0, ".")
from paper_1609_04809_b200 import gmg  # noqa: E402
from paper_1609_04809_b200.levels import StructuredSetup  # noqa: E402

nc, L, kind = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
prob = int(sys.argv[4]) if len(sys.argv) > 4 else 0
s = StructuredSetup(3, nc, L, 1, 0, prob, seed=2024, materialize=False)
h = gmg.Hierarchy.from_setups([s])
ms, by = h.time_sweep(L - 1, kind, 5)
print(f"sweep kind {kind}: {ms * 1e3:.0f} us, {by / ms / 1e6:.0f} GB/s on stored bytes ({by / 1e9:.2f} GB)")
