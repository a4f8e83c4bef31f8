"""The storage / load-policy variants of the row kernels, bit-exact against the oracle.

At the default settings every operator whose values allow it is index-encoded (8-bit /
16-bit value indices, table in shared memory), the coarser levels that fit L2 are read
with the caching load policy and the finest with evict-first loads + row prefetch, and
the bottom kernel reads decoded fp64 copies.  Here the parity suite is re-run in a
subprocess whose PF_* environment sets those options on every hierarchy it creates
(pf_hierarchy_set_option) under the other storage / load-policy
combinations, so every kernel variant is compared with the oracle bit for bit on the
same cases.
"""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)

VARIANTS = {
    # only >= 2M-entry operators index-encoded: the small hierarchies run fp64 operators
    # (cached below the finest) and the bottom kernel its native fp64 views; the cycle
    # residual and restriction as separate launches on every level
    "fp64_small_levels": {"PF_VALUE_INDEX_MIN": "2097152", "PF_FUSED_RR_ROWS": "0"},
    # index-encoded, table through L1, every level streamed (evict-first + prefetch), the
    # fused residual + restriction on every level whose R rows fit a warp
    "index_l1_streamed": {"PF_VTAB_SMEM": "0", "PF_CACHED_MAX_BYTES": "0", "PF_FUSED_RR_ROWS": "100000000"},
    # fp64 everywhere, every level streamed
    "fp64_streamed": {"PF_VALUE_INDEX": "0", "PF_CACHED_MAX_BYTES": "0"},
    # the opt-in TMA-staged colour sweep (pf_sweep_tma.cuh) on every level whose rows fit it,
    # index-encoded and fp64 operators
    "sor_tma_everywhere": {"PF_SOR_TMA": "1", "PF_SOR_TMA_MIN_ROWS": "0", "PF_SOR_TMA_BPS": "2"},
    "sor_tma_fp64": {"PF_SOR_TMA": "1", "PF_SOR_TMA_MIN_ROWS": "0", "PF_VALUE_INDEX": "0"},
    # the colour-interleaved block schedule (RowMap) of the Jacobi / residual passes on every
    # level with 2-8 colours (default: only where x exceeds 64 MB)
    "interleave_everywhere": {"PF_INTERLEAVE_MIN_BYTES": "0"},
    # the bottom levels unstaged (operators and vectors in global memory) in the cooperative
    # kernel, no wide-row kernels (every mid-size launch takes the group-pipelined rows) and
    # no slice-split Jacobi / residual for the long (Q2) rows
    "bottom_unstaged_no_wide": {"PF_BOTTOM_STAGE": "0", "PF_WIDE_MAX_ROWS": "0", "PF_SPLIT_ROWS_MAX": "0"},
    # staged bottom levels inside the cooperative kernel (not the one-block kernel), wide
    # rows on every launch that fits them, damped Jacobi through the bottom kernel too
    "bottom_staged_cooperative_wide_all": {"PF_BOTTOM_BLOCK_KERNEL": "0", "PF_WIDE_MAX_ROWS": "100000000",
                                           "PF_BOTTOM_JACOBI": "1"},
    # ... through the one-block bottom kernel, and the solve graph's older shape (IF node
    # inside the WHILE body)
    "bottom_block_kernel_jacobi": {"PF_BOTTOM_JACOBI": "1", "PF_SOLVE_GRAPH_IF": "1"},
    # the opt-in block-window row kernels (pf_window.cuh: a block's x cover staged in shared
    # memory, 16-bit window offsets, the diagonal through a private signed-zero slot) on every
    # level, colour sweeps included; fp64 and index-encoded operators
    "block_windows": {"PF_WIN": "1", "PF_WIN_MIN_ROWS": "0", "PF_WIN_KERNELS": "2"},
    "block_windows_fp64": {"PF_WIN": "1", "PF_WIN_MIN_ROWS": "0", "PF_WIN_KERNELS": "2", "PF_VALUE_INDEX": "0"},
    # memory checking: a 4 KB 0xFF guard zone after every device buffer (a read past an
    # array feeds NaN / -1 into the bit-exact comparisons; a write past one is reported
    # when the buffer is freed)
    "guard_zones": {"PF_GUARD": "1", "_files": "test_gpu_parity.py test_gpu_fe.py test_gpu_colorwise.py "
                    "test_gpu_heat.py test_gpu_assembly.py test_gpu_golden.py test_gpu_peer.py"},
}


# The opt-in TMA sweep and the pure load-policy variants run with PF_RUN_SLOW=1 (each
# re-runs the parity suite in a subprocess; the default GPU run keeps the layout, launch
# structure and memory-checking variants).
SLOW = {"sor_tma_everywhere", "sor_tma_fp64", "index_l1_streamed", "interleave_everywhere", "block_windows_fp64"}


@pytest.mark.parametrize("name", [pytest.param(n, marks=[pytest.mark.slow, pytest.mark.skipif(
    os.environ.get("PF_RUN_SLOW") != "1", reason="PF_RUN_SLOW=1")]) if n in SLOW else n for n in sorted(VARIANTS)])
def test_parity_suite_under_variant(cuda, name):
    env = dict(os.environ)
    v = dict(VARIANTS[name])
    files = v.pop("_files", None)
    env.update(v)
    cmd = [sys.executable, "-m", "pytest", "-q", "-x", "-m", "gpu", "-p", "no:cacheprovider"]
    if files:  # a whole-suite variant
        cmd += [os.path.join(HERE, f) for f in files.split()]
    else:
        cmd += [os.path.join(HERE, "test_gpu_parity.py"), os.path.join(HERE, "test_gpu_fe.py"),
                os.path.join(HERE, "test_gpu_colorwise.py"), "-k", "bit_exact or solve or lognormal or colorwise"]
    r = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=900)
    tail = "\n".join((r.stdout + r.stderr).splitlines()[-25:])
    assert r.returncode == 0, f"{name}:\n{tail}"
    assert " passed" in r.stdout, tail
    assert "[pf guard]" not in r.stdout + r.stderr, f"{name}: a kernel wrote past a device buffer"


def test_guard_zone_catches_a_planted_overrun(cuda):
    """The guard-zone check itself: one element written past a guarded buffer is caught."""
    import ctypes as C

    from paper_1609_04809_b200 import _lib
    det = C.c_int(0)
    _lib.check(_lib.lib().pf_debug_guard_selftest(0, C.byref(det)))
    assert det.value == 1
