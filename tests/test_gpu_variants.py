"""The storage / load-policy variants of the row kernels, bit-exact against the oracle.

At the default settings only operators with >= 2M stored entries get 8-bit / 16-bit value
indices (the finest levels of C2-sized hierarchies), so the small hierarchies of the
parity suite run the fp64 kernels on their finest level.  Here the parity suite is re-run
in a subprocess (the settings are read once per process) with every operator
index-encoded, so the value-table kernels — table in shared memory (kVKSmem) or read
through L1, with the streamed (evict-first + row prefetch) or the cached load policy —
are compared with the oracle bit for bit on the same cases as the fp64 ones.
"""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)

VARIANTS = {
    # every operator index-encoded, value table in shared memory, coarse levels cached
    "index_smem_cached": {"PF_VALUE_INDEX_MIN": "0"},
    # index-encoded, table through L1, every level streamed (evict-first + prefetch)
    "index_l1_streamed": {"PF_VALUE_INDEX_MIN": "0", "PF_VTAB_SMEM": "0", "PF_CACHED_MAX_BYTES": "0"},
    # fp64 everywhere, every level streamed
    "fp64_streamed": {"PF_VALUE_INDEX": "0", "PF_CACHED_MAX_BYTES": "0"},
}


@pytest.mark.parametrize("name", sorted(VARIANTS))
def test_parity_suite_under_variant(cuda, name):
    env = dict(os.environ)
    env.update(VARIANTS[name])
    cmd = [sys.executable, "-m", "pytest", "-q", "-x", "-m", "gpu", "-p", "no:cacheprovider",
           os.path.join(HERE, "test_gpu_parity.py"), os.path.join(HERE, "test_gpu_fe.py"),
           "-k", "bit_exact or solve or lognormal"]
    r = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=900)
    tail = "\n".join((r.stdout + r.stderr).splitlines()[-25:])
    assert r.returncode == 0, f"{name}:\n{tail}"
    assert " passed" in r.stdout, tail
