"""Test configuration: `gpu` marks tests that need a B200 (run with -m gpu on the GPU box);
everything else runs on the CPU container (-m "not gpu")."""
import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")
    config.addinivalue_line("markers", "slow: long-running (full BASELINE sizes)")


@pytest.fixture(scope="session")
def cuda():
    """Fail loudly (not skip) when a gpu-marked test runs without a device."""
    import torch
    if not torch.cuda.is_available():
        pytest.fail("gpu test run without a CUDA device")
    return torch.cuda.get_device_name(0)


@pytest.fixture(scope="session")
def ref_lib():
    from oracle import ref
    if not ref.available():
        pytest.skip("reference oracle oracle/_ref not built")
    return ref


def _ensure_built():
    """Build libpf_gpu.so and the oracle checkers if they are missing (nvcc cross-compiles
    without a GPU; the reference oracle only where /root/reference exists)."""
    import subprocess
    lib = os.path.join(ROOT, "paper_1609_04809_b200", "libpf_gpu.so")
    if not os.path.exists(lib):
        subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "paper_1609_04809_b200", "csrc")], check=True)
    orc = os.path.join(ROOT, "oracle", "libpf_oracle.so")
    ref = os.path.join(ROOT, "oracle", "_ref", "libparfem_ref.so")
    if not os.path.exists(orc) or (not os.path.exists(ref) and os.path.isdir("/root/reference/proj")):
        subprocess.run(["make", "-s", "-j8", "-C", os.path.join(ROOT, "oracle")], check=True)


_ensure_built()
