# SPDX-License-Identifier: Apache-2.0
import os
import sys

import numpy as np
import pytest

# Colocated worlds (tests/colo.py) run every rank's kernels concurrently on one device, each rank on
# its own streams: give each stream its own hardware queue so no rank's barrier-waiting kernel can
# sit in front of another rank's work (set before CUDA initialises in this process).
# Kernels must also be loaded eagerly: a kernel loaded lazily while another rank's kernel spins at
# a barrier on the same device stalls the world (gf_comm_connect_colocated refuses lazy loading).
os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")
os.environ.setdefault("CUDA_MODULE_LOADING", "EAGER")

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)
GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs the sm_100a kernels)")
    config.addinivalue_line("markers", "multigpu(n): needs n GPUs on one box")


def _cuda_ok():
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:  # pragma: no cover
        return False


def pytest_runtest_setup(item):
    if item.get_closest_marker("gpu") and not _cuda_ok():
        pytest.skip("no CUDA device in this container (run under gpurun)")
    m = item.get_closest_marker("multigpu")
    if m:
        import torch
        need = m.args[0]
        if torch.cuda.device_count() < need:
            pytest.skip(f"needs {need} GPUs, have {torch.cuda.device_count()}")


@pytest.fixture(scope="session")
def oracle():
    from oracle.oracle import Oracle
    return Oracle()


@pytest.fixture(scope="session")
def reference():
    from oracle.oracle import Reference
    if not Reference.available():
        pytest.skip("oracle/_ref not built")
    return Reference()


@pytest.fixture(scope="session")
def golden():
    cache = {}

    def load(name):
        # eager dict: NpzFile reads lazily and is not safe to share across rank threads
        if name not in cache:
            with np.load(os.path.join(GOLDEN, name)) as z:
                cache[name] = {k: z[k] for k in z.files}
        return cache[name]
    return load


@pytest.fixture(scope="session")
def gf():
    """The product's C-ABI (fails loudly if the native library is missing)."""
    from paper_1902_06855_b200 import capi
    capi.lib()
    return capi
