# SPDX-License-Identifier: Apache-2.0
"""The reference's OWN C++ test programs, compiled unchanged against the B200 drop-in.

tests/cpp/Makefile builds /root/reference/proj/tests/{acceptance,test_*}.cpp with our gflow
headers + libgflow_b200.so (doctest subset: tests/cpp/doctest_shim) into tests/_reftests/ (built
here by __graft_entry__.build(); the binaries travel to the GPU box). Each program's own
checks decide: exit 0 and every doctest case passed; acceptance prints 12 PASS lines.
The codec and transport suites need no GPU; the others drive GradientPool / collectives /
FusionEngine / SparseState / train_worker on the B200, ranks as threads.
"""
import os
import subprocess

import pytest

BIN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "_reftests")


def run_suite(name, timeout):
    exe = os.path.join(BIN, name)
    if not os.path.exists(exe):
        pytest.skip(f"{exe} not built (make -C tests/cpp needs /root/reference)")
    env = dict(os.environ)
    env.setdefault("GFLOW_PORT_BASE", str(30000 + (os.getpid() % 2000) * 10))
    # the driver's default kernel loading (conftest.py switches this process to EAGER for the
    # colocated worlds; the reference's suites time pool construction, criterion 1: < 1 s)
    env.pop("CUDA_MODULE_LOADING", None)
    p = subprocess.run([exe], capture_output=True, text=True, timeout=timeout, env=env)
    out = p.stdout + p.stderr
    assert p.returncode == 0, f"{name} exit {p.returncode}\n{out[-6000:]}"
    return out


@pytest.mark.parametrize("name", ["test_half", "test_transport"])
def test_reference_host_suites(name):
    out = run_suite(name, 300)
    assert "Status: SUCCESS" in out, out[-3000:]


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["test_pool", "test_collectives", "test_fusion", "test_sparse", "test_trainer"])
def test_reference_device_suites(name):
    out = run_suite(name, 600)
    assert "Status: SUCCESS" in out, out[-3000:]


@pytest.mark.gpu
def test_reference_acceptance_12_criteria():
    out = run_suite("acceptance", 900)
    passed = [line for line in out.splitlines() if line.startswith("criterion") and "[PASS]" in line]
    assert len(passed) == 12, out[-6000:]
    assert "ALL CRITERIA PASSED" in out
