"""Test configuration. ``-m gpu`` tests need a B200 and call the product through the
C-ABI; everything else runs on CPU (oracle pinning, host-side decomposition, ABI symbols,
multi-process host logic over gloo). The oracle under ../oracle is imported only here,
as the checker."""
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))
GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA (sm_100a) device; run with -m gpu")
    config.addinivalue_line("markers", "slow: larger configurations")


def pytest_collection_modifyitems(config, items):
    """A device-side wait that never completes would block the whole run inside a C call, where a
    signal cannot reach it: give every GPU test a watchdog thread (pytest-timeout, when present)
    that dumps the stacks and ends the process instead."""
    if not config.pluginmanager.hasplugin("timeout"):
        return
    for item in items:
        if item.get_closest_marker("gpu") and not item.get_closest_marker("timeout"):
            item.add_marker(pytest.mark.timeout(300, method="thread"))


@pytest.fixture(scope="session")
def port():
    """The plain-C restatement (always buildable; travels to the GPU box)."""
    import pyoracle
    if pyoracle.PORT is None:
        subprocess_build()
        import importlib
        importlib.reload(pyoracle)
    assert pyoracle.PORT is not None, "oracle/_port not built (make -C oracle port)"
    pyoracle.PORT.set_threads(os.cpu_count() or 1)
    return pyoracle.PORT


@pytest.fixture(scope="session")
def ref():
    """The unmodified reference compiled out of tree, when it was built (CPU container)."""
    import pyoracle
    if pyoracle.REF is None:
        pytest.skip("reference oracle (oracle/_ref) not built here")
    pyoracle.REF.set_threads(os.cpu_count() or 1)
    return pyoracle.REF


def subprocess_build():
    import subprocess
    subprocess.run(["make", "-C", os.path.join(ROOT, "oracle"), "port"], check=True,
                   capture_output=True)


@pytest.fixture(scope="session")
def golden():
    def load(name):
        return np.load(os.path.join(GOLDEN, name), allow_pickle=False)
    return load


@pytest.fixture(scope="session")
def ctx():
    import torch
    if not torch.cuda.is_available():
        pytest.fail("gpu test run without a CUDA device")
    from paper_1508_02977_b200 import flowfem
    return flowfem.default_context()


def rel_l2(a, b):
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    d = np.linalg.norm((a - b).ravel())
    n = np.linalg.norm(b.ravel())
    return d / n if n > 0 else d
