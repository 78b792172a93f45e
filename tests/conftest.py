import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and the built libfmtgp_b200.so")
    config.addinivalue_line("markers", "slow: long-running (full-size configurations)")


def _ensure_ref():
    """The reference oracle is built from /root/reference when present (this container);
    on the GPU box the prebuilt oracle/_ref/libfmtgp_ref.so travels with the snapshot."""
    from oracle import ref
    if not ref.available() and os.path.isdir("/root/reference/proj/src"):
        subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "oracle"), "ref"], check=True)
    return ref


@pytest.fixture(scope="session")
def ref():
    r = _ensure_ref()
    if not r.available():
        pytest.skip("reference oracle unavailable (oracle/_ref not built and /root/reference absent)")
    return r


@pytest.fixture(scope="session")
def port():
    from oracle import port as p
    p.ensure_built()
    return p
