import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); runs the product path")
    config.addinivalue_line("markers", "slow: long-running")


def _ensure_built():
    """Build the product library and the oracles if they are missing (nvcc/g++ are in
    the image; the reference sources are only needed for oracle/_ref, which is
    prebuilt when the repo is shipped to a GPU box)."""
    import shutil
    have_tools = shutil.which("nvcc") and shutil.which("make")
    lib = os.path.join(ROOT, "paper_1908_06869_b200", "lib", "libxsp.so")
    if have_tools or not os.path.exists(lib):  # incremental: a no-op when up to date
        subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "paper_1908_06869_b200"), "-j8"], check=True)
    if have_tools or not os.path.exists(os.path.join(ROOT, "oracle", "lib", "libxsp_oracle.so")):
        subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "oracle"), "port"], check=True)
    ref = os.path.join(ROOT, "oracle", "_ref", "libxsp_ref.so")
    if not os.path.exists(ref) and os.path.exists("/root/reference/proj/src"):
        subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "oracle"), "ref", "-j8"], check=True)


_ensure_built()


@pytest.fixture(scope="session")
def engine():
    from paper_1908_06869_b200 import Engine
    e = Engine(0)
    yield e
    e.close()


@pytest.fixture(scope="session")
def has_ref():
    from oracle import ref
    if not ref.available():
        pytest.skip("oracle/_ref not built (needs /root/reference at build time)")
    return True
