import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")
    config.addinivalue_line("markers", "slow: long-running CPU test")


def pytest_sessionstart(session):
    """The C-ABI library is a build artefact (git-ignored): build it when it is missing, so a fresh
    checkout can run either suite (nvcc cross-compiles sm_100a without a GPU)."""
    lib = os.path.join(ROOT, "paper_2205_05158_b200", "libfdpd.so")
    if not os.path.exists(lib) and not os.environ.get("FDPD_LIB"):
        from paper_2205_05158_b200 import build
        build.build()
