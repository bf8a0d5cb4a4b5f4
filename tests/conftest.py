import os
import sys

# Tensor-parallel tests run several ranks of a TP group inside ONE process on one GPU.  With the
# default lazy module loading, a kernel's first launch can wait for the device to go idle --
# which never happens while a peer rank's exchange wait spins for this rank's next GEMM.  Load
# every kernel at context creation instead (must be set before CUDA initialises).
os.environ.setdefault("CUDA_MODULE_LOADING", "EAGER")

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs through the C-ABI library)")
    config.addinivalue_line("markers", "slow: long-running CPU test")
    config.addinivalue_line("markers", "gpu_long: long GPU parity run (minutes of fp64 oracle work); "
                                       "runs only with SART_LONG_GPU_TESTS=1")


def pytest_collection_modifyitems(config, items):
    """The default `-m gpu` tier stays well inside the round-end limit; the long parity runs
    (variants of paths the default tier already covers, at more steps / more geometries) are
    skipped unless SART_LONG_GPU_TESTS=1 -- their logs are committed under profiles/."""
    import pytest
    if os.environ.get("SART_LONG_GPU_TESTS") == "1":
        return
    skip = pytest.mark.skip(reason="long GPU parity run: set SART_LONG_GPU_TESTS=1 (logs in profiles/)")
    for it in items:
        if "gpu_long" in it.keywords:
            it.add_marker(skip)
