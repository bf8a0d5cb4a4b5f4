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
