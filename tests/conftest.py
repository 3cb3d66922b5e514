import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 (run with -m gpu on the GPU box)")
    config.addinivalue_line("markers", "slow: large-size property tests")


def _ensure_built():
    oracle_so = os.path.join(ROOT, "oracle", "_build", "libstrassen_oracle.so")
    if not os.path.exists(oracle_so):
        subprocess.run(["make", "-C", os.path.join(ROOT, "oracle"), "-s"], check=True)
    lib_so = os.path.join(ROOT, "paper_1605_01078_b200", "libstrassen_b200.so")
    if not os.path.exists(lib_so):
        subprocess.run(["make", "-C", os.path.join(ROOT, "paper_1605_01078_b200", "csrc"), "-s",
                        "-j4"], check=True)


_ensure_built()


@pytest.fixture(scope="session")
def cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.fail("GPU test selected but no CUDA device is visible")
    return torch.device("cuda:0")
