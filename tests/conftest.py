import glob
import os
import sys

import numpy as np
import pytest

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)
GOLDEN_DIR = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200)")


def golden_names():
    return sorted(os.path.basename(p)[len("golden_"):-len(".npz")]
                  for p in glob.glob(os.path.join(GOLDEN_DIR, "golden_*.npz"))
                  if not os.path.basename(p).startswith(("golden_task_", "golden_codec")))


def load_golden(name):
    return dict(np.load(os.path.join(GOLDEN_DIR, f"golden_{name}.npz")))


@pytest.fixture(scope="session")
def oracle_mod():
    from oracle import oracle
    oracle.build()
    return oracle
