"""Pytest configuration: markers and shared fixtures.

``-m "not gpu"`` runs the oracle pins, host logic, ABI-export and gloo
multi-process tests (CPU only).  ``-m gpu`` runs the CUDA parity tests, which
call the C-ABI library through ``paper_2108_12050_b200``.
"""
import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); calls the CUDA path through the C-ABI")
    config.addinivalue_line("markers", "slow: longer CPU test")


@pytest.fixture(scope="session")
def golden_dir():
    return os.path.join(ROOT, "tests", "golden")
