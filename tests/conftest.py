"""pytest configuration: the ``gpu`` marker and the repo root on sys.path.

``-m "not gpu"`` runs here (no GPU): the oracle against its pins, host logic,
and that the C-ABI library loads and exports every symbol ``include/sw2d.h``
declares.  ``-m gpu`` (a B200) runs the parity tests through the C ABI.
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line(
        "markers", "gpu: needs a CUDA GPU (B200, sm_100a); parity through the C ABI")
