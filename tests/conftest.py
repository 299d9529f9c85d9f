"""Shared pytest configuration.

Markers: ``gpu`` — needs a B200 (run on the GPU box with ``-m gpu``); every
other test runs on CPU (``-m "not gpu"``).
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: requires a CUDA B200 device")
    config.addinivalue_line("markers", "slow: long-running CPU test")
