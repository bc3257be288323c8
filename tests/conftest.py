import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100) device; runs through libvp_b200.so")
    # the shared objects are built in-tree; build them if a fresh checkout lacks them
    need = [os.path.join(ROOT, "paper_2205_04401_b200", "libvp_b200.so"),
            os.path.join(ROOT, "oracle", "liboracle.so")]
    if not all(os.path.exists(p) for p in need):
        subprocess.run(["make", "-C", ROOT, "all"], check=True)
    if os.path.isdir("/root/reference/proj/include") and not os.path.exists(
            os.path.join(ROOT, "oracle", "_ref", "libvpref.so")):
        subprocess.run(["make", "-C", ROOT, "ref"], check=True)
