import math
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); parity tests through the C-ABI")
    config.addinivalue_line("markers", "slow: long-running CPU test")


# Backbone constants of PAPER.md P:159-167, retyped here from the paper so the
# geometry pins do not read them from the code under test.
BB_THETA = {0: math.pi - 2.1186, 1: math.pi - 1.9391, 2: math.pi - 2.0610}  # C-N, N-CA, CA-C
BB_D = {0: 1.330, 1: 1.460, 2: 1.525}


def dihedral(p0, p1, p2, p3):
    """IUPAC / praxeolitic dihedral angle (radians) of four points."""
    b0, b1, b2 = p0 - p1, p2 - p1, p3 - p2
    b1n = b1 / np.linalg.norm(b1)
    v = b0 - np.dot(b0, b1n) * b1n
    w = b2 - np.dot(b2, b1n) * b1n
    return math.atan2(float(np.dot(np.cross(b1n, v), w)), float(np.dot(v, w)))


def bond_angle(a, b, c):
    u, v = a - b, c - b
    return math.acos(max(-1.0, min(1.0, float(np.dot(u, v) / (np.linalg.norm(u) * np.linalg.norm(v))))))


def angdiff(a, b):
    """Smallest signed difference of two angles."""
    return (a - b + math.pi) % (2 * math.pi) - math.pi


@pytest.fixture(scope="session")
def oracle_lib():
    import oracle

    oracle.build()
    return oracle


@pytest.fixture(scope="session")
def table():
    import synth

    return synth.load_residue_table()


@pytest.fixture(scope="session")
def table_chi5():
    import synth

    return synth.load_residue_table("chi5")
