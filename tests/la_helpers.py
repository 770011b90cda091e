"""Shared test helpers (golden fixture access)."""

import os

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = os.path.join(ROOT, "tests", "golden", "golden.npz")
FIXTURES = ["ex_a", "ex_b", "ex_c", "ex_d", "ex_e"]


def load_golden():
    return dict(np.load(GOLDEN))


def fixture_case(golden, name):
    """(b, c, v, gamma list, decay, expected) of a canonical fixture EX-A..EX-E."""
    g = golden
    return (g[f"fx_{name}_b"], g[f"fx_{name}_c"], g[f"fx_{name}_v"], list(g[f"fx_{name}_gamma"]),
            bool(g[f"fx_{name}_decay"]), g[f"fx_{name}_expected"])
