"""Shared helpers for the test suite."""
import numpy as np


def rel_err(a, b):
    den = np.linalg.norm(b)
    return float(np.linalg.norm(np.asarray(a) - np.asarray(b)) / (den if den > 0 else 1.0))
