"""Helpers shared by the test modules (imported as a top-level module;
pytest puts tests/ on sys.path)."""

import os

import numpy as np

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def load_golden(name):
    return np.load(os.path.join(GOLDEN, name), allow_pickle=False)


def have_cuda():
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False
