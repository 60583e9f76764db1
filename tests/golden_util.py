"""Fixture helpers shared by the test modules (tests/ is on sys.path)."""

from pathlib import Path

import numpy as np

GOLDEN = Path(__file__).resolve().parent / "golden"


def load_fixture(name):
    return dict(np.load(GOLDEN / name, allow_pickle=False))
