"""Reader for tests/golden/golden_v1.npz (written by tests/golden/make_golden.py
from the reference library itself)."""
import os

import numpy as np

from oracle_lib import Fmt

PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden",
                    "golden_v1.npz")


def load():
    return np.load(PATH)


def quantize_cases(z=None):
    z = load() if z is None else z
    for i, row in enumerate(z["meta"]):
        fmt = Fmt(*[int(v) for v in row[1:9]])
        mode, seed, call, st, ndim = (int(v) for v in row[9:14])
        x, y = z[f"x{i}"], z[f"y{i}"]
        yield i, fmt, mode, seed, call, st, x, y
