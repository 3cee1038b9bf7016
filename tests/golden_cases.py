"""Shared loader for the reference-generated fixtures (tests/golden/*.npz)."""

import glob
import os

import numpy as np

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def names():
    return sorted(os.path.splitext(os.path.basename(p))[0]
                  for p in glob.glob(os.path.join(GOLDEN, "*.npz")))


def load(name):
    with np.load(os.path.join(GOLDEN, f"{name}.npz")) as z:
        return {k: z[k] for k in z.files}


def system(rec):
    from paper_0810_1119_b200.linalg import SymSystem
    return SymSystem.from_pairs(rec["diag"], rec["pair_i"], rec["pair_j"], rec["pair_v"],
                                rec["rhs"])


def load_serial(name):
    """Serial-schedule fixtures (tests/golden/make_golden_serial.py)."""
    with np.load(os.path.join(GOLDEN, "serial", f"{name}.npz")) as z:
        return {k: z[k] for k in z.files}
