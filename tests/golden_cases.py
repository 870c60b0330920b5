"""Loader for tests/golden (fixtures produced by the reference via make_golden.py)."""
from __future__ import annotations

import hashlib
import json
from pathlib import Path

import numpy as np

from shapes import shape_from_key

HERE = Path(__file__).resolve().parent / "golden"
COST = ("additions", "multiplications", "mask_multiplications", "rotations", "bootstraps",
        "power_of_two_rotations")


class Case(dict):
    def arr(self, name):
        return self["_arrays"][f"c{self['_i']}_{name}"]

    def shape(self, name):
        return shape_from_key(self[name])


def load():
    index = json.loads((HERE / "golden_index.json").read_text())
    arrays = np.load(HERE / "golden.npz")
    out = []
    for i, meta in enumerate(index):
        c = Case(meta)
        c["_i"] = i
        c["_arrays"] = arrays
        out.append(c)
    return out


def cost_tuple(c) -> tuple:
    return tuple(int(getattr(c, f)) for f in COST)


def bitwise_equal(a, b) -> bool:
    a = np.ascontiguousarray(a, dtype=np.float64)
    b = np.ascontiguousarray(b, dtype=np.float64)
    return a.shape == b.shape and np.array_equal(a.view(np.uint64), b.view(np.uint64))


def digest(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a, dtype=np.float64).tobytes()).hexdigest()
