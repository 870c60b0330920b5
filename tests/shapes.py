"""Random shape / data generators and sentinel fuzzing for the tests.

Modelled on the reference's own test helpers (random_pack_shape
tests/test_tile_tensor.cpp:21-51, fuzz_unused_slots :60-79,
fuzz_unknown_regions :82-102, all under /root/reference/proj/).  Python's
``random.Random`` / numpy generators replace mt19937; the draws differ from
the reference's but follow the same distributions.
"""
from __future__ import annotations

import random

import numpy as np

from paper_2011_01805_b200 import DimSpec, TileTensorShape


def random_pack_shape(rng: random.Random, slots: int, rank: int,
                      allow_replication: bool = True) -> TileTensorShape:
    t = [1] * rank
    remaining = slots
    for i in range(rank - 1):
        divisors = []
        x = 1
        while x <= remaining:
            divisors.append(x)
            x *= 2
        t[i] = rng.choice(divisors)
        remaining //= t[i]
    t[rank - 1] = remaining
    dims = []
    for i in range(rank):
        pick = rng.randint(0, 3)
        if allow_replication and pick == 0:
            dims.append(DimSpec(1, t[i], t[i]))
        elif allow_replication and pick == 1 and t[i] > 1:
            dims.append(DimSpec(1, rng.randint(1, t[i]), t[i]))
        else:
            dims.append(DimSpec(rng.randint(1, 12), 1, t[i]))
    return TileTensorShape(dims)


def partner_shape(rng: random.Random, sa: TileTensorShape) -> TileTensorShape:
    """Elementwise partner sharing tile extents (test_tile_tensor.cpp:227-245)."""
    dims = []
    for d in sa.dims():
        k = rng.randint(0, 2)
        if k == 0:
            dims.append(DimSpec(d.n, 1, d.t))
        elif k == 1:
            dims.append(DimSpec(1, d.t, d.t))
        else:
            dims.append(DimSpec(rng.randint(1, 12), 1, d.t))
    return TileTensorShape(dims)


def random_tensor(rng: np.random.Generator, extents, lo=-2.0, hi=2.0) -> np.ndarray:
    return rng.uniform(lo, hi, size=extents).astype(np.float64)


def logical_box(shape: TileTensorShape) -> np.ndarray:
    """j[flat, h, i] for every tile and slot h < tile_slots (Eq. 1)."""
    ext = shape.external_extents()
    rank = shape.rank()
    ts = shape.tile_slots()
    n_tiles = shape.tile_count()
    flat = np.arange(n_tiles)
    h = np.arange(ts)
    out = np.zeros((n_tiles, ts, rank), dtype=np.int64)
    es = 1
    tstride = 1
    tstr = []
    estr = []
    for i in range(rank - 1, -1, -1):
        tstr.insert(0, tstride)
        estr.insert(0, es)
        tstride *= shape.dim(i).t
        es *= ext[i]
    for i in range(rank):
        d = shape.dim(i)
        l = (flat // estr[i]) % ext[i]
        m = (h // tstr[i]) % d.t
        if d.interleaved:
            out[:, :, i] = m[None, :] * ext[i] + l[:, None]
        else:
            out[:, :, i] = l[:, None] * d.t + m[None, :]
    return out


def used_mask(shape: TileTensorShape, s: int) -> np.ndarray:
    """[tiles, s] bool: slot holds data (inside every dim's used range)."""
    j = logical_box(shape)
    used = np.array([d.used() for d in shape.dims()])
    m = np.zeros((shape.tile_count(), s), dtype=bool)
    m[:, :shape.tile_slots()] = np.all(j < used[None, None, :], axis=2)
    return m


def fuzz_unused_slots(shape: TileTensorShape, tiles: np.ndarray, seed: int) -> np.ndarray:
    rng = np.random.default_rng(seed)
    out = tiles.copy()
    s = tiles.shape[1]
    garbage = ~used_mask(shape, s)
    garbage[:, shape.tile_slots():] = False
    out[garbage] = rng.uniform(-100, 100, size=int(garbage.sum()))
    return out


def fuzz_unknown_regions(shape: TileTensorShape, tiles: np.ndarray, seed: int) -> np.ndarray:
    if not shape.has_unknown():
        return tiles
    rng = np.random.default_rng(seed)
    out = tiles.copy()
    j = logical_box(shape)
    garbage = np.zeros((shape.tile_count(), tiles.shape[1]), dtype=bool)
    g = np.zeros(j.shape[:2], dtype=bool)
    for i, d in enumerate(shape.dims()):
        if d.unknown:
            g |= j[:, :, i] >= d.used()
    garbage[:, :shape.tile_slots()] = g
    out[garbage] = rng.uniform(-100, 100, size=int(garbage.sum()))
    return out


def shape_key(shape: TileTensorShape) -> list:
    """Flat int encoding for fixtures: [rank, relaxed, (n,d,t,unknown,interleaved)*rank]."""
    out = [shape.rank(), int(shape.relaxed())]
    for d in shape.dims():
        out += [d.n, d.d, d.t, int(d.unknown), int(d.interleaved)]
    return out


def shape_from_key(key) -> TileTensorShape:
    key = [int(x) for x in key]
    rank, relaxed = key[0], key[1]
    dims = []
    for i in range(rank):
        n, d, t, u, il = key[2 + 5 * i: 7 + 5 * i]
        dims.append(DimSpec(n, d, t, bool(u), bool(il)))
    return TileTensorShape(dims, bool(relaxed))
