"""The five BASELINE.json configurations as concrete, seeded inputs.

Uniform inputs come from the counter-based generator shared by host and
device (``uniform`` here == ``tt_fill_uniform`` on the GPU ==
``or_fill_uniform`` in the oracle), so any slab of a tensor can be generated
independently and bit-identically anywhere.  Normal draws (configs 3 and 4)
are made on the host with numpy's PCG64 and uploaded (device
log/cos differ from libm).

No public dataset is involved: the paper's MNIST/CryptoNets data is not
needed and seeded synthetic tensors of the configured shapes stand in.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

_M1 = np.uint64(0xBF58476D1CE4E5B9)
_M2 = np.uint64(0x94D049BB133111EB)
_GOLD = np.uint64(0x9E3779B97F4A7C15)


def _splitmix64(x: np.ndarray) -> np.ndarray:
    with np.errstate(over="ignore"):
        x = x + _GOLD
        x = (x ^ (x >> np.uint64(30))) * _M1
        x = (x ^ (x >> np.uint64(27))) * _M2
        return x ^ (x >> np.uint64(31))


def uniform_at(index: np.ndarray, seed: int, lo: float, hi: float) -> np.ndarray:
    """Values of the shared generator at arbitrary flat indices."""
    key = _splitmix64(np.array([seed], dtype=np.uint64))[0]
    u = _splitmix64(np.asarray(index, dtype=np.uint64) ^ key)
    frac = (u >> np.uint64(11)).astype(np.float64) * (2.0 ** -53)
    return lo + (hi - lo) * frac


def uniform(count: int, seed: int, lo: float, hi: float, offset: int = 0) -> np.ndarray:
    return uniform_at(np.arange(offset, offset + count, dtype=np.uint64), seed, lo, hi)


def normal(shape, seed: int, sigma: float) -> np.ndarray:
    return np.random.default_rng(seed).normal(0.0, sigma, size=shape)


# ---- config 5: the throughput sweep -------------------------------------------------

C5_X_SHAPE = "[2048/16,2048/32,512/32]"
C5_W_SHAPE = "[*/16,2048/32,512/32]"
C5_SLOTS = 16384
C5_SEED_X = 13
C5_SEED_W = 14
C5_DIMS = (2048, 2048, 512)


def c5_x_slab(d1: slice = slice(None), d2: slice = slice(None), d3: slice = slice(None),
              rank_offset: int = 0) -> np.ndarray:
    """Dense slab X[d1, d2, d3] of config 5's input (seed 13, U[-1,1]).
    `rank_offset` selects rank r's block of a weak-scaled global tensor."""
    n1, n2, n3 = C5_DIMS
    i1 = np.arange(n1)[d1]
    i2 = np.arange(n2)[d2]
    i3 = np.arange(n3)[d3]
    idx = (i1[:, None, None] * (n2 * n3) + i2[None, :, None] * n3 + i3[None, None, :])
    return uniform_at(idx.astype(np.uint64) + np.uint64(rank_offset), C5_SEED_X, -1.0, 1.0)


def c5_w(d2: slice = slice(None), d3: slice = slice(None)) -> np.ndarray:
    """Dense W [1, 2048, 512] of config 5 (seed 14, U[-1,1])."""
    _, n2, n3 = C5_DIMS
    i2 = np.arange(n2)[d2]
    i3 = np.arange(n3)[d3]
    idx = i2[:, None] * n3 + i3[None, :]
    return uniform_at(idx.astype(np.uint64), C5_SEED_W, -1.0, 1.0)[None, :, :]


# ---- configs 1-4 ---------------------------------------------------------------------


@dataclass
class Case:
    name: str
    slots: int
    tensors: dict      # name -> dense numpy array
    shapes: dict       # name -> shape string


def config1() -> Case:
    a = uniform(100 * 200, 1, -1.0, 1.0).reshape(100, 200)
    b = uniform(100 * 200, 2, -1.0, 1.0).reshape(100, 200)
    return Case("c1", 512, {"A": a, "B": b},
                {"A": "[100/16,200/32]", "B": "[100/16,200/32]"})


def config2() -> Case:
    m = uniform(1024 * 4096, 3, -1.0, 1.0).reshape(1024, 4096)
    v = uniform(4096, 4, -1.0, 1.0).reshape(1, 4096)
    return Case("c2", 8192, {"M": m, "V": v}, {"M": "[1024/64,4096/128]", "V": "[*/64,4096/128]"})


def config3() -> Case:
    """A(512x1024) B(1024x768) C(768x256), normal(0, 1/sqrt(k)), k the inner dim."""
    a = normal((512, 1024), 5, 1.0 / np.sqrt(1024))
    b = normal((1024, 768), 6, 1.0 / np.sqrt(768))
    c = normal((768, 256), 7, 1.0 / np.sqrt(256))
    return Case("c3", 8192, {
        "A3": a.reshape(512, 1024, 1),             # [512/16,1024/32,*/16]
        "Bt3": b.T.copy().reshape(768, 1024, 1),   # [768/16,1024/32,*/16]  (B transposed)
        "C3": c.reshape(768, 1, 256),              # [768/16,*/32,256/16]
        "B3": b.reshape(1, 1024, 768),             # [*/16,1024/32,768/16]  (literal 3a)
        "Ct3": c.T.copy().reshape(1, 256, 768),    # [*/16,256/32,768/16]   (literal 3a)
        "A": a, "B": b, "C": c,
    }, {
        "A3": "[512/16,1024/32,*/16]", "Bt3": "[768/16,1024/32,*/16]", "C3": "[768/16,*/32,256/16]",
        "B3": "[*/16,1024/32,768/16]", "Ct3": "[*/16,256/32,768/16]",
    })


def config4(interleaved: bool = False) -> Case:
    """FC 784->100, square, FC 100->10 on a 4096-sample batch (batch in tile dim 3)."""
    x = uniform(784 * 4096, 8, 0.0, 1.0).reshape(784, 4096)
    w1 = normal((100, 784), 9, 0.1)
    w2 = normal((10, 100), 10, 0.1)
    b1 = normal((100,), 11, 0.01)
    b2 = normal((10,), 12, 0.01)
    batch = "4096~/256" if interleaved else "4096/256"
    return Case("c4" + ("~" if interleaved else ""), 8192, {
        "X": x.reshape(784, 1, 4096),
        "W1t": w1.T.copy().reshape(784, 100, 1),
        "b1": b1.reshape(1, 100, 1),
        "W2": w2.reshape(10, 100, 1),
        "b2": b2.reshape(10, 1, 1),
        "x": x, "w1": w1, "w2": w2, "b1v": b1, "b2v": b2,
    }, {
        "X": f"[784/32,1,{batch}]",
        "W1t": "[784/32,100,*/256]",
        "b1": "[*/32,100,*/256]",
        "W2": "[10/32,100,*/256]",
        "b2": "[10/32,1,*/256]",
    })


def dense_forward_c4(case: Case) -> np.ndarray:
    """Plain float64 forward pass (nn_forward semantics) for config 4: [10, 4096]."""
    t = case.tensors
    h = t["w1"] @ t["x"] + t["b1v"][:, None]
    h = h * h
    return t["w2"] @ h + t["b2v"][:, None]
