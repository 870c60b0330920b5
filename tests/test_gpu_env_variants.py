"""GPU parity of the matmul-path kernel variants selected by environment knobs.

The knobs (TT_GEMM_TMA, TT_GEMM_DYNAMIC, TT_GEMM_CFG, TT_GEMM_BC, TT_GEMM_ORDER,
TT_TREE_SMEM, TT_ROW_ROWS, TT_TREE_TMA, TT_FOLD_RING, TT_FOLD_BLK) are read once when the native library loads, so each variant
runs in its own subprocess; every one must give the oracle's tiles bit for bit.
The chain is the reference's matmul_b -> matmul_a (tests/test_linalg.cpp:157-178)
on 8192-slot 16x32x16 tiles, at a size where both stages take the GEMM fold
and both tree passes (column tree for dim 1, row tree for dim 2).
"""
import hashlib
import json
import os
import subprocess
import sys
from pathlib import Path

import numpy as np
import pytest

from paper_2011_01805_b200 import parse_shape

pytestmark = pytest.mark.gpu

ROOT = Path(__file__).resolve().parents[1]
S = 8192
SHAPES = {"Bt": "[48/16,64/32,*/16]", "C": "[48/16,*/32,40/16]", "A": "[40/16,64/32,*/16]"}

SCRIPT = r"""
import hashlib, json, sys
import numpy as np
sys.path.insert(0, sys.argv[1])
import paper_2011_01805_b200 as tt
from paper_2011_01805_b200 import TileTensor, parse_shape
shapes = json.loads(sys.argv[2])
S = tt.Session(8192, 8)
T = {}
for i, (k, v) in enumerate(sorted(shapes.items())):
    sh = parse_shape(v)
    rng = np.random.default_rng(100 + i)
    T[k] = TileTensor(sh, rng.uniform(-1, 1, size=(sh.tile_count(), 8192)), S)
s1 = tt.matmul_b(T["Bt"], T["C"])
r = tt.matmul_a(T["A"], s1)
F = {}
for i, (k, v) in enumerate(sorted(json.loads(sys.argv[3]).items())):
    sh = parse_shape(v)
    rng = np.random.default_rng(200 + i)
    F[k] = TileTensor(sh, rng.uniform(-1, 1, size=(sh.tile_count(), 8192)), S)
folds = [tt.tt_mul_sum(F["M"], F["V"], 1), tt.tt_mul_sum(F["M"], F["W"], 1), tt.tt_sum(F["M"], 1),
         tt.tt_mul_sum(F["N"], F["U"], 1), tt.tt_mul_sum(F["U"], F["N"], 1)]
h = lambda t: hashlib.sha256(np.ascontiguousarray(t.tiles()).tobytes()).hexdigest()
print(json.dumps({"s1": h(s1), "r": h(r), "folds": [h(f) for f in folds]}))
"""
# few-group folds (t = 1 summed dim, 40 steps): the plain and the cp.async-ring fold
# N x U: two groups along dim 2 that share U's tiles (the group-blocked ring fold)
FOLD_SHAPES = {"M": "[40,2/2,4096/4096]", "V": "[40,2/2,4096/4096]", "W": "[*,2/2,4096/4096]",
               "N": "[40,4/2,4096/4096]", "U": "[40,*/2,4096/4096]"}

VARIANTS = [
    {},
    {"TT_GEMM_TMA": "0"},
    {"TT_GEMM_TMA": "0", "TT_GEMM_BC": "16"},
    {"TT_GEMM_TMA": "0", "TT_GEMM_SLOTS": "64"},
    {"TT_GEMM_DYNAMIC": "0"},
    {"TT_GEMM_ORDER": "1"},
    {"TT_GEMM_CFG": "1"},
    {"TT_GEMM_CFG": "2"},
    {"TT_GEMM_CFG": "3"},
    {"TT_GEMM_CFG": "4"},
    {"TT_GEMM_CFG": "5"},
    {"TT_GEMM_CFG": "6"},
    {"TT_GEMM_CFG": "7"},
    {"TT_GEMM_CFG": "8"},
    {"TT_GEMM_CFG": "9"},
    {"TT_GEMM_CFG": "10"},
    {"TT_GEMM_CFG": "11"},
    {"TT_GEMM_WAIT": "0"},
    {"TT_GEMM_WAIT": "2"},
    {"TT_GEMM_GRID": "200"},
    {"TT_GEMM_CFG": "11", "TT_GEMM_DYNAMIC": "0"},
    {"TT_TREE_SMEM": "1"},
    {"TT_FOLD_RING": "1"},
    {"TT_FOLD_RING": "0"},
    {"TT_FOLD_BLK": "0"},
    {"TT_ROW_CHAIN": "2"},
    {"TT_ROW_CHAIN": "4"},
    {"TT_ROW_ROWS": "16"},
    {"TT_ROW_ROWS": "64"},
    {"TT_TREE_TMA": "1"},
    {"TT_TREE_TMA": "2"},
    {"TT_PDL": "0"},
    {"TT_PDL_OVERSUB": "1"},
    {"TT_GEMM_LATE": "0"},
]


def _digest(x):
    return hashlib.sha256(np.ascontiguousarray(x, dtype=np.float64).tobytes()).hexdigest()


@pytest.fixture(scope="module")
def expected(oracle):
    T = {}
    for i, (k, v) in enumerate(sorted(SHAPES.items())):
        sh = parse_shape(v)
        rng = np.random.default_rng(100 + i)
        T[k] = (sh, rng.uniform(-1, 1, size=(sh.tile_count(), S)))
    s1s, s1t, _ = oracle.mul_sum(*T["Bt"], *T["C"], S, 1)
    rs, rt, _ = oracle.mul_sum(*T["A"], s1s, s1t, S, 2)
    F = {}
    for i, (k, v) in enumerate(sorted(FOLD_SHAPES.items())):
        sh = parse_shape(v)
        rng = np.random.default_rng(200 + i)
        F[k] = (sh, rng.uniform(-1, 1, size=(sh.tile_count(), S)))
    folds = [oracle.mul_sum(*F["M"], *F["V"], S, 1)[1], oracle.mul_sum(*F["M"], *F["W"], S, 1)[1],
             oracle.sum(*F["M"], S, 1)[1], oracle.mul_sum(*F["N"], *F["U"], S, 1)[1],
             oracle.mul_sum(*F["U"], *F["N"], S, 1)[1]]
    return {"s1": _digest(s1t), "r": _digest(rt), "folds": [_digest(f) for f in folds]}


@pytest.mark.parametrize("env", VARIANTS, ids=lambda e: ",".join(f"{k}={v}" for k, v in e.items())
                         or "default")
def test_matmul_chain_variant(gpu, expected, env):
    full = dict(os.environ)
    full.update(env)
    out = subprocess.run([sys.executable, "-c", SCRIPT, str(ROOT), json.dumps(SHAPES),
                          json.dumps(FOLD_SHAPES)],
                         env=full, capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    got = json.loads(out.stdout.strip().splitlines()[-1])
    assert got == expected, f"{env}: {got} vs {expected}"
