"""The persistent chain kernel (csrc/kernels/chain.cuh): tile matmuls as fold
units + in-tile tree items from one dependency-ordered queue, alone
(tt_linalg_product) and as a two-product chain (tt_linalg_chain2).

Checked bit for bit against the CPU oracle (the reference's tt_sum(tt_mul)
restated, oracle/tt_oracle.c) on random GEMM-shaped products: column-local
trees (matmul_b: sum over tile dim 1), row-local trees (matmul_a: sum over
tile dim 2), partial 16-tile blocks, several slot counts -- and counters /
chain indices equal to the two separate calls.  Reference forms:
inc/linalg.hpp:41-73, chain tests/test_linalg.cpp:157-178.
"""
import os
import subprocess
import sys
from pathlib import Path

import numpy as np
import pytest

import paper_2011_01805_b200 as tt
from golden_cases import bitwise_equal
from paper_2011_01805_b200 import configs

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parents[1]


@pytest.fixture(autouse=True)
def chain_on():
    tt.set_chain_kernel(True)
    yield
    tt.set_chain_kernel(False)


def _cost(c):
    return (c.additions, c.multiplications, c.mask_multiplications, c.rotations,
            c.bootstraps, c.power_of_two_rotations)


def _pack(oracle, rng, shape_text, s):
    sh = tt.parse_shape(shape_text)
    dense = rng.standard_normal(size=sh.tensor_extents())
    return sh, oracle.pack(dense, sh, s)


# (tile t1 x t2 x t3, K, N2, N3, M) -- matmul_b(Bt[K/t1,N2/t2,*/t3], C[K/t1,*/t2,N3/t3])
# then matmul_a(A[M/t1,N2/t2,*/t3], R1[*/t1,N2/t2,N3/t3])
CASES = [
    ((16, 32, 16), 768, 1024, 256, 512),   # config 3 (3b) itself
    ((8, 8, 8), 40, 160, 136, 72),         # 512 slots, partial blocks (20 x 17)
    ((8, 16, 8), 64, 400, 96, 200),        # 1024 slots, 25 x 12 output tiles
    ((16, 16, 8), 48, 96, 280, 48),        # 2048 slots, 35 j-tiles
]


@pytest.mark.parametrize("case", CASES)
def test_chain_and_single_products_bitwise(gpu, oracle, case):
    (t1, t2, t3), K, N2, N3, M = case
    s = t1 * t2 * t3
    rng = np.random.default_rng(K * 7 + N3)
    sbt, bt = _pack(oracle, rng, f"[{K}/{t1},{N2}/{t2},*/{t3}]", s)
    sc, c = _pack(oracle, rng, f"[{K}/{t1},*/{t2},{N3}/{t3}]", s)
    sa, a = _pack(oracle, rng, f"[{M}/{t1},{N2}/{t2},*/{t3}]", s)
    s1, w1, k1 = oracle.mul_sum(sbt, bt, sc, c, s, 1)       # matmul_b
    s2, w2, k2 = oracle.mul_sum(sa, a, s1, w1, s, 2)        # matmul_a(A, R1)
    S = tt.Session(s, 8)
    TBt, TC, TA = (tt.TileTensor(sbt, bt, S), tt.TileTensor(sc, c, S), tt.TileTensor(sa, a, S))
    # separate calls (each one chain-kernel launch when eligible)
    S.reset_counters()
    r1 = tt.matmul_b(TBt, TC)
    r2 = tt.matmul_a(TA, r1)
    sep = _cost(S.cost_report())
    assert tt.format_shape(r1.shape()) == tt.format_shape(s1)
    assert tt.format_shape(r2.shape()) == tt.format_shape(s2)
    assert bitwise_equal(r1.tiles(), w1)
    assert bitwise_equal(r2.tiles(), w2)
    # the fused two-product chain
    S.reset_counters()
    f1, f2 = tt.linalg_chain("matmul_b", TBt, TC, "matmul_a", TA)
    assert _cost(S.cost_report()) == sep == tuple(np.add(_cost(k1), _cost(k2)))
    assert bitwise_equal(f1.tiles(), w1)
    assert bitwise_equal(f2.tiles(), w2)
    assert (f1.chain_index(), f2.chain_index()) == (r1.chain_index(), r2.chain_index()) == (7, 6)
    # repeated launches reuse the self-resetting counter blocks
    for _ in range(3):
        g1, g2 = tt.linalg_chain("matmul_b", TBt, TC, "matmul_a", TA)
    assert bitwise_equal(g2.tiles(), w2) and bitwise_equal(g1.tiles(), w1)


def test_chain_first_result_on_the_left_is_the_two_calls(gpu, oracle):
    # matmul_b's result [*/8,40/8,56/8] cannot be matmul_a's LEFT operand (its
    # dim 3 is not replicated, linalg.hpp:32-37): the chain runs the first
    # call, then raises the second call's ShapeError, as the two calls would
    s = 512
    rng = np.random.default_rng(77)
    sbt, bt = _pack(oracle, rng, "[24/8,40/8,*/8]", s)
    sc, c = _pack(oracle, rng, "[24/8,*/8,56/8]", s)
    sx, x = _pack(oracle, rng, "[*/8,40/8,56/8]", s)
    S = tt.Session(s, 8)
    TBt, TC, TX = tt.TileTensor(sbt, bt, S), tt.TileTensor(sc, c, S), tt.TileTensor(sx, x, S)
    S.reset_counters()
    with pytest.raises(tt.ShapeError):
        tt.linalg_chain("matmul_b", TBt, TC, "matmul_a", TX, first_is_right=False)
    assert S.cost_report().multiplications == 3 * 5 * 7


def test_chain_errors_match_two_calls(gpu):
    S = tt.Session(512, 8)
    bt = tt.pack(np.ones((8, 8, 1)), tt.parse_shape("[8/8,8/8,*/8]"), S)
    c = tt.pack(np.ones((8, 1, 8)), tt.parse_shape("[8/8,*/8,8/8]"), S)
    bad = tt.pack(np.ones((8, 8, 8)), tt.parse_shape("[8/8,8/8,8/8]"), S)
    with pytest.raises(tt.ShapeError):     # first product invalid: nothing runs
        tt.linalg_chain("matmul_b", bt, bad, "matmul_a", bt)
    S.reset_counters()
    with pytest.raises(tt.ShapeError):     # second invalid: the first ran and counted
        tt.linalg_chain("matmul_b", bt, c, "matmul_a", bad)
    assert S.cost_report().multiplications == 1


def test_chain_depth_exhaustion(gpu):
    S = tt.Session(512, 1)
    bt = tt.pack(np.ones((8, 8, 1)), tt.parse_shape("[8/8,8/8,*/8]"), S)
    c = tt.pack(np.ones((8, 1, 8)), tt.parse_shape("[8/8,*/8,8/8]"), S)
    a = tt.pack(np.ones((8, 8, 1)), tt.parse_shape("[8/8,8/8,*/8]"), S)
    with pytest.raises(tt.DepthExhaustedError):
        tt.linalg_chain("matmul_b", bt, c, "matmul_a", a)


def test_config3_chain_kernel_off_is_identical(gpu, tmp_path):
    """TT_CHAIN=1 (the chain kernel) and 0 (GEMM fold + tree passes) give the same bits."""
    code = (
        "import sys, numpy as np; sys.path.insert(0, %r);"
        "import paper_2011_01805_b200 as tt; from paper_2011_01805_b200 import configs;"
        "c3 = configs.config3(); S = tt.Session(8192, 8);"
        "T = {k: tt.pack(c3.tensors[k], tt.parse_shape(v), S) for k, v in c3.shapes.items() if k in ('A3','Bt3','C3')};"
        "r = tt.matmul_a(T['A3'], tt.matmul_b(T['Bt3'], T['C3']));"
        "np.save(sys.argv[1], r.tiles())" % str(ROOT))
    outs = []
    for flag in ("0", "1"):
        f = tmp_path / f"c3_{flag}.npy"
        env = dict(os.environ, TT_CHAIN=flag)
        proc = subprocess.run([sys.executable, "-c", code, str(f)], env=env, capture_output=True,
                              text=True, timeout=600)
        assert proc.returncode == 0, proc.stderr[-2000:]
        outs.append(np.load(f))
    assert bitwise_equal(outs[0], outs[1])
