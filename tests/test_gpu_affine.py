"""tt_mul_sum_affine (one fully connected stage of cryptonets_infer's tiled branch,
nn.hpp:468-490: tt_sum(tt_mul(a, b)), + bias, square) against the three-call
composition on the GPU -- tiles bit for bit, result shape, chain index, cost
counters and errors -- over every path the tail can take: fused into the column
tree pass (config 4 layer 1), the row-shift tree pass (matmul_a shapes), a
separate epilogue pass after the fused group kernels and the tiny single-launch
reduction, a degenerate sum, and the composition fallbacks (bias broadcasting
the sum to a larger grid, a square that exhausts the depth, incompatible bias)."""
import numpy as np
import pytest

import paper_2011_01805_b200 as tt
from golden_cases import bitwise_equal
from paper_2011_01805_b200 import configs, parse_shape

pytestmark = pytest.mark.gpu


def _rand(shape, seed):
    return np.random.default_rng(seed).uniform(-1, 1, size=shape)


def _compose(a, b, dim, c, square):
    r = tt.tt_mul_sum(a, b, dim)
    if c is not None:
        r = tt.tt_add(r, c)
    if square:
        r = tt.tt_mul(r, r)
    return r


def _check(S, a, b, dim, c, square):
    S.reset_counters()
    want = _compose(a, b, dim, c, square)
    want_cost = S.cost_report()
    S.reset_counters()
    got = tt.tt_mul_sum_affine(a, b, dim, c, square=square)
    got_cost = S.cost_report()
    assert tt.format_shape(got.shape()) == tt.format_shape(want.shape())
    assert got.chain_index() == want.chain_index()
    assert bitwise_equal(got.tiles(), want.tiles())
    assert got_cost == want_cost, (got_cost, want_cost)
    return got


def _pack(S, spec, dense_shape, seed):
    return tt.pack(_rand(dense_shape, seed), parse_shape(spec), S)


@pytest.mark.parametrize("square", [False, True])
def test_config4_layer1_column_tree(gpu, oracle, square):
    case = configs.config4(False)
    S = tt.Session(8192, 8)
    T = {k: tt.pack(case.tensors[k], parse_shape(v), S) for k, v in case.shapes.items()}
    got = _check(S, T["W1t"], T["X"], 1, T["b1"], square)
    # and against the CPU oracle's composition
    s = 8192
    ps = {k: parse_shape(v) for k, v in case.shapes.items()}
    p = {k: oracle.pack(case.tensors[k], ps[k], s) for k in ("W1t", "X", "b1")}
    s1, o1, _ = oracle.mul_sum(ps["W1t"], p["W1t"], ps["X"], p["X"], s, 1)
    s2, o2, _ = oracle.elementwise(0, s1, o1, ps["b1"], p["b1"], s)
    if square:
        s2, o2, _ = oracle.elementwise(1, s2, o2, s2, o2, s)
    assert bitwise_equal(got.tiles(), o2)


@pytest.mark.parametrize("bias", ["[64/16,*/32,*/16]", "[64/16,*/32,64/16]", None])
def test_matmul_a_row_tree(gpu, bias):
    S = tt.Session(8192, 8)
    a = _pack(S, "[64/16,128/32,*/16]", (64, 128, 1), 1)
    b = _pack(S, "[*/16,128/32,64/16]", (1, 128, 64), 2)
    c = None
    if bias is not None:
        dshape = tuple(1 if "*" in d else int(d.split("/")[0]) for d in bias[1:-1].split(","))
        c = _pack(S, bias, dshape, 3)
    for square in (False, True):
        _check(S, a, b, 2, c, square)


def test_config1_single_launch(gpu):
    c1 = configs.config1()
    S = tt.Session(512, 8)
    a = tt.pack(c1.tensors["A"], parse_shape(c1.shapes["A"]), S)
    b = tt.pack(c1.tensors["B"], parse_shape(c1.shapes["B"]), S)
    c = _pack(S, "[100/16,*/32]", (100, 1), 4)
    for square in (False, True):
        _check(S, a, b, 2, c, square)
    _check(S, a, b, 2, None, True)


@pytest.mark.parametrize("dim", [1, 2, 3])
def test_group_kernels_separate_tail(gpu, dim):
    """c5-like shapes: the fused group kernels (TMA ring / window) end the
    reduction, the tail runs as its own in-place pass."""
    S = tt.Session(16384, 8)
    x = _pack(S, "[256/16,256/32,64/32]", (256, 256, 64), 5)
    w = _pack(S, "[*/16,256/32,64/32]", (1, 256, 64), 6)
    r = tt.tt_mul_sum(x, w, dim)
    dense = tuple(1 if d.n == 1 else d.n for d in r.shape().dims())
    spec = tt.format_shape(r.shape()).replace("1?", "1")
    c = _pack(S, spec, dense, 7)
    _check(S, x, w, dim, c, True)


def test_degenerate_sum(gpu):
    S = tt.Session(512, 8)
    a = _pack(S, "[*/16,200/32]", (1, 200), 8)
    b = _pack(S, "[*/16,200/32]", (1, 200), 9)
    c = _pack(S, "[*/16,200/32]", (1, 200), 10)
    _check(S, a, b, 1, c, True)


def test_composition_fallbacks(gpu):
    S = tt.Session(512, 8)
    a = _pack(S, "[64/16,64/32]", (64, 64), 11)
    b = _pack(S, "[64/16,64/32]", (64, 64), 12)
    # the bias broadcasts the sum [*/16,64/32] (1 x 2 tiles) to 4 x 2 tiles
    big = _pack(S, "[64/16,64/32]", (64, 64), 13)
    got = _check(S, a, b, 1, big, True)
    assert got.shape().tile_count() == 8
    # incompatible bias: the same ShapeError as the composition's tt_add
    bad = _pack(S, "[64/16,64/32]", (64, 64), 14)
    with pytest.raises(tt.ShapeError) as e1:
        _compose(a, b, 2, bad, True)
    S.reset_counters()
    with pytest.raises(tt.ShapeError) as e2:
        tt.tt_mul_sum_affine(a, b, 2, bad, square=True)
    assert str(e1.value) == str(e2.value)


def test_square_exhausts_depth(gpu):
    S = tt.Session(512, 1)  # packed tensors have chain index 1; after the product 0
    a = _pack(S, "[64/16,64/32]", (64, 64), 15)
    b = _pack(S, "[64/16,64/32]", (64, 64), 16)
    c = _pack(S, "[64/16,*/32]", (64, 1), 17)
    S.reset_counters()
    with pytest.raises(tt.DepthExhaustedError) as e1:
        _compose(a, b, 2, c, True)
    want_cost = S.cost_report()
    S.reset_counters()
    with pytest.raises(tt.DepthExhaustedError) as e2:
        tt.tt_mul_sum_affine(a, b, 2, c, square=True)
    assert S.cost_report() == want_cost
    assert str(e1.value) == str(e2.value)
    # without the square the stage itself is fine
    _check(S, a, b, 2, c, False)



def _pack_random(S, shape, nrng):
    ext = tuple(d.n for d in shape.dims())
    return tt.pack(nrng.uniform(-2, 2, size=ext), shape, S)


@pytest.mark.parametrize("s", [16, 64, 512, 8192])
def test_random_shapes_match_composition(gpu, s):
    """Random operand pairs (the reference's random_pack_shape / partner draws),
    every summed dim, random bias partners of the sum's shape (compatible or
    not) and square on/off: the fused call equals the composition in tiles,
    shape, chain, counters -- or raises the same error."""
    import random
    from shapes import partner_shape, random_pack_shape
    rng = random.Random(9000 + s)
    nrng = np.random.default_rng(s)
    S = tt.Session(s, 8)
    runs = errors = 0
    for _ in range(40 if s < 8192 else 12):
        sa = random_pack_shape(rng, s, rng.randint(1, 3))
        sb = partner_shape(rng, sa)
        a, b = _pack_random(S, sa, nrng), _pack_random(S, sb, nrng)
        dim = rng.randint(1, sa.rank())
        try:
            so = tt.sum_result_shape(tt.elementwise_result_shape(sa, sb, tt.OpKind.mul), dim)
        except tt.ShapeError:
            continue
        plain = tt.TileTensorShape([tt.DimSpec(d.n, d.d, d.t) for d in so.dims()])
        sc = partner_shape(rng, plain)
        c = _pack_random(S, sc, nrng)
        square = rng.random() < 0.5
        S.reset_counters()
        try:
            want = _compose(a, b, dim, c, square)
            werr = None
        except (tt.ShapeError, tt.DepthExhaustedError) as e:
            want, werr = None, e
        want_cost = S.cost_report()
        S.reset_counters()
        if werr is not None:
            with pytest.raises(type(werr)) as ge:
                tt.tt_mul_sum_affine(a, b, dim, c, square=square)
            assert str(ge.value) == str(werr)
            errors += 1
            continue
        got = tt.tt_mul_sum_affine(a, b, dim, c, square=square)
        assert S.cost_report() == want_cost
        assert tt.format_shape(got.shape()) == tt.format_shape(want.shape())
        assert got.chain_index() == want.chain_index()
        assert bitwise_equal(got.tiles(), want.tiles()), (tt.format_shape(sa), tt.format_shape(sb), dim)
        runs += 1
    assert runs >= 5


# ---- tt_mul_sum_clean: clean_unknowns(tt_sum(tt_mul(a, b), dim)) ---------------------


def _check_clean(S, a, b, dim):
    S.reset_counters()
    want = tt.clean_unknowns(tt.tt_mul_sum(a, b, dim))
    want_cost = S.cost_report()
    S.reset_counters()
    got = tt.tt_mul_sum_clean(a, b, dim)
    assert S.cost_report() == want_cost, (S.cost_report(), want_cost)
    assert tt.format_shape(got.shape()) == tt.format_shape(want.shape())
    assert got.chain_index() == want.chain_index()
    assert bitwise_equal(got.tiles(), want.tiles())
    return got


def test_clean_seam_config3_literal(gpu, oracle):
    """matmul_a(A, B) -> clean_unknowns (config 3's literal chain): GEMM fold +
    row-shift tree with the mask in its store; bitwise vs the oracle too."""
    c3 = configs.config3()
    s = 8192
    S = tt.Session(s, 8)
    sh = {k: parse_shape(c3.shapes[k]) for k in ("A3", "B3")}
    T = {k: tt.pack(c3.tensors[k], sh[k], S) for k in sh}
    got = _check_clean(S, T["A3"], T["B3"], 2)
    assert tt.format_shape(got.shape()) == "[512/16,1/32,768/16]"
    p = {k: oracle.pack(c3.tensors[k], sh[k], s) for k in sh}
    so, o, _ = oracle.mul_sum(sh["A3"], p["A3"], sh["B3"], p["B3"], s, 2)
    sc, oc, _ = oracle.clean_unknowns(so, o, s)
    assert bitwise_equal(got.tiles(), oc)


def test_clean_seam_paths(gpu):
    # c1: two cut dims (100 = 6 x 16 + 4 rows, and the summed 1?/32), one launch
    c1 = configs.config1()
    S = tt.Session(512, 8)
    a = tt.pack(c1.tensors["A"], parse_shape(c1.shapes["A"]), S)
    b = tt.pack(c1.tensors["B"], parse_shape(c1.shapes["B"]), S)
    _check_clean(S, a, b, 2)
    _check_clean(S, a, b, 1)
    # config-5-like group kernels (TMA ring / window), every dim
    S = tt.Session(16384, 8)
    x = _pack(S, "[200/16,256/32,64/32]", (200, 256, 64), 21)
    w = _pack(S, "[*/16,256/32,64/32]", (1, 256, 64), 22)
    for dim in (1, 2, 3):
        _check_clean(S, x, w, dim)
    # config 2: matvec (fold + row tree), and no '?' (clean is the identity)
    c2 = configs.config2()
    S = tt.Session(8192, 8)
    m = tt.pack(c2.tensors["M"], parse_shape(c2.shapes["M"]), S)
    v = tt.pack(c2.tensors["V"], parse_shape(c2.shapes["V"]), S)
    _check_clean(S, m, v, 2)
    _check_clean(S, m, m, 1)


def test_clean_seam_depth(gpu):
    S = tt.Session(512, 1)  # the product leaves chain 0: clean must fail after it
    a = _pack(S, "[64/16,64/32]", (64, 64), 23)
    b = _pack(S, "[64/16,64/32]", (64, 64), 24)
    S.reset_counters()
    with pytest.raises(tt.DepthExhaustedError) as e1:
        tt.clean_unknowns(tt.tt_mul_sum(a, b, 2))
    want = S.cost_report()
    S.reset_counters()
    with pytest.raises(tt.DepthExhaustedError) as e2:
        tt.tt_mul_sum_clean(a, b, 2)
    assert S.cost_report() == want and str(e1.value) == str(e2.value)


@pytest.mark.parametrize("s", [16, 64, 512, 8192])
def test_clean_seam_random(gpu, s):
    import random
    from shapes import partner_shape, random_pack_shape
    rng = random.Random(7000 + s)
    nrng = np.random.default_rng(70 + s)
    S = tt.Session(s, 8)
    runs = 0
    for _ in range(40 if s < 8192 else 12):
        sa = random_pack_shape(rng, s, rng.randint(1, 3))
        sb = partner_shape(rng, sa)
        a, b = _pack_random(S, sa, nrng), _pack_random(S, sb, nrng)
        dim = rng.randint(1, sa.rank())
        try:
            tt.sum_result_shape(tt.elementwise_result_shape(sa, sb, tt.OpKind.mul), dim)
        except tt.ShapeError:
            continue
        _check_clean(S, a, b, dim)
        runs += 1
    assert runs >= 5


@pytest.mark.parametrize("square", [False, True])
def test_config4_layer2_ring_fold_tail(gpu, square):
    """Config 4's second layer: a fold-only reduction (t2 = 1) over 100 steps whose
    streamed operand (100 MiB) takes the cp.async-ring fold -- the tail (+ bias,
    square) is applied in the fold's store, no separate pass.  Bias broadcast along
    the batch tiles, and a bias-free square."""
    S = tt.Session(8192, 8)
    nrng = np.random.default_rng(44)
    sw, sh = parse_shape("[10/32,100,*/256]"), parse_shape("[*/32,100,4096/256]")
    w = tt.TileTensor(sw, nrng.uniform(-1, 1, size=(sw.tile_count(), 8192)), S)
    h = tt.TileTensor(sh, nrng.uniform(-1, 1, size=(sh.tile_count(), 8192)), S)
    b = _pack(S, "[10/32,1,*/256]", (10, 1, 1), 45)
    launches0 = S.launches()
    got = _check(S, w, h, 2, b, square)
    assert got.shape().tile_count() == 16
    _check(S, w, h, 2, None, True)
    # the fused call is one launch (the composition before it: fold + add (+ mul))
    S.reset_counters()
    n0 = S.launches()
    tt.tt_mul_sum_affine(w, h, 2, b, square=square)
    assert S.launches() - n0 == 1, S.launches() - n0
    assert launches0 >= 0
