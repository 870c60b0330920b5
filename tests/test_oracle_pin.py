"""Pin the CPU oracle (oracle/tt_oracle.c) before trusting it.

1. Every golden fixture (outputs of the reference itself, tests/golden) is
   reproduced bit for bit, counters included.
2. The reference's own known-answer tests, restated from its test sources
   (paths under /root/reference/proj/tests/), hold for the oracle.
3. When the reference library is built here (oracle/_ref), random cases are
   compared live against it.
"""
import random

import numpy as np
import pytest

from golden_cases import bitwise_equal, cost_tuple, digest, load
from paper_2011_01805_b200 import DimSpec, TileTensorShape, configs, parse_shape
from shapes import partner_shape, random_pack_shape

CASES = load()
LINALG_DIM = {0: 2, 1: 1, 2: 2, 3: 1}


def by_kind(kind):
    return [c for c in CASES if c["kind"] == kind]


def test_golden_pack(oracle):
    for c in by_kind("pack"):
        got = oracle.pack(c.arr("dense"), c.shape("shape"), c["s"])
        assert bitwise_equal(got, c.arr("tiles"))
        assert bitwise_equal(oracle.unpack(c.shape("shape"), c["s"], got), c.arr("dense"))


def test_golden_elementwise(oracle):
    for c in by_kind("elementwise"):
        so, out, cost = oracle.elementwise(c["op"], c.shape("sa"), c.arr("ta"), c.shape("sb"),
                                           c.arr("tb"), c["s"])
        assert so == c.shape("so")
        assert bitwise_equal(out, c.arr("out"))
        assert cost_tuple(cost) == tuple(c.arr("cost"))


def test_golden_sum(oracle):
    n = 0
    for c in by_kind("sum"):
        so, out, cost = oracle.sum(c.shape("shape"), c.arr("tiles"), c["s"], c["dim"], c["variant"])
        assert so == c.shape("so")
        assert bitwise_equal(out, c.arr("out")), (c["dim"], c["variant"])
        assert cost_tuple(cost) == tuple(c.arr("cost"))
        n += 1
    assert n > 150
    for c in by_kind("sum_error"):
        with pytest.raises(Exception) as ei:
            oracle.sum(c.shape("shape"), c.arr("tiles"), c["s"], c["dim"], c["variant"])
        assert ei.value.code == c["code"]


def test_golden_products(oracle):
    for c in by_kind("linalg"):
        so, out, cost = oracle.mul_sum(c.shape("sa"), c.arr("ta"), c.shape("sb"), c.arr("tb"),
                                       c["s"], LINALG_DIM[c["which"]])
        assert so == c.shape("so")
        assert bitwise_equal(out, c.arr("out"))
        assert cost_tuple(cost) == tuple(c.arr("cost"))


def test_golden_clean_replicate(oracle):
    for c in by_kind("clean"):
        so, out, cost = oracle.clean_unknowns(c.shape("shape"), c.arr("tiles"), c["s"])
        assert so == c.shape("so") and bitwise_equal(out, c.arr("out"))
        assert cost_tuple(cost) == tuple(c.arr("cost"))
    for c in by_kind("replicate"):
        so, out, cost = oracle.replicate_dim(c.shape("shape"), c.arr("tiles"), c["s"], c["dim"])
        assert so == c.shape("so") and bitwise_equal(out, c.arr("out"))
        assert cost_tuple(cost) == tuple(c.arr("cost"))


def test_golden_tile_schedules(oracle):
    for c in by_kind("strided"):
        out, cost = oracle.sum_tile_strided(c.arr("tile"), c["n"], c["stride"], c["variant"])
        assert bitwise_equal(out, c.arr("out")) and cost_tuple(cost) == tuple(c.arr("cost"))
    for c in by_kind("rotate"):
        out, cost = oracle.rotate(c.arr("tile"), c["offset"])
        assert bitwise_equal(out, c.arr("out")) and cost_tuple(cost) == tuple(c.arr("cost"))


def test_golden_configs(oracle):
    c1 = next(c for c in by_kind("config") if c["name"] == "c1")
    case = configs.config1()
    sA = parse_shape(case.shapes["A"])
    pa, pb = oracle.pack(case.tensors["A"], sA, 512), oracle.pack(case.tensors["B"], sA, 512)
    so, out, cost = oracle.mul_sum(sA, pa, sA, pb, 512, 2)
    assert so == c1.shape("so") and bitwise_equal(out, c1.arr("out"))
    assert cost_tuple(cost)[:4] == (77, 49, 0, 35)  # SURVEY 8(d) c1 counters
    c2g = next(c for c in by_kind("config_digest") if c["name"] == "c2")
    case = configs.config2()
    sM, sV = parse_shape(case.shapes["M"]), parse_shape(case.shapes["V"])
    pm, pv = oracle.pack(case.tensors["M"], sM, 8192), oracle.pack(case.tensors["V"], sV, 8192)
    so, out, cost = oracle.mul_sum(sM, pm, sV, pv, 8192, 2)
    assert digest(out) == c2g["digest"]
    assert cost_tuple(cost)[:4] == (608, 512, 0, 112)


# ---- reference KATs restated from the reference's test sources ----------------------


def test_kat_pack_figures(oracle):
    """tests/test_tile_tensor.cpp:152-181."""
    v = np.array([1.0, 2, 3, 4, 5])
    t = oracle.pack(v, parse_shape("[5/2,*/4]"), 8)
    assert t.tolist() == [[1, 1, 1, 1, 2, 2, 2, 2], [3, 3, 3, 3, 4, 4, 4, 4], [5, 5, 5, 5, 0, 0, 0, 0]]
    assert oracle.pack(v, parse_shape("[5/2,*3/4]"), 8)[0].tolist() == [1, 1, 1, 0, 2, 2, 2, 0]
    m = np.random.default_rng(67).uniform(-2, 2, (5, 6))
    tm = oracle.pack(m, parse_shape("[5/2,6/4]"), 8)
    assert tm.shape == (6, 8)
    assert tm[0][1] == m[0, 1] and tm[0][5] == m[1, 1] and tm[4][4] == 0.0
    assert oracle.pack(np.array([42.5]), parse_shape("[*/4]"), 4).tolist() == [[42.5] * 4]


def test_kat_rotate_and_schedules(oracle):
    """tests/test_backend.cpp:32-45 and tests/test_rotate_sum.cpp:117-154."""
    t = np.array([1.0, 2, 3, 4])
    assert oracle.rotate(t, 1)[0].tolist() == [2, 3, 4, 1]
    assert oracle.rotate(t, -1)[0].tolist() == [4, 1, 2, 3]
    assert oracle.rotate(t, 5)[0].tolist() == [2, 3, 4, 1]
    for off in (0, 4, -8):
        out, c = oracle.rotate(t, off)
        assert out.tolist() == [1, 2, 3, 4] and c.rotations == 0
    tile = np.array([1.0, 2, 3, 4, 10, 20, 30, 40])
    rows, _ = oracle.sum_tile_strided(tile, 2, 4, -1)       # sum_tile_dim dim 1 of [2,4]
    assert rows.tolist() == [11, 22, 33, 44, 11, 22, 33, 44]
    cols, _ = oracle.sum_tile_strided(tile, 4, 1, -1)       # dim 2
    assert cols[0] == 10 and cols[4] == 100
    whole, _ = oracle.sum_tile_strided(tile, 8, 1, -1)
    assert whole.tolist() == [110] * 8
    r, c = oracle.replicate_tile_dim(np.array([5.0, 0, 0, 0, 7, 0, 0, 0]), [2, 4], 2)
    assert r.tolist() == [5, 5, 5, 5, 7, 7, 7, 7] and c.rotations == 2
    r2, c2 = oracle.replicate_tile_dim(np.array([3.0, 0, 0, 0, 0, 0]), [6], 1)
    assert r2.tolist() == [3] * 6 and c2.rotations == 3


def test_kat_running_sums_all_schedules(oracle):
    """tests/test_rotate_sum.cpp:30-45: every schedule yields the running-sum
    vector exactly on integer tiles."""
    rng = np.random.default_rng(41)
    for s in (16, 64, 256):
        v = rng.integers(-50, 51, s).astype(np.float64)
        for n in rng.integers(1, s + 1, 40):
            want = np.array([sum(v[(j + i) % s] for i in range(n)) for j in range(s)])
            for var in (0, 1, 2):
                if var == 2 and n & (n - 1):
                    continue
                got, _ = oracle.sum_tile_strided(v, int(n), 1, var)
                assert np.array_equal(got, want)


def test_kat_rotation_counts(oracle):
    """tests/test_rotate_sum.cpp:47-78 (closed forms, 1190 -> 14, 2048 -> 11)."""
    import paper_2011_01805_b200 as tt
    v = np.random.default_rng(43).integers(-50, 51, 4096).astype(np.float64)
    for n in range(1, 129):
        _, c0 = oracle.sum_tile_strided(v, n, 1, 0)
        _, c1 = oracle.sum_tile_strided(v, n, 1, 1)
        assert c0.rotations == tt.rotations_left_to_right(n)
        assert c1.rotations == tt.rotations_right_to_left(n)
        assert c0.additions == c0.rotations and c1.additions == c1.rotations
    assert tt.rotations_left_to_right(1190) == 14 and tt.rotations_right_to_left(1190) == 14
    assert tt.rotations_left_to_right(2048) == 11 and tt.rotations_right_to_left(2048) == 11
    _, c = oracle.sum_tile_strided(v, 1190, 1, 1)
    assert c.rotations == 14 and c.power_of_two_rotations == 14


def test_kat_table_one_and_small_sum(oracle):
    """tests/test_tile_tensor.cpp:487-507 and the shape-rule example."""
    from paper_2011_01805_b200 import format_shape
    a = np.random.default_rng(113).uniform(-2, 2, (4, 3, 5))
    shape = parse_shape("[4,3/8,5/16]")
    t = oracle.pack(a, shape, 128)
    want = ["[1,3/8,5/16]", "[4,*/8,5/16]", "[4,3/8,1?/16]"]
    for dim in (1, 2, 3):
        so, out, _ = oracle.sum(shape, t, 128, dim)
        assert format_shape(so) == want[dim - 1]
        assert oracle.max_rel_diff(oracle.unpack(so, 128, out), oracle.dense_sum(a, dim)) < 1e-9
    small = oracle.pack(np.array([[1.0, 2], [3, 4]]), parse_shape("[2/2,2/2]"), 4)
    so, out, _ = oracle.sum(parse_shape("[2/2,2/2]"), small, 4, 2)
    assert format_shape(so) == "[2/2,1?/2]"
    assert oracle.unpack(so, 4, out).tolist() == [[3.0], [7.0]]


def test_kat_added_garbage(oracle):
    """tests/test_tile_tensor.cpp:266-288: [18/8,4/16] (+|*) [*/8,4/16]."""
    from paper_2011_01805_b200 import format_shape
    rng = np.random.default_rng(79)
    m, v = rng.uniform(-2, 2, (18, 4)), rng.uniform(-2, 2, (1, 4))
    sm, sv = parse_shape("[18/8,4/16]"), parse_shape("[*/8,4/16]")
    tm, tv = oracle.pack(m, sm, 128), oracle.pack(v, sv, 128)
    so, out, _ = oracle.elementwise(0, sm, tm, sv, tv, 128)
    assert format_shape(so) == "[18?/8,4/16]"
    assert out[2][3 * 16 + 2] == v[0, 2]  # logical (19, 2): welded row 19 holds v
    so, out, _ = oracle.elementwise(1, sm, tm, sv, tv, 128)
    assert format_shape(so) == "[18/8,4/16]"
    assert out[2][2 * 16 + 2] == 0.0
    assert oracle.max_rel_diff(oracle.unpack(so, 128, out), oracle.dense_elementwise(1, m, v)) < 1e-9


def test_homomorphisms_against_dense(oracle):
    """Criterion 5 (tests/acceptance_main.cpp:205-292): unpack(op(pack)) == dense op."""
    rng = random.Random(5005)
    nrng = np.random.default_rng(5005)
    for it in range(200):
        s = 1 << rng.randint(2, 5)
        sa = random_pack_shape(rng, s, rng.randint(1, 3))
        a = nrng.uniform(-1, 1, sa.tensor_extents())
        ta = oracle.pack(a, sa, s)
        for dim in range(1, sa.rank() + 1):
            so, out, _ = oracle.sum(sa, ta, s, dim)
            assert oracle.max_rel_diff(oracle.unpack(so, s, out), oracle.dense_sum(a, dim)) < 1e-9


# ---- live comparison against the reference (this container only) ---------------------


def test_live_against_reference(oracle, ref):
    rng = random.Random(99)
    nrng = np.random.default_rng(99)
    for it in range(150):
        s = 1 << rng.randint(2, 6)
        sh = random_pack_shape(rng, s, rng.randint(1, 4))
        a = nrng.uniform(-1, 1, sh.tensor_extents())
        assert bitwise_equal(oracle.pack(a, sh, s), ref.pack(a, sh, s))
        tiles = nrng.uniform(-5, 5, (sh.tile_count(), s))
        for dim in range(1, sh.rank() + 1):
            for v in (-1, 0, 1):
                r1, r2 = oracle.sum(sh, tiles, s, dim, v), ref.sum(sh, tiles, s, dim, v)
                assert r1[0] == r2[0] and bitwise_equal(r1[1], r2[1])
                assert cost_tuple(r1[2]) == cost_tuple(r2[2])
        sb = partner_shape(rng, sh)
        tb = nrng.uniform(-5, 5, (sb.tile_count(), s))
        for op in (0, 1):
            try:
                r2 = ref.elementwise(op, sh, tiles, sb, tb, s)
            except Exception:
                with pytest.raises(Exception):
                    oracle.elementwise(op, sh, tiles, sb, tb, s)
                continue
            r1 = oracle.elementwise(op, sh, tiles, sb, tb, s)
            assert r1[0] == r2[0] and bitwise_equal(r1[1], r2[1])


def _golden_digest(name):
    return next(c for c in CASES if c["kind"] == "config_digest" and c["name"] == name)


def test_golden_config3_and_4_full_size(oracle):
    """Full-size configs 3 and 4: the oracle reproduces the reference's digests."""
    c3 = configs.config3()
    s = 8192
    sh = {k: parse_shape(v) for k, v in c3.shapes.items()}
    p = {k: oracle.pack(c3.tensors[k], sh[k], s) for k in sh}
    s1, o1, _ = oracle.mul_sum(sh["Bt3"], p["Bt3"], sh["C3"], p["C3"], s, 1)
    assert digest(o1) == _golden_digest("c3b_stage1")["digest"]
    s2, o2, _ = oracle.mul_sum(sh["A3"], p["A3"], s1, o1, s, 2)
    assert digest(o2) == _golden_digest("c3b")["digest"]
    c4 = configs.config4(False)
    sh4 = {k: parse_shape(v) for k, v in c4.shapes.items()}
    p4 = {k: oracle.pack(c4.tensors[k], sh4[k], s) for k in sh4}
    h1, t1, _ = oracle.mul_sum(sh4["W1t"], p4["W1t"], sh4["X"], p4["X"], s, 1)
    h2, t2, _ = oracle.elementwise(0, h1, t1, sh4["b1"], p4["b1"], s)
    h3, t3, _ = oracle.elementwise(1, h2, t2, h2, t2, s)
    h4, t4, _ = oracle.mul_sum(sh4["W2"], p4["W2"], h3, t3, s, 2)
    h5, t5, _ = oracle.elementwise(0, h4, t4, sh4["b2"], p4["b2"], s)
    assert digest(t5) == _golden_digest("c4")["digest"]


def test_golden_config5_slabs(oracle):
    s5 = configs.C5_SLOTS
    sw = parse_shape(configs.C5_W_SHAPE)
    pw = oracle.pack(configs.c5_w(), sw, s5)
    assert digest(pw) == _golden_digest("c5_w_pack")["digest"]
    ss = TileTensorShape([DimSpec(32, 1, 16), DimSpec(2048, 1, 32), DimSpec(512, 1, 32)])
    px = oracle.pack(configs.c5_x_slab(slice(0, 32)), ss, s5)
    assert digest(px) == _golden_digest("c5_x_pack_slab")["digest"]
    for dim in (2, 3):
        _, out, _ = oracle.mul_sum(ss, px, sw, pw, s5, dim)
        assert digest(out) == _golden_digest(f"c5_dim{dim}_slab")["digest"]
