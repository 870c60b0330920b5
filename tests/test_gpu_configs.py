"""GPU parity on the reference's golden fixtures and on BASELINE.json's five
configurations (full size), against the CPU oracle (and the reference's own
digests).  Bit-exact wherever the reference's operation order is reproduced;
dense-oracle agreement within 1e-12 relative where a value is compared with a
differently-associated plain computation.
"""
import numpy as np
import pytest

import paper_2011_01805_b200 as tt
from golden_cases import bitwise_equal, cost_tuple, digest, load
from paper_2011_01805_b200 import TileTensor, configs, parse_shape

pytestmark = pytest.mark.gpu
LINALG = {0: tt.matvec_a, 1: tt.matvec_b, 2: tt.matmul_a, 3: tt.matmul_b}
_S = {}


def session(s):
    if s not in _S:
        _S[s] = tt.Session(s, 8)
    return _S[s]


def test_golden_fixtures_on_gpu(gpu):
    n = 0
    for c in load():
        k = c["kind"]
        if k in ("parse", "config", "config_digest"):
            continue
        S = session(c["s"])
        S.reset_counters()
        if k == "pack":
            t = tt.pack(c.arr("dense"), c.shape("shape"), S)
            assert bitwise_equal(t.tiles(), c.arr("tiles"))
            assert bitwise_equal(tt.unpack(t), c.arr("dense"))
            continue
        if k == "elementwise":
            r = tt.tt_elementwise(TileTensor(c.shape("sa"), c.arr("ta"), S),
                                  TileTensor(c.shape("sb"), c.arr("tb"), S), tt.OpKind(c["op"]))
        elif k == "sum":
            v = None if c["variant"] < 0 else tt.SumVariant(c["variant"])
            r = tt.tt_sum(TileTensor(c.shape("shape"), c.arr("tiles"), S), c["dim"], v)
        elif k == "sum_error":
            v = tt.SumVariant(c["variant"])
            with pytest.raises(ValueError):
                tt.tt_sum(TileTensor(c.shape("shape"), c.arr("tiles"), S), c["dim"], v)
            continue
        elif k == "linalg":
            r = LINALG[c["which"]](TileTensor(c.shape("sa"), c.arr("ta"), S),
                                   TileTensor(c.shape("sb"), c.arr("tb"), S))
        elif k == "clean":
            r = tt.clean_unknowns(TileTensor(c.shape("shape"), c.arr("tiles"), S))
        elif k == "replicate":
            r = tt.replicate_dim(TileTensor(c.shape("shape"), c.arr("tiles"), S), c["dim"])
        elif k == "strided":
            out = tt.sum_tile_strided(S, c.arr("tile"), c["n"], c["stride"], tt.SumVariant(c["variant"]))
            assert bitwise_equal(out.cpu().numpy()[0], c.arr("out"))
            assert cost_tuple(S.cost_report()) == tuple(c.arr("cost"))
            continue
        elif k == "rotate":
            out = tt.tiles_rotate(S, c.arr("tile"), c["offset"])
            assert bitwise_equal(out.cpu().numpy()[0], c.arr("out"))
            assert cost_tuple(S.cost_report()) == tuple(c.arr("cost"))
            continue
        else:
            raise AssertionError(k)
        assert r.shape() == c.shape("so"), k
        assert bitwise_equal(r.tiles(), c.arr("out")), k
        assert cost_tuple(S.cost_report()) == tuple(c.arr("cost")), k
        n += 1
    assert n > 200


def test_config1(gpu, oracle):
    """100x200 (x) 100x200, [100/16,200/32], sum dim 2 -> [100/16,1?/32]."""
    golden = next(c for c in load() if c["kind"] == "config" and c["name"] == "c1")
    case = configs.config1()
    S = tt.Session(512, 8)
    sA = parse_shape(case.shapes["A"])
    r = tt.tt_mul_sum(tt.pack(case.tensors["A"], sA, S), tt.pack(case.tensors["B"], sA, S), 2)
    assert tt.format_shape(r.shape()) == "[100/16,1?/32]"
    assert bitwise_equal(r.tiles(), golden.arr("out"))
    c = S.cost_report()
    assert (c.additions, c.multiplications, c.rotations) == (77, 49, 35)
    dense = oracle.dense_sum(oracle.dense_elementwise(1, case.tensors["A"], case.tensors["B"]), 2)
    assert oracle.max_rel_diff(tt.unpack(r), dense) < 1e-12


def test_config2_matvec(gpu, oracle):
    golden = next(c for c in load() if c["kind"] == "config_digest" and c["name"] == "c2")
    case = configs.config2()
    S = tt.Session(8192, 8)
    M = tt.pack(case.tensors["M"], parse_shape(case.shapes["M"]), S)
    V = tt.pack(case.tensors["V"], parse_shape(case.shapes["V"]), S)
    S.reset_counters()
    r = tt.matvec_a(M, V)
    assert tt.format_shape(r.shape()) == "[1024/64,1?/128]"
    assert digest(r.tiles()) == golden["digest"]
    c = S.cost_report()
    assert (c.additions, c.multiplications, c.rotations) == (608, 512, 112)
    got = tt.unpack(r).reshape(-1)
    assert bitwise_equal(got, golden.arr("unpacked").reshape(-1))
    want = oracle.dense_matmul(case.tensors["M"], case.tensors["V"].reshape(4096, 1)).reshape(-1)
    assert oracle.max_rel_diff(got, want) < 1e-12


def test_config3_chains(gpu, oracle):
    """A(512x1024) B(1024x768) C(768x256), 3-D tiles 16x32x16.  '3b' is the
    reference's zero-processing chain (tests/test_linalg.cpp:157-178):
    matmul_b(B^T, C) then matmul_a(A, .).  '3a' is the literal chain with the
    clean + replicate seam."""
    case = configs.config3()
    s = 8192
    S = tt.Session(s, 8)
    T = {k: tt.pack(case.tensors[k], parse_shape(v), S) for k, v in case.shapes.items()}
    S.reset_counters()
    s1 = tt.matmul_b(T["Bt3"], T["C3"])
    r = tt.matmul_a(T["A3"], s1)
    assert tt.format_shape(s1.shape()) == "[*/16,1024/32,256/16]"
    assert tt.format_shape(r.shape()) == "[512/16,1?/32,256/16]"
    # oracle: the same two-line bodies on the host
    p = {k: oracle.pack(case.tensors[k], parse_shape(v), s) for k, v in case.shapes.items()}
    so1, o1, c1 = oracle.mul_sum(parse_shape(case.shapes["Bt3"]), p["Bt3"],
                                 parse_shape(case.shapes["C3"]), p["C3"], s, 1)
    assert bitwise_equal(s1.tiles(), o1)
    so2, o2, c2 = oracle.mul_sum(parse_shape(case.shapes["A3"]), p["A3"], so1, o1, s, 2)
    assert bitwise_equal(r.tiles(), o2)
    assert cost_tuple(S.cost_report())[:4] == tuple(np.add(cost_tuple(c1), cost_tuple(c2)))[:4]
    # pinned to the reference's own outputs (tests/golden, made by oracle/_ref)
    gold = {c["name"]: c for c in load() if c["kind"] == "config_digest"}
    assert digest(s1.tiles()) == gold["c3b_stage1"]["digest"]
    assert digest(r.tiles()) == gold["c3b"]["digest"]
    abc = case.tensors["A"] @ case.tensors["B"] @ case.tensors["C"]
    got = tt.unpack(r).reshape(512, 256)
    assert oracle.max_rel_diff(got, abc) < 1e-12
    # literal '3a': matmul_a(A, B) -> clean -> replicate dim 2 -> x C^T, sum dim 3
    ra = tt.matmul_a(T["A3"], T["B3"])
    assert tt.format_shape(ra.shape()) == "[512/16,1?/32,768/16]"
    rep = tt.replicate_dim(tt.clean_unknowns(ra), 2)
    assert tt.format_shape(rep.shape()) == "[512/16,*/32,768/16]"
    r3a = tt.tt_mul_sum(rep, T["Ct3"], 3)
    assert digest(r3a.tiles()) == gold["c3a"]["digest"]
    assert tt.format_shape(r3a.shape()) == "[512/16,256/32,1?/16]"
    assert oracle.max_rel_diff(tt.unpack(r3a).reshape(512, 256), abc) < 1e-12
    # bitwise against the oracle composition of the same chain
    sa, oa, _ = oracle.mul_sum(parse_shape(case.shapes["A3"]), p["A3"],
                               parse_shape(case.shapes["B3"]), p["B3"], s, 2)
    assert bitwise_equal(ra.tiles(), oa)
    sc, oc, _ = oracle.clean_unknowns(sa, oa, s)
    sr, orr, _ = oracle.replicate_dim(sc, oc, s, 2)
    assert bitwise_equal(rep.tiles(), orr)


@pytest.mark.parametrize("interleaved", [False, True])
def test_config4_fc_square_fc(gpu, oracle, interleaved):
    """784 -> 100 -> square -> 10 on a 4096-sample batch in tile dim 3
    (composition of cryptonets_infer's FC/square stages, nn.hpp:468-490, on
    the full batch).  The `~` variant interleaves the batch dimension; since
    no rotation crosses samples its logits equal the plain variant bit for bit."""
    case = configs.config4(interleaved)
    plain = configs.config4(False)
    s = 8192
    S = tt.Session(s, 8)
    sh = {k: parse_shape(v) for k, v in case.shapes.items()}
    T = {k: tt.pack(case.tensors[k], sh[k], S) for k in sh}
    h = tt.tt_mul_sum(T["W1t"], T["X"], 1)                 # odd stage: sum dim 1
    assert tt.format_shape(h.shape()) == ("[*/32,100,4096~/256]" if interleaved
                                          else "[*/32,100,4096/256]")
    h = tt.tt_add(h, T["b1"])
    h = tt.tt_mul(h, h)                                     # square activation
    y = tt.tt_mul_sum(T["W2"], h, 2)                        # even stage: sum dim 2 (t = 1)
    y = tt.tt_add(y, T["b2"])
    logits = tt.unpack(y).reshape(10, 4096)
    dense = configs.dense_forward_c4(plain)
    assert oracle.max_rel_diff(logits, dense) < 1e-12
    # oracle composition (plain layout) -- bitwise
    ps = {k: parse_shape(v) for k, v in plain.shapes.items()}
    p = {k: oracle.pack(plain.tensors[k], ps[k], s) for k in ps}
    s1, o1, _ = oracle.mul_sum(ps["W1t"], p["W1t"], ps["X"], p["X"], s, 1)
    s2, o2, _ = oracle.elementwise(0, s1, o1, ps["b1"], p["b1"], s)
    s3, o3, _ = oracle.elementwise(1, s2, o2, s2, o2, s)
    s4, o4, _ = oracle.mul_sum(ps["W2"], p["W2"], s3, o3, s, 2)
    s5, o5, _ = oracle.elementwise(0, s4, o4, ps["b2"], p["b2"], s)
    want = oracle.unpack(s5, s, o5).reshape(10, 4096)
    assert bitwise_equal(logits, want)
    if not interleaved:
        assert bitwise_equal(y.tiles(), o5)
        gold = next(c for c in load() if c["kind"] == "config_digest" and c["name"] == "c4")
        assert digest(y.tiles()) == gold["digest"]


@pytest.mark.slow
def test_config5_full_size_slabs(gpu, oracle):
    """X [2048/16,2048/32,512/32] (16 GiB) x W [*/16,2048/32,512/32], sums
    over each dim at full size on the GPU; slabs of the results (tile
    boundaries align, so they are bitwise slices) are checked against the
    oracle run on the matching input slab."""
    import torch
    S = tt.Session(configs.C5_SLOTS, 8)
    sx, sw = parse_shape(configs.C5_X_SHAPE), parse_shape(configs.C5_W_SHAPE)
    x = torch.empty(configs.C5_DIMS, dtype=torch.float64, device="cuda")
    w = torch.empty((1, 2048, 512), dtype=torch.float64, device="cuda")
    tt.fill_uniform(S, x, configs.C5_SEED_X, -1.0, 1.0)
    tt.fill_uniform(S, w, configs.C5_SEED_W, -1.0, 1.0)
    X, W = tt.pack(x, sx, S), tt.pack(w, sw, S)
    del x
    s = configs.C5_SLOTS
    # pack: the first two external rows of dim 1 are the pack of X[0:32]
    xs = configs.c5_x_slab(slice(0, 32))
    ss = tt.TileTensorShape([tt.DimSpec(32, 1, 16), tt.DimSpec(2048, 1, 32), tt.DimSpec(512, 1, 32)])
    px = oracle.pack(xs, ss, s)
    assert bitwise_equal(X.data()[:2048].cpu().numpy(), px)
    pw = oracle.pack(configs.c5_w(), sw, s)
    assert bitwise_equal(W.tiles(), pw)
    gold = {c["name"]: c for c in load() if c["kind"] == "config_digest"}
    assert digest(W.tiles()) == gold["c5_w_pack"]["digest"]
    assert digest(X.data()[:2048].cpu().numpy()) == gold["c5_x_pack_slab"]["digest"]
    for dim, ntiles in ((2, 32), (3, 128)):
        r = tt.tt_mul_sum(X, W, dim)
        so, want, _ = oracle.mul_sum(ss, px, sw, pw, s, dim)
        got = r.data()[:ntiles].cpu().numpy()
        assert bitwise_equal(got, want), dim
        assert digest(got) == gold[f"c5_dim{dim}_slab"]["digest"]
    # dim 1 spans all of X: slab along dim 2 (external index l2 = 0)
    r1 = tt.tt_mul_sum(X, W, 1)
    xs2 = configs.c5_x_slab(slice(None), slice(0, 32))
    ss2 = tt.TileTensorShape([tt.DimSpec(2048, 1, 16), tt.DimSpec(32, 1, 32), tt.DimSpec(512, 1, 32)])
    sw2 = tt.TileTensorShape([tt.DimSpec(1, 16, 16), tt.DimSpec(32, 1, 32), tt.DimSpec(512, 1, 32)])
    so, want, _ = oracle.mul_sum(ss2, oracle.pack(xs2, ss2, s), sw2,
                                 oracle.pack(configs.c5_w(slice(0, 32)), sw2, s), s, 1)
    assert tt.format_shape(r1.shape()) == "[*/16,2048/32,512/32]"
    assert bitwise_equal(r1.data()[:16].cpu().numpy(), want)
    assert digest(r1.data()[:16].cpu().numpy()) == gold["c5_dim1_slab"]["digest"]
    # the replicated result unpacks to the dense sum (1e-12)
    got = tt.unpack(r1)[0, :32, :]
    dense = (xs2 * configs.c5_w(slice(0, 32))).sum(axis=0)
    assert oracle.max_rel_diff(got, dense) < 1e-12
    # middle and last slabs: groups the persistent grids reach in later loop
    # iterations (group index >= 148), the last external rows / columns and
    # the sliding-window wrap on the final chunks
    r2, r3 = tt.tt_mul_sum(X, W, 2), tt.tt_mul_sum(X, W, 3)
    ss1 = tt.TileTensorShape([tt.DimSpec(16, 1, 16), tt.DimSpec(2048, 1, 32), tt.DimSpec(512, 1, 32)])
    for row in (64, 97, 127):                      # external rows of dim 1
        px = oracle.pack(configs.c5_x_slab(slice(16 * row, 16 * row + 16)), ss1, s)
        assert bitwise_equal(X.data()[1024 * row:1024 * (row + 1)].cpu().numpy(), px), row
        for dim, r, per in ((2, r2, 16), (3, r3, 64)):
            _, want, _ = oracle.mul_sum(ss1, px, sw, pw, s, dim)
            assert bitwise_equal(r.data()[per * row:per * (row + 1)].cpu().numpy(), want), (dim, row)
    for l2 in (31, 63):                            # external columns of dim 2
        cols = slice(32 * l2, 32 * l2 + 32)
        px2 = oracle.pack(configs.c5_x_slab(slice(None), cols), ss2, s)
        so, want, _ = oracle.mul_sum(ss2, px2, sw2, oracle.pack(configs.c5_w(cols), sw2, s), s, 1)
        assert bitwise_equal(r1.data()[16 * l2:16 * (l2 + 1)].cpu().numpy(), want), l2
