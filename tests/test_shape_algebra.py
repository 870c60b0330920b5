"""Shape notation and algebra of the product library (host code, no GPU).

KATs restated from /root/reference/proj/tests/test_shape.cpp (cited per
test), the reference's parse/format outputs from tests/golden, and random
agreement with the oracle's restatement of the rules (and the reference
itself when oracle/_ref is built).
"""
import random

import numpy as np

import pytest

import paper_2011_01805_b200 as tt
from golden_cases import load
from paper_2011_01805_b200 import (DimSpec, OpKind, ShapeError, ShapeParseError, TileTensorShape,
                                   elementwise_result_shape, external_shape, format_shape,
                                   parse_shape, sum_result_shape)


def ds(n, d, t, unknown=False):
    return DimSpec(n, d, t, unknown)


def test_parse_defaults():  # test_shape.cpp:57-68
    assert parse_shape("[5,6/8]").dims() == (ds(5, 1, 1), ds(6, 1, 8))
    assert parse_shape("[5/2,*3/4]").dims() == (ds(5, 1, 2), ds(1, 3, 4))
    assert parse_shape("[5/2,1?/4]").dims() == (ds(5, 1, 2), ds(1, 1, 4, True))
    assert parse_shape("[*/4,5/8]").dims() == (ds(1, 4, 4), ds(5, 1, 8))
    assert parse_shape("[2,5/8]").dims() == (ds(2, 1, 1), ds(5, 1, 8))
    assert parse_shape("[18?/8,4/16]").dims() == (ds(18, 1, 8, True), ds(4, 1, 16))
    assert parse_shape(" [ 5 / 2 , * 3 / 4 ] ").dims() == parse_shape("[5/2,*3/4]").dims()


def test_parse_errors_with_position():  # test_shape.cpp:70-86
    for bad in ["[*5/4]", "[2*3/8]", "[0/4]", "[5/0]", "[5/2", "[]", "[5/2,]", "[?/4]",
                "[5/2] junk"]:
        with pytest.raises(ShapeParseError):
            parse_shape(bad)
    with pytest.raises(ShapeParseError) as e:
        parse_shape("[5/2,*3/")
    assert e.value.position() == 8


def test_golden_parse_cases():
    """Every parse/format outcome recorded from the reference (tests/golden)."""
    for c in (c for c in load() if c["kind"] == "parse"):
        if c["rc"] == 0:
            shape = parse_shape(c["text"])
            assert shape == c.shape("shape")
            assert format_shape(shape) == c["formatted"]
        else:
            with pytest.raises(ShapeParseError) as e:
                parse_shape(c["text"])
            assert e.value.position() == c["pos"], c["text"]


def test_canonical_printing():  # test_shape.cpp:88-104
    assert format_shape(TileTensorShape([ds(2, 1, 1), ds(5, 1, 8)])) == "[2,5/8]"
    assert format_shape(TileTensorShape([ds(1, 4, 4), ds(5, 1, 8)])) == "[*/4,5/8]"
    assert format_shape(TileTensorShape([ds(1, 3, 4), ds(5, 1, 8)])) == "[*3/4,5/8]"
    assert format_shape(TileTensorShape([ds(5, 1, 2), ds(1, 1, 4, True)])) == "[5/2,1?/4]"
    assert format_shape(TileTensorShape([ds(1, 1, 1)])) == "[1]"
    assert format_shape(parse_shape("[2/1,5/8]")) == "[2,5/8]"
    for messy in ["[2/1,5/8]", " [ *4 / 4 ] ", "[1*3/4]", "[05/02]", "[*8/8,1?/2]"]:
        once = format_shape(parse_shape(messy))
        assert format_shape(parse_shape(once)) == once
    assert format_shape(parse_shape(" [ *4 / 4 ] ")) == "[*/4]"
    assert format_shape(parse_shape("[1*3/4]")) == "[*3/4]"


def _random_shape(rng, slots):
    rank = rng.randint(1, 4)
    t = [1] * rank
    rem = slots
    for i in range(rank - 1):
        opts = []
        x = 1
        while x <= rem:
            opts.append(x)
            x *= 2
        t[i] = rng.choice(opts)
        rem //= t[i]
    t[-1] = rem
    dims = []
    for ti in t:
        k = rng.randint(0, 3)
        if k == 0:
            dims.append(ds(1, ti, ti))
        elif k == 1 and ti > 1:
            dims.append(ds(1, rng.randint(1, ti), ti))
        elif k == 2:
            dims.append(ds(1, 1, ti, True))
        else:
            dims.append(ds(rng.randint(1, 12), 1, ti))
    return TileTensorShape(dims)


def test_round_trip_and_minimal_covers():  # test_shape.cpp:106-136
    rng = random.Random(20260809)
    for _ in range(500):
        shape = _random_shape(rng, 1 << rng.randint(0, 6))
        text = format_shape(shape)
        assert parse_shape(text) == shape and format_shape(parse_shape(text)) == text
        for d, e in zip(shape.dims(), shape.external_extents()):
            assert (e - 1) * d.t < d.used() <= e * d.t


def test_external_shape():  # test_shape.cpp:118-122
    assert external_shape(parse_shape("[5/2,6/4]")) == [3, 2]
    assert external_shape(parse_shape("[50/16,20/2,255/32]")) == [4, 10, 8]
    assert external_shape(parse_shape("[*/4,5/8]")) == [1, 1]


def test_elementwise_result_shapes():  # test_shape.cpp:138-164
    a, b = parse_shape("[18/8,4/16]"), parse_shape("[*/8,4/16]")
    assert format_shape(elementwise_result_shape(a, b, OpKind.add)) == "[18?/8,4/16]"
    assert format_shape(elementwise_result_shape(a, b, OpKind.mul)) == "[18/8,4/16]"
    for x, y in [("[5/8]", "[6/8]"), ("[5/8]", "[5/4]"), ("[5/8]", "[5/8,2]"),
                 ("[18/8,4/16]", "[*3/8,4/16]")]:
        with pytest.raises(ShapeError):
            elementwise_result_shape(parse_shape(x), parse_shape(y), OpKind.add)
    assert format_shape(elementwise_result_shape(parse_shape("[1?/4]"), parse_shape("[1/4]"),
                                                 OpKind.mul)) == "[1/4]"
    assert format_shape(elementwise_result_shape(parse_shape("[1?/4]"), parse_shape("[*/4]"),
                                                 OpKind.mul)) == "[1?/4]"
    assert format_shape(elementwise_result_shape(parse_shape("[16/8]"), parse_shape("[*/8]"),
                                                 OpKind.add)) == "[16?/8]"
    assert format_shape(elementwise_result_shape(parse_shape("[16/8]"), parse_shape("[*/8]"),
                                                 OpKind.mul)) == "[16/8]"


def test_summation_rules():  # test_shape.cpp:222-250 ; acceptance criterion 7
    shape = parse_shape("[4,3/8,5/16]")
    assert format_shape(sum_result_shape(shape, 1)) == "[1,3/8,5/16]"
    assert format_shape(sum_result_shape(shape, 2)) == "[4,*/8,5/16]"
    assert format_shape(sum_result_shape(shape, 3)) == "[4,3/8,1?/16]"
    for bad in (0, 4):
        with pytest.raises(ShapeError):
            sum_result_shape(shape, bad)
    assert format_shape(sum_result_shape(parse_shape("[4?/8,2]"), 1)) == "[1?/8,2]"
    assert format_shape(sum_result_shape(parse_shape("[*/8,4/16]"), 1)) == "[*/8,4/16]"
    assert format_shape(sum_result_shape(parse_shape("[4/8,*3/16]"), 2)) == "[4/8,*3/16]"
    relaxed = TileTensorShape(parse_shape("[4/4,3/2]").dims(), True)
    assert format_shape(sum_result_shape(relaxed, 1)) == "[1?/4,3/2]"
    rng = random.Random(123)
    for _ in range(300):
        s = _random_shape(rng, 1 << rng.randint(0, 5))
        for dim in range(1, s.rank() + 1):
            once = sum_result_shape(s, dim)
            assert sum_result_shape(once, dim) == once and once.tile_slots() == s.tile_slots()


def test_slot_accounting():  # test_shape.cpp:252-257
    shape = parse_shape("[5/2,6/4]")
    assert shape.used_slots() == 30 and shape.total_slots() == 48 and shape.tile_count() == 6


def test_logical_index_map():  # test_tile_tensor.cpp:106-150
    shape = parse_shape("[5/2,6/4]")
    assert tt.logical_indices(shape, [1, 0], 5) == [3, 1]
    assert tt.logical_indices(shape, [0, 0], 0) == [0, 0]
    assert tt.logical_indices(parse_shape("[3,4]"), [2, 3], 0) == [2, 3]
    with pytest.raises(ShapeError):
        tt.logical_indices(shape, [3, 0], 0)
    with pytest.raises(ShapeError):
        tt.logical_indices(shape, [0, 0], 8)
    rng = random.Random(61)
    for _ in range(50):
        sh = _random_shape(rng, 1 << rng.randint(0, 5))
        sh = TileTensorShape([DimSpec(d.n, d.d, d.t) for d in sh.dims()])
        ext = sh.external_extents()
        seen = set()
        import itertools
        for l in itertools.product(*[range(e) for e in ext]):
            for h in range(sh.tile_slots()):
                j = tt.logical_indices(sh, list(l), h)
                assert tt.slot_of(sh, j) == (list(l), h)
                seen.add(tuple(j))
        assert len(seen) == sh.tile_count() * sh.tile_slots()


def test_agrees_with_oracle_rules(oracle):
    rng = random.Random(99)
    for _ in range(400):
        a = _random_shape(rng, 1 << rng.randint(0, 5))
        dims = []
        for d in a.dims():
            k = rng.randint(0, 3)
            dims.append(DimSpec(d.n, 1 if d.n > 1 else d.d, d.t, rng.random() < 0.25) if k == 0 else
                        DimSpec(1, d.t, d.t) if k == 1 else DimSpec(1, 1, d.t, True) if k == 2 else
                        DimSpec(rng.randint(1, 12), 1, d.t))
        b = TileTensorShape(dims)
        for op in (OpKind.add, OpKind.mul):
            try:
                want = oracle.elementwise_result_shape(a, b, int(op))
            except Exception:
                with pytest.raises(ShapeError):
                    elementwise_result_shape(a, b, op)
                continue
            assert elementwise_result_shape(a, b, op) == want
        for dim in range(1, a.rank() + 1):
            assert sum_result_shape(a, dim) == oracle.sum_result_shape(a, dim)


def test_interleaved_notation():
    """The builder's `~` token (not in the reference)."""
    s = parse_shape("[784/32,1,4096~/256]")
    assert s.dim(2).interleaved and format_shape(s) == "[784/32,1,4096~/256]"
    assert parse_shape("[9~?/4]").dim(0) == DimSpec(9, 1, 4, True, True)
    assert format_shape(parse_shape("[9?~/4]")) == "[9~?/4]"
    with pytest.raises(ShapeParseError):
        parse_shape("[*~/4]")  # replication cannot be interleaved
    # j -> tile j mod e, in-tile coordinate j div e
    assert tt.logical_indices(parse_shape("[10~/4]"), [1], 2) == [2 * 3 + 1]
    assert tt.slot_of(parse_shape("[10~/4]"), [7]) == ([1], 2)
    with pytest.raises(ShapeError):
        elementwise_result_shape(parse_shape("[8~/4]"), parse_shape("[8/4]"), OpKind.add)
    assert format_shape(elementwise_result_shape(parse_shape("[8~/4]"), parse_shape("[*/4]"),
                                                 OpKind.mul)) == "[8~/4]"


# Known answers of the builder's `~` tiling, worked by
# hand: element j of an n~/t dim with e = ceil(n/t) external tiles sits in tile
# j mod e at in-tile coordinate j div e; slots past n stay +0.0.
INTERLEAVED_KATS = [
    # (shape, dense values, expected tiles)
    ("[10~/4]", list(range(10)), [[0, 3, 6, 9], [1, 4, 7, 0], [2, 5, 8, 0]]),
    ("[8~/4]", list(range(1, 9)), [[1, 3, 5, 7], [2, 4, 6, 8]]),
    # 2-D: dim 1 plain [3/2] (tiles by rows 0-1, 2), dim 2 interleaved [5~/2] (e = 3)
    ("[3/2,5~/2]", [[r * 10 + c for c in range(5)] for r in range(3)],
     [[0, 3, 10, 13], [1, 4, 11, 14], [2, 0, 12, 0],
      [20, 23, 0, 0], [21, 24, 0, 0], [22, 0, 0, 0]]),
]


@pytest.mark.parametrize("text,dense,want", INTERLEAVED_KATS)
def test_interleaved_pack_kats(oracle, text, dense, want):
    sh = parse_shape(text)
    s = len(want[0])
    got = oracle.pack(np.asarray(dense, dtype=np.float64), sh, s)
    assert got.tolist() == [[float(v) for v in row] for row in want]
    assert oracle.unpack(sh, s, got).tolist() == np.asarray(dense, dtype=np.float64).tolist()


def test_interleaved_sum_kat(oracle):
    """tt_sum over a `~` dim: the external fold adds the e tiles in order, then the
    in-tile power-of-two tree; [8~/4] holding 1..8 -> every slot 36, shape [*/4]."""
    sh = parse_shape("[8~/4]")
    tiles = oracle.pack(np.arange(1, 9, dtype=np.float64), sh, 4)
    so, out, cost = oracle.sum(sh, tiles, 4, 1)
    assert format_shape(so) == "[*/4]"
    assert out.tolist() == [[36.0, 36.0, 36.0, 36.0]]
    assert (cost.additions, cost.rotations) == (1 + 2, 2)


def test_high_rank_shapes(oracle):
    # the reference has no rank limit; this build holds up to TT_MAX_RANK (16) dims
    from paper_2011_01805_b200._abi import TT_MAX_RANK
    assert TT_MAX_RANK == 16
    text = "[" + ",".join(["3/2"] * 12) + "]"
    sh = parse_shape(text)
    assert sh.rank() == 12 and format_shape(sh) == text
    assert sh.tile_count() == 2 ** 12
    r = tt.sum_result_shape(tt.elementwise_result_shape(sh, sh, OpKind.mul), 7)
    assert format_shape(r) == "[" + ",".join(["3/2"] * 6 + ["1?/2"] + ["3/2"] * 5) + "]"
    dense = np.arange(3 ** 12, dtype=np.float64).reshape((3,) * 12)
    want = oracle.pack(dense, sh, 4096)
    assert want.shape == (2 ** 12, 4096)
    with pytest.raises(ShapeError):
        parse_shape("[" + ",".join(["2"] * 17) + "]")
