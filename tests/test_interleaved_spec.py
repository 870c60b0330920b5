"""Known answers of the `~` (interleaved) tiling specification, DESIGN.md section 6
(rules I1-I12).  The reference has no `~` (inc/shape.hpp:164-213), so these are
the builder's own definition: parity is UNPINNED -- every expected value below
is worked by hand from the rule it tests, not produced by either
implementation.  Each KAT runs twice: on the CPU oracle (oracle/tt_oracle.c,
the restatement the GPU parity tests compare against) and on the CUDA path.
"""
import numpy as np
import pytest

import paper_2011_01805_b200 as tt
from paper_2011_01805_b200 import DimSpec, OpKind, TileTensorShape, format_shape, parse_shape


def _cost(c):
    return (c.additions, c.multiplications, c.mask_multiplications, c.rotations)


class _Gpu:
    """The same calls through the CUDA path (one session per slot count)."""

    def __init__(self):
        self.sessions = {}

    def S(self, s):
        if s not in self.sessions:
            self.sessions[s] = tt.Session(s, 8)
        return self.sessions[s]

    def pack(self, dense, shape, s):
        return tt.pack(np.asarray(dense, dtype=np.float64), shape, self.S(s)).tiles()

    def unpack(self, shape, s, tiles):
        return tt.unpack(tt.TileTensor(shape, tiles, self.S(s)))

    def _run(self, s, fn):
        S = self.S(s)
        S.reset_counters()
        r = fn(S)
        return r.shape(), r.tiles(), S.cost_report()

    def elementwise(self, op, sa, ta, sb, tb, s):
        return self._run(s, lambda S: tt.tt_elementwise(tt.TileTensor(sa, ta, S),
                                                        tt.TileTensor(sb, tb, S), OpKind(op)))

    def sum(self, shape, tiles, s, dim):
        return self._run(s, lambda S: tt.tt_sum(tt.TileTensor(shape, tiles, S), dim))

    def mul_sum(self, sa, ta, sb, tb, s, dim):
        return self._run(s, lambda S: tt.tt_mul_sum(tt.TileTensor(sa, ta, S),
                                                    tt.TileTensor(sb, tb, S), dim))

    def clean_unknowns(self, shape, tiles, s):
        return self._run(s, lambda S: tt.clean_unknowns(tt.TileTensor(shape, tiles, S)))

    def replicate_dim(self, shape, tiles, s, dim):
        return self._run(s, lambda S: tt.replicate_dim(tt.TileTensor(shape, tiles, S), dim))


@pytest.fixture(params=["oracle", pytest.param("gpu", marks=pytest.mark.gpu)])
def impl(request):
    if request.param == "oracle":
        return request.getfixturevalue("oracle")
    request.getfixturevalue("gpu")
    return _Gpu()


def _tiles(rows):
    return np.asarray(rows, dtype=np.float64)


# I1 notation: `n~/t`, printed before `?`; no replication (d = 1) -- test_shape_algebra.py
# I2 index map: j = m * e + l (tile l = j mod e, in-tile coordinate m = j div e)
def test_i2_index_map():
    sh = parse_shape("[10~/4]")  # e = 3
    assert [tt.logical_indices(sh, [l], m)[0] for l in range(3) for m in range(4)] == \
        [0, 3, 6, 9, 1, 4, 7, 10, 2, 5, 8, 11]
    assert tt.slot_of(sh, [8]) == ([2], 2)


# I3 pack / unpack: slots with j >= n stay +0.0; unpack reads them back (tile l, coordinate m)
def test_i3_pack_unpack(impl):
    sh = parse_shape("[6~/4]")
    got = impl.pack(np.arange(1, 7), sh, 4)
    assert got.tolist() == [[1, 3, 5, 0], [2, 4, 6, 0]]
    assert impl.unpack(sh, 4, got).tolist() == [1, 2, 3, 4, 5, 6]


# I4 relaxed shapes: the interleaved map fills the first prod(t) slots, the rest stay 0
def test_i4_relaxed(impl):
    sh = TileTensorShape([DimSpec(5, 1, 4, False, True)], relaxed=True)
    got = impl.pack(np.arange(1, 6), sh, 8)
    assert got.tolist() == [[1, 3, 5, 0, 0, 0, 0, 0], [2, 4, 0, 0, 0, 0, 0, 0]]


# I5 elementwise: `~` with `~` (same n) keeps `~`; tile l meets tile l
def test_i5_elementwise_same(impl):
    sh = parse_shape("[8~/4]")
    a, b = _tiles([[1, 3, 5, 7], [2, 4, 6, 8]]), _tiles([[10, 30, 50, 70], [20, 40, 60, 80]])
    so, out, cost = impl.elementwise(0, sh, a, sh, b, 4)
    assert format_shape(so) == "[8~/4]" and out.tolist() == [[11, 33, 55, 77], [22, 44, 66, 88]]
    assert _cost(cost)[0] == 2


# I6 elementwise: `~` with a fully replicated operand broadcasts it; `~` with a plain
# (non-replicated) tiling is a ShapeError
def test_i6_elementwise_broadcast_and_mismatch(impl):
    sa, sb = parse_shape("[8~/4]"), parse_shape("[*/4]")
    so, out, _ = impl.elementwise(1, sa, _tiles([[1, 3, 5, 7], [2, 4, 6, 8]]), sb,
                                  _tiles([[2, 2, 2, 2]]), 4)
    assert format_shape(so) == "[8~/4]" and out.tolist() == [[2, 6, 10, 14], [4, 8, 12, 16]]
    with pytest.raises(Exception):
        impl.elementwise(0, sa, np.zeros((2, 4)), parse_shape("[8/4]"), np.zeros((2, 4)), 4)


# I7 unknown (`?`) on `~`: used extents that differ make the result `~?`; the used
# slots of tile l are m < ceil((n - l) / e)
def test_i7_unknown_then_clean(impl):
    sa, sb = parse_shape("[6~/4]"), parse_shape("[*/4]")
    a = _tiles([[1, 3, 5, 0], [2, 4, 6, 0]])
    so, out, _ = impl.elementwise(0, sa, a, sb, _tiles([[10, 10, 10, 10]]), 4)
    assert format_shape(so) == "[6~?/4]"
    assert out.tolist() == [[11, 13, 15, 10], [12, 14, 16, 10]]
    # I8 clean_unknowns masks exactly the slots with j >= n (mask multiplication per tile)
    sc, cl, cost = impl.clean_unknowns(so, out, 4)
    assert format_shape(sc) == "[6~/4]"
    assert cl.tolist() == [[11, 13, 15, 0], [12, 14, 16, 0]]
    assert _cost(cost)[2] == 2
    # I9 a sum over an unknown `~` dim needs clean_unknowns first
    with pytest.raises(Exception):
        impl.sum(so, out, 4, 1)


# I10 sum over a dim of a tensor with a `~` dim elsewhere: the `~` dim is untouched
X = _tiles([[0, 2, 10, 12], [1, 3, 11, 13]])  # [2/2,4~/2] of X[r][c] = 10 r + c


def test_i10_sum_other_dim_keeps_tilde(impl):
    sh = parse_shape("[2/2,4~/2]")
    assert impl.pack([[0, 1, 2, 3], [10, 11, 12, 13]], sh, 4).tolist() == X.tolist()
    so, out, cost = impl.sum(sh, X, 4, 1)
    assert format_shape(so) == "[*/2,4~/2]"
    assert out.tolist() == [[10, 14, 10, 14], [12, 16, 12, 16]]
    assert (_cost(cost)[0], _cost(cost)[3]) == (2, 2)


# I11 sum over a `~` dim: the external fold adds tiles l = 0 .. e-1 in order, then the
# in-tile power-of-two tree; the result dim is not interleaved
def test_i11_sum_over_tilde(impl):
    sh = parse_shape("[2/2,4~/2]")
    so, out, cost = impl.sum(sh, X, 4, 2)
    assert format_shape(so) == "[2/2,1?/2]"
    assert out.tolist() == [[6, 26, 46, 26]]
    assert (_cost(cost)[0], _cost(cost)[3]) == (2, 1)
    s1, o1, _ = impl.sum(parse_shape("[8~/4]"), _tiles([[1, 3, 5, 7], [2, 4, 6, 8]]), 4, 1)
    assert format_shape(s1) == "[*/4]" and o1.tolist() == [[36, 36, 36, 36]]


# I12 the matvec / matmul forms: a `~` dim that is not summed rides through the
# product and the sum (config 4's batch dim)
def test_i12_product_with_tilde_batch(impl):
    sa, sb = parse_shape("[2/2,4~/2]"), parse_shape("[2/2,*/2]")
    b = impl.pack([[1], [2]], sb, 4)
    assert b.tolist() == [[1, 1, 2, 2]]
    so, out, _ = impl.mul_sum(sa, X, sb, b, 4, 1)
    assert format_shape(so) == "[*/2,4~/2]"
    assert out.tolist() == [[20, 26, 20, 26], [23, 29, 23, 29]]


# I13 replicate_dim on a `~` dim (n = 1: e = 1, interleaving is the identity):
# the right-to-left schedule copies slot 0 everywhere; the result is `*/t`, not `~`
def test_i13_replicate(impl):
    so, out, cost = impl.replicate_dim(parse_shape("[1~/4]"), _tiles([[5, 0, 0, 0]]), 4, 1)
    assert format_shape(so) == "[*/4]" and out.tolist() == [[5, 5, 5, 5]]
    assert _cost(cost)[3] == 2


# I14 what `~` does not take: block sharding of a `~` dim, exact fold chains over one
@pytest.mark.gpu
def test_i14_refusals(gpu):
    with pytest.raises(tt.ShapeError):
        tt.shard_plan(parse_shape("[8~/4]"), 1, 2, 0)
    S = tt.Session(4, 8)
    x = tt.pack(np.arange(1, 9, dtype=np.float64), parse_shape("[8~/4]"), S)
    with pytest.raises(ValueError):
        tt.mul_fold(x, None, 1)


def test_i14_shard_refusal_cpu():
    with pytest.raises(tt.ShapeError):
        tt.shard_plan(parse_shape("[8~/4]"), 1, 2, 0)
