"""The packing methods, the alternating pipeline and the tile-extent search
(inc/linalg.hpp:77-294) on the GPU ops, against the reference itself
(oracle/_ref: the same functions compiled from /root/reference): identical
output tiles bit for bit and identical cost counters, for random chains and
every tile factorisation; plus the reference's own behavioural KATs
(tests/test_linalg.cpp:181-326) restated.
"""
import numpy as np
import pytest

import paper_2011_01805_b200 as tt
from paper_2011_01805_b200 import OperandRole, PackingMethod

pytestmark = pytest.mark.gpu


def _cost_tuple(c):
    return (c.additions, c.multiplications, c.mask_multiplications, c.rotations, c.bootstraps,
            c.power_of_two_rotations)


def _chain(rng, widths):
    ms = [rng.uniform(-1, 1, size=(widths[i + 1], widths[i])) for i in range(len(widths) - 1)]
    return ms, rng.uniform(-1, 1, size=widths[0])


def _dense_chain(ms, v):
    x = v
    for m in ms:
        x = m @ x
    return x


@pytest.mark.parametrize("s", [8, 16, 32])
def test_pipeline_matches_reference_bitwise(gpu, ref, s):
    rng = np.random.default_rng(5150 + s)
    for stages in (1, 2, 3, 4):
        for _ in range(3):
            widths = [int(x) for x in rng.integers(1, 2 * s, size=stages + 1)]
            ms, v = _chain(rng, widths)
            t1 = 1
            while t1 <= s:
                tile = (t1, s // t1)
                S = tt.Session(s, 16)
                got = tt.pipeline(ms, v, tile, S)
                ws, wt, wc = ref.pipeline(ms, v, tile, s, depth=16)
                assert got.out.shape() == ws, (widths, tile)
                assert np.array_equal(got.out.tiles().view(np.uint64), wt.view(np.uint64)), \
                    (widths, tile)
                assert _cost_tuple(got.cost) == _cost_tuple(wc), (widths, tile)
                t1 *= 2


def test_score_tile_factorizations_matches_reference(gpu, ref):
    rng = np.random.default_rng(239)
    for widths, s in (([6, 4, 5], 16), ([7, 5, 9, 7], 32), ([3, 8, 2], 8)):
        ms, v = _chain(rng, widths)
        got = tt.score_tile_factorizations(ms, v, s, 8)
        want = ref.score_tile_factorizations(ms, v, s, 8)
        assert len(got) == len(want)
        # keys in the same order; ties (equal keys) may be listed in any order
        assert [(c.cost.rotations, c.cost.total_ops()) for c in got] == [(w[1], w[2]) for w in want]
        assert sorted((c.t1, c.cost.rotations, c.cost.total_ops()) for c in got) == sorted(want)


def test_pack_for_method_kats(gpu):
    rng = np.random.default_rng(217)
    m = rng.uniform(-1, 1, size=(5, 3))
    v = rng.uniform(-1, 1, size=3)
    for method in (PackingMethod.row_order(), PackingMethod.column_order(),
                   PackingMethod.input_packing(), PackingMethod.general([4, 4])):
        S = tt.Session(16, 8)
        inp = method.kind == PackingMethod.Kind.input_packing
        tm = tt.pack_for_method(m, OperandRole.lhs if inp else OperandRole.matrix, method, S)
        tv = tt.pack_for_method(v, OperandRole.rhs if inp else OperandRole.vector, method, S)
        r = tt.tt_sum(tt.tt_mul(tm, tv), tt.sum_dim_for(method))
        np.testing.assert_allclose(tt.unpack_vector(r), m @ v, rtol=1e-9, atol=1e-12)
    S = tt.Session(16, 8)
    batch = rng.uniform(-1, 1, size=(3, 7))
    tw = tt.pack_for_method(m, OperandRole.matrix, PackingMethod.batch_packing(), S)
    tb = tt.pack_for_method(batch, OperandRole.vector, PackingMethod.batch_packing(), S)
    assert tt.format_shape(tw.shape()) == "[5,3,*/16]"
    assert tt.format_shape(tb.shape()) == "[3,7/16]"
    S.reset_counters()
    r = tt.tt_sum(tt.tt_mul(tw, tt.with_leading_unit_dim(tb)), 2)
    assert S.cost_report().rotations == 0
    np.testing.assert_allclose(tt.unpack(r).reshape(5, 7), m @ batch, rtol=1e-9, atol=1e-12)
    # input packing: smallest divisor of s fitting the contracted extent
    tm = tt.pack_for_method(rng.uniform(size=(4, 3)), OperandRole.lhs,
                            PackingMethod.input_packing(), S)
    assert tt.format_shape(tm.shape()) == "[3/4,4/4]"
    with pytest.raises(tt.ShapeError):
        tt.pack_for_method(rng.uniform(size=(2, 17)), OperandRole.lhs,
                           PackingMethod.input_packing(), S)
    # general packing fills every slot
    S2 = tt.Session(1024, 2)
    big = rng.uniform(-1, 1, size=(768, 768))
    g = tt.pack_for_method(big, OperandRole.matrix, PackingMethod.general([4, 256]), S2)
    assert g.tile_count() == 576 and g.shape().used_slots() == g.shape().total_slots()
    assert tt.pack_for_method(big, OperandRole.matrix, PackingMethod.row_order(),
                              S2).tile_count() == 768


def test_pipeline_kats(gpu):
    rng = np.random.default_rng(251)
    S = tt.Session(8, 8)
    v3 = np.array([1.0, 2.0, 3.0])
    res = tt.pipeline([np.eye(3), np.eye(3)], v3, (2, 4), S)
    np.testing.assert_allclose(tt.unpack_vector(res.out), v3, rtol=1e-12)
    m, v = rng.uniform(-1, 1, size=(5, 6)), rng.uniform(-1, 1, size=6)
    one = tt.pipeline([m], v, (2, 4), S)
    assert tt.format_shape(one.out.shape()) == "[*/2,5/4]"
    assert one.cost.mask_multiplications == 0
    S16 = tt.Session(16, 16)
    ms, v4 = _chain(rng, [4, 5, 7, 6, 3])
    four = tt.pipeline(ms, v4, (4, 4), S16)
    np.testing.assert_allclose(tt.unpack_vector(four.out), _dense_chain(ms, v4), rtol=1e-9,
                               atol=1e-12)
    assert four.cost.mask_multiplications == 2  # one seam: [7/4,1?/4] -> two tiles masked
    two = tt.pipeline(ms[:2], v4, (4, 4), S16)
    assert two.cost.mask_multiplications == 0
    with pytest.raises(tt.ShapeError):
        tt.pipeline([rng.uniform(size=(3, 4))], rng.uniform(size=5), (2, 4), S)
    with pytest.raises(tt.ShapeError):
        tt.pipeline([rng.uniform(size=(3, 4))], rng.uniform(size=4), (3, 4), S)
    shallow = tt.Session(8, 2)
    with pytest.raises(tt.DepthExhaustedError, match="stage"):
        tt.pipeline([rng.uniform(size=(4, 4))] * 3, rng.uniform(size=4), (2, 4), shallow)
