"""GPU parity: the sm_100a kernels (through the C-ABI) vs the CPU oracle.

Bit-exact for every slot of every tile (including '?' crossover garbage and
replicas) and identical cost counters -- the bar of SURVEY 8(c).  Inputs are
seeded; tile contents are random over ALL slots (not just packed data) so
the kernels must reproduce the reference's full-tile semantics.
"""
import random

import numpy as np
import pytest
import torch

import paper_2011_01805_b200 as tt
from paper_2011_01805_b200 import DimSpec, TileTensor, TileTensorShape, parse_shape, format_shape
from oracle_lib import CheckerError
from shapes import (fuzz_unknown_regions, partner_shape, random_pack_shape, random_tensor,
                    used_mask)

pytestmark = pytest.mark.gpu


def bits(x):
    return np.ascontiguousarray(x, dtype=np.float64).view(np.uint64)


def assert_bitwise(got, want, what=""):
    got = np.asarray(got)
    want = np.asarray(want)
    assert got.shape == want.shape, f"{what}: shape {got.shape} vs {want.shape}"
    g, w = bits(got), bits(want)
    if not np.array_equal(g, w):
        idx = np.argwhere(g != w)
        first = tuple(idx[0])
        raise AssertionError(f"{what}: {len(idx)} slots differ, first at {first}: "
                             f"{got[first]!r} vs {want[first]!r}")


def same_cost(a: tt.CostReport, b) -> bool:
    return (a.additions, a.multiplications, a.mask_multiplications, a.rotations,
            a.power_of_two_rotations) == (b.additions, b.multiplications, b.mask_multiplications,
                                          b.rotations, b.power_of_two_rotations)


_SESSIONS = {}


def session(s, depth=8):
    key = (s, depth)
    if key not in _SESSIONS:
        _SESSIONS[key] = tt.Session(s, depth)
    return _SESSIONS[key]


def test_pack_unpack_random_shapes(gpu, oracle):
    rng = random.Random(4004)
    nrng = np.random.default_rng(4004)
    for it in range(300):
        s = rng.choice([8, 16, 32, 64])
        S = session(s)
        shape = random_pack_shape(rng, s, rng.randint(1, 4))
        a = random_tensor(nrng, shape.tensor_extents())
        t = tt.pack(a, shape, S)
        assert_bitwise(t.tiles(), oracle.pack(a, shape, s), f"pack {format_shape(shape)}")
        assert_bitwise(tt.unpack(t), a, f"unpack {format_shape(shape)}")


def test_unpack_ignores_unused_slots(gpu, oracle):
    rng = random.Random(71)
    nrng = np.random.default_rng(71)
    for it in range(100):
        s = rng.choice([8, 16, 32, 64])
        S = session(s)
        shape = random_pack_shape(rng, s, rng.randint(1, 4))
        a = random_tensor(nrng, shape.tensor_extents())
        tiles = oracle.pack(a, shape, s)
        # garbage everywhere outside the used box; replicas keep their values
        garbage = ~used_mask(shape, s)
        tiles[garbage] = nrng.uniform(-100, 100, size=int(garbage.sum()))
        t = TileTensor(shape, tiles, S)
        assert_bitwise(tt.unpack(t), a, f"unpack fuzzed {format_shape(shape)}")


@pytest.mark.parametrize("op", [tt.OpKind.add, tt.OpKind.mul])
def test_elementwise_random(gpu, oracle, op):
    rng = random.Random(73 + int(op))
    nrng = np.random.default_rng(73 + int(op))
    done = 0
    while done < 150:
        s = 1 << rng.randint(2, 5)
        S = session(s)
        sa = random_pack_shape(rng, s, rng.randint(1, 3))
        sb = partner_shape(rng, sa)
        try:
            want_shape = oracle.elementwise_result_shape(sa, sb, int(op))
        except Exception:
            with pytest.raises(tt.ShapeError):
                tt.elementwise_result_shape(sa, sb, op)
            continue
        ta = nrng.uniform(-3, 3, size=(sa.tile_count(), s))
        tb = nrng.uniform(-3, 3, size=(sb.tile_count(), s))
        S.reset_counters()
        got = tt.tt_elementwise(TileTensor(sa, ta, S), TileTensor(sb, tb, S), op)
        ws, wt, wc = oracle.elementwise(int(op), sa, ta, sb, tb, s)
        assert got.shape() == ws
        assert_bitwise(got.tiles(), wt, f"ew {format_shape(sa)} {format_shape(sb)}")
        assert same_cost(S.cost_report(), wc)
        done += 1


def test_sum_every_dim_every_variant(gpu, oracle):
    rng = random.Random(89)
    nrng = np.random.default_rng(89)
    for it in range(120):
        s = 1 << rng.randint(2, 6)
        S = session(s)
        rank = rng.randint(1, 3)
        shape = random_pack_shape(rng, s, rank)
        tiles = nrng.uniform(-5, 5, size=(shape.tile_count(), s))
        T = TileTensor(shape, tiles, S)
        for dim in range(1, rank + 1):
            for variant in (None, tt.SumVariant.left_to_right, tt.SumVariant.right_to_left,
                            tt.SumVariant.power_of_two):
                v = -1 if variant is None else int(variant)
                try:
                    ws, wt, wc = oracle.sum(shape, tiles, s, dim, v)
                except Exception:
                    with pytest.raises(ValueError):
                        tt.tt_sum(T, dim, variant)
                    continue
                S.reset_counters()
                got = tt.tt_sum(T, dim, variant)
                assert got.shape() == ws
                assert_bitwise(got.tiles(), wt, f"sum {format_shape(shape)} dim {dim} v {v}")
                assert same_cost(S.cost_report(), wc), (S.cost_report(), wc)


def test_sum_boundary_split(gpu, oracle):
    """'?' dims whose used extent is not a multiple of t (tile_tensor.hpp:302-343)."""
    nrng = np.random.default_rng(97)
    cases = ["[18?/8,1]", "[5/2,1?/4]", "[13?/4,3/2]", "[7?/8]", "[3,11?/4]", "[2/2,9?/4,1]",
             "[1?/8]", "[29?/32]", "[6/2,5?/4]"]
    for text in cases:
        shape = parse_shape(text)
        s = shape.tile_slots()
        S = session(s)
        tiles = nrng.uniform(-5, 5, size=(shape.tile_count(), s))
        for dim in range(1, shape.rank() + 1):
            for v in (-1, 0, 1):
                ws, wt, wc = oracle.sum(shape, tiles, s, dim, v)
                S.reset_counters()
                got = tt.tt_sum(TileTensor(shape, tiles, S), dim,
                                None if v < 0 else tt.SumVariant(v))
                assert got.shape() == ws
                assert_bitwise(got.tiles(), wt, f"split {text} dim {dim} v {v}")
                assert same_cost(S.cost_report(), wc)


def test_mul_sum_matches_composition(gpu, oracle):
    """Fused tt_sum(tt_mul(a,b)) == the two-step oracle, incl. counters."""
    rng = random.Random(6006)
    nrng = np.random.default_rng(6006)
    for s in (8, 16, 32):
        S = session(s)
        t1 = 1
        while t1 <= s:
            t2 = 1
            while t1 * t2 <= s:
                t3 = s // (t1 * t2)
                a, b, c = rng.randint(1, 9), rng.randint(1, 9), rng.randint(1, 9)
                forms = [
                    (TileTensorShape([DimSpec(a, 1, t1), DimSpec(b, 1, t2), DimSpec(1, t3, t3)]),
                     TileTensorShape([DimSpec(1, t1, t1), DimSpec(b, 1, t2), DimSpec(c, 1, t3)]), 2),
                    (TileTensorShape([DimSpec(b, 1, t1), DimSpec(a, 1, t2), DimSpec(1, t3, t3)]),
                     TileTensorShape([DimSpec(b, 1, t1), DimSpec(1, t2, t2), DimSpec(c, 1, t3)]), 1),
                ]
                for sa, sb, dim in forms:
                    ta = nrng.uniform(-2, 2, size=(sa.tile_count(), s))
                    tb = nrng.uniform(-2, 2, size=(sb.tile_count(), s))
                    ws, wt, wc = oracle.mul_sum(sa, ta, sb, tb, s, dim)
                    S.reset_counters()
                    got = tt.tt_mul_sum(TileTensor(sa, ta, S), TileTensor(sb, tb, S), dim)
                    assert got.shape() == ws
                    assert_bitwise(got.tiles(), wt, f"mulsum {format_shape(sa)}x{format_shape(sb)}")
                    assert same_cost(S.cost_report(), wc)
                t2 *= 2
            t1 *= 2


def test_clean_and_replicate(gpu, oracle):
    nrng = np.random.default_rng(107)
    # the first four: small tiles; the rest: 4096-slot chunks of the chunked
    # clean kernel with cut dims of in-tile stride below, at and above 512
    # slots (its per-thread / per-chunk split of the mask coordinates)
    for text, s in [("[5/2,1?/4]", 8), ("[18?/8,4/16]", 128), ("[3?/4,2/2,7?/4]", 32),
                    ("[1?/8,3/4]", 32),
                    ("[40/16,70/32,1?/32]", 16384), ("[40/16,1?/32,70/32]", 16384),
                    ("[1?/16,70/32,40/32]", 16384), ("[20?/16,3?/32,7?/32]", 16384),
                    ("[9/8,5?/16,100?/32]", 4096), ("[13?/64,2/2,19?/32]", 4096),
                    ("[3/4,5?/1024,2?/4]", 16384)]:
        shape = parse_shape(text)
        S = session(s)
        tiles = nrng.uniform(-5, 5, size=(shape.tile_count(), s))
        ws, wt, wc = oracle.clean_unknowns(shape, tiles, s)
        S.reset_counters()
        got = tt.clean_unknowns(TileTensor(shape, tiles, S))
        assert got.shape() == ws
        assert_bitwise(got.tiles(), wt, f"clean {text}")
        assert same_cost(S.cost_report(), wc)
        assert got.chain_index() == S.max_chain_index() - 1
    # the last group reaches the mirrored register tree passes (replicate
    # schedules rotate by -e*stride): shuffles (stride < 32), row shifts, and
    # the column-local kind (t * stride == s)
    for text, s, dim in [("[5/2,1/4]", 8, 2), ("[7/4,1/8]", 32, 2), ("[1/8,3/4]", 32, 1),
                         ("[3/2,1/6,2/2]", 24, 2), ("[4,1/16,5/32]", 512, 2),
                         ("[4,3/16,1/32]", 512, 3), ("[2,1/32,3/16]", 512, 2),
                         ("[5,1/16,2/32,3/32]", 16384, 2), ("[3,2/16,1/32,2/32]", 16384, 3),
                         ("[3,2/16,2/32,1/32]", 16384, 4)]:
        shape = parse_shape(text)
        S = session(s)
        tiles = nrng.uniform(-5, 5, size=(shape.tile_count(), s))
        ws, wt, wc = oracle.replicate_dim(shape, tiles, s, dim)
        S.reset_counters()
        got = tt.replicate_dim(TileTensor(shape, tiles, S), dim)
        assert got.shape() == ws
        assert_bitwise(got.tiles(), wt, f"replicate {text}")
        assert same_cost(S.cost_report(), wc)


def test_tile_primitives(gpu, oracle):
    nrng = np.random.default_rng(41)
    for s in (16, 64, 256, 4096):
        S = session(s, 2)
        tile = nrng.integers(-50, 51, size=s).astype(np.float64)
        for n in sorted({1, 2, 3, 7, s // 2, s, min(s, 1190)} | {int(x) for x in nrng.integers(1, s + 1, 6)}):
            for v in (0, 1, 2):
                if v == 2 and n & (n - 1):
                    with pytest.raises(ValueError):
                        tt.sum_tile_flat(S, tile, n, tt.SumVariant(v))
                    continue
                want, wc = oracle.sum_tile_strided(tile, n, 1, v)
                S.reset_counters()
                got = tt.sum_tile_flat(S, tile, n, tt.SumVariant(v)).cpu().numpy()[0]
                assert_bitwise(got, want, f"flat sum s={s} n={n} v={v}")
                assert same_cost(S.cost_report(), wc)
        for off in (1, -1, 5, s - 1, 3 * s + 2, -8 * s):
            want, wc = oracle.rotate(tile, off)
            S.reset_counters()
            got = tt.tiles_rotate(S, tile, off).cpu().numpy()[0]
            assert_bitwise(got, want, f"rotate {off}")
            assert same_cost(S.cost_report(), wc)


def test_kat_backend_rotate(gpu):
    """tests/test_backend.cpp:32-45 (reference KAT)."""
    S = tt.Session(4, 3)
    t = np.array([1.0, 2, 3, 4])
    assert list(tt.tiles_rotate(S, t, 1).cpu().numpy()[0]) == [2, 3, 4, 1]
    assert list(tt.tiles_rotate(S, t, -1).cpu().numpy()[0]) == [4, 1, 2, 3]
    assert list(tt.tiles_rotate(S, t, 5).cpu().numpy()[0]) == [2, 3, 4, 1]
    assert S.cost_report().rotations == 3
    for off in (0, 4, -8):
        assert list(tt.tiles_rotate(S, t, off).cpu().numpy()[0]) == [1, 2, 3, 4]
    assert S.cost_report().rotations == 3


def test_kat_pack_figures(gpu):
    """tests/test_tile_tensor.cpp:152-181 (reference KAT)."""
    S = tt.Session(8, 4)
    v = np.array([1.0, 2, 3, 4, 5])
    tv = tt.pack(v, parse_shape("[5/2,*/4]"), S)
    assert tv.tile_count() == 3
    assert tv.tiles().tolist() == [[1, 1, 1, 1, 2, 2, 2, 2], [3, 3, 3, 3, 4, 4, 4, 4],
                                   [5, 5, 5, 5, 0, 0, 0, 0]]
    assert tt.pack(v, parse_shape("[5/2,*3/4]"), S).tile_at(0).tolist() == [1, 1, 1, 0, 2, 2, 2, 0]
    with pytest.raises(tt.ShapeError):
        tt.pack(v, parse_shape("[5/2,1?/4]"), S)
    with pytest.raises(tt.ShapeError):
        tt.pack(v, parse_shape("[5/2]"), S)
    with pytest.raises(tt.ShapeError):
        tt.pack(np.zeros(6), parse_shape("[5/2,*/4]"), S)


def test_kat_small_summation(gpu):
    """tests/test_tile_tensor.cpp:500-507."""
    S = tt.Session(4, 4)
    ta = tt.pack(np.array([[1.0, 2], [3, 4]]), parse_shape("[2/2,2/2]"), S)
    r = tt.tt_sum(ta, 2)
    assert format_shape(r.shape()) == "[2/2,1?/2]"
    assert tt.unpack(r).tolist() == [[3.0], [7.0]]


def test_depth_exhaustion(gpu):
    """tests/test_tile_tensor.cpp:478-485."""
    S = tt.Session(4, 1)
    ta = tt.pack(np.array([[1.0, 2], [3, 4]]), parse_shape("[2/2,2/2]"), S)
    sq = tt.tt_mul(ta, ta)
    with pytest.raises(tt.DepthExhaustedError):
        tt.tt_mul(sq, sq)


@pytest.mark.parametrize("path", ["auto", "tma", "regs", "generic", "window"])
def test_fused_large_tiles_every_path(gpu, oracle, path):
    """Config-5-like tiles (s = 16384 and 8192): every reduction kernel path
    (TMA ring, register tree, generic interpreter) and both group regimes
    (few groups -> split fold + tree, many groups -> single pass), with B
    broadcast along the summed dim (W-like) and not."""
    nrng = np.random.default_rng(5005)
    cases = [
        ("[512/16,256/32,64/32]", "[*/16,256/32,64/32]", 16384),
        ("[64/16,64/32,128/32]", "[64/16,64/32,*/32]", 16384),
        ("[256/16,512/32,32/16]", "[*/16,512/32,32/16]", 8192),
    ]
    tt.set_kernel_path(path)
    try:
        for xa, xb, s in cases:
            S = session(s)
            sa, sb = parse_shape(xa), parse_shape(xb)
            ta = nrng.uniform(-1, 1, size=(sa.tile_count(), s))
            tb = nrng.uniform(-1, 1, size=(sb.tile_count(), s))
            A, B = TileTensor(sa, ta, S), TileTensor(sb, tb, S)
            for dim in (1, 2, 3):
                ws, wt, wc = oracle.mul_sum(sa, ta, sb, tb, s, dim)
                S.reset_counters()
                got = tt.tt_mul_sum(A, B, dim)
                assert got.shape() == ws
                assert_bitwise(got.tiles(), wt, f"{path} {xa} x {xb} dim {dim}")
                assert same_cost(S.cost_report(), wc)
                # tt_sum alone on the same tensor
                ws2, wt2, _ = oracle.sum(sa, ta, s, dim)
                assert_bitwise(tt.tt_sum(A, dim).tiles(), wt2, f"{path} sum {xa} dim {dim}")
    finally:
        tt.set_kernel_path("auto")


@pytest.mark.parametrize("path", ["auto", "regs"])
def test_pack_unpack_plain_shapes_tma_and_gather(gpu, oracle, path):
    """Plain shapes take the TMA tensor-map pack/unpack (auto); `regs` forces
    the gather kernels.  Edge tiles exercise TMA out-of-bounds zero fill."""
    rng = random.Random(1234)
    nrng = np.random.default_rng(1234)
    tt.set_kernel_path(path)
    try:
        for it in range(150):
            s = rng.choice([16, 64, 256, 1024])
            S = session(s)
            rank = rng.randint(1, 4)
            shape = random_pack_shape(rng, s, rank, allow_replication=False)
            dims = list(shape.dims())
            # make the innermost extent even half the time (TMA eligibility)
            if rng.random() < 0.5 and dims[-1].n % 2:
                dims[-1] = DimSpec(dims[-1].n + 1, 1, dims[-1].t)
            shape = TileTensorShape(dims)
            a = random_tensor(nrng, shape.tensor_extents())
            t = tt.pack(a, shape, S)
            assert_bitwise(t.tiles(), oracle.pack(a, shape, s), f"{path} pack {format_shape(shape)}")
            assert_bitwise(tt.unpack(t), a, f"{path} unpack {format_shape(shape)}")
        for text, s in [("[100/16,200/32]", 512), ("[1024/64,4096/128]", 8192),
                        ("[50/16,20/2,255/32]", 1024), ("[13/4,30/8,6/2]", 64)]:
            shape = parse_shape(text)
            S = session(s)
            a = random_tensor(nrng, shape.tensor_extents())
            t = tt.pack(a, shape, S)
            assert_bitwise(t.tiles(), oracle.pack(a, shape, s), f"{path} pack {text}")
            assert_bitwise(tt.unpack(t), a, f"{path} unpack {text}")
    finally:
        tt.set_kernel_path("auto")


@pytest.mark.parametrize("path", ["auto", "window", "generic"])
def test_tile_matmul_gemm_paths(gpu, oracle, path):
    """Products with two broadcast dims (matmul_a / matmul_b) at sizes that
    take the GEMM-style blocked fold, the fused column tree (sum over dim 1
    with t = 16) and the row-shift tree pass; partial 16x16 blocks included."""
    nrng = np.random.default_rng(777)
    cases = [  # (A shape, B shape, summed dim, slots)
        ("[40/16,24/8,*/8]", "[40/16,*/8,20/8]", 1, 1024),     # matmul_b, t1 = 16: fused column tree
        ("[36/8,50/16,*/8]", "[*/8,50/16,40/8]", 2, 1024),     # matmul_a, t2 = 16: row-shift pass
        ("[100/16,70/8,*/16]", "[100/16,*/8,33/16]", 1, 2048),
        ("[24/4,96/32,*/16]", "[*/4,96/32,24/16]", 2, 2048),
    ]
    tt.set_kernel_path(path)
    try:
        for xa, xb, dim, s in cases:
            S = session(s)
            sa, sb = parse_shape(xa), parse_shape(xb)
            ta = nrng.uniform(-1, 1, size=(sa.tile_count(), s))
            tb = nrng.uniform(-1, 1, size=(sb.tile_count(), s))
            ws, wt, wc = oracle.mul_sum(sa, ta, sb, tb, s, dim)
            S.reset_counters()
            f = tt.matmul_b if dim == 1 else tt.matmul_a
            got = f(TileTensor(sa, ta, S), TileTensor(sb, tb, S))
            assert got.shape() == ws
            assert_bitwise(got.tiles(), wt, f"{path} {xa} x {xb}")
            assert same_cost(S.cost_report(), wc)
    finally:
        tt.set_kernel_path("auto")


def test_huge_tiles(gpu, oracle):
    """Tiles too large for shared memory (s = 2^20 and 2^21 slots, 8-16 MiB
    per tile): every op still runs (split fold + global-scratch schedule,
    gather pack) and matches the oracle bit for bit -- the reference allows
    any slot count below 2^31."""
    nrng = np.random.default_rng(2024)
    for text_a, text_b, s in [("[3/1024,5/1024]", "[*/1024,5/1024]", 1 << 20),
                              ("[2/2048,2/1024]", "[2/2048,*/1024]", 1 << 21)]:
        S = session(s)
        sa, sb = parse_shape(text_a), parse_shape(text_b)
        ta = nrng.uniform(-1, 1, size=(sa.tile_count(), s))
        tb = nrng.uniform(-1, 1, size=(sb.tile_count(), s))
        A, B = TileTensor(sa, ta, S), TileTensor(sb, tb, S)
        for dim in (1, 2):
            ws, wt, wc = oracle.mul_sum(sa, ta, sb, tb, s, dim)
            S.reset_counters()
            got = tt.tt_mul_sum(A, B, dim)
            assert got.shape() == ws
            assert_bitwise(got.tiles(), wt, f"huge {text_a} dim {dim}")
            assert same_cost(S.cost_report(), wc)
        dense = nrng.uniform(-1, 1, size=sa.tensor_extents())
        packed = tt.pack(dense, sa, S)
        assert_bitwise(packed.tiles(), oracle.pack(dense, sa, s), f"huge pack {text_a}")
        assert_bitwise(tt.unpack(packed), dense, f"huge unpack {text_a}")


def test_rotate_all_kernel_forms(gpu):
    """Session::rotate (backend.hpp:150-163): out[j] = in[(j + r) mod s] through
    the aligned shuffle form (s % 512 == 0), the chunked form and the
    per-slot form, for offsets across segment and tile boundaries."""
    nrng = np.random.default_rng(31337)
    for s in (16, 96, 1024 + 64, 512, 1024, 16384):
        S = session(s)
        tiles = nrng.uniform(-1, 1, size=(7, s))
        for off in (1, 5, 31, 32, 33, 511, 512, s - 1, s + 7, -3, -s - 1):
            r = ((off % s) + s) % s
            got = tt.tiles_rotate(S, tiles, off)
            want = np.roll(tiles, -r, axis=1)
            assert_bitwise(got.detach().cpu().numpy(), want, f"rotate s={s} off={off}")


def test_fold_chain_matches_single_pass(gpu, oracle):
    """tt_mul_fold continuing an accumulator (the exact cross-GPU chain of
    sharding.chain_mul_sum, run here as slabs on one GPU): slab 0 folded from
    its first product, slab 1 from slab 0's accumulators in chunks, then the
    in-tile schedule once -- bit-identical to tt_mul_sum on the whole tensor,
    with the same counters in total."""
    nrng = np.random.default_rng(4242)
    for gx, gw, s in [("[64/4,8/2,6/2]", "[*/4,8/2,6/2]", 16),
                      ("[256/16,64/32,32/32]", "[*/16,64/32,32/32]", 16384),
                      ("[96/16,32/32,16/16]", "[96/16,32/32,16/16]", 8192)]:
        S = session(s)
        sx, sw = parse_shape(gx), parse_shape(gw)
        xd = nrng.uniform(-1, 1, size=sx.tensor_extents())
        wd = nrng.uniform(-1, 1, size=sw.tensor_extents())
        X, W = tt.pack(xd, sx, S), tt.pack(wd, sw, S)
        S.reset_counters()
        want = tt.tt_mul_sum(X, W, 1)
        c_want = S.cost_report()
        w_shared = sw.dim(0).n == 1
        S.reset_counters()
        parts, init = [], None
        for p in (tt_shard(sx, 2, 0), tt_shard(sx, 2, 1)):
            Xs = tt.pack(xd[p[1]], p[0], S)
            Ws = W if w_shared else tt.pack(wd[p[1]], p[0], S)
            fs = tt.fold_shape(p[0], Ws.shape(), 1)
            n_out = fs.tile_count()
            cuts = [0, n_out // 3, n_out]
            chunks = [tt.mul_fold(Xs, Ws, 1, (lo, hi), None if init is None else init[lo:hi])[0]
                      for lo, hi in zip(cuts, cuts[1:])]
            init = torch.cat(chunks)
        got = tt.tt_sum(tt.TileTensor(fs, init, S), 1)
        assert got.shape() == want.shape()
        assert_bitwise(got.tiles(), want.tiles(), f"fold chain {gx}")
        c = S.cost_report()
        assert (c.additions, c.multiplications, c.rotations) == \
            (c_want.additions, c_want.multiplications, c_want.rotations)
    with pytest.raises(tt.ShapeError):
        tt.mul_fold(X, W, 9)


def tt_shard(shape, world, rank):
    from paper_2011_01805_b200 import sharding
    p = sharding.plan(shape, 1, world, rank)
    return p.local_shape, p.dense_slices()


def _big_shape(rng, s, rank):
    """A random pack shape over a large slot count with few tiles."""
    from paper_2011_01805_b200 import DimSpec, TileTensorShape
    t = [1] * rank
    rem = s
    for i in range(rank - 1):
        t[i] = rng.choice([x for x in (1, 2, 4, 8, 16, 32, 64, 128) if x <= rem])
        rem //= t[i]
    t[rank - 1] = rem
    dims = []
    for i in range(rank):
        pick = rng.randint(0, 4)
        if pick == 0:
            dims.append(DimSpec(1, t[i], t[i]))
        elif pick == 1 and t[i] > 1:
            dims.append(DimSpec(1, rng.randint(1, t[i]), t[i]))
        else:
            dims.append(DimSpec(rng.randint(1, 3 * t[i]), 1, t[i]))
    return TileTensorShape(dims)


def test_random_large_slot_counts(gpu, oracle):
    """Random shapes over 512..16384-slot tiles (the chunked elementwise /
    clean / rotate kernels, TMA pack, window and register tree passes, split
    folds): pack, elementwise, every sum variant, fused product sums,
    clean_unknowns and replicate_dim -- all bitwise vs the oracle."""
    rng = random.Random(8128)
    nrng = np.random.default_rng(8128)
    cases = 0
    seen = {"ew": 0, "sum": 0, "clean": 0, "replicate": 0, "mul_sum": 0}
    while cases < 40:
        s = rng.choice([512, 1024, 2048, 4096, 8192, 16384])
        S = session(s)
        sa = _big_shape(rng, s, rng.randint(2, 3))
        if sa.tile_count() > 64:
            continue
        dense = nrng.uniform(-2, 2, size=sa.tensor_extents())
        A = tt.pack(dense, sa, S)
        assert_bitwise(A.tiles(), oracle.pack(dense, sa, s), f"pack {format_shape(sa)}")
        sb = partner_shape(rng, sa)
        tb = nrng.uniform(-2, 2, size=(sb.tile_count(), s))
        B = TileTensor(sb, tb, S)
        ta = A.tiles()
        try:
            oracle.elementwise_result_shape(sa, sb, 1)
            ok = True
        except Exception:
            ok = False
        if ok:
            for op in (tt.OpKind.add, tt.OpKind.mul):
                ws, wt, _ = oracle.elementwise(int(op), sa, ta, sb, tb, s)
                got = tt.tt_elementwise(A, B, op)
                assert_bitwise(got.tiles(), wt, f"ew {format_shape(sa)} {format_shape(sb)}")
                seen["ew"] += 1
        for dim in range(1, sa.rank() + 1):
            for variant in (None, tt.SumVariant.left_to_right):
                v = -1 if variant is None else int(variant)
                try:
                    ws, wt, wc = oracle.sum(sa, ta, s, dim, v)
                except Exception:
                    continue
                S.reset_counters()
                got = tt.tt_sum(A, dim, variant)
                assert got.shape() == ws
                assert_bitwise(got.tiles(), wt, f"sum {format_shape(sa)} dim {dim} v {v}")
                assert same_cost(S.cost_report(), wc)
                seen["sum"] += 1
                if got.shape().has_unknown():
                    cs, ct, _ = oracle.clean_unknowns(ws, wt, s)
                    C = tt.clean_unknowns(got)
                    assert_bitwise(C.tiles(), ct, f"clean {format_shape(ws)}")
                    seen["clean"] += 1
                    d = got.shape().dim(dim - 1)
                    if d.n == 1 and d.t > 1:
                        rs, rt, _ = oracle.replicate_dim(cs, ct, s, dim)
                        R = tt.replicate_dim(C, dim)
                        assert_bitwise(R.tiles(), rt, f"replicate {format_shape(cs)} dim {dim}")
                        seen["replicate"] += 1
            if ok:
                try:
                    ws, wt, wc = oracle.mul_sum(sa, ta, sb, tb, s, dim)
                except Exception:
                    continue
                got = tt.tt_mul_sum(A, B, dim)
                assert_bitwise(got.tiles(), wt, f"mul_sum {format_shape(sa)} x {format_shape(sb)} {dim}")
                seen["mul_sum"] += 1
        cases += 1
    print(seen)
    assert seen["sum"] >= 40 and seen["clean"] >= 5 and seen["replicate"] >= 3 and seen["mul_sum"] >= 10


def test_interleaved_random(gpu, oracle):
    """The builder's `~` tiling (not in the reference, so
    checked against the C restatement's own definition): random shapes with
    interleaved dims through pack, unpack, elementwise with `~` / broadcast
    partners, sums over every dim (clean first when '?'), bit for bit."""
    from paper_2011_01805_b200 import DimSpec, TileTensorShape
    rng = random.Random(777)
    nrng = np.random.default_rng(777)
    done = 0
    while done < 60:
        s = rng.choice([16, 32, 64, 512])
        rank = rng.randint(1, 3)
        t = [1] * rank
        rem = s
        for i in range(rank - 1):
            t[i] = rng.choice([x for x in (1, 2, 4, 8) if x <= rem])
            rem //= t[i]
        t[-1] = rem
        dims = [DimSpec(rng.randint(1, 3 * ti), 1, ti, False, rng.random() < 0.6) for ti in t]
        try:
            sa = TileTensorShape(dims)
        except tt.ShapeError:
            continue
        S = session(s)
        dense = nrng.uniform(-2, 2, size=sa.tensor_extents())
        A = tt.pack(dense, sa, S)
        assert_bitwise(A.tiles(), oracle.pack(dense, sa, s), f"pack {format_shape(sa)}")
        assert_bitwise(tt.unpack(A), dense, f"unpack {format_shape(sa)}")
        # partner: same interleaving or fully replicated per dim
        pdims = [DimSpec(d.n, 1, d.t, False, d.interleaved) if rng.random() < 0.6
                 else DimSpec(1, d.t, d.t) for d in sa.dims()]
        sb = TileTensorShape(pdims)
        tb = nrng.uniform(-2, 2, size=(sb.tile_count(), s))
        ta = A.tiles()
        for op in (tt.OpKind.add, tt.OpKind.mul):
            try:
                ws, wt, _ = oracle.elementwise(int(op), sa, ta, sb, tb, s)
            except Exception:
                with pytest.raises(tt.ShapeError):
                    tt.tt_elementwise(A, TileTensor(sb, tb, S), op)
                continue
            got = tt.tt_elementwise(A, TileTensor(sb, tb, S), op)
            assert got.shape() == ws
            assert_bitwise(got.tiles(), wt, f"ew {format_shape(sa)} {format_shape(sb)}")
        for dim in range(1, rank + 1):
            try:
                ws, wt, wc = oracle.sum(sa, ta, s, dim)
            except Exception:
                with pytest.raises((tt.ShapeError, ValueError)):
                    tt.tt_sum(A, dim)
                continue
            S.reset_counters()
            got = tt.tt_sum(A, dim)
            assert got.shape() == ws
            assert_bitwise(got.tiles(), wt, f"sum {format_shape(sa)} dim {dim}")
            assert same_cost(S.cost_report(), wc)
        done += 1


def test_relaxed_and_variants_random(gpu, oracle):
    """Relaxed shapes (tile extents multiply to less than s; the remaining
    slots are never touched by the reference's pack) and explicit sum
    variants (left-to-right, right-to-left, power-of-two where legal) over
    large tiles, including '?' boundary splits: bitwise vs the oracle."""
    from paper_2011_01805_b200 import DimSpec, TileTensorShape
    rng = random.Random(99)
    nrng = np.random.default_rng(99)
    seen = 0
    while seen < 40:
        s = rng.choice([64, 512, 4096])
        rank = rng.randint(1, 3)
        budget = s // rng.choice([1, 2, 4])
        t = []
        rem = budget
        for i in range(rank - 1):
            ti = rng.choice([x for x in (1, 2, 3, 4, 8) if x <= rem])
            t.append(ti)
            rem //= ti
        t.append(max(1, rem))
        dims = [DimSpec(rng.randint(1, 2 * ti + 1), 1, ti) for ti in t]
        relaxed = int(np.prod(t)) != s
        try:
            sa = TileTensorShape(dims, relaxed)
        except tt.ShapeError:
            continue
        if sa.tile_slots() > s:
            continue
        S = session(s)
        dense = nrng.uniform(-2, 2, size=sa.tensor_extents())
        A = tt.pack(dense, sa, S)
        assert_bitwise(A.tiles(), oracle.pack(dense, sa, s), f"pack {format_shape(sa)} relaxed={relaxed}")
        assert_bitwise(tt.unpack(A), dense, f"unpack {format_shape(sa)}")
        ta = A.tiles()
        for dim in range(1, rank + 1):
            for variant in (tt.SumVariant.left_to_right, tt.SumVariant.right_to_left,
                            tt.SumVariant.power_of_two):
                try:
                    ws, wt, wc = oracle.sum(sa, ta, s, dim, int(variant))
                except Exception:
                    continue
                S.reset_counters()
                got = tt.tt_sum(A, dim, variant)
                assert got.shape() == ws
                assert_bitwise(got.tiles(), wt, f"sum {format_shape(sa)} dim {dim} {variant}")
                assert same_cost(S.cost_report(), wc)
                if ws.has_unknown():
                    cs, ct, _ = oracle.clean_unknowns(ws, wt, s)
                    assert_bitwise(tt.clean_unknowns(got).tiles(), ct, f"clean {format_shape(ws)}")
        seen += 1


def test_odd_and_tiny_slot_counts(gpu, oracle):
    """s = 1, odd and non-power-of-two slot counts take the scalar fallbacks
    of every vectorised kernel (pack, elementwise, clean, rotate, folds)."""
    from paper_2011_01805_b200 import DimSpec, TileTensorShape
    nrng = np.random.default_rng(135)
    for s, texts in [(1, ["[5]", "[3,4]"]), (3, ["[7/3]", "[2,5/3]"]), (5, ["[11/5,2]"]),
                     (6, ["[7/2,5/3]", "[4/3,*/2]"]), (7, ["[15/7]"]), (9, ["[10/3,4/3]"]),
                     (97, ["[200/97]"]), (1000, ["[3/10,250/100]"])]:
        S = session(s)
        for text in texts:
            sa = parse_shape(text)
            dense = nrng.uniform(-2, 2, size=sa.tensor_extents())
            A = tt.pack(dense, sa, S)
            assert_bitwise(A.tiles(), oracle.pack(dense, sa, s), f"pack {text} s={s}")
            assert_bitwise(tt.unpack(A), dense, f"unpack {text} s={s}")
            ta = A.tiles()
            for op in (tt.OpKind.add, tt.OpKind.mul):
                ws, wt, _ = oracle.elementwise(int(op), sa, ta, sa, ta, s)
                assert_bitwise(tt.tt_elementwise(A, A, op).tiles(), wt, f"ew {text} s={s}")
            for dim in range(1, sa.rank() + 1):
                ws, wt, wc = oracle.sum(sa, ta, s, dim)
                S.reset_counters()
                got = tt.tt_sum(A, dim)
                assert_bitwise(got.tiles(), wt, f"sum {text} dim {dim} s={s}")
                assert same_cost(S.cost_report(), wc)
                ms, mt, _ = oracle.mul_sum(sa, ta, sa, ta, s, dim)
                assert_bitwise(tt.tt_mul_sum(A, A, dim).tiles(), mt, f"mul_sum {text} {dim} s={s}")
                if ws.has_unknown():
                    cs, ct, _ = oracle.clean_unknowns(ws, wt, s)
                    assert_bitwise(tt.clean_unknowns(got).tiles(), ct, f"clean {text} s={s}")
            for off in (1, s // 2 + 1, -1):
                r = ((off % s) + s) % s
                want = np.roll(ta, -r, axis=1)
                got = tt.tiles_rotate(S, ta, off)
                assert_bitwise(got.detach().cpu().numpy(), want, f"rotate s={s} off={off}")


def test_interleaved_kats_on_gpu(gpu):
    """The `~` known answers of tests/test_shape_algebra.py through the CUDA pack /
    unpack and the fused fold + tree (no oracle involved: hand-worked values)."""
    from test_shape_algebra import INTERLEAVED_KATS
    for text, dense, want in INTERLEAVED_KATS:
        sh = parse_shape(text)
        s = len(want[0])
        S = session(s)
        t = tt.pack(np.asarray(dense, dtype=np.float64), sh, S)
        assert t.tiles().tolist() == [[float(v) for v in row] for row in want], text
        assert tt.unpack(t).tolist() == np.asarray(dense, dtype=np.float64).tolist()
    S = session(4)
    S.reset_counters()
    r = tt.tt_sum(tt.pack(np.arange(1, 9, dtype=np.float64), parse_shape("[8~/4]"), S), 1)
    assert tt.format_shape(r.shape()) == "[*/4]"
    assert r.tiles().tolist() == [[36.0, 36.0, 36.0, 36.0]]
    c = S.cost_report()
    assert (c.additions, c.rotations) == (3, 2)


@pytest.mark.parametrize("case", [
    # (a shape, b shape): b broadcast along dims 1 (and 3), a broadcast along dim 2;
    # > 64 MiB of output, so the L2-hinted broadcast kernel runs;
    # the broadcast operand on either side, one or two broadcast dims
    ("[640/16,64/32,256/32]", "[*/16,64/32,256/32]"),
    ("[*/16,640/32,256/32]", "[64/16,640/32,256/32]"),
    ("[96/16,64/32,1504/32]", "[*/16,64/32,*/32]"),
    # even innermost broadcast extent with two broadcast dims (paired items), either side
    ("[96/16,64/32,1536/32]", "[*/16,64/32,*/32]"),
    ("[*/16,64/32,*/32]", "[96/16,64/32,1536/32]"),
])
@pytest.mark.parametrize("op", [tt.OpKind.add, tt.OpKind.mul], ids=["add", "mul"])
def test_broadcast_elementwise_large(gpu, oracle, case, op):
    s = 16 * 32 * 32
    S = session(s)
    sa, sb = parse_shape(case[0]), parse_shape(case[1])
    nrng = np.random.default_rng(11 + int(op))
    ta = nrng.uniform(-3, 3, size=(sa.tile_count(), s))
    tb = nrng.uniform(-3, 3, size=(sb.tile_count(), s))
    got = tt.tt_elementwise(TileTensor(sa, ta, S), TileTensor(sb, tb, S), op)
    ws, wt, _ = oracle.elementwise(int(op), sa, ta, sb, tb, s)
    assert got.shape() == ws
    assert got.tiles().nbytes > (64 << 20)
    assert_bitwise(got.tiles(), wt, f"ew {case}")


def test_high_rank_pack_sum_unpack(gpu, oracle):
    # rank 12 (TT_MAX_RANK = 16; the reference has no limit): pack, fused
    # multiply + sum over a middle dim, elementwise with a broadcast, unpack
    s = 4096
    S = session(s)
    sh = parse_shape("[" + ",".join(["3/2"] * 12) + "]")
    nrng = np.random.default_rng(1212)
    dense = nrng.uniform(-1, 1, size=(3,) * 12)
    T = tt.pack(dense, sh, S)
    assert_bitwise(T.tiles(), oracle.pack(dense, sh, s), "rank-12 pack")
    assert_bitwise(tt.unpack(T), dense, "rank-12 unpack")
    for dim in (1, 7, 12):
        got = tt.tt_mul_sum(T, T, dim)
        ws, wt, _ = oracle.mul_sum(sh, T.tiles(), sh, T.tiles(), s, dim)
        assert got.shape() == ws
        assert_bitwise(got.tiles(), wt, f"rank-12 mul_sum dim {dim}")
    sb = parse_shape("[" + ",".join(["3/2"] * 5 + ["*/2"] + ["3/2"] * 6) + "]")
    tb = nrng.uniform(-1, 1, size=(sb.tile_count(), s))
    got = tt.tt_elementwise(T, TileTensor(sb, tb, S), tt.OpKind.mul)
    ws, wt, _ = oracle.elementwise(int(tt.OpKind.mul), sh, T.tiles(), sb, tb, s)
    assert got.shape() == ws
    assert_bitwise(got.tiles(), wt, "rank-12 broadcast mul")


def test_dependent_launch_chain(gpu, oracle):
    # 300 back-to-back operators, each reading the previous one's result (and
    # some overwriting a block the one before read): with programmatic dependent
    # launch every kernel is dispatched while its predecessor drains, so any
    # early read / early write would show in the bits.  Same chain on the oracle.
    s = 512
    S = tt.Session(s, 1000)  # ~200 multiplications deep
    sh = parse_shape("[40/16,60/32]")
    nrng = np.random.default_rng(300)
    x = nrng.uniform(-1, 1, size=(sh.tile_count(), s))
    y = nrng.uniform(-1, 1, size=(sh.tile_count(), s))
    c = nrng.uniform(0.4, 0.6, size=(sh.tile_count(), s))   # X <- (X + Y) * c stays bounded
    d = nrng.uniform(0.9, 1.0, size=(sh.tile_count(), s))
    X, Y = TileTensor(sh, x, S), TileTensor(sh, y, S)
    C, D = TileTensor(sh, c, S), TileTensor(sh, d, S)
    wx, wy = x, y
    sums = []
    for i in range(300):
        if i % 3 == 0:
            X = tt.tt_elementwise(X, Y, tt.OpKind.add)
            _, wx, _ = oracle.elementwise(int(tt.OpKind.add), sh, wx, sh, wy, s)
        elif i % 3 == 1:
            X = tt.tt_elementwise(X, C, tt.OpKind.mul)
            _, wx, _ = oracle.elementwise(int(tt.OpKind.mul), sh, wx, sh, c, s)
        else:
            Y = tt.tt_elementwise(Y, D, tt.OpKind.mul)
            _, wy, _ = oracle.elementwise(int(tt.OpKind.mul), sh, wy, sh, d, s)
            Y = tt.tt_elementwise(Y, X, tt.OpKind.add)
            _, wy, _ = oracle.elementwise(int(tt.OpKind.add), sh, wy, sh, wx, s)
            Y = tt.tt_elementwise(Y, C, tt.OpKind.mul)
            _, wy, _ = oracle.elementwise(int(tt.OpKind.mul), sh, wy, sh, c, s)
        if i % 25 == 24:  # a reduction in the chain
            sums.append((tt.tt_sum(X, 2), oracle.sum(sh, wx, s, 2)[1]))
    assert np.isfinite(wx).all() and np.isfinite(wy).all()
    assert_bitwise(X.tiles(), wx, "dependent chain X")
    assert_bitwise(Y.tiles(), wy, "dependent chain Y")
    for k, (got, want) in enumerate(sums):
        assert_bitwise(got.tiles(), want, f"dependent chain sum {k}")


def test_tile_matmul_random_shapes(gpu, oracle):
    """Random products with two broadcast dims (the GEMM-shaped fold): both summed
    dims, block counts that cross the 16 x 16 group blocks with partial edge blocks,
    fold lengths that are not a multiple of the ring's 4-step stages, partial tiles
    ('?' results), and zero to two further group dims -- bitwise and counter parity."""
    rng = random.Random(20241021)
    nrng = np.random.default_rng(4242)
    done = 0
    while done < 36:
        rank = rng.choice([3, 3, 4, 5])
        s = rng.choice([256, 512, 1024])
        # tile dims: powers of two with product s
        logs = [0] * rank
        for _ in range(s.bit_length() - 1):
            logs[rng.randrange(rank)] += 1
        t = [1 << l for l in logs]
        dim = rng.choice([1, 2])           # the summed (fold) dim
        other = 2 if dim == 1 else 1        # A varies, B broadcasts
        third = 3                           # B varies, A broadcasts
        ext = [1] * rank
        ext[dim - 1] = rng.randint(1, 13)
        ext[other - 1] = rng.choice([1, 2, 5, 15, 16, 17, 31, 33, 40])
        ext[third - 1] = rng.choice([1, 3, 8, 16, 18, 23, 32, 37])
        for i in range(3, rank):
            ext[i] = rng.randint(1, 3)
        if ext[0] * ext[1] * ext[2] * int(np.prod(ext[3:])) > 16000:
            continue
        n = [rng.randint((e - 1) * ti + 1, e * ti) for e, ti in zip(ext, t)]
        da, db = [], []
        for i in range(rank):
            if i == other - 1:
                da.append(DimSpec(n[i], 1, t[i]))
                db.append(DimSpec(1, t[i], t[i]) if t[i] > 1 and rng.random() < 0.8 else DimSpec(1, 1, t[i]))
            elif i == third - 1:
                da.append(DimSpec(1, t[i], t[i]) if t[i] > 1 and rng.random() < 0.8 else DimSpec(1, 1, t[i]))
                db.append(DimSpec(n[i], 1, t[i]))
            else:
                da.append(DimSpec(n[i], 1, t[i]))
                db.append(DimSpec(n[i], 1, t[i]))
        sa, sb = TileTensorShape(da), TileTensorShape(db)
        try:
            ta = nrng.uniform(-1, 1, size=(sa.tile_count(), s))
            tb = nrng.uniform(-1, 1, size=(sb.tile_count(), s))
            ws, wt, wc = oracle.mul_sum(sa, ta, sb, tb, s, dim)
        except CheckerError:
            continue
        S = session(s)
        S.reset_counters()
        got = tt.tt_mul_sum(TileTensor(sa, ta, S), TileTensor(sb, tb, S), dim)
        what = f"{format_shape(sa)} x {format_shape(sb)} sum {dim} (s={s})"
        assert got.shape() == ws, what
        assert_bitwise(got.tiles(), wt, what)
        assert same_cost(S.cost_report(), wc), what
        done += 1


def test_few_group_shared_operand_folds(gpu, oracle):
    """Small folds over few groups in which one operand is the same for every group
    along a dim (matvec forms: the group-blocked ring fold): both orientations, fold
    lengths below and above the ring depth, a further group dim, large and small tiles."""
    nrng = np.random.default_rng(99)
    cases = [  # (A shape, B shape, summed dim, slots)
        ("[1024/64,4096/128]", "[*/64,4096/128]", 2, 8192),        # config 2
        ("[*/64,640/128]", "[384/64,640/128]", 2, 8192),           # the shared operand first
        ("[128/32,66/2,*/4]", "[*/32,66/2,8/4]", 2, 256),          # 33 steps, both dims broadcast
        ("[20/2,7,48/128]", "[*/2,7,48/128]", 2, 256),             # t2 = 1: fold only, 7 steps
        ("[12/2,300/8,5/16]", "[*/2,300/8,5/16]", 2, 256),         # odd third dim: partial tiles
        ("[8/4,100/4,3,6/64]", "[8/4,100/4,3,*/64]", 2, 1024),     # shared along the last dim
        ("[6/2,9/2,2/64]", "[*/2,9/2,2/64]", 2, 256),              # 5 steps: shorter than the ring
        ("[64/16,2048/512]", "[*/16,2048/512]", 2, 8192),
    ]
    for xa, xb, dim, s in cases:
        S = session(s)
        sa, sb = parse_shape(xa), parse_shape(xb)
        ta = nrng.uniform(-1, 1, size=(sa.tile_count(), s))
        tb = nrng.uniform(-1, 1, size=(sb.tile_count(), s))
        ws, wt, wc = oracle.mul_sum(sa, ta, sb, tb, s, dim)
        S.reset_counters()
        got = tt.tt_mul_sum(TileTensor(sa, ta, S), TileTensor(sb, tb, S), dim)
        assert got.shape() == ws, f"{xa} x {xb}"
        assert_bitwise(got.tiles(), wt, f"{xa} x {xb}")
        assert same_cost(S.cost_report(), wc), f"{xa} x {xb}"
