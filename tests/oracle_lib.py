"""ctypes wrappers over the CPU checkers (TEST INFRASTRUCTURE ONLY).

* :class:`Oracle` -- ``oracle/_build/libttoracle.so``, the C restatement.
* :class:`Ref` -- ``oracle/_ref/libttref.so``, the unmodified reference
  headers compiled in this container (absent on the GPU box).

Both expose the same methods so a test can run one case through either.
Shapes are :class:`paper_2011_01805_b200.TileTensorShape` (converted with
``to_c``); tiles are numpy ``float64`` arrays ``[tile_count, s]``.
"""
from __future__ import annotations

import ctypes
from pathlib import Path

import numpy as np

from paper_2011_01805_b200._abi import CCost, CShape, TT_MAX_RANK
from paper_2011_01805_b200.tiletensor import TileTensorShape, CostReport

ROOT = Path(__file__).resolve().parents[1]
ORACLE_LIB = ROOT / "oracle" / "_build" / "libttoracle.so"
REF_LIB = ROOT / "oracle" / "_ref" / "libttref.so"

_D = ctypes.POINTER(ctypes.c_double)
_SP = ctypes.POINTER(CShape)
_CP = ctypes.POINTER(CCost)
_I64P = ctypes.POINTER(ctypes.c_int64)


def _dp(a: np.ndarray):
    return a.ctypes.data_as(_D)


def _cost(c: CCost) -> CostReport:
    return CostReport(c.additions, c.multiplications, c.mask_multiplications, c.rotations,
                      c.bootstraps, c.power_of_two_rotations)


def _sh(shape) -> CShape:
    return shape.to_c() if isinstance(shape, TileTensorShape) else shape


class CheckerError(RuntimeError):
    def __init__(self, code: int, msg: str = ""):
        super().__init__(f"checker error {code}: {msg}")
        self.code = code


class _Base:
    prefix = ""

    def __init__(self, path: Path):
        if not path.exists():
            raise FileNotFoundError(path)
        self.lib = ctypes.CDLL(str(path))

    def _f(self, name):
        return getattr(self.lib, self.prefix + name)

    def _rc(self, rc):
        if rc != 0:
            raise CheckerError(rc, self._err())

    def _err(self):
        return ""

    # --- ops ---------------------------------------------------------------------
    def pack(self, dense, shape, s):
        dense = np.ascontiguousarray(dense, dtype=np.float64).reshape(-1)
        out = np.empty((shape.tile_count(), s), dtype=np.float64)
        self._pack(dense, shape, s, out)
        return out

    def unpack(self, shape, s, tiles):
        tiles = np.ascontiguousarray(tiles, dtype=np.float64)
        out = np.empty(shape.tensor_extents(), dtype=np.float64)
        self._rc(self._f("unpack")(ctypes.byref(_sh(shape)), ctypes.c_int64(s), _dp(tiles),
                                   _dp(out)))
        return out

    def elementwise(self, op, sa, ta, sb, tb, s):
        ta = np.ascontiguousarray(ta, dtype=np.float64)
        tb = np.ascontiguousarray(tb, dtype=np.float64)
        so = CShape()
        self._rc(self._shape_ew(sa, sb, op, so))
        shape = TileTensorShape.from_c(so)
        out = np.empty((shape.tile_count(), s), dtype=np.float64)
        c = CCost()
        self._rc(self._f("elementwise")(int(op), ctypes.byref(_sh(sa)), _dp(ta),
                                        ctypes.byref(_sh(sb)), _dp(tb), ctypes.c_int64(s),
                                        ctypes.byref(so), _dp(out), ctypes.byref(c)))
        return TileTensorShape.from_c(so), out, _cost(c)

    def sum(self, shape, tiles, s, dim, variant=-1):
        tiles = np.ascontiguousarray(tiles, dtype=np.float64)
        so = CShape()
        self._rc(self._shape_sum(shape, dim, so))
        res = TileTensorShape.from_c(so)
        out = np.empty((max(res.tile_count(), shape.tile_count()), s), dtype=np.float64)
        c = CCost()
        self._rc(self._f("sum")(ctypes.byref(_sh(shape)), _dp(tiles), ctypes.c_int64(s),
                                int(dim), int(variant), ctypes.byref(so), _dp(out),
                                ctypes.byref(c)))
        res = TileTensorShape.from_c(so)
        return res, out[:res.tile_count()].copy(), _cost(c)

    def mul_sum(self, sa, ta, sb, tb, s, dim, variant=-1):
        sp, prod, c1 = self.elementwise(1, sa, ta, sb, tb, s)
        so, out, c2 = self.sum(sp, prod, s, dim, variant)
        total = CostReport(*(getattr(c1, f) + getattr(c2, f) for f in (
            "additions", "multiplications", "mask_multiplications", "rotations", "bootstraps",
            "power_of_two_rotations")))
        return so, out, total

    def clean_unknowns(self, shape, tiles, s):
        tiles = np.ascontiguousarray(tiles, dtype=np.float64)
        out = np.empty_like(tiles)
        so = CShape()
        c = CCost()
        self._rc(self._f("clean_unknowns")(ctypes.byref(_sh(shape)), _dp(tiles),
                                           ctypes.c_int64(s), ctypes.byref(so), _dp(out),
                                           ctypes.byref(c)))
        return TileTensorShape.from_c(so), out, _cost(c)

    def replicate_dim(self, shape, tiles, s, dim):
        tiles = np.ascontiguousarray(tiles, dtype=np.float64)
        out = np.empty_like(tiles)
        so = CShape()
        c = CCost()
        self._rc(self._f("replicate_dim")(ctypes.byref(_sh(shape)), _dp(tiles),
                                          ctypes.c_int64(s), int(dim), ctypes.byref(so),
                                          _dp(out), ctypes.byref(c)))
        return TileTensorShape.from_c(so), out, _cost(c)

    def rotate(self, tile, offset):
        tile = np.ascontiguousarray(tile, dtype=np.float64)
        out = np.empty_like(tile)
        c = CCost()
        self._rotate(tile, offset, out, c)
        return out, _cost(c)

    def sum_tile_strided(self, tile, n, stride, variant=-1):
        tile = np.ascontiguousarray(tile, dtype=np.float64)
        out = np.empty_like(tile)
        c = CCost()
        self._rc(self._f("sum_tile_strided")(_dp(tile), ctypes.c_int64(tile.size),
                                             ctypes.c_int64(n), ctypes.c_int64(stride),
                                             int(variant), _dp(out), ctypes.byref(c)))
        return out, _cost(c)

    def replicate_tile_dim(self, tile, extents, dim):
        tile = np.ascontiguousarray(tile, dtype=np.float64)
        out = np.empty_like(tile)
        ext = (ctypes.c_int64 * len(extents))(*extents)
        c = CCost()
        self._rc(self._f("replicate_tile_dim")(_dp(tile), ctypes.c_int64(tile.size), ext,
                                               len(extents), int(dim), _dp(out),
                                               ctypes.byref(c)))
        return out, _cost(c)

    def elementwise_result_shape(self, a, b, op):
        so = CShape()
        self._rc(self._shape_ew(a, b, op, so))
        return TileTensorShape.from_c(so)

    def sum_result_shape(self, shape, dim):
        so = CShape()
        self._rc(self._shape_sum(shape, dim, so))
        return TileTensorShape.from_c(so)


class Oracle(_Base):
    """The C restatement oracle/tt_oracle.c."""

    prefix = "or_"

    def __init__(self, path: Path = ORACLE_LIB):
        super().__init__(path)
        L = self.lib
        L.or_max_rel_diff.restype = ctypes.c_double
        L.or_tile_count.restype = ctypes.c_int64
        L.or_tile_slots.restype = ctypes.c_int64

    def _pack(self, dense, shape, s, out):
        self._rc(self.lib.or_pack(_dp(dense), ctypes.byref(_sh(shape)), ctypes.c_int64(s),
                                  _dp(out)))

    def _shape_ew(self, a, b, op, so):
        return self.lib.or_elementwise_result_shape(ctypes.byref(_sh(a)), ctypes.byref(_sh(b)),
                                                    int(op), ctypes.byref(so))

    def _shape_sum(self, shape, dim, so):
        return self.lib.or_sum_result_shape(ctypes.byref(_sh(shape)), int(dim), ctypes.byref(so))

    def _rotate(self, tile, offset, out, c):
        self.lib.or_rotate(_dp(tile), ctypes.c_int64(offset), _dp(out), ctypes.c_int64(tile.size),
                           ctypes.byref(c))

    def fill_uniform(self, count, seed, lo, hi, offset=0):
        out = np.empty(count, dtype=np.float64)
        self.lib.or_fill_uniform(_dp(out), ctypes.c_int64(count), ctypes.c_uint64(seed),
                                 ctypes.c_int64(offset), ctypes.c_double(lo), ctypes.c_double(hi))
        return out

    # dense oracle (dense.hpp:107-198)
    def dense_elementwise(self, op, a, b):
        a = np.ascontiguousarray(a, dtype=np.float64)
        b = np.ascontiguousarray(b, dtype=np.float64)
        r = a.ndim
        ea = (ctypes.c_int64 * r)(*a.shape)
        eb = (ctypes.c_int64 * r)(*b.shape)
        eo = (ctypes.c_int64 * r)()
        out = np.empty([max(x, y) for x, y in zip(a.shape, b.shape)], dtype=np.float64)
        self._rc(self.lib.or_dense_elementwise(int(op), _dp(a), ea, _dp(b), eb, r, _dp(out), eo))
        return out

    def dense_sum(self, a, dim):
        a = np.ascontiguousarray(a, dtype=np.float64)
        r = a.ndim
        ea = (ctypes.c_int64 * r)(*a.shape)
        shape = list(a.shape)
        shape[dim - 1] = 1
        out = np.empty(shape, dtype=np.float64)
        self._rc(self.lib.or_dense_sum(_dp(a), ea, r, int(dim), _dp(out)))
        return out

    def dense_matmul(self, a, b):
        a = np.ascontiguousarray(a, dtype=np.float64)
        b = np.ascontiguousarray(b, dtype=np.float64)
        m, k = a.shape
        k2, n = b.shape
        assert k == k2
        out = np.empty((m, n), dtype=np.float64)
        self.lib.or_dense_matmul(_dp(a), _dp(b), ctypes.c_int64(m), ctypes.c_int64(k),
                                 ctypes.c_int64(n), _dp(out))
        return out

    def max_rel_diff(self, a, b):
        a = np.ascontiguousarray(a, dtype=np.float64).reshape(-1)
        b = np.ascontiguousarray(b, dtype=np.float64).reshape(-1)
        if a.shape != b.shape:
            return float("inf")
        return float(self.lib.or_max_rel_diff(_dp(a), _dp(b), ctypes.c_int64(a.size)))


class Ref(_Base):
    """The reference itself (oracle/_ref/libttref.so)."""

    prefix = "ref_"

    def __init__(self, path: Path = REF_LIB):
        super().__init__(path)
        self.lib.ref_last_error.restype = ctypes.c_char_p

    def _err(self):
        return self.lib.ref_last_error().decode()

    def _pack(self, dense, shape, s, out):
        c = CCost()
        self._rc(self.lib.ref_pack(_dp(dense), ctypes.byref(_sh(shape)), ctypes.c_int64(s),
                                   _dp(out), ctypes.byref(c)))

    def _shape_ew(self, a, b, op, so):
        return self.lib.ref_elementwise_result_shape(ctypes.byref(_sh(a)), ctypes.byref(_sh(b)),
                                                     int(op), ctypes.byref(so))

    def _shape_sum(self, shape, dim, so):
        return self.lib.ref_sum_result_shape(ctypes.byref(_sh(shape)), int(dim), ctypes.byref(so))

    def _rotate(self, tile, offset, out, c):
        self._rc(self.lib.ref_rotate(_dp(tile), ctypes.c_int64(tile.size), ctypes.c_int64(offset),
                                     _dp(out), ctypes.byref(c)))

    def mul_sum(self, sa, ta, sb, tb, s, dim, variant=-1):
        ta = np.ascontiguousarray(ta, dtype=np.float64)
        tb = np.ascontiguousarray(tb, dtype=np.float64)
        prod = self.elementwise_result_shape(sa, sb, 1)
        res = self.sum_result_shape(prod, dim)
        out = np.empty((max(res.tile_count(), prod.tile_count()), s), dtype=np.float64)
        so = CShape()
        c = CCost()
        self._rc(self.lib.ref_mul_sum(ctypes.byref(_sh(sa)), _dp(ta), ctypes.byref(_sh(sb)),
                                      _dp(tb), ctypes.c_int64(s), int(dim), int(variant),
                                      ctypes.byref(so), _dp(out), ctypes.byref(c)))
        res = TileTensorShape.from_c(so)
        return res, out[:res.tile_count()].copy(), _cost(c)

    def nn_run(self, which, spec, seed, batch, tile=(1, 1, 1), slots=1, depth=8):
        """nn_forward (which=0) / cryptonets_infer (which=1) of the reference on
        parse_network(spec, seed): (logits [out, n], cost)."""
        batch = np.ascontiguousarray(batch, dtype=np.float64)
        cap = 1 << 20
        out = np.empty(cap, dtype=np.float64)
        rows = ctypes.c_int64()
        c = CCost()
        t = (ctypes.c_int64 * 3)(*tile)
        self._rc(self.lib.ref_nn_run(int(which), spec.encode(), ctypes.c_uint64(seed), _dp(batch),
                                     ctypes.c_int64(batch.shape[0]), ctypes.c_int64(batch.shape[1]),
                                     t, ctypes.c_int64(slots), ctypes.c_int64(depth), _dp(out),
                                     ctypes.c_int64(cap), ctypes.byref(rows), ctypes.byref(c)))
        r = rows.value
        return out[:r * batch.shape[1]].reshape(r, batch.shape[1]).copy(), _cost(c)

    def nn_params(self, spec, seed):
        """parse_network's seeded weights and biases, flattened in layer order."""
        cap = 1 << 20
        out = np.empty(cap, dtype=np.float64)
        n = ctypes.c_int64()
        self._rc(self.lib.ref_nn_params(spec.encode(), ctypes.c_uint64(seed), _dp(out),
                                        ctypes.c_int64(cap), ctypes.byref(n)))
        return out[:n.value].copy()

    @staticmethod
    def _chain_args(matrices, v):
        mats = [np.ascontiguousarray(m, dtype=np.float64) for m in matrices]
        flat = np.ascontiguousarray(np.concatenate([m.reshape(-1) for m in mats]))
        rows = (ctypes.c_int64 * len(mats))(*[m.shape[0] for m in mats])
        cols = (ctypes.c_int64 * len(mats))(*[m.shape[1] for m in mats])
        v = np.ascontiguousarray(np.asarray(v, dtype=np.float64).reshape(-1))
        return mats, flat, rows, cols, v

    def pipeline(self, matrices, v, tile, s, depth=8):
        """The reference's pipeline (linalg.hpp:213-260): (shape, tiles, cost)."""
        mats, flat, rows, cols, v = self._chain_args(matrices, v)
        cap = 4 * (max(max(m.shape) for m in mats) + v.size) + 8
        out = np.empty((cap, s), dtype=np.float64)
        so = CShape()
        c = CCost()
        self._rc(self.lib.ref_pipeline(_dp(flat), rows, cols, len(mats), _dp(v),
                                       ctypes.c_int64(v.size), ctypes.c_int64(tile[0]),
                                       ctypes.c_int64(tile[1]), ctypes.c_int64(s),
                                       ctypes.c_int64(depth), ctypes.byref(so), _dp(out),
                                       ctypes.byref(c)))
        res = TileTensorShape.from_c(so)
        return res, out[:res.tile_count()].copy(), _cost(c)

    def score_tile_factorizations(self, matrices, v, s, depth=8):
        """[(t1, rotations, total_ops)] in the reference's order (linalg.hpp:279-294)."""
        mats, flat, rows, cols, v = self._chain_args(matrices, v)
        cap = 256
        trip = (ctypes.c_int64 * (3 * cap))()
        n = ctypes.c_int()
        self._rc(self.lib.ref_score_tile_factorizations(
            _dp(flat), rows, cols, len(mats), _dp(v), ctypes.c_int64(v.size), ctypes.c_int64(s),
            ctypes.c_int64(depth), trip, cap, ctypes.byref(n)))
        return [(trip[3 * i], trip[3 * i + 1], trip[3 * i + 2]) for i in range(min(n.value, cap))]

    def linalg(self, which, sa, ta, sb, tb, s):
        ta = np.ascontiguousarray(ta, dtype=np.float64)
        tb = np.ascontiguousarray(tb, dtype=np.float64)
        prod = self.elementwise_result_shape(sa, sb, 1)
        out = np.empty((prod.tile_count(), s), dtype=np.float64)
        so = CShape()
        c = CCost()
        self._rc(self.lib.ref_linalg(int(which), ctypes.byref(_sh(sa)), _dp(ta),
                                     ctypes.byref(_sh(sb)), _dp(tb), ctypes.c_int64(s),
                                     ctypes.byref(so), _dp(out), ctypes.byref(c)))
        res = TileTensorShape.from_c(so)
        return res, out[:res.tile_count()].copy(), _cost(c)

    def parse(self, text):
        so = CShape()
        pos = ctypes.c_int64()
        rc = self.lib.ref_shape_parse(text.encode(), ctypes.byref(so), ctypes.byref(pos))
        return rc, (TileTensorShape.from_c(so) if rc == 0 else None), pos.value

    def format(self, shape):
        buf = ctypes.create_string_buffer(512)
        self._rc(self.lib.ref_shape_format(ctypes.byref(_sh(shape)), buf, 512))
        return buf.value.decode()


def load_oracle():
    return Oracle()


def load_ref():
    """The reference library, or None when it is not built (e.g. on the GPU box)."""
    try:
        return Ref()
    except (FileNotFoundError, OSError):
        return None
