"""Python mirror of the reference tile-tensor API over the B200 C-ABI.

Same names, argument meaning and error behaviour as the reference's
``namespace tiletensor`` (/root/reference/proj/include/tiletensor/*.hpp), so
tests read like the reference's own.  Every operator calls
``libtiletensor_b200.so`` (include/tiletensor_b200.h) through ctypes; slot
arithmetic runs only in the sm_100a kernels.  There is no CPU path: importing
works without a GPU (the shape algebra is host code in the library), but
creating a :class:`Session` raises :class:`NoDeviceError` when no CUDA device
is present, and every op fails loudly if the native library is missing.

Device memory is held in ``torch`` CUDA tensors (plumbing only): a
:class:`TileTensor` owns one ``float64`` tensor of shape ``[tile_count, s]``.
"""
from __future__ import annotations

import ctypes
import enum
from dataclasses import dataclass, field
from pathlib import Path
from typing import Optional, Sequence

import numpy as np

from . import _abi
from ._abi import TT_MAX_RANK, CCost, CShape, lib

# ---- errors (shape.hpp:21-35, backend.hpp:18-21) -------------------------------


class ShapeError(RuntimeError):
    pass


class ShapeParseError(ShapeError):
    def __init__(self, msg: str, position: int):
        super().__init__(msg)
        self._position = position

    def position(self) -> int:
        return self._position


class DepthExhaustedError(RuntimeError):
    pass


class CudaError(RuntimeError):
    pass


class NoDeviceError(RuntimeError):
    pass


def _check(rc: int) -> None:
    if rc == 0:
        return
    msg = lib().tt_last_error().decode()
    if rc == 1:
        raise ShapeError(msg)
    if rc == 2:
        raise ShapeParseError(msg, int(lib().tt_last_error_position()))
    if rc == 3:
        raise DepthExhaustedError(msg)
    if rc == 4:
        raise ValueError(msg)  # std::invalid_argument
    if rc == 5:
        raise IndexError(msg)  # std::out_of_range
    if rc == 7:
        raise CudaError(msg)
    if rc == 8:
        raise NoDeviceError(msg)
    raise RuntimeError(msg)


# ---- shapes (shape.hpp:37-138) ---------------------------------------------------


class OpKind(enum.IntEnum):
    add = 0
    mul = 1


class SumVariant(enum.IntEnum):
    left_to_right = 0
    right_to_left = 1
    power_of_two = 2


@dataclass(frozen=True)
class DimSpec:
    n: int = 1
    d: int = 1
    t: int = 1
    unknown: bool = False
    interleaved: bool = False  # the builder's `~` extension

    def used(self) -> int:
        return self.n * self.d

    def fully_replicated(self) -> bool:
        return self.n == 1 and self.d == self.t


def _ceil_div(a: int, b: int) -> int:
    return (a + b - 1) // b


# shapes decoded from C structs, by struct bytes (shapes are immutable values)
_FROM_C_CACHE: dict = {}


class TileTensorShape:
    """TileTensorShape shape.hpp:72-138 (validated by the native library)."""

    __slots__ = ("_dims", "_relaxed", "_c", "_tiles", "_hash")

    def __init__(self, dims: Sequence[DimSpec], relaxed: bool = False):
        self._dims = tuple(dims)
        self._relaxed = bool(relaxed)
        self._c = None
        self._tiles = None
        self._hash = None
        _check(lib().tt_shape_check(ctypes.byref(self.to_c())))

    # construction helpers
    def to_c(self) -> CShape:
        """The C struct (cached: shapes are immutable and the C ABI takes them const)."""
        if self._c is None:
            self._c = self._make_c()
        return self._c

    def _make_c(self) -> CShape:
        c = CShape()
        c.rank = len(self._dims)
        c.relaxed = 1 if self._relaxed else 0
        if c.rank > TT_MAX_RANK:
            raise ShapeError(f"rank {c.rank} exceeds the supported maximum {TT_MAX_RANK}")
        for i, d in enumerate(self._dims):
            c.dims[i].n, c.dims[i].d, c.dims[i].t = d.n, d.d, d.t
            c.dims[i].unknown = 1 if d.unknown else 0
            c.dims[i].interleaved = 1 if d.interleaved else 0
        return c

    @classmethod
    def from_c(cls, c: CShape) -> "TileTensorShape":
        key = bytes(c)
        obj = _FROM_C_CACHE.get(key)
        if obj is not None:
            return obj
        obj = cls.__new__(cls)
        obj._dims = tuple(
            DimSpec(c.dims[i].n, c.dims[i].d, c.dims[i].t, bool(c.dims[i].unknown),
                    bool(c.dims[i].interleaved)) for i in range(c.rank))
        obj._relaxed = bool(c.relaxed)
        obj._c = None
        obj._tiles = None
        obj._hash = None
        if len(_FROM_C_CACHE) >= 4096:
            _FROM_C_CACHE.clear()
        _FROM_C_CACHE[key] = obj
        return obj

    def rank(self) -> int:
        return len(self._dims)

    def dims(self) -> tuple:
        return self._dims

    def dim(self, i: int) -> DimSpec:
        return self._dims[i]

    def relaxed(self) -> bool:
        return self._relaxed

    def tile_slots(self) -> int:
        p = 1
        for d in self._dims:
            p *= d.t
        return p

    def tensor_extents(self) -> list:
        return [d.n for d in self._dims]

    def external_extents(self) -> list:
        return [_ceil_div(d.used(), d.t) for d in self._dims]

    def tile_count(self) -> int:
        if self._tiles is None:
            p = 1
            for e in self.external_extents():
                p *= e
            self._tiles = p
        return self._tiles

    def used_slots(self) -> int:
        p = 1
        for d in self._dims:
            p *= d.used()
        return p

    def total_slots(self) -> int:
        return self.tile_count() * self.tile_slots()

    def has_unknown(self) -> bool:
        return any(d.unknown for d in self._dims)

    def with_dim(self, i: int, ds: DimSpec) -> "TileTensorShape":
        dims = list(self._dims)
        dims[i] = ds
        return TileTensorShape(dims, self._relaxed)

    def __eq__(self, other) -> bool:
        return (isinstance(other, TileTensorShape) and self._dims == other._dims
                and self._relaxed == other._relaxed)

    def __hash__(self):
        if self._hash is None:
            self._hash = hash((self._dims, self._relaxed))
        return self._hash

    def __repr__(self) -> str:
        return f"TileTensorShape({format_shape(self)}{', relaxed' if self._relaxed else ''})"


def parse_shape(text: str) -> TileTensorShape:  # shape.hpp:250
    c = CShape()
    _check(lib().tt_shape_parse(text.encode(), ctypes.byref(c)))
    return TileTensorShape.from_c(c)


def format_shape(shape: TileTensorShape) -> str:  # shape.hpp:256
    buf = ctypes.create_string_buffer(64 * TT_MAX_RANK + 64)
    _check(lib().tt_shape_format(ctypes.byref(shape.to_c()), buf, len(buf)))
    return buf.value.decode()


def external_shape(shape: TileTensorShape) -> list:  # shape.hpp:280
    return shape.external_extents()


def elementwise_result_shape(a: TileTensorShape, b: TileTensorShape, op) -> TileTensorShape:
    out = CShape()
    _check(lib().tt_shape_elementwise_result(ctypes.byref(a.to_c()), ctypes.byref(b.to_c()),
                                             int(op), ctypes.byref(out)))
    return TileTensorShape.from_c(out)


def sum_result_shape(shape: TileTensorShape, dim: int) -> TileTensorShape:
    out = CShape()
    _check(lib().tt_shape_sum_result(ctypes.byref(shape.to_c()), int(dim), ctypes.byref(out)))
    return TileTensorShape.from_c(out)


def logical_indices(shape: TileTensorShape, tile_index: Sequence[int], h: int) -> list:
    if len(tile_index) != shape.rank():
        raise ShapeError("tile index rank mismatch")
    ti = (ctypes.c_int64 * TT_MAX_RANK)(*tile_index)
    j = (ctypes.c_int64 * TT_MAX_RANK)()
    _check(lib().tt_logical_indices(ctypes.byref(shape.to_c()), ti, int(h), j))
    return [j[i] for i in range(shape.rank())]


def slot_of(shape: TileTensorShape, j: Sequence[int]):
    if len(j) != shape.rank():
        raise ShapeError("logical index rank mismatch")
    jj = (ctypes.c_int64 * TT_MAX_RANK)(*j)
    l = (ctypes.c_int64 * TT_MAX_RANK)()
    h = ctypes.c_int64()
    _check(lib().tt_slot_of(ctypes.byref(shape.to_c()), jj, l, ctypes.byref(h)))
    return [l[i] for i in range(shape.rank())], h.value


def rotations_left_to_right(n: int) -> int:
    return int(lib().tt_rotations_left_to_right(n))


def rotations_right_to_left(n: int) -> int:
    return int(lib().tt_rotations_right_to_left(n))


# ---- cost report (backend.hpp:28-63) ---------------------------------------------


@dataclass
class CostReport:
    additions: int = 0
    multiplications: int = 0
    mask_multiplications: int = 0
    rotations: int = 0
    bootstraps: int = 0
    power_of_two_rotations: int = 0

    def to_text(self, extended: bool = False) -> str:
        out = (f"additions={self.additions}\nmultiplications={self.multiplications}\n"
               f"mask_multiplications={self.mask_multiplications}\nrotations={self.rotations}\n"
               f"bootstraps={self.bootstraps}\n")
        if extended:
            out += f"power_of_two_rotations={self.power_of_two_rotations}\n"
        return out

    def since(self, base: "CostReport") -> "CostReport":
        return CostReport(*(getattr(self, f) - getattr(base, f) for f in _COST_FIELDS))

    def total_ops(self) -> int:
        return (self.additions + self.multiplications + self.mask_multiplications +
                self.rotations + self.bootstraps)


_COST_FIELDS = ("additions", "multiplications", "mask_multiplications", "rotations", "bootstraps",
                "power_of_two_rotations")

# ---- session ------------------------------------------------------------------------


_RAW_STREAM = None  # torch._C._cuda_getCurrentRawStream, bound on first Session


def _current_raw_stream(device: int) -> int:
    """cudaStream_t of torch's current stream on `device` (the raw accessor
    when this torch has it: ~10x cheaper than building a Stream object)."""
    torch = _torch()
    raw = getattr(torch._C, "_cuda_getCurrentRawStream", None)
    if raw is not None:
        return int(raw(device))
    return torch.cuda.current_stream(device).cuda_stream


def _torch():
    import torch  # plumbing: device memory + streams
    return torch


class Session:
    """Session backend.hpp:83-204, bound to one CUDA device.

    Ops run on torch's current stream of that device at call time, so they are
    ordered with the torch allocations that hold their operands.
    """

    def __init__(self, slot_count: int, max_chain_index: int, device: int = 0):
        self._ptr = ctypes.c_void_p()
        _check(lib().tt_session_create(int(slot_count), int(max_chain_index), int(device),
                                       ctypes.byref(self._ptr)))
        self._slots = int(slot_count)
        self._depth = int(max_chain_index)
        self._device = int(device)
        self._stream = None  # stream last bound to the native session
        self._tdev = _torch().device("cuda", self._device)
        global _RAW_STREAM
        if _RAW_STREAM is None:
            _RAW_STREAM = getattr(_torch()._C, "_cuda_getCurrentRawStream", None)

    def __del__(self):
        p = getattr(self, "_ptr", None)
        if p and p.value:
            try:
                lib().tt_session_destroy(p)
            except Exception:
                pass
            self._ptr = None

    def _h(self) -> int:
        """The session handle as an int (fast path), bound to torch's current stream."""
        stream = _RAW_STREAM(self._device) if _RAW_STREAM is not None else _current_raw_stream(self._device)
        if stream != self._stream:
            _check(lib().tt_session_set_stream(self._ptr, ctypes.c_void_p(stream)))
            self._stream = stream
        return self._ptr.value

    @property
    def handle(self):
        stream = _current_raw_stream(self._device)
        if stream != self._stream:  # re-bind only when torch's current stream changed
            _check(lib().tt_session_set_stream(self._ptr, ctypes.c_void_p(stream)))
            self._stream = stream
        return self._ptr

    def slot_count(self) -> int:
        return self._slots

    def max_chain_index(self) -> int:
        return self._depth

    def device(self):
        return self._tdev

    def cost_report(self) -> CostReport:
        c = CCost()
        lib().tt_session_cost(self._ptr, ctypes.byref(c))
        return CostReport(*(getattr(c, f) for f in _COST_FIELDS))

    def reset_counters(self) -> None:
        lib().tt_session_reset_counters(self._ptr)

    def launches(self) -> int:
        return int(lib().tt_session_launches(self._ptr))

    def synchronize(self) -> None:
        _torch().cuda.synchronize(self._device)

    def count_bootstraps(self, n: int) -> None:
        lib().tt_session_count_bootstraps(self._ptr, int(n))

    # allocation helper
    def empty_tiles(self, count: int):
        torch = _torch()
        return torch.empty((int(count), self._slots), dtype=torch.float64, device=self._tdev)


def _ptr(t) -> ctypes.c_void_p:
    return ctypes.c_void_p(t.data_ptr()) if t is not None else ctypes.c_void_p(0)


def _as_device(x, session: Session):
    torch = _torch()
    if isinstance(x, torch.Tensor):
        t = x.to(device=session.device(), dtype=torch.float64)
    else:
        t = torch.from_numpy(np.ascontiguousarray(np.asarray(x, dtype=np.float64))).to(
            session.device())
    return t.contiguous()


# ---- tile tensors (tile_tensor.hpp:130-165) -------------------------------------------


class _Block:
    """A result block from the session's tile cache (tt_tiles_alloc): released
    back to the cache (stream-ordered reuse, tt_tiles_release) when the last
    reference -- the TileTensor, or a torch view made by data() -- goes away."""
    __slots__ = ("ptr", "session", "__weakref__")

    def __init__(self, ptr: int, session: "Session"):
        self.ptr = ptr
        self.session = session

    def __del__(self):
        try:
            h = self.session._ptr
            if h and h.value:
                _fastmod().release(h.value, self.ptr)
        except Exception:
            pass


class _CudaArray:
    """__cuda_array_interface__ view of a _Block for torch.as_tensor (torch keeps
    a reference to this object, hence to the block, for the tensor's life)."""

    def __init__(self, block: _Block, shape):
        self._block = block
        self.__cuda_array_interface__ = {"shape": tuple(shape), "typestr": "<f8",
                                         "data": (block.ptr, False), "version": 3,
                                         "strides": None, "stream": None}


class TileTensor:
    """Shape + one device array [tile_count, s] + Session + chain index.

    The array is a torch tensor, or (fast-path operator results) a block of
    the session's tile cache that data() exposes as a torch tensor on demand."""

    __slots__ = ("_shape", "_t", "_block", "_p", "_session", "_chain")

    def __init__(self, shape: TileTensorShape, tiles, session: Session, chain: Optional[int] = None):
        torch = _torch()
        if not isinstance(tiles, torch.Tensor) or tiles.device.type != "cuda":
            tiles = _as_device(tiles, session)
        tiles = tiles.reshape(-1, session.slot_count()) if tiles.numel() else tiles.reshape(
            0, session.slot_count())
        if tiles.shape[0] != shape.tile_count():
            raise ShapeError("tile count does not match external shape")
        self._shape = shape
        self._t = tiles.contiguous()
        self._block = None
        self._p = self._t.data_ptr()
        self._session = session
        self._chain = session.max_chain_index() if chain is None else int(chain)

    @classmethod
    def _wrap(cls, shape: TileTensorShape, tiles, session: Session, chain: int) -> "TileTensor":
        """An operator result: `tiles` is a fresh contiguous [tile_count, s]
        device array from Session.empty_tiles (no validation needed)."""
        obj = cls.__new__(cls)
        obj._shape = shape
        obj._t = tiles
        obj._block = None
        obj._p = tiles.data_ptr()
        obj._session = session
        obj._chain = int(chain)
        return obj

    @classmethod
    def _wrap_block(cls, shape: TileTensorShape, ptr: int, session: Session, chain: int) -> "TileTensor":
        obj = cls.__new__(cls)
        obj._shape = shape
        obj._t = None
        obj._block = _Block(ptr, session)
        obj._p = ptr
        obj._session = session
        obj._chain = chain
        return obj

    def shape(self) -> TileTensorShape:
        return self._shape

    def session(self) -> Session:
        return self._session

    def tile_count(self) -> int:
        return self._shape.tile_count()

    def data(self):
        """The device array [tile_count, s] (torch float64)."""
        if self._t is None:
            n = self._shape.tile_count()
            self._t = _torch().as_tensor(_CudaArray(self._block, (n, self._session._slots)),
                                         device=self._session._tdev)
        return self._t

    def tiles(self) -> np.ndarray:
        """Host copy of every tile, [tile_count, s] (TileTensor::tiles)."""
        return self.data().detach().cpu().numpy()

    def tile_at(self, flat: int) -> np.ndarray:
        return self.data()[flat].detach().cpu().numpy()

    def chain_index(self) -> int:
        return self._chain


def _dptr(t: TileTensor) -> ctypes.c_void_p:
    """Device address of a tile tensor's array (no torch view needed)."""
    return ctypes.c_void_p(t._p)


class _Out:
    """An operator's result storage: a block of the session's tile cache
    (tt_tiles_alloc: the same block the next call of that shape reuses), or a
    torch tensor while the stream is being captured into a CUDA graph.  A block
    not handed to a TileTensor (the call raised) is released on collection."""
    __slots__ = ("s", "n", "ptr", "t", "owned")

    def __init__(self, s: Session, n: int):
        self.s, self.n = s, max(int(n), 1)
        p = ctypes.c_void_p()
        _check(lib().tt_tiles_alloc(s.handle, self.n * s._slots * 8, ctypes.byref(p)))
        if p.value:
            self.ptr, self.t, self.owned = p.value, None, True
        else:
            self.t = s.empty_tiles(self.n)
            self.ptr, self.owned = self.t.data_ptr(), False

    def c(self) -> ctypes.c_void_p:
        return ctypes.c_void_p(self.ptr)

    def wrap(self, shape: TileTensorShape, chain: int) -> TileTensor:
        n = shape.tile_count()
        if n > self.n:  # host-side sizing and the C-ABI disagree: never hand out a short array
            raise ShapeError(f"result has {n} tiles, {self.n} allocated")
        if self.t is not None:
            return TileTensor._wrap(shape, self.t if n == self.t.shape[0] else self.t[:n], self.s, chain)
        self.owned = False
        return TileTensor._wrap_block(shape, self.ptr, self.s, int(chain))

    def __del__(self):
        if getattr(self, "owned", False):
            try:
                _fastmod().release(self.s._ptr.value, self.ptr)
            except Exception:
                pass


def with_leading_unit_dim(t: TileTensor) -> TileTensor:  # tile_tensor.hpp:158-165
    dims = [DimSpec()] + list(t.shape().dims())
    return TileTensor(TileTensorShape(dims, t.shape().relaxed()), t.data(), t.session(),
                      t.chain_index())


def _same_session(a: TileTensor, b: TileTensor) -> Session:
    if a.session() is not b.session():
        raise ValueError("operands belong to different sessions")  # tile_tensor.hpp:245-246
    return a.session()


def pack(tensor, shape: TileTensorShape, session: Session) -> TileTensor:
    """pack tile_tensor.hpp:167-220; `tensor` is a numpy array or torch tensor
    whose element count equals prod(n_i) (reshaped like the reference)."""
    arr = tensor
    want = 1
    for e in shape.tensor_extents():
        want *= e
    size = int(np.prod(arr.shape)) if hasattr(arr, "shape") else len(arr)
    if shape.has_unknown():
        raise ShapeError("pack target shape may not contain '?': " + format_shape(shape))
    if size != want:
        raise ShapeError(f"tensor of {size} values cannot pack into {format_shape(shape)}")
    torch = _torch()
    if (isinstance(arr, torch.Tensor) and arr.device.type == "cpu" and arr.is_pinned()
            and arr.dtype == torch.float64 and arr.is_contiguous() and want * 8 >= _STAGED_MIN):
        staged = _pack_staged(arr, shape, session)
        if staged is not None:
            return staged
    dense = _as_device(arr, session).reshape(-1)
    out = session.empty_tiles(shape.tile_count())
    _check(lib().tt_pack(session.handle, _ptr(dense), ctypes.byref(shape.to_c()), _ptr(out)))
    return TileTensor(shape, out, session)


_STAGED_MIN = 512 << 20   # pinned inputs from this size on are copied and packed in slabs
_STAGED_SLAB = 512 << 20  # bytes per slab (two device staging buffers)


def _pack_staged(host, shape: TileTensorShape, session: Session):
    """pack() of a large pinned host tensor with the host-to-device copy
    overlapped: the dense rows go over PCIe in slabs of whole external rows of
    dim 1 (a copy stream, two device staging buffers), and each slab is packed
    into its contiguous range of output tiles on the session stream while the
    next slab is in flight.  The tiles are those of one pack() of the whole
    tensor (the slab's rows are a pack of the sub-shape with dim 1 cut to them).
    None when the shape cannot be cut that way (the caller packs in one piece).
    Returns after the last copy has been issued and completed (the host tensor
    may be released then); the packs stay queued on the stream."""
    torch = _torch()
    d0 = shape.dim(0)
    if shape.relaxed() or d0.d != 1 or d0.interleaved or d0.n == 1 or shape.rank() < 2:
        return None
    row_elems = 1
    for e in shape.tensor_extents()[1:]:
        row_elems *= e
    rows_per_tile = d0.t
    tile_rows = max(1, _STAGED_SLAB // (row_elems * 8 * rows_per_tile))  # external rows per slab
    slab_rows = tile_rows * rows_per_tile
    if slab_rows >= d0.n:
        return None
    tiles_per_row = shape.tile_count() // shape.external_extents()[0]
    s = session.slot_count()
    out = session.empty_tiles(shape.tile_count())
    flat = host.reshape(-1)
    dev = session.device()
    main = torch.cuda.current_stream(dev)
    copy = torch.cuda.Stream(device=dev)
    bufs = [torch.empty(slab_rows * row_elems, dtype=torch.float64, device=dev) for _ in range(2)]
    freed = [None, None]
    rest = [DimSpec(d.n, d.d, d.t, d.unknown, d.interleaved) for d in shape.dims()[1:]]
    r0, k = 0, 0
    while r0 < d0.n:
        r1 = min(d0.n, r0 + slab_rows)
        buf = bufs[k % 2]
        n = (r1 - r0) * row_elems
        with torch.cuda.stream(copy):
            if freed[k % 2] is not None:
                copy.wait_event(freed[k % 2])       # its previous slab has been packed
            buf[:n].copy_(flat[r0 * row_elems:r1 * row_elems], non_blocking=True)
            landed = torch.cuda.Event()
            landed.record(copy)
        main.wait_event(landed)
        sub = TileTensorShape([DimSpec(r1 - r0, 1, d0.t)] + rest)
        dst = out[(r0 // d0.t) * tiles_per_row:]
        _check(lib().tt_pack(session.handle, _ptr(buf), ctypes.byref(sub.to_c()), _ptr(dst)))
        freed[k % 2] = torch.cuda.Event()
        freed[k % 2].record(main)
        r0, k = r1, k + 1
    copy.synchronize()
    for b in bufs:
        b.record_stream(main)  # the staging buffers outlive the queued packs
    return TileTensor(shape, out, session)


def unpack_device(t: TileTensor):
    """unpack onto the device (torch tensor of the shape's n_i)."""
    torch = _torch()
    s = t.session()
    ext = t.shape().tensor_extents()
    out = torch.empty(ext, dtype=torch.float64, device=s.device())
    _check(lib().tt_unpack(s.handle, ctypes.byref(t.shape().to_c()), _dptr(t), _ptr(out)))
    return out


def unpack(t: TileTensor) -> np.ndarray:
    """unpack tile_tensor.hpp:222-242 -> host numpy array.  The dense result is
    copied into page-locked host memory (torch's caching host allocator): a
    device-to-host copy into fresh pageable memory runs at ~2 GB/s (page
    faults), into pinned memory at PCIe rate (config 5's 32 MiB dim-3 sum:
    15 ms -> 0.6 ms)."""
    torch = _torch()
    dev = unpack_device(t)
    try:
        host = torch.empty(dev.shape, dtype=dev.dtype, pin_memory=True)
    except RuntimeError:  # the host cannot pin: pageable copy
        return dev.cpu().numpy()
    host.copy_(dev)
    return host.numpy()


# result tile counts by (op, operand shapes, dim): sizing an output costs a
# shape-rule evaluation through the C-ABI, which dominates small ops' host time
def fold_shape(a: TileTensorShape, b: Optional[TileTensorShape], dim: int) -> TileTensorShape:
    """Shape of tt_mul_fold's accumulated tiles: the product (a alone when b
    is None) with `dim` reduced to one external tile."""
    out = CShape()
    _check(lib().tt_fold_shape(ctypes.byref(a.to_c()), ctypes.byref(b.to_c()) if b else None,
                               int(dim), ctypes.byref(out)))
    return TileTensorShape.from_c(out)


def mul_fold(a: TileTensor, b: Optional[TileTensor], dim: int, out_range=None, init=None):
    """Partial left fold of tt_sum(tt_mul(a, b), dim) over output tiles
    out_range = (begin, end) (default: all), continuing from `init` (device
    tiles [end - begin, s]) when given -- the building block of exact
    cross-GPU chains (sharding.chain_mul_sum).  Returns (tiles, chain)."""
    s = a.session() if b is None else _same_session(a, b)
    fs = fold_shape(a.shape(), b.shape() if b is not None else None, dim)
    n_out = fs.tile_count()
    begin, end = (0, n_out) if out_range is None else (int(out_range[0]), int(out_range[1]))
    acc = s.empty_tiles(max(end - begin, 0))
    chain = ctypes.c_int64()
    if init is not None and tuple(init.shape) != (end - begin, s.slot_count()):
        raise ValueError("init must hold one tile per output tile of the range")
    _check(lib().tt_mul_fold(s.handle, ctypes.byref(a.shape().to_c()), _dptr(a),
                             a.chain_index(),
                             ctypes.byref(b.shape().to_c()) if b is not None else None,
                             _dptr(b) if b is not None else ctypes.c_void_p(0),
                             b.chain_index() if b is not None else 0, int(dim), begin, end,
                             _ptr(init), _ptr(acc), ctypes.byref(chain)))
    return acc, chain.value


_RESULT_TILES: dict = {}


def _result_tiles(key, compute) -> int:
    n = _RESULT_TILES.get(key)
    if n is None:
        n = compute()
        if len(_RESULT_TILES) >= 4096:
            _RESULT_TILES.clear()
        _RESULT_TILES[key] = n
    return n


# ---- small-op fast path -------------------------------------------------------------
# An operator's result shape, tile count and C structs depend only on its
# operand shapes and arguments, so after the first call with a given key they
# are reused: the repeat call is one torch allocation and ONE C-ABI call (which
# still validates everything -- depth, slots -- before launching) with no
# result-shape round trip.  The C side accepts a null out_shape / out_chain.

class _Call:
    __slots__ = ("nbytes", "shape", "ca", "cb", "v", "keep")

    def __init__(self, nbytes, shape, ca, cb, v, keep):
        self.nbytes, self.shape, self.ca, self.cb, self.v, self.keep = nbytes, shape, ca, cb, v, keep


_FAST: dict = {}


def _remember(key, shape: TileTensorShape, ca, cb, v, slots: int) -> None:
    """ca / cb: the operands' cached tt_shape structs (immutable, owned by their
    TileTensorShape, kept alive here); passed to the C-ABI by address."""
    if len(_FAST) >= 4096:
        _FAST.clear()
    nbytes = max(1, shape.tile_count()) * slots * 8
    _FAST[key] = _Call(nbytes, shape, ctypes.addressof(ca),
                       ctypes.addressof(cb) if cb is not None else 0, -1 if v is None else v, (ca, cb))


def _fastmod():
    """The CPython fast-call module (csrc/tt_pyfast.c) over the same C-ABI."""
    global _FASTMOD
    if _FASTMOD is None:
        lib()
        from . import _ttfast
        _FASTMOD = _ttfast
    return _FASTMOD


_FASTMOD = None


_F64 = None


def _empty(s: "Session", n: int):
    global _F64
    torch = _torch()
    if _F64 is None:
        _F64 = torch.float64
    return torch.empty((n, s._slots), dtype=_F64, device=s._tdev)


def tt_elementwise(a: TileTensor, b: TileTensor, op) -> TileTensor:
    s = a._session
    if b._session is s:
        e = _FAST.get(("ew", op, a._shape, b._shape, s._slots))
        if e is not None:
            p = _fastmod().elementwise_new(s._h(), int(op), e.ca, a._p, a._chain, e.cb, b._p,
                                           b._chain, e.nbytes)
            if p < 0:
                _check(-p)
            if p:
                chain = min(a._chain, b._chain) - (1 if int(op) == int(OpKind.mul) else 0)
                return TileTensor._wrap_block(e.shape, p, s, chain)
    r = _tt_elementwise(a, b, op)
    _remember(("ew", op, a._shape, b._shape, s._slots), r._shape, a._shape.to_c(), b._shape.to_c(),
              None, s._slots)
    return r


def _tt_elementwise(a: TileTensor, b: TileTensor, op) -> TileTensor:
    s = _same_session(a, b)
    so = CShape()
    chain = ctypes.c_int64()
    n_out = _result_tiles(("ew", int(op), a.shape(), b.shape()),
                          lambda: elementwise_result_shape(a.shape(), b.shape(), op).tile_count())
    out = _Out(s, n_out)
    _check(lib().tt_elementwise(s.handle, int(op), ctypes.byref(a.shape().to_c()), _dptr(a),
                                a.chain_index(), ctypes.byref(b.shape().to_c()), _dptr(b),
                                b.chain_index(), ctypes.byref(so), out.c(), ctypes.byref(chain)))
    return out.wrap(TileTensorShape.from_c(so), chain.value)


def tt_add(a: TileTensor, b: TileTensor) -> TileTensor:
    return tt_elementwise(a, b, OpKind.add)


def tt_mul(a: TileTensor, b: TileTensor) -> TileTensor:
    return tt_elementwise(a, b, OpKind.mul)


def _variant(v) -> int:
    return -1 if v is None else int(v)


def tt_sum(t: TileTensor, dim: int, variant: Optional[SumVariant] = None) -> TileTensor:
    """tt_sum tile_tensor.hpp:286-347."""
    key = ("sum", t._shape, dim, variant, t._session._slots)
    e = _FAST.get(key)
    if e is not None:
        s = t._session
        p = _fastmod().sum_new(s._h(), e.ca, t._p, dim, e.v, e.nbytes)
        if p < 0:
            _check(-p)
        if p:
            return TileTensor._wrap_block(e.shape, p, s, t._chain)
    r = _tt_sum(t, dim, variant)
    _remember(key, r._shape, t._shape.to_c(), None, _variant(variant), t._session._slots)
    return r


def _tt_sum(t: TileTensor, dim: int, variant: Optional[SumVariant] = None) -> TileTensor:
    s = t.session()
    n_out = _result_tiles(("sum", t.shape(), int(dim)),
                          lambda: sum_result_shape(t.shape(), dim).tile_count())
    out = _Out(s, n_out)
    so = CShape()
    _check(lib().tt_sum(s.handle, ctypes.byref(t.shape().to_c()), _dptr(t), int(dim),
                        _variant(variant), ctypes.byref(so), out.c()))
    return out.wrap(TileTensorShape.from_c(so), t.chain_index())


def tt_mul_sum(a: TileTensor, b: TileTensor, dim: int,
               variant: Optional[SumVariant] = None) -> TileTensor:
    """tt_sum(tt_mul(a, b), dim) fused: one pass, product never stored."""
    s = a._session
    if b._session is s:
        e = _FAST.get(("mulsum", a._shape, b._shape, dim, variant, s._slots))
        if e is not None:
            p = _fastmod().mul_sum_new(s._h(), e.ca, a._p, a._chain, e.cb, b._p, b._chain, dim, e.v,
                                       e.nbytes)
            if p < 0:
                _check(-p)
            if p:
                return TileTensor._wrap_block(e.shape, p, s, min(a._chain, b._chain) - 1)
    r = _tt_mul_sum(a, b, dim, variant)
    _remember(("mulsum", a._shape, b._shape, dim, variant, s._slots), r._shape, a._shape.to_c(),
              b._shape.to_c(), _variant(variant), s._slots)
    return r


def _tt_mul_sum(a: TileTensor, b: TileTensor, dim: int,
                variant: Optional[SumVariant] = None) -> TileTensor:
    s = _same_session(a, b)
    n_out = _result_tiles(("mulsum", a.shape(), b.shape(), int(dim)), lambda: sum_result_shape(
        elementwise_result_shape(a.shape(), b.shape(), OpKind.mul), dim).tile_count())
    out = _Out(s, n_out)
    so = CShape()
    chain = ctypes.c_int64()
    _check(lib().tt_mul_sum(s.handle, ctypes.byref(a.shape().to_c()), _dptr(a),
                            a.chain_index(), ctypes.byref(b.shape().to_c()), _dptr(b),
                            b.chain_index(), int(dim), _variant(variant), ctypes.byref(so),
                            out.c(), ctypes.byref(chain)))
    return out.wrap(TileTensorShape.from_c(so), chain.value)


def tt_mul_sum_clean(a: TileTensor, b: TileTensor, dim: int,
                     variant: Optional[SumVariant] = None) -> TileTensor:
    """clean_unknowns(tt_sum(tt_mul(a, b), dim)) with the mask applied in the
    reduction's last pass (pipeline()'s odd -> even seam, linalg.hpp:213-260).
    Shapes, chain index, counters and errors equal the two-call composition."""
    s = _same_session(a, b)
    n_out = _result_tiles(("mulsum", a.shape(), b.shape(), int(dim)), lambda: sum_result_shape(
        elementwise_result_shape(a.shape(), b.shape(), OpKind.mul), dim).tile_count())
    out = _Out(s, n_out)
    so = CShape()
    chain = ctypes.c_int64()
    _check(lib().tt_mul_sum_clean(s.handle, ctypes.byref(a.shape().to_c()), _dptr(a),
                                  a.chain_index(), ctypes.byref(b.shape().to_c()), _dptr(b),
                                  b.chain_index(), int(dim), _variant(variant), ctypes.byref(so),
                                  out.c(), ctypes.byref(chain)))
    return out.wrap(TileTensorShape.from_c(so), chain.value)


def tt_mul_sum_affine(a: TileTensor, b: TileTensor, dim: int, c: Optional[TileTensor] = None,
                      square: bool = False, variant: Optional[SumVariant] = None) -> TileTensor:
    """One fully connected stage of cryptonets_infer's tiled branch (nn.hpp:468-490):
    tt_sum(tt_mul(a, b), dim), then tt_add(., c) when c is given, then tt_mul(., .) when
    square -- the tail fused into the reduction's tree pass.  Shapes, chain index,
    counters and errors equal the three-call composition."""
    s = _same_session(a, b)
    if c is not None:
        _same_session(a, c)

    def count():
        r = sum_result_shape(elementwise_result_shape(a.shape(), b.shape(), OpKind.mul), dim)
        if c is not None:
            r = elementwise_result_shape(r, c.shape(), OpKind.add)
        return r.tile_count()
    n_out = _result_tiles(("mulsum_affine", a.shape(), b.shape(), int(dim),
                           None if c is None else c.shape()), count)
    out = _Out(s, n_out)
    so = CShape()
    chain = ctypes.c_int64()
    _check(lib().tt_mul_sum_affine(
        s.handle, ctypes.byref(a.shape().to_c()), _dptr(a), a.chain_index(),
        ctypes.byref(b.shape().to_c()), _dptr(b), b.chain_index(), int(dim), _variant(variant),
        None if c is None else ctypes.byref(c.shape().to_c()), None if c is None else _dptr(c),
        0 if c is None else c.chain_index(), 1 if square else 0, ctypes.byref(so), out.c(),
        ctypes.byref(chain)))
    return out.wrap(TileTensorShape.from_c(so), chain.value)


_PRODUCT_TILES: dict = {}


def _product(which: int, a: TileTensor, b: TileTensor, variant) -> TileTensor:
    s = a._session
    if b._session is s:
        e = _FAST.get(("prod", which, a._shape, b._shape, variant, s._slots))
        if e is not None:
            p = _fastmod().product_new(s._h(), which, e.ca, a._p, a._chain, e.cb, b._p, b._chain,
                                       e.v, e.nbytes)
            if p < 0:
                _check(-p)
            if p:
                return TileTensor._wrap_block(e.shape, p, s, min(a._chain, b._chain) - 1)
    r = _product_slow(which, a, b, variant)
    _remember(("prod", which, a._shape, b._shape, variant, s._slots), r._shape, a._shape.to_c(),
              b._shape.to_c(), _variant(variant), s._slots)
    return r


def _product_slow(which: int, a: TileTensor, b: TileTensor, variant) -> TileTensor:
    s = _same_session(a, b)
    so = CShape()
    chain = ctypes.c_int64()
    # allocate from the worst case (the product's summed shape) after validation
    key = (which, a.shape(), b.shape())
    n_out = _PRODUCT_TILES.get(key)
    if n_out is None:
        try:
            prod = elementwise_result_shape(a.shape(), b.shape(), OpKind.mul)
            dim = 2 if which in (0, 2) else 1
            n_out = sum_result_shape(prod, dim).tile_count()
        except ShapeError:
            n_out = 0
        if len(_PRODUCT_TILES) >= 4096:
            _PRODUCT_TILES.clear()
        _PRODUCT_TILES[key] = n_out
    out = _Out(s, max(n_out, 1))
    _check(lib().tt_linalg_product(s.handle, which, ctypes.byref(a.shape().to_c()),
                                   _dptr(a), a.chain_index(),
                                   ctypes.byref(b.shape().to_c()), _dptr(b),
                                   b.chain_index(), _variant(variant), ctypes.byref(so),
                                   out.c(), ctypes.byref(chain)))
    return out.wrap(TileTensorShape.from_c(so), chain.value)


def matvec_a(m: TileTensor, v: TileTensor, variant=None) -> TileTensor:  # linalg.hpp:41
    return _product(0, m, v, variant)


def matvec_b(m_transposed: TileTensor, v: TileTensor, variant=None) -> TileTensor:  # :49
    return _product(1, m_transposed, v, variant)


def matmul_a(m1: TileTensor, m2: TileTensor, variant=None) -> TileTensor:  # :57
    return _product(2, m1, m2, variant)


def matmul_b(m1_transposed: TileTensor, m2: TileTensor, variant=None) -> TileTensor:  # :66
    return _product(3, m1_transposed, m2, variant)


_PRODUCTS = {"matvec_a": 0, "matvec_b": 1, "matmul_a": 2, "matmul_b": 3}


def linalg_chain(first: str, a: TileTensor, b: TileTensor, second: str, x: TileTensor,
                 first_is_right: bool = True, variant=None):
    """Two consecutive products in ONE launch (tt_linalg_chain2):
    r1 = first(a, b); r2 = second(x, r1) (first_is_right) or second(r1, x).
    E.g. config 3's zero-repack chain matmul_a(A, matmul_b(Bt, C)) is
    linalg_chain("matmul_b", Bt, C, "matmul_a", A) -- the reference's own
    two-call chain (tests/test_linalg.cpp:157-178).  Returns (r1, r2), bit for
    bit, counter for counter and error for error the two calls' results; the
    second product's units start on a slot chunk as soon as the first
    product's trees covering it are done (no kernel boundary between them)."""
    w1, w2 = _PRODUCTS[first], _PRODUCTS[second]
    s = _same_session(a, b)
    _same_session(a, x)
    d1 = 2 if w1 in (0, 2) else 1
    d2 = 2 if w2 in (0, 2) else 1
    try:
        s1 = sum_result_shape(elementwise_result_shape(a.shape(), b.shape(), OpKind.mul), d1)
        l2, r2s = (x.shape(), s1) if first_is_right else (s1, x.shape())
        n2 = sum_result_shape(elementwise_result_shape(l2, r2s, OpKind.mul), d2).tile_count()
        n1 = s1.tile_count()
    except ShapeError:  # let the C-ABI raise the reference's error for the calls
        n1 = n2 = 0
    out1, out2 = _Out(s, n1), _Out(s, n2)
    so1, so2 = CShape(), CShape()
    c1, c2 = ctypes.c_int64(), ctypes.c_int64()
    _check(lib().tt_linalg_chain2(s.handle, w1, ctypes.byref(a.shape().to_c()), _dptr(a),
                                  a.chain_index(), ctypes.byref(b.shape().to_c()), _dptr(b),
                                  b.chain_index(), w2, ctypes.byref(x.shape().to_c()), _dptr(x),
                                  x.chain_index(), 1 if first_is_right else 0, _variant(variant),
                                  ctypes.byref(so1), out1.c(), ctypes.byref(c1), ctypes.byref(so2),
                                  out2.c(), ctypes.byref(c2)))
    return (out1.wrap(TileTensorShape.from_c(so1), c1.value),
            out2.wrap(TileTensorShape.from_c(so2), c2.value))


def clean_unknowns(t: TileTensor) -> TileTensor:  # tile_tensor.hpp:352-386
    s = t.session()
    out = s.empty_tiles(t.tile_count())
    so = CShape()
    chain = ctypes.c_int64()
    _check(lib().tt_clean_unknowns(s.handle, ctypes.byref(t.shape().to_c()), _dptr(t),
                                   t.chain_index(), ctypes.byref(so), _ptr(out),
                                   ctypes.byref(chain)))
    return TileTensor._wrap(TileTensorShape.from_c(so), out, s, chain.value)


def replicate_dim(t: TileTensor, dim: int) -> TileTensor:  # tile_tensor.hpp:391-420
    s = t.session()
    out = s.empty_tiles(t.tile_count())
    so = CShape()
    _check(lib().tt_replicate_dim(s.handle, ctypes.byref(t.shape().to_c()), _dptr(t),
                                  int(dim), ctypes.byref(so), _ptr(out)))
    return TileTensor._wrap(TileTensorShape.from_c(so), out, s, t.chain_index())


# ---- tile-level primitives over [n, s] device arrays (backend.hpp / rotate_sum.hpp) ----


def _tiles_arg(session: Session, tiles):
    t = _as_device(tiles, session)
    return t.reshape(-1, session.slot_count())


def tiles_rotate(session: Session, tiles, offset: int):
    """Session::rotate backend.hpp:152-163 on every row of `tiles`."""
    src = _tiles_arg(session, tiles)
    out = session.empty_tiles(src.shape[0])
    _check(lib().tt_tiles_rotate(session.handle, _ptr(src), int(offset), _ptr(out), src.shape[0]))
    return out


def tiles_binary(session: Session, op, a, b):
    """Session::add / Session::mul backend.hpp:117-136 row by row."""
    ta, tb = _tiles_arg(session, a), _tiles_arg(session, b)
    out = session.empty_tiles(ta.shape[0])
    _check(lib().tt_tiles_binary(session.handle, int(op), _ptr(ta), _ptr(tb), _ptr(out),
                                 ta.shape[0], None, None, None))
    return out


def tiles_mask_mul(session: Session, a, mask):
    """Session::mask_mul backend.hpp:138-148 (one mask row per tile)."""
    ta, tm = _tiles_arg(session, a), _tiles_arg(session, mask)
    if tm.shape != ta.shape:
        raise ValueError("mask length does not match slot count")
    out = session.empty_tiles(ta.shape[0])
    _check(lib().tt_tiles_mask_mul(session.handle, _ptr(ta), _ptr(tm), _ptr(out), ta.shape[0],
                                   None, None))
    return out


def sum_tile_strided(session: Session, tiles, n: int, stride: int, variant) -> object:
    """sum_tile_strided rotate_sum.hpp:44-90 on every row."""
    src = _tiles_arg(session, tiles)
    out = session.empty_tiles(src.shape[0])
    _check(lib().tt_sum_tile_strided(session.handle, _ptr(src), int(n), int(stride),
                                     _variant(variant), _ptr(out), src.shape[0]))
    return out


def sum_tile_flat(session: Session, tiles, n: int, variant) -> object:  # rotate_sum.hpp:92
    return sum_tile_strided(session, tiles, n, 1, variant)


def sum_tile_dim(session: Session, tiles, tile_extents: Sequence[int], dim: int,
                 variant: Optional[SumVariant] = None):
    src = _tiles_arg(session, tiles)
    out = session.empty_tiles(src.shape[0])
    ext = (ctypes.c_int64 * len(tile_extents))(*tile_extents)
    _check(lib().tt_sum_tile_dim(session.handle, _ptr(src), ext, len(tile_extents), int(dim),
                                 _variant(variant), _ptr(out), src.shape[0]))
    return out


def replicate_tile_dim(session: Session, tiles, tile_extents: Sequence[int], dim: int):
    src = _tiles_arg(session, tiles)
    out = session.empty_tiles(src.shape[0])
    ext = (ctypes.c_int64 * len(tile_extents))(*tile_extents)
    _check(lib().tt_replicate_tile_dim(session.handle, _ptr(src), ext, len(tile_extents),
                                       int(dim), _ptr(out), src.shape[0]))
    return out


def auto_variant(n: int) -> SumVariant:  # rotate_sum.hpp:99-101
    return SumVariant.power_of_two if n > 0 and n & (n - 1) == 0 else SumVariant.right_to_left


def fill_uniform(session: Session, out, seed: int, lo: float, hi: float, offset: int = 0):
    """Device generator, bit-identical to oracle or_fill_uniform."""
    _check(lib().tt_fill_uniform(session.handle, _ptr(out), out.numel(), ctypes.c_uint64(seed),
                                 int(offset), float(lo), float(hi)))
    return out


def shard_plan(shape: TileTensorShape, shard_dim: int, world: int, rank: int):
    """Block partition of external dim `shard_dim` (1-based): (begin, end, local shape)."""
    b, e = ctypes.c_int64(), ctypes.c_int64()
    out = CShape()
    _check(lib().tt_shard_plan(ctypes.byref(shape.to_c()), int(shard_dim), int(world), int(rank),
                               ctypes.byref(b), ctypes.byref(e), ctypes.byref(out)))
    return b.value, e.value, TileTensorShape.from_c(out)


KERNEL_PATHS = {"auto": 0, "tma": 1, "regs": 2, "generic": 3, "window": 4}


def set_kernel_path(path: str) -> None:
    """Force the reduction kernel path (identical results, different speed)."""
    _check(lib().tt_set_kernel_path(KERNEL_PATHS[path]))


def set_chain_kernel(on: bool) -> None:
    """Run GEMM-shaped products (and linalg_chain) on the persistent chain
    kernel (csrc/kernels/chain.cuh); identical results, off by default."""
    _check(lib().tt_set_chain_kernel(1 if on else 0))


def chain_kernel() -> bool:
    return bool(lib().tt_chain_kernel())


def kernel_path() -> str:
    v = int(lib().tt_kernel_path())
    return {b: a for a, b in KERNEL_PATHS.items()}[v]


def device_count() -> int:
    n = ctypes.c_int()
    lib().tt_device_count(ctypes.byref(n))
    return n.value


# ---- packing methods, the alternating pipeline, tile-extent search ---------------------
# (linalg.hpp:77-294).  Host orchestration of the device ops above: packs,
# fused matvec passes, clean_unknowns and replicate_dim.


class PackingMethod:  # linalg.hpp:77-89
    class Kind(enum.Enum):
        row_order = 0
        column_order = 1
        input_packing = 2
        batch_packing = 3
        general = 4

    def __init__(self, kind: "PackingMethod.Kind", tile: Sequence[int] = ()):
        self.kind = kind
        self.tile = list(tile)

    @staticmethod
    def row_order():
        return PackingMethod(PackingMethod.Kind.row_order)

    @staticmethod
    def column_order():
        return PackingMethod(PackingMethod.Kind.column_order)

    @staticmethod
    def input_packing():
        return PackingMethod(PackingMethod.Kind.input_packing)

    @staticmethod
    def batch_packing():
        return PackingMethod(PackingMethod.Kind.batch_packing)

    @staticmethod
    def general(tile: Sequence[int]):
        return PackingMethod(PackingMethod.Kind.general, tile)


class OperandRole(enum.Enum):  # linalg.hpp:91
    matrix = 0
    vector = 1
    lhs = 2
    rhs = 3


def sum_dim_for(method: PackingMethod) -> int:  # linalg.hpp:94-96
    return 1 if method.kind == PackingMethod.Kind.input_packing else 2


def _smallest_divisor_at_least(s: int, b: int) -> int:  # linalg.hpp:100-105
    for t in range(max(b, 1), s + 1):
        if s % t == 0:
            return t
    return s


def _shape2(n1, d1, t1, n2, d2, t2) -> TileTensorShape:
    return TileTensorShape([DimSpec(n1, d1, t1), DimSpec(n2, d2, t2)])


def pack_for_method(m, role: OperandRole, method: PackingMethod, session: Session) -> TileTensor:
    """pack_for_method linalg.hpp:114-199 (m: numpy array)."""
    K = PackingMethod.Kind
    m = np.asarray(m, dtype=np.float64)
    s = session.slot_count()
    if method.kind == K.batch_packing:
        if role in (OperandRole.matrix, OperandRole.lhs):
            if m.ndim != 2:
                raise ShapeError("batch packing expects a rank-2 weight matrix")
            a, b = m.shape
            return pack(m.reshape(a, b, 1),
                        TileTensorShape([DimSpec(a, 1, 1), DimSpec(b, 1, 1), DimSpec(1, s, s)]),
                        session)
        if m.ndim != 2:
            raise ShapeError("batch packing expects data of shape [x, n]")
        x, n = m.shape
        if n > s:
            raise ShapeError("batch size exceeds the slot count")
        return pack(m, TileTensorShape([DimSpec(x, 1, 1), DimSpec(n, 1, s)]), session)
    t1, t2 = 1, s
    if method.kind == K.column_order:
        t1, t2 = s, 1
    elif method.kind == K.input_packing:
        b = m.shape[1] if role in (OperandRole.lhs, OperandRole.matrix) else m.shape[0]
        if b > s:
            raise ShapeError("input packing requires the contracted extent <= slot count")
        t1 = _smallest_divisor_at_least(s, b)
        t2 = s // t1
    elif method.kind == K.general:
        if len(method.tile) != 2:
            raise ShapeError("general packing here expects two tile extents")
        t1, t2 = method.tile
        if t1 * t2 != s:
            raise ShapeError("tile extents must multiply to the slot count")
    transposed = (method.kind == K.input_packing or
                  role in (OperandRole.lhs, OperandRole.rhs))
    if role == OperandRole.matrix:
        if m.ndim != 2:
            raise ShapeError("matrix role expects a rank-2 tensor")
        mm = np.ascontiguousarray(m.T) if transposed else m
        return pack(mm, _shape2(mm.shape[0], 1, t1, mm.shape[1], 1, t2), session)
    if role == OperandRole.lhs:
        if m.ndim != 2:
            raise ShapeError("lhs role expects a rank-2 tensor")
        mt = np.ascontiguousarray(m.T)
        return pack(mt, _shape2(mt.shape[0], 1, t1, mt.shape[1], 1, t2), session)
    b = m.size
    if role == OperandRole.vector and not transposed:
        return pack(m.reshape(1, b), _shape2(1, t1, t1, b, 1, t2), session)
    return pack(m.reshape(b, 1), _shape2(b, 1, t1, 1, t2, t2), session)


def unpack_vector(t: TileTensor) -> np.ndarray:  # linalg.hpp:263-266
    return unpack(t).reshape(-1)


@dataclass
class PipelineResult:
    out: TileTensor
    cost: CostReport


def pipeline(matrices: Sequence, v, tile: Sequence[int], session: Session) -> PipelineResult:
    """pipeline linalg.hpp:213-260: M_k(...(M_2(M_1 v))); odd stages pack the
    matrix transposed and sum dim 1, even stages sum dim 2 and, before a next
    stage, clean_unknowns + replicate_dim(2) when the output is not replicated."""
    if len(matrices) == 0:
        raise ShapeError("pipeline needs at least one matrix")
    t1, t2 = int(tile[0]), int(tile[1])
    if t1 * t2 != session.slot_count():
        raise ShapeError("tile extents must multiply to the slot count")
    v = np.asarray(v, dtype=np.float64).reshape(-1)
    mats = [np.asarray(m, dtype=np.float64) for m in matrices]
    width = v.size
    for k, m in enumerate(mats):
        if m.ndim != 2 or m.shape[1] != width:
            raise ShapeError(f"pipeline stage {k + 1}: matrix extents do not chain")
        width = m.shape[0]
    before = session.cost_report()
    data = pack(v.reshape(-1, 1), _shape2(v.size, 1, t1, 1, t2, t2), session)
    for k, m in enumerate(mats):
        try:
            if k % 2 == 0:  # odd stage k + 1
                mt = np.ascontiguousarray(m.T)
                tm = pack(mt, _shape2(mt.shape[0], 1, t1, mt.shape[1], 1, t2), session)
                data = matvec_b(tm, data)
            else:
                tm = pack(m, _shape2(m.shape[0], 1, t1, m.shape[1], 1, t2), session)
                if k + 1 < len(mats):
                    # matvec_a + clean_unknowns in one pass (operands valid by
                    # construction: the same result, counters and errors)
                    data = tt_mul_sum_clean(tm, data, 2)
                    if data.shape().dim(1).d < t2:
                        data = replicate_dim(data, 2)
                else:
                    data = matvec_a(tm, data)
        except DepthExhaustedError as e:
            raise DepthExhaustedError(f"pipeline stage {k + 1}: {e}") from None
    return PipelineResult(data, session.cost_report().since(before))


@dataclass
class TileChoice:
    t1: int
    t2: int
    cost: CostReport


def score_tile_factorizations(matrices: Sequence, v, s: int, depth: int,
                              device: int = 0) -> list:
    """score_tile_factorizations linalg.hpp:279-294: the pipeline under every
    t1 * t2 = s in a scratch session, ordered by rotations then total ops."""
    out = []
    for t1 in range(1, s + 1):
        if s % t1:
            continue
        scratch = Session(s, depth, device)
        res = pipeline(matrices, v, (t1, s // t1), scratch)
        out.append(TileChoice(t1, s // t1, res.cost))
    out.sort(key=lambda c: (c.cost.rotations, c.cost.total_ops()))
    return out


__all__ = [n for n in dir() if not n.startswith("_")]
