"""Neural-network layer of the tile-tensor API (mirror of inc/nn.hpp).

Host orchestration over the device ops of `tiletensor`: im2col lowering and
weight layout happen on the host in plaintext (as in the reference); every
tile operation -- pack, fused multiply + sum, add, square, clean_unknowns,
replicate_dim and the batch-packed affine fold -- runs on the GPU.

  im2col                      nn.hpp:30-54
  ConvLayer/FcLayer/...       nn.hpp:57-89
  parse_network               nn.hpp:138-185   (seeded weights: std::mt19937_64 +
                                                uniform_real_distribution(-0.5, 0.5))
  cryptonets_network          nn.hpp:187-196
  nn_forward                  nn.hpp:202-257   (plaintext oracle, same left folds)
  infer_batch_packed          nn.hpp:270-346   (one tt_batch_affine pass per layer)
  cryptonets_infer            nn.hpp:350-507

The reference's bootstrap_lower_bound and handcrafted-plan checker
(nn.hpp:511-700) are planning tools off the hot path (SURVEY.md section 2:
out of scope) and are not mirrored.
"""
from __future__ import annotations

import ctypes
import io
from dataclasses import dataclass, field
from pathlib import Path
from typing import List, Optional, Sequence, Union

import numpy as np

from . import tiletensor as tt
from ._abi import lib
from .tiletensor import (CostReport, DepthExhaustedError, DimSpec, ShapeError, TileTensor,
                         TileTensorShape, _check, _ptr)

# ---- seeded parameters: libstdc++'s mt19937_64 + uniform_real_distribution ---------

_M64 = (1 << 64) - 1


class Mt19937_64:
    """std::mt19937_64 (the 64-bit Mersenne Twister of the C++ standard)."""

    def __init__(self, seed: int):
        self.mt = [0] * 312
        self.mt[0] = seed & _M64
        for i in range(1, 312):
            prev = self.mt[i - 1]
            self.mt[i] = (6364136223846793005 * (prev ^ (prev >> 62)) + i) & _M64
        self.idx = 312

    def _twist(self):
        mt = self.mt
        for i in range(312):
            x = (mt[i] & 0xFFFFFFFF80000000) | (mt[(i + 1) % 312] & 0x7FFFFFFF)
            xa = x >> 1
            if x & 1:
                xa ^= 0xB5026F5AA96619E9
            mt[i] = mt[(i + 156) % 312] ^ xa
        self.idx = 0

    def __call__(self) -> int:
        if self.idx >= 312:
            self._twist()
        y = self.mt[self.idx]
        self.idx += 1
        y ^= (y >> 29) & 0x5555555555555555
        y ^= (y << 17) & 0x71D67FFFEDA60000
        y ^= (y << 37) & 0xFFF7EEE000000000
        y ^= y >> 43
        return y & _M64


def _uniform(rng: Mt19937_64, a: float, b: float) -> float:
    # generate_canonical<double, 53> over a 64-bit engine: one draw / 2^64
    u = float(rng()) / 18446744073709551616.0
    if u >= 1.0:
        u = np.nextafter(1.0, 0.0)
    return u * (b - a) + a


def random_tensor(shape: Sequence[int], rng: Mt19937_64) -> np.ndarray:
    """nn.hpp:92-99 detail::random_tensor: U[-0.5, 0.5) in row-major order."""
    n = int(np.prod(shape)) if len(shape) else 1
    return np.array([_uniform(rng, -0.5, 0.5) for _ in range(n)], dtype=np.float64).reshape(shape)


# ---- dense text format (dense.hpp:200-242) ------------------------------------------


def read_tensor(src: Union[str, io.TextIOBase]) -> np.ndarray:
    """`shape: n1 ... nk` then row-major values; '#' lines are comments."""
    lines = src.splitlines() if isinstance(src, str) else src.read().splitlines()
    shape = None
    values: List[float] = []
    for line in lines:
        text = line.strip(" \t\r")
        if not text or text.startswith("#"):
            continue
        if shape is None:
            parts = text.split()
            if parts[0] != "shape:":
                raise RuntimeError("tensor file must start with a 'shape:' line")
            shape = [int(x) for x in parts[1:]]
            continue
        for tok in text.split():
            try:
                values.append(float(tok))
            except ValueError:
                raise RuntimeError("malformed value in tensor file") from None
    if not shape:
        raise RuntimeError("tensor file has no shape line")
    if int(np.prod(shape)) != len(values):
        raise ShapeError("tensor file: value count does not match its shape")
    return np.array(values, dtype=np.float64).reshape(shape)


def write_tensor(t: np.ndarray) -> str:
    """Text of write_tensor: shape line, then rows of the last extent, %.17g."""
    t = np.asarray(t, dtype=np.float64)
    row = t.shape[-1] if t.ndim else 1
    out = ["shape:" + "".join(f" {e}" for e in t.shape) + "\n"]
    flat = t.reshape(-1)
    for i, v in enumerate(flat):
        out.append(format(float(v), ".17g"))
        out.append("\n" if (i + 1) % row == 0 else " ")
    return "".join(out)


# ---- network description ----------------------------------------------------------


@dataclass
class ConvLayer:  # nn.hpp:57-61
    filters: int = 1
    kh: int = 1
    kw: int = 1
    stride: int = 1
    pad: int = 0
    weights: np.ndarray = field(default_factory=lambda: np.zeros((1, 1)))  # [filters, kh*kw]
    bias: np.ndarray = field(default_factory=lambda: np.zeros(1))          # [filters]


@dataclass
class FcLayer:  # nn.hpp:63-67
    inp: int = 1
    out: int = 1
    weights: np.ndarray = field(default_factory=lambda: np.zeros((1, 1)))  # [out, in]
    bias: np.ndarray = field(default_factory=lambda: np.zeros(1))          # [out]


@dataclass
class SquareLayer:  # nn.hpp:69
    pass


@dataclass
class MeanPoolLayer:  # nn.hpp:71-73
    window: int = 1


@dataclass
class NetworkSpec:  # nn.hpp:77-89
    input_h: int = 0
    input_w: int = 0
    layers: list = field(default_factory=list)

    def input_size(self) -> int:
        if self.input_h > 0 and self.input_w > 0:
            return self.input_h * self.input_w
        for layer in self.layers:
            if isinstance(layer, FcLayer):
                return layer.inp
        raise ShapeError("network has no declared input size")


def _kv(tokens, key):
    for tok in tokens:
        if tok.startswith(key + "="):
            return tok[len(key) + 1:]
    return None


def _kv_int(tokens, key, line) -> int:
    v = _kv(tokens, key)
    if v is None:
        raise RuntimeError(f"missing '{key}=' in: {line}")
    return int(v)


def _load_or_random(tokens, key, shape, base_dir: str, rng: Mt19937_64) -> np.ndarray:
    path = _kv(tokens, key)
    if path is not None:
        full = path if not base_dir else str(Path(base_dir) / path)
        try:
            text = Path(full).read_text()
        except OSError:
            raise RuntimeError(f"cannot open weight file {full}") from None
        t = read_tensor(text)
        if t.size != int(np.prod(shape)):
            raise RuntimeError(f"weight file {full} has wrong element count")
        return t.reshape(shape)
    return random_tensor(shape, rng)


def parse_network(text: str, base_dir: str = "", seed: int = 0) -> NetworkSpec:
    """nn.hpp:138-185: `input h= w=`, `conv filters= kh= kw= stride= pad=`,
    `act square`, `fc in= out=`, `pool mean window=`; layers without
    weights=/bias= files get seeded random parameters (in file order)."""
    net = NetworkSpec()
    rng = Mt19937_64(seed)
    for line in text.splitlines():
        tokens = line.split()
        if not tokens or tokens[0].startswith("#"):
            continue
        kind = tokens[0]
        if kind == "input":
            net.input_h = _kv_int(tokens, "h", line)
            net.input_w = _kv_int(tokens, "w", line)
        elif kind == "conv":
            c = ConvLayer(_kv_int(tokens, "filters", line), _kv_int(tokens, "kh", line),
                          _kv_int(tokens, "kw", line), _kv_int(tokens, "stride", line),
                          _kv_int(tokens, "pad", line))
            c.weights = _load_or_random(tokens, "weights", (c.filters, c.kh * c.kw), base_dir, rng)
            c.bias = _load_or_random(tokens, "bias", (c.filters,), base_dir, rng)
            net.layers.append(c)
        elif kind == "fc":
            f = FcLayer(_kv_int(tokens, "in", line), _kv_int(tokens, "out", line))
            f.weights = _load_or_random(tokens, "weights", (f.out, f.inp), base_dir, rng)
            f.bias = _load_or_random(tokens, "bias", (f.out,), base_dir, rng)
            net.layers.append(f)
        elif kind == "act":
            if len(tokens) < 2 or tokens[1] != "square":
                raise RuntimeError("only the square activation is supported: " + line)
            net.layers.append(SquareLayer())
        elif kind == "pool":
            net.layers.append(MeanPoolLayer(_kv_int(tokens, "window", line)))
        else:
            raise RuntimeError(f"unknown layer kind '{kind}'")
    if not net.layers:
        raise RuntimeError("network file declares no layers")
    return net


CRYPTONETS_SPEC = ("input h=28 w=28\n"
                   "conv filters=5 kh=5 kw=5 stride=2 pad=1\n"
                   "act square\n"
                   "fc in=845 out=100\n"
                   "act square\n"
                   "fc in=100 out=10\n")


def cryptonets_network(seed: int) -> NetworkSpec:  # nn.hpp:187-196
    return parse_network(CRYPTONETS_SPEC, "", seed)


# ---- im2col and the plaintext forward pass ----------------------------------------


def _conv_grid(h, w, c: ConvLayer):
    gh = (h + 2 * c.pad - c.kh) // c.stride + 1
    gw = (w + 2 * c.pad - c.kw) // c.stride + 1
    return gh, gw


def _im2col_index(h: int, w: int, kh: int, kw: int, stride: int, pad: int) -> np.ndarray:
    """[windows, kh*kw] source pixel index (y*w + x), -1 outside the input."""
    if kh < 1 or kw < 1 or stride < 1 or pad < 0:
        raise ShapeError("im2col: invalid filter geometry")
    if h + 2 * pad < kh or w + 2 * pad < kw:
        raise ShapeError("im2col: no valid window")
    gh = (h + 2 * pad - kh) // stride + 1
    gw = (w + 2 * pad - kw) // stride + 1
    gy, gx, ky, kx = np.meshgrid(np.arange(gh), np.arange(gw), np.arange(kh), np.arange(kw),
                                 indexing="ij")
    y = gy * stride - pad + ky
    x = gx * stride - pad + kx
    idx = np.where((y >= 0) & (y < h) & (x >= 0) & (x < w), y * w + x, -1)
    return idx.reshape(gh * gw, kh * kw)


def im2col(img: np.ndarray, kh: int, kw: int, stride: int, pad: int) -> np.ndarray:
    """nn.hpp:30-54: row r = the filter window at grid position r, zero padded."""
    img = np.asarray(img, dtype=np.float64)
    if img.ndim != 2:
        raise ShapeError("im2col expects a rank-2 input")
    idx = _im2col_index(img.shape[0], img.shape[1], kh, kw, stride, pad)
    flat = np.concatenate([img.reshape(-1), [0.0]])
    return flat[np.where(idx < 0, flat.size - 1, idx)]


def nn_forward(net: NetworkSpec, batch: np.ndarray) -> np.ndarray:
    """nn.hpp:202-257, the plaintext oracle: batch [features, samples] ->
    logits [out, samples].  Same left folds as the reference (bias first, then
    += w * x in input order), vectorised over samples and outputs only."""
    batch = np.asarray(batch, dtype=np.float64)
    if batch.ndim != 2:
        raise ShapeError("batch must be [features, samples]")
    v = batch.copy()  # [features, n]
    for layer in net.layers:
        if isinstance(layer, ConvLayer):
            c = layer
            if net.input_h * net.input_w != v.shape[0]:
                raise ShapeError("conv input size mismatch")
            idx = _im2col_index(net.input_h, net.input_w, c.kh, c.kw, c.stride, c.pad)
            padded = np.concatenate([v, np.zeros((1, v.shape[1]))])
            m1 = padded[np.where(idx < 0, v.shape[0], idx)]  # [windows, kk, n]
            acc = np.broadcast_to(c.bias[None, :, None], (idx.shape[0], c.filters, v.shape[1])).copy()
            for b in range(c.kh * c.kw):
                acc = acc + m1[:, b, None, :] * c.weights[None, :, b, None]
            v = acc.reshape(idx.shape[0] * c.filters, v.shape[1])  # window-major
        elif isinstance(layer, FcLayer):
            f = layer
            if v.shape[0] != f.inp:
                raise ShapeError("fc input size mismatch")
            acc = np.broadcast_to(f.bias[:, None], (f.out, v.shape[1])).copy()
            for i in range(f.inp):
                acc = acc + f.weights[:, i, None] * v[i][None, :]
            v = acc
        elif isinstance(layer, SquareLayer):
            v = v * v
        else:
            raise ShapeError("mean pooling is not executable here (plan fixture only)")
    return v


# ---- tiled inference ----------------------------------------------------------------


def _is_torch(x) -> bool:
    return type(x).__module__.startswith("torch")


@dataclass
class InferResult:  # nn.hpp:260-263
    logits: np.ndarray
    cost: CostReport


def _batch_affine(session: tt.Session, data, chain: int, n_in: int, row_ptr, src, w, bias):
    n_out = len(bias)
    out = session.empty_tiles(max(n_out, 1))
    rp = np.ascontiguousarray(row_ptr, dtype=np.int64)
    sr = np.ascontiguousarray(src, dtype=np.int64)
    ww = np.ascontiguousarray(w, dtype=np.float64)
    bb = np.ascontiguousarray(bias, dtype=np.float64)
    co = ctypes.c_int64()
    p64 = ctypes.POINTER(ctypes.c_int64)
    pd = ctypes.POINTER(ctypes.c_double)
    _check(lib().tt_batch_affine(session.handle, _ptr(data), int(n_in), int(n_out),
                                 rp.ctypes.data_as(p64), sr.ctypes.data_as(p64),
                                 ww.ctypes.data_as(pd), bb.ctypes.data_as(pd), _ptr(out),
                                 int(chain), ctypes.byref(co)))
    return out[:n_out], co.value


def _batch_packed_plan(net: NetworkSpec) -> list:
    """The batch-packed branch's layers as device work: ("affine", n_in, row_ptr,
    src, w, bias) -- one tt_batch_affine pass, taps in the reference's order --
    or ("square",).  Layer-size errors are raised when the layer is reached."""
    plan = []
    n_tiles = net.input_size()
    for layer in net.layers:
        if isinstance(layer, ConvLayer):
            c = layer
            h, w = net.input_h, net.input_w
            idx = _im2col_index(h, w, c.kh, c.kw, c.stride, c.pad)  # [windows, kk]
            windows, kk = idx.shape
            # output (window, filter): taps over (ky, kx) in order, padding skipped
            valid = idx >= 0
            counts = np.repeat(valid.sum(axis=1), c.filters)
            row_ptr = np.concatenate([[0], np.cumsum(counts)])
            src = np.concatenate([np.tile(idx[wi][valid[wi]], c.filters) for wi in range(windows)])
            wts = np.concatenate([c.weights[:, valid[wi]].reshape(-1) for wi in range(windows)])
            bias = np.tile(c.bias, windows)
            plan.append(("affine", h * w, row_ptr, src, wts, bias))
            n_tiles = len(bias)
        elif isinstance(layer, FcLayer):
            f = layer
            if n_tiles != f.inp:
                plan.append(("error", ShapeError("fc input size mismatch")))
                break
            row_ptr = np.arange(f.out + 1, dtype=np.int64) * f.inp
            src = np.tile(np.arange(f.inp, dtype=np.int64), f.out)
            plan.append(("affine", f.inp, row_ptr, src, np.asarray(f.weights).reshape(-1),
                         np.asarray(f.bias)))
            n_tiles = f.out
        elif isinstance(layer, SquareLayer):
            plan.append(("square",))
        else:
            plan.append(("error", ShapeError("unsupported layer for inference")))
            break
    return plan


def _arrays(row_ptr, src, w, bias):
    return (np.ascontiguousarray(row_ptr, dtype=np.int64), np.ascontiguousarray(src, dtype=np.int64),
            np.ascontiguousarray(w, dtype=np.float64), np.ascontiguousarray(bias, dtype=np.float64))


def _square(session: tt.Session, data, chain: int):
    # session.mul(t, t) per tile (chains are uniform across the layer)
    if chain < 1:
        raise DepthExhaustedError("multiplication at chain index 0 (bootstrap required)")
    out = session.empty_tiles(data.shape[0])
    _check(lib().tt_tiles_binary(session.handle, int(tt.OpKind.mul), _ptr(data), _ptr(data),
                                 _ptr(out), int(data.shape[0]), None, None, None))
    return out, chain - 1


def _run_batch_packed(plan: list, batch, session: tt.Session, affine) -> InferResult:
    before = session.cost_report()
    if not _is_torch(batch):  # a device-resident torch batch is packed in place (no host copy)
        batch = np.asarray(batch, dtype=np.float64)
    n = int(batch.shape[1])
    s = session.slot_count()
    packed = tt.pack(batch, TileTensorShape([DimSpec(int(batch.shape[0]), 1, 1), DimSpec(n, 1, s)]),
                     session)
    data, chain = packed.data(), packed.chain_index()
    for layer_no, step in enumerate(plan, start=1):
        try:
            if step[0] == "affine":
                data, chain = affine(layer_no - 1, step, data, chain)
            elif step[0] == "square":
                data, chain = _square(session, data, chain)
            else:
                raise step[1]
        except DepthExhaustedError as e:
            raise DepthExhaustedError(f"layer {layer_no}: {e}") from None
    shape = TileTensorShape([DimSpec(int(data.shape[0]), 1, 1), DimSpec(n, 1, s)])
    logits = tt.unpack(TileTensor(shape, data, session, chain))
    return InferResult(logits, session.cost_report().since(before))


def infer_batch_packed(net: NetworkSpec, batch: np.ndarray, session: tt.Session) -> InferResult:
    """nn.hpp:270-346: every network scalar is one tile carrying it for all
    samples; each conv / fc layer is ONE device pass (tt_batch_affine) that
    folds bias + w * x in the reference's order; zero rotations."""
    if int(batch.shape[0]) != net.input_size():
        raise ShapeError("batch feature size mismatch")

    def affine(i, step, data, chain):
        _, n_in, row_ptr, src, w, bias = step
        if data.shape[0] != n_in:
            raise ShapeError("fc input size mismatch")
        return _batch_affine(session, data, chain, n_in, row_ptr, src, w, bias)
    return _run_batch_packed(_batch_packed_plan(net), batch, session, affine)


class CompiledBatchPacked:
    """cryptonets_infer's batch-packed branch (tile [1, 1, s]) for repeated
    inference with fixed weights: the network's layers are turned into tap lists
    and uploaded once (tt_affine_layer_create); each infer() is then the pack,
    one device pass per layer and the unpack.  Logits and counters equal
    cryptonets_infer(net, batch, (1, 1, s), session) bit for bit.  The weights
    are captured at construction (later edits to `net` are not seen)."""

    def __init__(self, net: NetworkSpec, session: tt.Session):
        self.session = session
        self.plan = _batch_packed_plan(net)
        self.n_in = net.input_size()
        self.layers = {}
        for i, step in enumerate(self.plan):
            if step[0] != "affine":
                continue
            _, n_in, row_ptr, src, w, bias = step
            rp, sr, ww, bb = _arrays(row_ptr, src, w, bias)
            h = ctypes.c_void_p()
            p64, pd = ctypes.POINTER(ctypes.c_int64), ctypes.POINTER(ctypes.c_double)
            _check(lib().tt_affine_layer_create(session.handle, int(n_in), len(bb),
                                                rp.ctypes.data_as(p64), sr.ctypes.data_as(p64),
                                                ww.ctypes.data_as(pd), bb.ctypes.data_as(pd),
                                                ctypes.byref(h)))
            self.layers[i] = (h, int(n_in), len(bb))

    def infer(self, batch) -> InferResult:
        if int(batch.shape[0]) != self.n_in:
            raise ShapeError("batch feature size mismatch")
        if int(batch.shape[1]) > self.session.slot_count():
            raise ShapeError("batch size exceeds the batch tile extent t3")

        def affine(i, step, data, chain):
            h, n_in, n_out = self.layers[i]
            if data.shape[0] != n_in:
                raise ShapeError("fc input size mismatch")
            out = self.session.empty_tiles(max(n_out, 1))
            co = ctypes.c_int64()
            _check(lib().tt_affine_layer_apply(self.session.handle, h, _ptr(data), _ptr(out),
                                               int(chain), ctypes.byref(co)))
            return out[:n_out], co.value
        return _run_batch_packed(self.plan, batch, self.session, affine)

    def close(self) -> None:
        for h, _, _ in self.layers.values():
            lib().tt_affine_layer_destroy(self.session.handle, h)
        self.layers = {}

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def cryptonets_infer(net: NetworkSpec, batch: np.ndarray, tile: Sequence[int],
                     session: tt.Session, lift_batch_limit: bool = False) -> InferResult:
    """nn.hpp:350-507: tile [t1, t2, t3], batch along the third dim.  A
    leading conv is folded client-side into a first-stage product (transposed
    im2col replicated per filter), fc stages alternate the two product forms
    with clean + replicate at even -> odd seams; t1 = t2 = 1 takes the
    batch-packed path.

    lift_batch_limit (SURVEY 8f "n > t3 lifted"; the reference throws):
    batches larger than t3 become several external tiles along the batch dim
    (no rotation crosses samples, so each sample's logits equal a reference
    run on its own t3-sized chunk bit for bit); the batch-packed path runs
    chunks of s samples."""
    t1, t2, t3 = (int(x) for x in tile)
    if t1 * t2 * t3 != session.slot_count():
        raise ShapeError("tile extents must multiply to the slot count")
    if len(batch.shape) != 2:
        raise ShapeError("batch must be [features, samples]")
    n = int(batch.shape[1])
    if n > t3 and not lift_batch_limit:
        raise ShapeError("batch size exceeds the batch tile extent t3")
    if int(batch.shape[0]) != net.input_size():
        raise ShapeError("batch feature size mismatch")
    if t1 == 1 and t2 == 1:
        if n <= t3:
            return infer_batch_packed(net, batch, session)
        parts = [infer_batch_packed(net, batch[:, k:k + t3], session) for k in range(0, n, t3)]
        total = CostReport()
        for r in parts:
            total = CostReport(*(getattr(total, f) + getattr(r.cost, f) for f in tt._COST_FIELDS))
        return InferResult(np.concatenate([r.logits for r in parts], axis=1), total)
    return _infer_tiled(net, batch, (t1, t2, t3), session, None)


def _infer_tiled(net: NetworkSpec, batch, tile, session: tt.Session, cache) -> InferResult:
    """The tiled branch of cryptonets_infer (nn.hpp:418-507).  cache: None, or a
    dict keeping the packed weight / bias tensors across calls (CompiledTiled)."""
    t1, t2, t3 = tile
    n = int(batch.shape[1])

    def cached(key, make):
        if cache is None:
            return make()
        if key not in cache:
            cache[key] = make()
        return cache[key]

    # the tiled path lays the batch out on the host (im2col, as the reference does)
    batch = np.asarray(batch.detach().cpu() if _is_torch(batch) else batch, dtype=np.float64)
    before = session.cost_report()

    def shape3(a, b, c):
        return TileTensorShape([DimSpec(*a), DimSpec(*b), DimSpec(*c)])

    def pack_weights(w2d, odd, perm):
        rows, cols = w2d.shape  # out, in
        if perm is not None and cols != len(perm):
            raise ShapeError(f"layer input extent {cols} does not match the convolution output "
                             f"{len(perm)}")
        src = w2d if perm is None else w2d[:, perm]
        if odd:  # [in/t1, out/t2, */t3]
            return tt.pack(np.ascontiguousarray(src.T).reshape(cols, rows, 1),
                           shape3((cols, 1, t1), (rows, 1, t2), (1, t3, t3)), session)
        return tt.pack(np.ascontiguousarray(src).reshape(rows, cols, 1),
                       shape3((rows, 1, t1), (cols, 1, t2), (1, t3, t3)), session)

    def pack_bias(b, odd):
        ln = b.size
        if odd:
            return tt.pack(b.reshape(1, ln, 1), shape3((1, t1, t1), (ln, 1, t2), (1, t3, t3)),
                           session)
        return tt.pack(b.reshape(ln, 1, 1), shape3((ln, 1, t1), (1, t2, t2), (1, t3, t3)), session)

    data: Optional[TileTensor] = None
    perm = None
    stage = 0
    fused_square = False
    for layer_no, layer in enumerate(net.layers, start=1):
        if fused_square:  # applied with the preceding linear stage
            fused_square = False
            continue
        try:
            if isinstance(layer, ConvLayer):
                c = layer
                if data is not None or stage != 0:
                    raise ShapeError("convolution is only supported as the first layer")
                stage += 1
                h, w = net.input_h, net.input_w
                idx = _im2col_index(h, w, c.kh, c.kw, c.stride, c.pad)
                windows, kk = idx.shape
                fold = c.filters * windows
                padded = np.concatenate([batch, np.zeros((1, n))])
                m1 = padded[np.where(idx < 0, batch.shape[0], idx)]  # [windows, kk, n]
                d3 = np.broadcast_to(m1.transpose(1, 0, 2)[:, None, :, :],
                                     (kk, c.filters, windows, n)).reshape(kk, fold, n)
                td = tt.pack(np.ascontiguousarray(d3), shape3((kk, 1, t1), (fold, 1, t2), (n, 1, t3)),
                             session)
                wf = np.broadcast_to(c.weights.T[:, :, None], (kk, c.filters, windows))
                bf = np.repeat(c.bias, windows)
                tw = cached((layer_no, "w"), lambda: tt.pack(
                    np.ascontiguousarray(wf).reshape(kk, fold, 1),
                    shape3((kk, 1, t1), (fold, 1, t2), (1, t3, t3)), session))
                tb = cached((layer_no, "b"), lambda: pack_bias(bf, True))
                nxt = net.layers[layer_no] if layer_no < len(net.layers) else None
                depth_after = min(min(tw.chain_index(), td.chain_index()) - 1, tb.chain_index())
                fused_square = isinstance(nxt, SquareLayer) and depth_after >= 1
                data = tt.tt_mul_sum_affine(tw, td, 1, tb, square=fused_square)
                # the oracle flattens window-major, the folded layout is filter-major
                perm = (np.arange(windows)[None, :] * c.filters +
                        np.arange(c.filters)[:, None]).reshape(-1)
            elif isinstance(layer, FcLayer):
                f = layer
                stage += 1
                odd = stage % 2 == 1
                if data is None:
                    if not odd:
                        raise RuntimeError("first stage must be odd")
                    data = tt.pack(batch.reshape(batch.shape[0], 1, n),
                                   shape3((batch.shape[0], 1, t1), (1, t2, t2), (n, 1, t3)), session)
                elif odd:
                    if data.shape().has_unknown():
                        data = tt.clean_unknowns(data)
                    if data.shape().dim(1).d < t2:
                        data = tt.replicate_dim(data, 2)
                tw = cached((layer_no, "w"), lambda: pack_weights(
                    np.asarray(f.weights, dtype=np.float64), odd, perm))
                perm = None
                tb = cached((layer_no, "b"), lambda: pack_bias(np.asarray(f.bias, dtype=np.float64), odd))
                # a following square activation runs in the same device pass
                # (tt_mul_sum_affine) unless it would exhaust the depth, which
                # must then be reported against the square layer itself
                nxt = net.layers[layer_no] if layer_no < len(net.layers) else None
                depth_after = min(min(tw.chain_index(), data.chain_index()) - 1, tb.chain_index())
                fused_square = isinstance(nxt, SquareLayer) and depth_after >= 1
                data = tt.tt_mul_sum_affine(tw, data, 1 if odd else 2, tb, square=fused_square)
            elif isinstance(layer, SquareLayer):
                if data is None:
                    raise ShapeError("activation before any linear layer")
                data = tt.tt_mul(data, data)
            else:
                raise ShapeError("unsupported layer for inference")
        except DepthExhaustedError as e:
            raise DepthExhaustedError(f"layer {layer_no}: {e}") from None
    if data is None:
        raise ShapeError("network has no linear layers")
    if perm is not None:
        raise ShapeError("network ends right after a convolution; add a linear layer")
    raw = tt.unpack(data)
    out_size = raw.shape[1] if stage % 2 == 1 else raw.shape[0]
    return InferResult(raw.reshape(out_size, n), session.cost_report().since(before))


class CompiledTiled:
    """cryptonets_infer's tiled branch (tile [t1, t2, t3], t1 * t2 > 1) for
    repeated inference: the weight and bias tensors are packed on the device
    by the first infer() and reused by later calls (only the batch is packed
    per call).  Logits and counters equal cryptonets_infer(net, batch, tile,
    session, lift_batch_limit) bit for bit; the weights are captured on first
    use."""

    def __init__(self, net: NetworkSpec, tile: Sequence[int], session: tt.Session,
                 lift_batch_limit: bool = False):
        t1, t2, t3 = (int(x) for x in tile)
        if t1 * t2 * t3 != session.slot_count():
            raise ShapeError("tile extents must multiply to the slot count")
        if t1 == 1 and t2 == 1:
            raise ShapeError("tile [1, 1, s] is the batch-packed branch: use CompiledBatchPacked")
        self.net, self.tile, self.session = net, (t1, t2, t3), session
        self.lift = lift_batch_limit
        self._cache: dict = {}

    def infer(self, batch) -> InferResult:
        if len(batch.shape) != 2:
            raise ShapeError("batch must be [features, samples]")
        if int(batch.shape[1]) > self.tile[2] and not self.lift:
            raise ShapeError("batch size exceeds the batch tile extent t3")
        if int(batch.shape[0]) != self.net.input_size():
            raise ShapeError("batch feature size mismatch")
        return _infer_tiled(self.net, batch, self.tile, self.session, self._cache)
