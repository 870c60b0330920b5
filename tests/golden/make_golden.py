"""Generate the golden fixtures from the REFERENCE itself (oracle/_ref).

Run here (where /root/reference exists and oracle/_ref/libttref.so is built):
    python tests/golden/make_golden.py
Writes tests/golden/golden.npz.  Every case stores its inputs, the
reference's outputs and counters.  Tests replay the cases through the C
restatement (not-gpu: pins the oracle) and through the CUDA kernels (gpu).
Large outputs are stored as SHA-256 digests of their bytes plus shapes.
"""
from __future__ import annotations

import hashlib
import json
import random
import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE.parent))
sys.path.insert(0, str(HERE.parents[1]))

from oracle_lib import Ref  # noqa: E402
from shapes import partner_shape, random_pack_shape, shape_key  # noqa: E402

from paper_2011_01805_b200 import DimSpec, TileTensorShape, parse_shape  # noqa: E402
from paper_2011_01805_b200 import configs  # noqa: E402

COST = ("additions", "multiplications", "mask_multiplications", "rotations", "bootstraps",
        "power_of_two_rotations")


def cost_vec(c):
    return np.array([getattr(c, f) for f in COST], dtype=np.int64)


def digest(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a, dtype=np.float64).tobytes()).hexdigest()


def main():
    ref = Ref()
    rng = random.Random(20201103)
    nrng = np.random.default_rng(20201103)
    arrays = {}
    index = []

    def add(kind, **kw):
        i = len(index)
        meta = {"kind": kind}
        for k, v in kw.items():
            if isinstance(v, np.ndarray):
                arrays[f"c{i}_{k}"] = v
            elif isinstance(v, TileTensorShape):
                meta[k] = shape_key(v)
            else:
                meta[k] = v
        index.append(meta)

    # pack / unpack over random shapes (criterion 4 style)
    for it in range(60):
        s = rng.choice([8, 16, 32, 64])
        shape = random_pack_shape(rng, s, rng.randint(1, 4))
        dense = nrng.uniform(-1, 1, size=shape.tensor_extents())
        add("pack", s=s, shape=shape, dense=dense, tiles=ref.pack(dense, shape, s))

    # elementwise with broadcasting (tests/test_tile_tensor.cpp:218-264)
    done = 0
    while done < 60:
        s = 1 << rng.randint(2, 5)
        sa = random_pack_shape(rng, s, rng.randint(1, 3))
        sb = partner_shape(rng, sa)
        op = rng.randint(0, 1)
        try:
            ref.elementwise_result_shape(sa, sb, op)
        except Exception:
            continue
        ta = nrng.uniform(-3, 3, size=(sa.tile_count(), s))
        tb = nrng.uniform(-3, 3, size=(sb.tile_count(), s))
        so, out, c = ref.elementwise(op, sa, ta, sb, tb, s)
        add("elementwise", s=s, op=op, sa=sa, sb=sb, ta=ta, tb=tb, so=so, out=out, cost=cost_vec(c))
        done += 1

    # tt_sum over every dim and variant on random full tiles (garbage everywhere)
    for it in range(40):
        s = 1 << rng.randint(2, 6)
        shape = random_pack_shape(rng, s, rng.randint(1, 3))
        tiles = nrng.uniform(-5, 5, size=(shape.tile_count(), s))
        for dim in range(1, shape.rank() + 1):
            for v in (-1, 0, 1, 2):
                try:
                    so, out, c = ref.sum(shape, tiles, s, dim, v)
                except Exception as e:
                    add("sum_error", s=s, shape=shape, tiles=tiles, dim=dim, variant=v,
                        code=int(getattr(e, "code", -1)))
                    continue
                add("sum", s=s, shape=shape, tiles=tiles, dim=dim, variant=v, so=so, out=out,
                    cost=cost_vec(c))

    # '?' boundary split (tile_tensor.hpp:302-343)
    for text in ["[18?/8,1]", "[5/2,1?/4]", "[13?/4,3/2]", "[7?/8]", "[3,11?/4]", "[29?/32]",
                 "[6/2,5?/4]", "[2/2,9?/4,1]"]:
        shape = parse_shape(text)
        s = shape.tile_slots()
        tiles = nrng.uniform(-5, 5, size=(shape.tile_count(), s))
        for dim in range(1, shape.rank() + 1):
            for v in (-1, 0, 1):
                so, out, c = ref.sum(shape, tiles, s, dim, v)
                add("sum", s=s, shape=shape, tiles=tiles, dim=dim, variant=v, so=so, out=out,
                    cost=cost_vec(c))

    # the four product forms (criterion 6 style, tiles random)
    for s in (8, 16, 32):
        for which in range(4):
            for it in range(3):
                a, b, c_ = rng.randint(1, 9), rng.randint(1, 9), rng.randint(1, 9)
                t1 = 1 << rng.randint(0, int(np.log2(s)))
                rest = s // t1
                if which < 2:
                    t2 = rest
                    if which == 0:
                        sa = TileTensorShape([DimSpec(a, 1, t1), DimSpec(b, 1, t2)])
                        sb = TileTensorShape([DimSpec(1, t1, t1), DimSpec(b, 1, t2)])
                    else:
                        sa = TileTensorShape([DimSpec(b, 1, t1), DimSpec(a, 1, t2)])
                        sb = TileTensorShape([DimSpec(b, 1, t1), DimSpec(1, t2, t2)])
                else:
                    t2 = 1 << rng.randint(0, int(np.log2(rest)))
                    t3 = rest // t2
                    if which == 2:
                        sa = TileTensorShape([DimSpec(a, 1, t1), DimSpec(b, 1, t2), DimSpec(1, t3, t3)])
                        sb = TileTensorShape([DimSpec(1, t1, t1), DimSpec(b, 1, t2), DimSpec(c_, 1, t3)])
                    else:
                        sa = TileTensorShape([DimSpec(b, 1, t1), DimSpec(a, 1, t2), DimSpec(1, t3, t3)])
                        sb = TileTensorShape([DimSpec(b, 1, t1), DimSpec(1, t2, t2), DimSpec(c_, 1, t3)])
                ta = nrng.uniform(-2, 2, size=(sa.tile_count(), s))
                tb = nrng.uniform(-2, 2, size=(sb.tile_count(), s))
                so, out, cst = ref.linalg(which, sa, ta, sb, tb, s)
                add("linalg", s=s, which=which, sa=sa, sb=sb, ta=ta, tb=tb, so=so, out=out,
                    cost=cost_vec(cst))

    # clean_unknowns / replicate_dim
    for text, s in [("[5/2,1?/4]", 8), ("[18?/8,4/16]", 128), ("[3?/4,2/2,7?/4]", 32)]:
        shape = parse_shape(text)
        tiles = nrng.uniform(-5, 5, size=(shape.tile_count(), s))
        so, out, c = ref.clean_unknowns(shape, tiles, s)
        add("clean", s=s, shape=shape, tiles=tiles, so=so, out=out, cost=cost_vec(c))
    for text, s, dim in [("[5/2,1/4]", 8, 2), ("[7/4,1/8]", 32, 2), ("[3/2,1/6,2/2]", 24, 2),
                         ("[4,1/16,5/32]", 512, 2)]:
        shape = parse_shape(text)
        tiles = nrng.uniform(-5, 5, size=(shape.tile_count(), s))
        so, out, c = ref.replicate_dim(shape, tiles, s, dim)
        add("replicate", s=s, shape=shape, tiles=tiles, dim=dim, so=so, out=out, cost=cost_vec(c))

    # single-tile schedules (rotate_sum.hpp), integer data as in test_rotate_sum.cpp
    for s in (16, 64, 256):
        tile = nrng.integers(-50, 51, size=s).astype(np.float64)
        for n in sorted({1, 2, 3, 5, 7, s // 2, s - 1, s}):
            for v in (0, 1, 2):
                if v == 2 and n & (n - 1):
                    continue
                out, c = ref.sum_tile_strided(tile, n, 1, v)
                add("strided", s=s, tile=tile, n=n, stride=1, variant=v, out=out, cost=cost_vec(c))
        for off in (1, -1, 5, s - 1, 3 * s + 2):
            out, c = ref.rotate(tile, off)
            add("rotate", s=s, tile=tile, offset=off, out=out, cost=cost_vec(c))

    # shape grammar: parse / format / positions
    for text in ["[5/2,*3/4]", "[5,6/8]", "[*/4,5/8]", "[18?/8,4/16]", " [ 5 / 2 , * 3 / 4 ] ",
                 "[2/1,5/8]", "[1*3/4]", "[05/02]", "[*8/8,1?/2]", "[*5/4]", "[2*3/8]", "[0/4]",
                 "[5/0]", "[5/2", "[]", "[5/2,]", "[?/4]", "[5/2] junk", "[5/2,*3/"]:
        rc, shape, pos = ref.parse(text)
        add("parse", text=text, rc=rc, pos=pos, shape=shape if shape else None,
            formatted=ref.format(shape) if shape else "")

    # configs 1 and 2 at full size (inputs regenerable from the shared generator)
    c1 = configs.config1()
    sA = parse_shape(c1.shapes["A"])
    pa, pb = ref.pack(c1.tensors["A"], sA, 512), ref.pack(c1.tensors["B"], sA, 512)
    so, out, c = ref.mul_sum(sA, pa, sA, pb, 512, 2)
    add("config", name="c1", so=so, out=out, cost=cost_vec(c))
    c2 = configs.config2()
    sM, sV = parse_shape(c2.shapes["M"]), parse_shape(c2.shapes["V"])
    pm, pv = ref.pack(c2.tensors["M"], sM, 8192), ref.pack(c2.tensors["V"], sV, 8192)
    so, out, c = ref.linalg(0, sM, pm, sV, pv, 8192)
    add("config_digest", name="c2", so=so, digest=digest(out), cost=cost_vec(c),
        unpacked=ref.unpack(so, 8192, out))

    np.savez_compressed(HERE / "golden.npz", **arrays)
    (HERE / "golden_index.json").write_text(json.dumps(index, indent=0))
    print(f"wrote {len(index)} cases, {len(arrays)} arrays")


if __name__ == "__main__":
    main()
