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

    # config 3 ('3b' chain and the literal '3a' chain), through the reference
    c3 = configs.config3()
    sh3 = {k: parse_shape(v) for k, v in c3.shapes.items()}
    p3 = {k: ref.pack(c3.tensors[k], sh3[k], 8192) for k in sh3}
    s1, o1, k1 = ref.linalg(3, sh3["Bt3"], p3["Bt3"], sh3["C3"], p3["C3"], 8192)
    s2, o2, k2 = ref.linalg(2, sh3["A3"], p3["A3"], s1, o1, 8192)
    add("config_digest", name="c3b_stage1", so=s1, digest=digest(o1), cost=cost_vec(k1))
    add("config_digest", name="c3b", so=s2, digest=digest(o2), cost=cost_vec(k2),
        unpacked=ref.unpack(s2, 8192, o2))
    sa, oa, ka = ref.linalg(2, sh3["A3"], p3["A3"], sh3["B3"], p3["B3"], 8192)
    sc, oc, _ = ref.clean_unknowns(sa, oa, 8192)
    sr, orr, _ = ref.replicate_dim(sc, oc, 8192, 2)
    s3, o3, _ = ref.mul_sum(sr, orr, sh3["Ct3"], p3["Ct3"], 8192, 3)
    add("config_digest", name="c3a", so=s3, digest=digest(o3), cost=cost_vec(ka))
    # config 4, composed FC -> square -> FC on the full batch
    c4 = configs.config4(False)
    sh4 = {k: parse_shape(v) for k, v in c4.shapes.items()}
    p4 = {k: ref.pack(c4.tensors[k], sh4[k], 8192) for k in sh4}
    h1, t1, _ = ref.mul_sum(sh4["W1t"], p4["W1t"], sh4["X"], p4["X"], 8192, 1)
    h2, t2, _ = ref.elementwise(0, h1, t1, sh4["b1"], p4["b1"], 8192)
    h3, t3, _ = ref.elementwise(1, h2, t2, h2, t2, 8192)
    h4, t4, _ = ref.mul_sum(sh4["W2"], p4["W2"], h3, t3, 8192, 2)
    h5, t5, _ = ref.elementwise(0, h4, t4, sh4["b2"], p4["b2"], 8192)
    add("config_digest", name="c4", so=h5, digest=digest(t5), cost=np.zeros(6, dtype=np.int64),
        unpacked=ref.unpack(h5, 8192, t5))
    # config 5 slabs: X[0:32] (sums over dims 2, 3) and X[:, 0:32] (sum over dim 1)
    s5 = configs.C5_SLOTS
    sw = parse_shape(configs.C5_W_SHAPE)
    pw = ref.pack(configs.c5_w(), sw, s5)
    add("config_digest", name="c5_w_pack", so=sw, digest=digest(pw), cost=np.zeros(6, dtype=np.int64))
    ss = TileTensorShape([DimSpec(32, 1, 16), DimSpec(2048, 1, 32), DimSpec(512, 1, 32)])
    px = ref.pack(configs.c5_x_slab(slice(0, 32)), ss, s5)
    add("config_digest", name="c5_x_pack_slab", so=ss, digest=digest(px), cost=np.zeros(6, dtype=np.int64))
    for dim in (2, 3):
        so, out, k = ref.mul_sum(ss, px, sw, pw, s5, dim)
        add("config_digest", name=f"c5_dim{dim}_slab", so=so, digest=digest(out), cost=cost_vec(k))
    ss2 = TileTensorShape([DimSpec(2048, 1, 16), DimSpec(32, 1, 32), DimSpec(512, 1, 32)])
    sw2 = TileTensorShape([DimSpec(1, 16, 16), DimSpec(32, 1, 32), DimSpec(512, 1, 32)])
    so, out, k = ref.mul_sum(ss2, ref.pack(configs.c5_x_slab(slice(None), slice(0, 32)), ss2, s5),
                             sw2, ref.pack(configs.c5_w(slice(0, 32)), sw2, s5), s5, 1)
    add("config_digest", name="c5_dim1_slab", so=so, digest=digest(out), cost=cost_vec(k))

    np.savez_compressed(HERE / "golden.npz", **arrays)
    (HERE / "golden_index.json").write_text(json.dumps(index, indent=0))
    print(f"wrote {len(index)} cases, {len(arrays)} arrays")


if __name__ == "__main__":
    main()
